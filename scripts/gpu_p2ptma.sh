cd $GRAFT_REPO_ROOT
for e in "DG_NONE=1" "DG_P2P_PULL=2" "DG_P2P_PULL=2 DG_TMA=2" "DG_TMA=2" "DG_P2P_KEEP_NC=0"; do
echo "-- $e"
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/round_timing.py --periods 1 --topology aer --nodes-per-gpu 2 --bucket-params 1300000000 2>&1 | grep -E "^\[|rror"
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 scripts/round_timing.py --periods 1 --topology static_exponential --nodes-per-gpu 2 --bucket-params 350000000 2>&1 | grep -E "^\[|rror"
done
