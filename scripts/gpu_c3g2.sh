cd $GRAFT_REPO_ROOT
for e in "DG_NONE=1" "DG_P2P_KEEP_NC=4" "DG_P2P_KEEP_NC=4 DG_TMA=2" "DG_P2P_KEEP_NC=4 DG_TMA=1" "DG_P2P_KEEP_NC=4 DG_COOP_MIN_NC=99"; do
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 scripts/round_timing.py --periods 1 --topology static_exponential --nodes-per-gpu 4 --bucket-params 350000000 2>&1 | grep -E "^\[|rror"
done
