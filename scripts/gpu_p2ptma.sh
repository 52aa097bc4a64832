cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|: ok|FAIL" | tail -4
for e in "DG_NONE=1" "DG_P2P_TMA=0"; do
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/round_timing.py --periods 1 --topology aer --nodes-per-gpu 2 --bucket-params 1300000000 2>&1 | grep -E "^\[|rror"
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 scripts/round_timing.py --periods 1 --topology static_exponential --nodes-per-gpu 2 --bucket-params 350000000 2>&1 | grep -E "^\[|rror"
env $e timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 scripts/round_timing.py --periods 1 --topology aer --nodes-per-gpu 4 --bucket-params 1300000000 2>&1 | grep -E "^\[|rror"
done
