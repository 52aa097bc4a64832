cd $GRAFT_REPO_ROOT
for args in "--topology static_exponential" "--topology aer --algo accum"; do
  echo "== sweep $args"; timeout 900 python scripts/sweep.py $args 2>&1
done
for v in "" build/variants/libdg_single2.so build/variants/libdg_single3.so build/variants/libdg_single4.so; do
  echo "-- 2 GPU exchange, lib=$v"
  DG_LIB=$v timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/round_timing.py --periods 1 2>&1 | grep -E "^\[|rror"
  DG_LIB=$v DG_WAVES=2 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 scripts/round_timing.py --periods 1 2>&1 | grep -E "^\[|rror"
done
