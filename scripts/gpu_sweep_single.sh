cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== static"; timeout 900 python scripts/sweep.py --topology static_exponential 2>&1 | grep -v waves
echo "== aer accum"; timeout 900 python scripts/sweep.py --topology aer --algo accum 2>&1 | grep -v waves
for v in "" build/variants/libdg_su1.so build/variants/libdg_su4.so; do
  echo "-- 2 GPU exchange, lib=$v"
  DG_LIB=$v timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/round_timing.py --periods 1 2>&1 | grep -E "^\[|rror"
done
