cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for args in "" "--topology static_exponential" "--topology aer --algo accum" "--topology one_peer_ring --algo accum"; do
  echo "== sweep $args"
  timeout 900 python scripts/sweep.py $args 2>&1
done > gpurun_out/sweep.log
cat gpurun_out/sweep.log
