cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py -x -q -p no:cacheprovider 2>&1 | tail -2
for args in "" "--topology static_exponential" "--topology aer --algo accum"; do
  echo "== sweep TMA (ws) $args"
  SWEEP_ENV="DG_TMA=2" timeout 900 python scripts/sweep.py $args 2>&1
done
