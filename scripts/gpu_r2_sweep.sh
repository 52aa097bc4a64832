#!/bin/bash
# round 2, 1 GPU: parity of every kernel path (new x-sharing loop), then the
# xshare variant sweep (build/variants: old loop / bulk prefetch / isfinite /
# just-in-time x) on configs 3 and 2, static AccumAdam and AER AccumAdam.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py tests/test_c_abi.py -m gpu -x -q 2>&1 | tail -3
for args in "--config 3" "--config 2" "--config 3 --algo accum" "--config 2 --topology aer --algo accum"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
