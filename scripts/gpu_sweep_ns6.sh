#!/bin/bash
# single-member-component occupancy variants (NS=6 instantiation, 3 CTAs/SM) on one GPU
cd "$(dirname "$0")/.."
for v in ns6m3; do
  DG_LIB=build/variants/libdg_$v.so timeout 600 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
done
for a in "--topology static_exponential" "--topology static_exponential --algo accum" "--topology aer --algo accum"; do
  echo "== $a"; SWEEP_ENV="X=1" timeout 900 python scripts/sweep.py $a --bucket-params 125000000
done
