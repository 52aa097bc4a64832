#!/bin/bash
# g/m/v software-prefetch variants (DG_PF_MIN_NS) on one GPU: parity + sweep.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in pf8 pf2; do
  DG_LIB=build/variants/libdg_$v.so timeout 600 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
done
for topo in static_exponential one_peer_exponential; do
  echo "== $topo dadam"; timeout 900 python scripts/sweep.py --topology $topo --bucket-params 125000000
done
echo "== aer accum"; timeout 900 python scripts/sweep.py --topology aer --algo accum --bucket-params 125000000
