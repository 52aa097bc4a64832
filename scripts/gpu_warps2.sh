#!/bin/bash
# warp-per-node kernel at 3 CTAs/SM (DG_WARPS_MIN_NC): parity + 1-GPU benches vs default
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py -m gpu -x -q -k "warps or default" 2>&1 | tail -1
for a in "--topology static_exponential --bucket-params 125000000" "--topology static_exponential --bucket-params 125000000 --algo accum" "--topology static_exponential --bucket-params 350000000" "--topology aer --algo accum --bucket-params 125000000"; do
  for w in 99 4; do
    DG_WARPS_MIN_NC=$w timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline $a | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$a warps_min=$w', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3))"
  done
done
DG_WARPS_MIN_NC=4 bash scripts/gpu_profile.sh static6w - --topology static_exponential --bucket-params 125000000
