#!/bin/bash
# warp-per-component kernel (DG_WARPS_*): parity + static-exponential / AER sweeps on one GPU
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_kernel_paths.py -m gpu -x -q -k "warps or default" 2>&1 | tail -2
run() {  # label, env..., -- bench args
  local label=$1; shift; local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 600 python bench.py --steps 30 --warmup 4 --no-e2e --no-cpu-baseline "$@" \
    | python -c "import json,sys; j=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('$label', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'frac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3))"
}
for a in "--topology static_exponential" "--topology static_exponential --algo accum" "--topology aer --algo accum"; do
  echo "== $a"
  run base X=1 -- $a --bucket-params 125000000
  for s in 0 1 4 16; do run warps_s$s DG_WARPS_MIN_NC=4 DG_WARPS_SYNC=$s -- $a --bucket-params 125000000; done
done
