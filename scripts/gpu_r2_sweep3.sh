#!/bin/bash
# round 2, 1 GPU: compute-sanitizer memcheck (one tool per call), then parity +
# sweep of the x-pipelining / staging / occupancy variants, config 1 with the
# pairs rule.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_r2_sanitize.sh memcheck
for v in build/variants/libdg_*.so; do
  DG_LIB=$v timeout 600 python tests/engine_parity_main.py 300001 > /tmp/p.log 2>&1; echo "parity $(basename $v) rc=$? $(tail -1 /tmp/p.log)"
done
for args in "--config 3" "--config 3 --algo accum" "--config 2 --topology aer --algo accum"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
for g in on off; do
  timeout 600 python bench.py --config 1 --graph $g --no-cpu-baseline --no-e2e 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('config 1 graph=$g', 'us/step', round(1e3*j['ms_per_step'],2), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3))
"
done
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('config 2 (pairs -> legacy)', 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3))
"
