#!/bin/bash
# round 2, 1 GPU: g/m/v staging variants (parity first, then sweep)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in build/variants/libdg_*.so; do
  for d in 5003 300001; do
    DG_LIB=$v timeout 600 python tests/engine_parity_main.py $d > /tmp/p.log 2>&1; echo "parity $(basename $v) d=$d rc=$? $(tail -1 /tmp/p.log)"
  done
  DG_LIB=$v timeout 600 python tests/guard_main.py 1003 > /tmp/p.log 2>&1; echo "guard $(basename $v) rc=$? $(tail -1 /tmp/p.log)"
done
for args in "--config 3" "--config 3 --algo accum" "--config 2 --topology aer --algo accum"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
for v in default libdg_xs_g1; do
  lib=build/variants/$v.so; [ $v = default ] && lib=paper_2410_11998_b200/libdg.so
  DG_LIB=$lib timeout 900 python bench.py --no-cpu-baseline --no-e2e 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('60-step config 3 $v', 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3), j['clocks'])
"
done
