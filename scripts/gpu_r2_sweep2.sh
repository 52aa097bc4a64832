#!/bin/bash
# round 2, 1 GPU: parity of the x-sharing variants (branch-free Adam direction,
# 32-bit indices), then the variant sweep and a DG_PREFETCH sweep (configs 3, 1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in build/variants/libdg_*.so; do
  for d in 5003 300001; do
    DG_LIB=$v timeout 600 python tests/engine_parity_main.py $d > /tmp/p.log 2>&1; echo "parity $(basename $v) d=$d rc=$? $(tail -1 /tmp/p.log)"
  done
  DG_LIB=$v timeout 600 python tests/graph_parity_main.py 5003 > /tmp/p.log 2>&1; echo "graph parity $(basename $v) rc=$? $(tail -1 /tmp/p.log)"
done
for args in "--config 3" "--config 2" "--config 3 --algo accum" "--config 2 --topology aer --algo accum"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
for pf in 0 2 3 4; do
  echo "== DG_PREFETCH=$pf"
  for args in "--config 3" "--config 1"; do
    DG_PREFETCH=$pf timeout 600 python bench.py $args --steps 30 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('  $args', 'ms', round(j['ms_per_step'],4), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3))
"
  done
done
