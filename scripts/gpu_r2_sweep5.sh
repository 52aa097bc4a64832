#!/bin/bash
# round 2, 1 GPU: occupancy / staging depth variants on top of the final kernel
cd "$(dirname "$0")/.."
for v in build/variants/libdg_*.so; do
  DG_LIB=$v timeout 600 python tests/engine_parity_main.py 300001 > /tmp/p.log 2>&1; echo "parity $(basename $v) rc=$? $(tail -1 /tmp/p.log)"
done
for args in "--config 3" "--config 3 --algo accum" "--config 5"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
