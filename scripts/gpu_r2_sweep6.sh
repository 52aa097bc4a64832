#!/bin/bash
# 1 GPU: config-3 kernel regression hunt (ShGroup layout, staging)
cd "$(dirname "$0")/.."
for v in build/variants/libdg_*.so; do
  DG_LIB=$v timeout 600 python tests/engine_parity_main.py 5003 > /tmp/p.log 2>&1; echo "parity $(basename $v) rc=$? $(tail -1 /tmp/p.log)"
done
timeout 1500 python scripts/sweep.py --config 3 2>&1
