#!/bin/bash
cd "$(dirname "$0")/.."
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
timeout 600 $TRN --nproc-per-node 4 --master-port 29691 scripts/round_timing.py --nodes-per-gpu 2 --bucket-params 125000000 --periods 20 --b2b 2>&1 | grep -E "rounds|b2b|rror"
for st in 18 60; do
  timeout 600 $TRN --nproc-per-node 4 --master-port 29692 bench.py --gpus 4 --config 2 --no-e2e --steps $st 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']; print('bench steps=$st', 'ms', round(j['ms_per_step'],3), 'kernel', round(r['kernel_ms_per_launch'],3), 'share', round(r['kernel_share_of_step'],3))
"
done
