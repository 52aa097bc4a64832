#!/bin/bash
# round 2, 2 GPUs: exchange-round kernel choice re-measured without start skew
cd "$(dirname "$0")/.."
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for c in 3 4 5 2; do
  for env in "DG_X=0" "DG_XSHARE_REMOTE=1" "DG_P2P_KEEP_NC=1" "DG_WARPS_MIN_NC=99"; do
    env $env timeout 900 $TRN --nproc-per-node 2 --master-port 29711 bench.py --gpus 2 --config $c --no-e2e --steps 30 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']
    print('g2 config $c $env', 'ms', round(j['ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0))
"
  done
done
