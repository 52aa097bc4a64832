#!/bin/bash
# config 2 at 4 GPUs: where do the inter-kernel gaps of the bench come from?
cd "$(dirname "$0")/.."
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
q() { grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']; print('$1', 'ms', round(j['ms_per_step'],3), 'kernel', round(r['kernel_ms_per_launch'],3), 'share', round(r['kernel_share_of_step'],3))
"; }
for n in 4 2; do
  devs=$(seq -s, 0 $((n - 1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 600 $TRN --nproc-per-node $n --master-port 29681 bench.py --gpus $n --config 2 --no-e2e 2>&1 | q "g$n clocks"
  CUDA_VISIBLE_DEVICES=$devs timeout 600 $TRN --nproc-per-node $n --master-port 29682 bench.py --gpus $n --config 2 --no-e2e --no-clocks 2>&1 | q "g$n no-clocks"
  CUDA_VISIBLE_DEVICES=$devs NCCL_PROTO=LL timeout 600 $TRN --nproc-per-node $n --master-port 29683 bench.py --gpus $n --config 2 --no-e2e --no-clocks 2>&1 | q "g$n no-clocks NCCL_PROTO=LL"
done
