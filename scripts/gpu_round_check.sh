#!/bin/bash
# 4-GPU box: full GPU suite + round benches + BASELINE configs + config-3 keep comparison
cd "$(dirname "$0")/.."
bash scripts/gpu_full.sh
bash scripts/gpu_configs.sh
echo "== config 3 @2 GPUs, singletons instead of kept 4-member components"
DG_P2P_KEEP_NC=0 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 12 --warmup 4 --no-e2e --nodes-per-gpu 4 --topology static_exponential --bucket-params 350000000 2>&1 | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.4e'%j['value'], j['ms_per_step'], j['step_roofline']['frac'])"
