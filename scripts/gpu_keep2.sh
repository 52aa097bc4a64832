#!/bin/bash
# 2 GPUs: keep only pair components in P2P exchange rounds (warp-per-node otherwise) -- parity + configs
cd "$(dirname "$0")/.."
for tr in p2p nccl; do
  MP_TRANSPORT=$tr timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29594 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|rror|: ok" | head -4
done
b() {
  local label=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595 bench.py --gpus 2 --steps 12 --warmup 4 --no-e2e "$@" 2>&1 | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); nv=j.get('nvlink') or {}; print('$label', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],2), 'sfrac', round(j['step_roofline']['frac'],3), 'nvl', nv.get('achieved'))"
}
b c3 --nodes-per-gpu 4 --topology static_exponential --bucket-params 350000000
b c4 --nodes-per-gpu 4 --topology aer --algo accum --bucket-params 1300000000
b c2 --nodes-per-gpu 4 --topology one_peer_exponential --bucket-params 125000000
b bench_g2 --nodes-per-gpu 8 --topology one_peer_exponential --bucket-params 125000000
