#!/bin/bash
# 2 GPUs: warp-per-node default -- multi-GPU parity (both transports) + configs 2/3/4 at 2 GPUs vs the old path
cd "$(dirname "$0")/.."
for tr in p2p nccl; do
  MP_TRANSPORT=$tr timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|rror|: ok" | head -4
done
b() {
  local label=$1; shift; local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 2 --steps 12 --warmup 4 --no-e2e "$@" 2>&1 | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); nv=j.get('nvlink') or {}; print('$label', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],2), 'sfrac', round(j['step_roofline']['frac'],3), 'nvl', nv.get('achieved'))"
}
for w in 4 99; do
  b c2_w$w DG_WARPS_MIN_NC=$w -- --nodes-per-gpu 4 --topology one_peer_exponential --bucket-params 125000000
  b c3_w$w DG_WARPS_MIN_NC=$w -- --nodes-per-gpu 4 --topology static_exponential --bucket-params 350000000
  b c4_w$w DG_WARPS_MIN_NC=$w -- --nodes-per-gpu 4 --topology aer --algo accum --bucket-params 1300000000
  b c2g8_w$w DG_WARPS_MIN_NC=$w -- --nodes-per-gpu 8 --topology one_peer_exponential --bucket-params 125000000
done
