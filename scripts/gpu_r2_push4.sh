#!/bin/bash
# 4 GPUs: P2P push exchange -- parity (+fault) and benches vs default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1"
DG_P2P_PUSH=1 MP_TRANSPORT=p2p MP_D=100003 MP_CHUNK=16384 timeout 900 $TRN --master-port 29741 tests/mp_parity_main.py \
   > gpurun_out/r2m_parity_push4.log 2>&1; echo "parity p2p push rc=$?"; grep -E "MISMATCH|Error" gpurun_out/r2m_parity_push4.log | head -5
DG_P2P_PUSH=1 MP_TRANSPORT=p2p MP_D=100003 DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TRN --master-port 29742 \
   tests/mp_parity_main.py > gpurun_out/r2m_parity_push4_fault.log 2>&1; echo "parity p2p push+fault rc=$?"
for c in 3 4 5 2; do
  for env in "DG_X=0" "DG_P2P_PUSH=1"; do
    env $env timeout 900 $TRN --master-port 29743 bench.py --gpus 4 --config $c --no-e2e --steps 30 2>&1 | grep -E "^\{|rror" | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): print(l.strip()); continue
    j=json.loads(l); r=j['roofline']
    print('g4 config $c $env', 'ms', round(j['ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(r['frac'],3))
"
  done
done
