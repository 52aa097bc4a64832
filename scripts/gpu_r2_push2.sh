#!/bin/bash
# 2 GPUs: P2P push exchange (DG_P2P_PUSH=1) -- parity (+fault, full-size config 4), benches vs default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
DG_P2P_PUSH=1 MP_TRANSPORT=p2p MP_D=100003 MP_CHUNK=16384 timeout 900 $TRN --master-port 29731 tests/mp_parity_main.py \
   > gpurun_out/r2l_parity_push.log 2>&1; echo "parity p2p push rc=$?"; grep -E "MISMATCH|Error" gpurun_out/r2l_parity_push.log | head -5
DG_P2P_PUSH=1 MP_TRANSPORT=p2p MP_D=100003 DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TRN --master-port 29732 \
   tests/mp_parity_main.py > gpurun_out/r2l_parity_push_fault.log 2>&1; echo "parity p2p push+fault rc=$?"; grep -E "MISMATCH|Error" gpurun_out/r2l_parity_push_fault.log | head -5
MP_TRANSPORT=p2p MP_D=1048576 MP_CHUNK=0 timeout 900 $TRN --master-port 29733 tests/mp_parity_main.py > gpurun_out/r2l_parity_default.log 2>&1; echo "parity default rc=$?"
for c in 2 3 4 5; do
  for env in "DG_X=0" "DG_P2P_PUSH=1"; do
    env $env timeout 900 $TRN --master-port 29734 bench.py --gpus 2 --config $c --no-e2e --steps 30 2>&1 | grep -E "^\{|rror" | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): print(l.strip()); continue
    j=json.loads(l); r=j['roofline']
    print('g2 config $c $env', 'ms', round(j['ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(r['frac'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0))
"
  done
done
DG_P2P_PUSH=1 MP_FULLSIZE=1 MP_TRANSPORT=p2p timeout 1500 $TRN --master-port 29735 tests/mp_parity_main.py > gpurun_out/r2l_fullsize_push.log 2>&1; echo "fullsize push rc=$?"; grep rank gpurun_out/r2l_fullsize_push.log | head -4
