#!/bin/bash
# final build, 2 GPUs: multi-GPU parity on every transport (+fault), DDP
cd "$(dirname "$0")/.."
TRN="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
for tr in p2p nccl; do
  for env in "DG_X=0" "DG_P2P_PUSH=1" "DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1"; do
    env $env MP_TRANSPORT=$tr MP_D=100003 MP_CHUNK=16384 timeout 900 $TRN --master-port 29761 tests/mp_parity_main.py > /tmp/mp.log 2>&1
    echo "parity $tr [$env] rc=$? $(grep -c MISMATCH /tmp/mp.log) mismatches"
  done
done
timeout 900 $TRN --master-port 29762 tests/mp_ddp_main.py > /tmp/ddp.log 2>&1; echo "ddp rc=$?"; grep rank /tmp/ddp.log | head -3
