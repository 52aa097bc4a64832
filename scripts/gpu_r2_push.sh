#!/bin/bash
# 2 GPUs: in-place P2P push variant -- parity (+fault) for push and pull, DDP, exchange, DDP bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
for pu in 1 0; do
  DG_INPLACE_PUSH=$pu MP_TRANSPORT=p2p MP_D=100003 MP_CHUNK=16384 timeout 900 $TRN --master-port 29721 tests/mp_parity_main.py \
     > gpurun_out/r2k_parity_push$pu.log 2>&1; echo "parity push=$pu rc=$?"; grep -E "MISMATCH" gpurun_out/r2k_parity_push$pu.log | head -5
  DG_INPLACE_PUSH=$pu MP_TRANSPORT=p2p MP_D=100003 DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TRN --master-port 29722 \
     tests/mp_parity_main.py > gpurun_out/r2k_parity_fault_push$pu.log 2>&1; echo "parity+fault push=$pu rc=$?"; grep -E "MISMATCH" gpurun_out/r2k_parity_fault_push$pu.log | head -5
  DG_INPLACE_PUSH=$pu timeout 900 $TRN --master-port 29723 tests/mp_ddp_main.py > gpurun_out/r2k_ddp_push$pu.log 2>&1; echo "ddp push=$pu rc=$?"; grep rank gpurun_out/r2k_ddp_push$pu.log | head -2
  DG_INPLACE_PUSH=$pu timeout 300 $TRN --master-port 29724 scripts/xchg_bw.py --range --transport p2p --tag "push=$pu" 2>&1 | grep -E "^xchg|rror" | head -2
done
timeout 900 $TRN --master-port 29725 scripts/ddp_bench.py > gpurun_out/r2k_ddp_bench.log 2>&1; echo "ddp_bench rc=$?"; grep "^|" gpurun_out/r2k_ddp_bench.log
