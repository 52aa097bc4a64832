#!/bin/bash
# round 2, 2 GPUs: in-place P2P transport (parity incl. fault injection, DDP
# wrapper, exchange bandwidth vs NCCL), P2P exchange-round kernel choice
# (legacy vs x-sharing), NVLink counter diagnostics.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1"
nvidia-smi nvlink -gt d -i 0 2>&1 | head -8
nvidia-smi nvlink -s -i 0 2>&1 | head -4
for tr in p2p nccl; do
  MP_TRANSPORT=$tr MP_D=100003 MP_CHUNK=16384 timeout 900 $TR --master-port 29621 tests/mp_parity_main.py \
     > gpurun_out/r2b_parity_g${N}_$tr.log 2>&1; echo "parity $tr rc=$?"; grep -E "MISMATCH|in-place|ok$" gpurun_out/r2b_parity_g${N}_$tr.log | head -14
  MP_TRANSPORT=$tr MP_D=100003 MP_CHUNK=16384 DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TR --master-port 29622 \
     tests/mp_parity_main.py > gpurun_out/r2b_parity_fault_g${N}_$tr.log 2>&1; echo "parity+fault $tr rc=$?"
done
DG_SIGNAL_KERNEL=1 MP_TRANSPORT=p2p MP_D=100003 timeout 900 $TR --master-port 29623 tests/mp_parity_main.py \
   > gpurun_out/r2b_parity_sigkernel.log 2>&1; echo "parity p2p signal-kernel rc=$?"
timeout 900 $TR --master-port 29624 tests/mp_ddp_main.py > gpurun_out/r2b_ddp.log 2>&1; echo "ddp rc=$?"; tail -4 gpurun_out/r2b_ddp.log
DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TR --master-port 29625 tests/mp_ddp_main.py > gpurun_out/r2b_ddp_fault.log 2>&1; echo "ddp+fault rc=$?"
for x in "--transport nccl" "--range --transport nccl" "--range --transport p2p"; do
  timeout 300 $TR --master-port 29626 scripts/xchg_bw.py $x --tag "$x" 2>&1 | grep -E "^xchg|rror" | head -3
done
DG_DIAG_SKIP_KERNEL=1 timeout 300 $TR --master-port 29627 scripts/xchg_bw.py --range --transport nccl --tag "nccl exchange only" 2>&1 | grep -E "^xchg|rror" | head -3
for c in 2 3 4; do
  for env in DG_XSHARE_REMOTE=0 DG_XSHARE_REMOTE=1; do
    env $env timeout 900 $TR --master-port 29628 bench.py --gpus $N --config $c --no-e2e > gpurun_out/r2b_bench_g${N}_c${c}_$env.log 2>&1; echo "bench config $c $env rc=$?"
    grep "^{" gpurun_out/r2b_bench_g${N}_c${c}_$env.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); n=j.get('nvlink_counters') or {}
    print('  value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'nvl(events)', (j.get('nvlink') or {}).get('achieved'), 'nvl(counters)', n.get('min_rx_GBps_over_exchange_kernels'), n.get('source') or n.get('unavailable'))
"
  done
done
