#!/bin/bash
# round 2, N GPUs (2 or 4): GPU suite incl. multi-GPU + fault-injection tests,
# 100-step full-size parity (configs 4/5) on every transport with per-rank
# pass lines kept, and benches with NVML NVLink counters.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1"
echo "GPUs: $N"
timeout 3000 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2_pytest_g$N.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2_pytest_g$N.log
for tr in p2p:1 p2p:2 nccl:1; do
  t=${tr%%:*}; pull=${tr##*:}
  DG_P2P_PULL=$pull MP_FULLSIZE=1 MP_TRANSPORT=$t timeout 1500 $TR --master-port 29611 tests/mp_parity_main.py \
    > gpurun_out/r2_fullsize_g${N}_${t}_pull${pull}.log 2>&1; echo "fullsize $t pull=$pull rc=$?"
  grep "rank" gpurun_out/r2_fullsize_g${N}_${t}_pull${pull}.log | tail -8
done
for c in 4 2 3 5; do
  timeout 900 $TR --master-port 29612 bench.py --gpus $N --config $c > gpurun_out/r2_bench_g${N}_c$c.log 2>&1; echo "bench config $c rc=$?"
  grep "^{" gpurun_out/r2_bench_g${N}_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); n=j.get('nvlink_counters') or {}
    print('config', j['config']['baseline_config'], 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'nvl_counter_GBps', n.get('min_rx_GBps_over_exchange_kernels'), n.get('source') or n.get('unavailable'))
"
done
timeout 900 $TR --master-port 29613 scripts/ddp_bench.py > gpurun_out/r2_ddp_bench_g$N.log 2>&1; echo "ddp_bench rc=$?"; grep "^|" gpurun_out/r2_ddp_bench_g$N.log
