#!/bin/bash
# round 2, 2 GPUs: benches of configs 2-5 at N=2 with the final kernel rules
# (config 5 = 32 resident nodes per GPU), in-place P2P parity + DDP recheck,
# Table-1 analogue on both transports.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1"
MP_TRANSPORT=p2p MP_D=100003 MP_CHUNK=16384 timeout 900 $TR --master-port 29651 tests/mp_parity_main.py \
   > gpurun_out/r2h_parity_p2p.log 2>&1; echo "parity p2p rc=$?"
for c in 2 3 4 5; do
  timeout 900 $TR --master-port 29652 bench.py --gpus $N --config $c > gpurun_out/r2h_bench_g${N}_c$c.log 2>&1; echo "bench config $c rc=$?"
  grep "^{" gpurun_out/r2h_bench_g${N}_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l)
    print('config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'bound', round(j['step_roofline']['bound_ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(j['roofline']['frac'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
done
for tr in p2p nccl; do
  timeout 900 $TR --master-port 29653 scripts/table1.py --transport $tr > gpurun_out/r2h_table1_$tr.log 2>&1; echo "table1 $tr rc=$?"; grep "^|" gpurun_out/r2h_table1_$tr.log
done
