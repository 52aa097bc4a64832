#!/bin/bash
# round 2, 4 GPUs: final multi-GPU bench lines, configs 2-5 at N=2 and N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for n in 2 4; do
  devs=$(seq -s, 0 $((n - 1)))
  for c in 2 3 4 5; do
    CUDA_VISIBLE_DEVICES=$devs timeout 900 $TRN --nproc-per-node $n --master-port 2970$c bench.py --gpus $n --config $c \
      > gpurun_out/r2j_bench_g${n}_c$c.log 2>&1; echo "bench g$n config $c rc=$?"
    grep "^{" gpurun_out/r2j_bench_g${n}_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']
    print('g$n config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'bound', round(j['step_roofline']['bound_ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(r['frac'],3), 'share', round(r['kernel_share_of_step'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
  done
done
