#!/bin/bash
# 4 GPUs: multi-GPU tests + default benches at 2 and 4 GPUs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m multigpu -q -p no:cacheprovider > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_mg.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n > gpurun_out/final_bench_g$n.log 2>&1; echo "bench$n rc=$?"
grep "^{" gpurun_out/final_bench_g$n.log | python -c "
import sys,json; j=json.loads(sys.stdin.read())
print('g$n', '%.4g'%j['value'], 'ms/step', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3), 'sfrac', round(j['step_roofline']['frac'],3), 'e2e', '%.3g'%j['e2e']['value'], 'clk', j['clocks'].get('sm_mhz'), j['clocks'].get('reasons'), 'nvl', (j.get('nvlink') or {}).get('achieved'))"
done
