#!/bin/bash
# round 2 final, 4 GPUs: full GPU suite (all multi-GPU transports incl. push variants,
# fault injection, DDP, full-size configs 4/5), final benches at N=2 and N=4, DDP bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
# the N=1 headline on GPU 0 first (bench + reference arm + one ncu capture of the hot kernel)
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2z_bench_g1.log 2>&1; echo "bench g1 rc=$?"
grep "^{" gpurun_out/r2z_bench_g1.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']; print('g1 config 3', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(r['frac'],3), j['clocks'])
"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/r2z_bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
CUDA_VISIBLE_DEVICES=0 timeout 600 $CMD > gpurun_out/r2z_short.log 2>&1 && \
CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xshare -s 3 -c 1 \
    -o gpurun_out/r2z_config3_full $CMD > gpurun_out/r2z_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 3300 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2z_pytest_g4.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|^ERROR" gpurun_out/r2z_pytest_g4.log | head; grep -E "passed|failed" gpurun_out/r2z_pytest_g4.log | tail -1
for n in 2 4; do
  devs=$(seq -s, 0 $((n - 1)))
  for c in 2 3 4 5; do
    CUDA_VISIBLE_DEVICES=$devs timeout 900 $TRN --nproc-per-node $n --master-port 2975$c bench.py --gpus $n --config $c \
      > gpurun_out/r2z_bench_g${n}_c$c.log 2>&1; echo "bench g$n config $c rc=$?"
    grep "^{" gpurun_out/r2z_bench_g${n}_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']
    print('g$n config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'bound', round(j['step_roofline']['bound_ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(r['frac'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
  done
done
timeout 900 $TRN --nproc-per-node 4 --master-port 29759 scripts/ddp_bench.py > gpurun_out/r2z_ddp_bench_g4.log 2>&1; echo "ddp_bench rc=$?"; grep "^|" gpurun_out/r2z_ddp_bench_g4.log
