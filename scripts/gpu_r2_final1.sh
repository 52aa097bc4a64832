#!/bin/bash
# round 2, 1 GPU: full GPU suite (verbose), smoke, default bench (config 3),
# reference arm, launch list + ncu --set full of the headline kernel, config 1
# small-bucket experiments.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2f_pytest_g1.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|error" gpurun_out/r2f_pytest_g1.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2f_bench_g1.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2f_bench_ref.log 2>&1; echo "ref rc=$?"
grep "^{" gpurun_out/r2f_bench_g1.log | head -c 1800; echo
grep "^{" gpurun_out/r2f_bench_ref.log | head -c 400; echo
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2f_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2f_launches_config3.csv $CMD > gpurun_out/r2f_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 $CMD > gpurun_out/r2f_short2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xshare -s 3 -c 1 \
    -o gpurun_out/r2f_config3_full $CMD > gpurun_out/r2f_ncu_full.log 2>&1; echo "ncu full rc=$?"
for c in 1 2 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2f_bench_g1_c$c.log 2>&1; echo "bench config $c rc=$?"
  grep "^{" gpurun_out/r2f_bench_g1_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],4), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
done
