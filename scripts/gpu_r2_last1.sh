#!/bin/bash
# round 2 last 1-GPU check: GPU suite, smoke, default bench, reference arm, ncu of the hot kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2y_pytest_g1.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r2y_pytest_g1.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2y_bench_g1.log 2>&1; echo "bench rc=$?"
grep "^{" gpurun_out/r2y_bench_g1.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); r=j['roofline']; print('g1 config 3', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(r['frac'],3), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
timeout 600 python bench.py --impl reference > gpurun_out/r2y_bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2y_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2y_launches_config3.csv $CMD > gpurun_out/r2y_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 $CMD > gpurun_out/r2y_short2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xshare -s 3 -c 1 \
    -o gpurun_out/r2y_config3_full $CMD > gpurun_out/r2y_ncu_full.log 2>&1; echo "ncu full rc=$?"
for c in 1 2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2y_bench_g1_c$c.log 2>&1; echo "bench config $c rc=$?"
done
