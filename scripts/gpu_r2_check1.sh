#!/bin/bash
# round 2, 1 GPU: new tests (padding canaries, kernel paths incl. 32/64 resident
# nodes, graphs, full size incl. > 2^30 buckets), benches of configs 3 (default),
# 1, 2 and 5 (64 nodes on one B200).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2g_pytest_g1.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|ERROR" gpurun_out/r2g_pytest_g1.log | head -10; grep -E "passed|failed" gpurun_out/r2g_pytest_g1.log | tail -1
timeout 900 python bench.py > gpurun_out/r2g_bench_g1.log 2>&1; echo "bench rc=$?"
grep "^{" gpurun_out/r2g_bench_g1.log | head -c 1500; echo
for c in 1 2 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2g_bench_g1_c$c.log 2>&1; echo "bench config $c rc=$?"
  grep "^{" gpurun_out/r2g_bench_g1_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],4), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'e2e %.3e'%j['e2e']['value'], j['clocks'])
"
done
