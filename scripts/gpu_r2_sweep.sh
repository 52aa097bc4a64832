#!/bin/bash
# round 2, 1 GPU: parity of every kernel path (new x-sharing loop), then the
# xshare variant sweep (build/variants: old loop / bulk prefetch / isfinite /
# just-in-time x) on configs 3 and 2, static AccumAdam and AER AccumAdam.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py tests/test_c_abi.py \
    tests/test_gpu_graph.py tests/test_gpu_consensus.py -m gpu -q 2>&1 | tail -4
for g in on off; do
  timeout 600 python bench.py --config 1 --graph $g --no-cpu-baseline > gpurun_out/r2_bench_c1_graph$g.log 2>&1; echo "config 1 graph=$g rc=$?"
  grep "^{" gpurun_out/r2_bench_c1_graph$g.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('  value %.4e'%j['value'], 'us/step', round(1e3*j['ms_per_step'],2), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'bound_us', round(1e3*j['step_roofline']['bound_ms_per_step'],2))
"
done
for args in "--config 3" "--config 2" "--config 3 --algo accum" "--config 2 --topology aer --algo accum"; do
  echo "== $args"
  timeout 1500 python scripts/sweep.py $args 2>&1
done
