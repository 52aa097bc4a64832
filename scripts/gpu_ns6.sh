#!/bin/bash
# NS=6 instantiation actually selected for static exponential: parity + 1-GPU static benches
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for a in "--bucket-params 125000000" "--bucket-params 125000000 --algo accum" "--bucket-params 350000000"; do
  timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline --topology static_exponential $a | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$a', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3))"
done
