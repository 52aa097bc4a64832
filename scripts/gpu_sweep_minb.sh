#!/bin/bash
# single-member-component CTA residency (DG_MINB_SINGLE) on one GPU + config 3 at full size
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -1
for a in "--topology static_exponential" "--topology static_exponential --algo accum"; do
  echo "== $a"; SWEEP_ENV="X=1" timeout 900 python scripts/sweep.py $a --bucket-params 125000000
done
echo "== config 3 (8 x 350M static exp)"
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --topology static_exponential --bucket-params 350000000 | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.4e'%j['value'], j['ms_per_step'], j['roofline']['frac'], j['step_roofline']['frac'])"
echo "== headline"
timeout 900 python bench.py --steps 30 --warmup 4 --no-e2e --no-cpu-baseline | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.4e'%j['value'], j['ms_per_step'], j['roofline']['frac'])"
