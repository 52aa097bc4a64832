#!/bin/bash
# round 2: shared-memory staged kernel -- parity, then staged vs legacy per topology, then knob sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py -m gpu -x -q 2>&1 | tail -3
q() { python -c "import json,sys; j=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$1', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3))"; }
for a in "--topology static_exponential --bucket-params 350000000" "--topology one_peer_exponential --bucket-params 125000000" "--topology static_exponential --bucket-params 125000000 --algo accum" "--topology aer --algo accum --bucket-params 125000000" "--topology one_peer_ring --algo accum --bucket-params 125000000"; do
  for env in "DG_STAGED=1" "DG_STAGED=0"; do
    env $env timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline $a 2>&1 | q "$a $env"
  done
done
for env in "DG_ST_STAGES=2" "DG_ST_STAGES=4" "DG_ST_TW=64" "DG_ST_TW=64 DG_ST_STAGES=2" "DG_ST_TW=128 DG_ST_STAGES=2" "DG_WAVES=0.5"; do
  env $env timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline --topology static_exponential --bucket-params 350000000 2>&1 | q "static350 $env"
done
