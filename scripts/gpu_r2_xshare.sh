#!/bin/bash
# round 2: x-sharing kernel -- parity on every kernel path, then prefetch / partition sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py -m gpu -x -q 2>&1 | tail -3
q() { python -c "import json,sys; j=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$1', '%.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3))"; }
b() { env $1 timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline $2 2>&1 | q "$2 $1"; }
for env in DG_PREFETCH=0 DG_PREFETCH=1 DG_PREFETCH=2 DG_PREFETCH=3 DG_PREFETCH=4 DG_PREFETCH=6 "DG_XS_CONTIG=1,DG_PREFETCH=2" "DG_XS_CONTIG=1,DG_PREFETCH=1"; do
  b "$(echo $env | tr ',' ' ')" "--topology static_exponential --bucket-params 350000000"
done
for env in DG_PREFETCH=0 DG_PREFETCH=1 DG_PREFETCH=2 DG_PREFETCH=4; do
  b $env "--topology one_peer_exponential --bucket-params 125000000"
  b $env "--topology static_exponential --bucket-params 125000000 --algo accum"
done
