#!/bin/bash
# round 2: ncu --set full of the x-sharing kernel (static exponential DAdam /
# AccumAdam, one-peer pairs, AER AccumAdam)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_profile.sh xs_static - --topology static_exponential --bucket-params 125000000
bash scripts/gpu_profile.sh xs_static_acc - --topology static_exponential --bucket-params 125000000 --algo accum
bash scripts/gpu_profile.sh xs_aer_acc - --topology aer --bucket-params 125000000 --algo accum
bash scripts/gpu_profile.sh lg_aer_acc DG_XSHARE=0 --topology aer --bucket-params 125000000 --algo accum
rm -f gpurun_out/*.ncu-rep
