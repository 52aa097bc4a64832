#!/bin/bash
# round 2: ncu --set full of the staged kernel (static exponential + pairs) and legacy pairs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_profile.sh st_static - --topology static_exponential --bucket-params 125000000
bash scripts/gpu_profile.sh st_pairs - --topology one_peer_exponential --bucket-params 125000000
bash scripts/gpu_profile.sh lg_pairs DG_STAGED=0 --topology one_peer_exponential --bucket-params 125000000
rm -f gpurun_out/*.ncu-rep
