cd $GRAFT_REPO_ROOT
bash scripts/gpu_profile.sh tma_static DG_TMA=2 --bucket-params 16000000 --topology static_exponential
bash scripts/gpu_profile.sh tma_pairs DG_TMA=2 --bucket-params 16000000
