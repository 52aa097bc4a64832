cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "bit_exact" 2>&1 | tail -3
bash scripts/gpu_configs.sh
