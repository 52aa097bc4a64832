cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_paths.py tests/test_gpu_ddp.py tests/test_gpu_consensus.py -x -q -p no:cacheprovider 2>&1 | tail -2
for a in "" "--topology static_exponential" "--topology aer --algo accum" "--topology one_peer_ring --algo accum"; do echo "== $a"; python scripts/sweep.py $a 2>&1 | grep default; done
