cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_fullsize.py tests/test_multigpu.py -v -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi.log
grep -E "PASS|FAIL|ERROR|rc=" gpurun_out/pytest_multi.log | tail -20
