cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ddp.py tests/test_gpu_allreduce.py -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 tests/mp_ddp_main.py 2>&1 | grep -E "rank|rror|Traceback" | head -20
