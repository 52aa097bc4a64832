cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_consensus.py tests/test_gpu_allreduce.py -q -p no:cacheprovider 2>&1 | tail -3
MP_TRANSPORT=p2p timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py > gpurun_out/mp_f23.log 2>&1; echo "mp rc=$?"
grep -E "MISMATCH|rank .: ok|failures" gpurun_out/mp_f23.log | tail -4
for tr in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516 scripts/table1.py --transport $tr 2>&1 | grep -E "^\||rror"
done
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 4 --steps 20 --warmup 4 --no-e2e --algo allreduce 2>&1 | grep "^{" | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('AR-Adam 4 GPUs', j['value'], j['ms_per_step'], j['roofline']['frac'], j['step_roofline']['frac'])"
timeout 600 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline --algo allreduce 2>&1 | grep "^{" | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('AR-Adam 1 GPU', j['value'], j['ms_per_step'], j['roofline']['frac'], j['step_roofline']['frac'])"
