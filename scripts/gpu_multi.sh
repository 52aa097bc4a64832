cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
export NCCL_DEBUG=WARN
for tr in p2p nccl; do
MP_TRANSPORT=$tr timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py > gpurun_out/mp_parity_$1_$tr.log 2>&1; echo "mp $tr rc=$?" >> gpurun_out/mp_parity_$1_$tr.log
grep -E "MISMATCH|ok|rc=|rror" gpurun_out/mp_parity_$1_$tr.log | tail -5
done
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29514 scripts/round_timing.py --periods 1 2>&1 | grep -E "^\[|rror"
DG_TRANSPORT=nccl timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29515 scripts/round_timing.py --periods 1 --chunk 26214400 2>&1 | grep -E "^\[|rror"
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $1 --steps 30 --warmup 4 --e2e-steps 2 > gpurun_out/bench_g$1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_g$1.log
grep -E "^\{" gpurun_out/bench_g$1.log | python -c "import sys,json; [print(json.dumps({k:j[k] for k in ('value','ms_per_step','n_gpus')}), json.dumps(j['roofline']['frac']), json.dumps(j['step_roofline'])) for j in map(json.loads, sys.stdin)]"
tail -3 gpurun_out/bench_g$1.log
