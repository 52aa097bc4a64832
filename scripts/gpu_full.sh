cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_g1.log 2>&1; echo "bench1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n > gpurun_out/bench_g$n.log 2>&1; echo "bench$n rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
for f in bench_g1 bench_g2 bench_g4 bench_ref; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json; j=json.loads(sys.stdin.read())
print('$f', '%.4g'%j['value'], 'ms/step', round(j['ms_per_step'],3), 'kfrac', j.get('roofline',{}).get('frac'), 'sfrac', (j.get('step_roofline') or {}).get('frac'), 'e2e', '%.3g'%j['e2e']['value'], 'clk', (j.get('clocks') or {}).get('sm_mhz'), (j.get('clocks') or {}).get('reasons'))"; done
