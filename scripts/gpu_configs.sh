# BASELINE.json configs 2-5 at 1/2/4 GPUs (strong scaling over a fixed node set)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name gpus nodes_per_gpu args...
  name=$1; n=$2; npg=$3; shift 3
  if [ $n -eq 1 ]; then
    out=$(timeout 900 python bench.py --steps 12 --warmup 4 --no-e2e --no-cpu-baseline --nodes-per-gpu $npg "$@" 2>&1 | grep "^{")
  else
    out=$(timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29540+n)) bench.py --gpus $n --steps 12 --warmup 4 --no-e2e --nodes-per-gpu $npg "$@" 2>&1 | grep "^{")
  fi
  echo "$out" | python -c "
import sys,json
try:
  j=json.loads(sys.stdin.read())
  nv=j.get('nvlink') or {}
  print('$name', 'G=$n', 'value=%.4g'%j['value'], 'ms=%.2f'%j['ms_per_step'], 'kfrac=%.3f'%j['roofline']['frac'], 'sfrac=%.3f'%j['step_roofline']['frac'], 'bound_ms=%.2f'%j['step_roofline']['bound_ms_per_step'], 'nvl=%s'%(('%.0f'%nv['achieved']) if nv else '-'))
except Exception as e: print('$name G=$n FAILED', e)
"
}
run config2_opexp_125M 1 8 --topology one_peer_exponential --bucket-params 125000000
run config2_opexp_125M 2 4 --topology one_peer_exponential --bucket-params 125000000
run config2_opexp_125M 4 2 --topology one_peer_exponential --bucket-params 125000000
run config3_static_350M 1 8 --topology static_exponential --bucket-params 350000000
run config3_static_350M 2 4 --topology static_exponential --bucket-params 350000000
run config3_static_350M 4 2 --topology static_exponential --bucket-params 350000000
run config4_aer_1.3B_accum 2 4 --topology aer --algo accum --bucket-params 1300000000
run config4_aer_1.3B_accum 4 2 --topology aer --algo accum --bucket-params 1300000000
run config5_64x125M 4 16 --topology one_peer_exponential --bucket-params 125000000
