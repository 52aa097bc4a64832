cd $GRAFT_REPO_ROOT
one() {  # label n npg env args
  label=$1; n=$2; npg=$3; envs=$4; shift 4
  out=$(env $envs timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29560+n)) bench.py --gpus $n --steps 8 --warmup 4 --no-e2e --nodes-per-gpu $npg "$@" 2>&1 | grep "^{")
  echo "$out" | python -c "
import sys,json
try:
  j=json.loads(sys.stdin.read()); print('$label G=$n [$envs]', 'ms=%.2f'%j['ms_per_step'], 'sfrac=%.3f'%j['step_roofline']['frac'])
except Exception as e: print('$label G=$n FAILED')"
}
for e in "DG_P2P_PULL=1" "DG_P2P_PULL=0" "DG_P2P_PULL=1 DG_PULL_STREAMS=1"; do
  one config3 2 4 "$e" --topology static_exponential --bucket-params 350000000
  one config3 4 2 "$e" --topology static_exponential --bucket-params 350000000
  one config4 2 4 "$e" --topology aer --algo accum --bucket-params 1300000000
  one config4 4 2 "$e" --topology aer --algo accum --bucket-params 1300000000
done
one config3 4 2 "DG_TRANSPORT=nccl" --topology static_exponential --bucket-params 350000000
one config4 4 2 "DG_TRANSPORT=nccl" --topology aer --algo accum --bucket-params 1300000000
