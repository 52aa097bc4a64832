#!/bin/bash
# round 2, 4 GPUs: benches of configs 2 and 4 with the final kernel rules at
# N=4, config 2 at N=2, per-round timing of config 2 at 2 and 4 GPUs with the
# exchange-round alternatives.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for c in 2 4; do
  timeout 900 $TRN --nproc-per-node 4 --master-port 29664 bench.py --gpus 4 --config $c > gpurun_out/r2i_bench_g4_c$c.log 2>&1; echo "bench g4 config $c rc=$?"
  grep "^{" gpurun_out/r2i_bench_g4_c$c.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l)
    print('g4 config $c', 'value %.4e'%j['value'], 'ms', round(j['ms_per_step'],3), 'bound', round(j['step_roofline']['bound_ms_per_step'],3), 'step', round(j['step_roofline']['frac'],3), 'kfrac', round(j['roofline']['frac'],3), 'nvl', round((j.get('nvlink') or {}).get('achieved') or 0), j['clocks'])
"
done
for n in 2 4; do
  npg=$((8 / n))
  devs=$(seq -s, 0 $((n - 1)))
  for env in "DG_X=0" "DG_P2P_KEEP_NC=1" "DG_P2P_PULL=2" "DG_XSHARE_PAIRS=1" "DG_XSHARE_REMOTE=1"; do
    env CUDA_VISIBLE_DEVICES=$devs $env timeout 600 $TRN --nproc-per-node $n --master-port 29665 scripts/round_timing.py \
      --nodes-per-gpu $npg --bucket-params 125000000 2>&1 | grep -E "rounds|rror" | sed "s/^/g$n config2 /"
  done
done
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TRN --nproc-per-node 2 --master-port 29666 bench.py --gpus 2 --config 2 > gpurun_out/r2i_bench_g2_c2.log 2>&1; echo "bench g2 config 2 rc=$?"
grep "^{" gpurun_out/r2i_bench_g2_c2.log | head -c 700; echo
