#!/bin/bash
# per-round timing of config 2 at 2 and 4 GPUs: isolated steps vs back to back
cd "$(dirname "$0")/.."
TRN="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
for n in 2 4; do
  npg=$((8 / n)); devs=$(seq -s, 0 $((n - 1)))
  for b in "" "--b2b"; do
    CUDA_VISIBLE_DEVICES=$devs timeout 600 $TRN --nproc-per-node $n --master-port 29671 scripts/round_timing.py \
      --nodes-per-gpu $npg --bucket-params 125000000 --periods 6 $b 2>&1 | grep -E "rounds|rror" | sed "s/^/g$n /"
  done
  CUDA_VISIBLE_DEVICES=$devs NCCL_DEBUG=WARN timeout 600 $TRN --nproc-per-node $n --master-port 29672 scripts/round_timing.py \
      --nodes-per-gpu $npg --bucket-params 125000000 --periods 6 --b2b 2>&1 | grep -E "rounds|rror" | sed "s/^/g$n again /"
done
