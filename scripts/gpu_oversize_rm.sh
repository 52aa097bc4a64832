#!/bin/bash
# 4 GPUs: multi-GPU parity incl. static exponential over 64 nodes (oversize plans), then f4 calibration
cd "$(dirname "$0")/.."
for tr in p2p nccl; do
  echo "== mp_parity $tr"
  MP_TRANSPORT=$tr timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|static_exponential\(64|rror|rank 0: ok" | head -12
done
echo "== rm_calibrate"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 scripts/rm_calibrate.py 2>&1 | grep -v Warning | tail -22
