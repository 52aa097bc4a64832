#!/bin/bash
# round 2: NCCL transport exchange bandwidth (2 GPUs), default vs tuned / registered buffers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
run() { local e=(); while [ "$1" != "--" ]; do e+=("$1"); shift; done; shift; env "${e[@]}" DG_DIAG_SKIP_KERNEL=1 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/xchg_bw.py 2>&1 | grep -E "^xchg|rror" | head -3; }
for extra in "" "--range"; do
run DG_X=0 -- $extra --tag default
run DG_NCCL_REGISTER=1 -- $extra --tag register
run NCCL_P2P_NVL_CHUNKSIZE=2097152 -- $extra --tag chunk2M
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 -- $extra --tag p2pch32
run NCCL_P2P_USE_CUDA_MEMCPY=1 -- $extra --tag cudamemcpy
run NCCL_P2P_USE_CUDA_MEMCPY=1 DG_NCCL_REGISTER=1 -- $extra --tag cudamemcpy_reg
run DG_NCCL_REGISTER=1 NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 NCCL_P2P_NVL_CHUNKSIZE=2097152 -- $extra --tag reg_ch32_2M
done
run DG_X=0 -- --chunk 131072000 --tag chunk500MB
run DG_NCCL_REGISTER=1 -- --chunk 131072000 --tag reg_chunk500MB
