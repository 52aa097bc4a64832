cd $GRAFT_REPO_ROOT
N=$1
run() { env "$@" timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 scripts/round_timing.py $EXTRA 2>&1 | grep -E "^\[|Error|error|WARN" | head -4; }
EXTRA="--periods 1" run DG_DIAG_SKIP_KERNEL=1
EXTRA="--periods 1 --chunk 26214400" run DG_DIAG_SKIP_KERNEL=1
EXTRA="--periods 1 --chunk 26214400" run DG_DIAG_SKIP_KERNEL=1 NCCL_P2P_NVL_CHUNKSIZE=4194304
EXTRA="--periods 1 --chunk 26214400" run DG_DIAG_SKIP_KERNEL=1 NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
EXTRA="--periods 1 --chunk 26214400" run DG_DIAG_SKIP_KERNEL=1 NCCL_P2P_USE_CUDA_MEMCPY=1 NCCL_DEBUG=WARN
EXTRA="--periods 1 --chunk 26214400" run NCCL_P2P_NVL_CHUNKSIZE=4194304
