#!/bin/bash
# 2 GPUs: exchange-round probe incl. the f1 in-place pair kernel, one GPU and both at once
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 build/nvl_probe_st2 125000000 5 2>&1 | tee gpurun_out/r2_nvl_probe_inplace.log
