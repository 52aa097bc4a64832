#!/bin/bash
# round 2, 1 GPU: ONE compute-sanitizer tool per gpurun call (B200_PROFILING.md):
#   bash scripts/gpu_r2_sanitize.sh memcheck|racecheck|synccheck|initcheck
# on the small shapes: every topology x algorithm through the default
# (x-sharing) kernel, the legacy/pingpong and TMA paths, CUDA-graph ranges.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tool=${1:-memcheck}
log=gpurun_out/r2_sanitize_$tool.log
: > $log
run() {
  echo "== $*" >> $log
  env "$@" >> $log 2>&1
  echo "rc=$?" >> $log
}
CS="compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20"
run timeout 1500 $CS python tests/engine_parity_main.py 1003
run DG_XSHARE=0 DG_PINGPONG_MIN_NC=1 timeout 1500 $CS python tests/engine_parity_main.py 1003
if [ "$tool" != "racecheck" ]; then
  run DG_XSHARE=0 DG_TMA=2 DG_PINGPONG_MIN_NC=0 timeout 1500 $CS python tests/engine_parity_main.py 1003
  run timeout 1500 $CS python tests/graph_parity_main.py 1003
fi
grep -E "^==|^rc=|ERROR SUMMARY|RACECHECK SUMMARY|^ok|mismatch" $log
