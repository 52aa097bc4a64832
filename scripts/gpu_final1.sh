#!/bin/bash
# 1 GPU: full GPU suite (multi-GPU tests skip), smoke, default bench, reference arm, headline ncu launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g1.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_g1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final_bench_g1.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo "ref rc=$?"
grep "^{" gpurun_out/final_bench_g1.log | head -c 1500; echo
grep "^{" gpurun_out/final_bench_ref.log | head -c 600; echo
