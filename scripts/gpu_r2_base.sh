#!/bin/bash
# round 2, 1 GPU: full GPU suite (T=100 full-size parity), smoke, default bench
# (config 3), reference arm, then the ncu launch list and one --set full capture
# of the x-sharing kernel on the same (short) bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_g1.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_g1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2_bench_g1.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
grep "^{" gpurun_out/r2_bench_g1.log | head -c 3000; echo
grep "^{" gpurun_out/r2_bench_ref.log | head -c 800; echo
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_config3.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 $CMD > gpurun_out/r2_short2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xshare -s 3 -c 1 \
    -o gpurun_out/r2_config3_full $CMD > gpurun_out/r2_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/r2_ncu_full.log
