cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cmd="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $cmd > gpurun_out/plain_launches.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $cmd > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 1200 bash scripts/gpu_profile.sh headline - 
timeout 900 bash scripts/gpu_profile.sh static_pp - --topology static_exponential
timeout 900 bash scripts/gpu_profile.sh aer_accum - --topology aer --algo accum
