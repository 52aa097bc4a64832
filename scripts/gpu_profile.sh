# usage: bash scripts/gpu_profile.sh <tag> <env-assignments|-> <bench args...>
# plain run first (must exit 0), then one ncu --set full capture of the fused
# kernel; the report is exported to text (raw metrics, details, source) so the
# results fit through gpurun's 64 MiB return limit.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=$1; shift; envs=$1; shift
[ "$envs" = "-" ] && envs=""
cmd="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $*"
env $envs timeout 300 $cmd > gpurun_out/plain_$tag.log 2>&1 && \
env $envs timeout 900 ncu --set full --clock-control none --import-source on -k regex:gossip_adam -s 2 -c 1 \
    -o /tmp/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
rc=$?
if [ -f /tmp/prof_$tag.ncu-rep ]; then
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/details_$tag.txt 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>&1
  sz=$(stat -c %s /tmp/prof_$tag.ncu-rep)
  [ "$sz" -lt 15000000 ] && cp /tmp/prof_$tag.ncu-rep gpurun_out/
fi
echo "$tag rc=$rc"
