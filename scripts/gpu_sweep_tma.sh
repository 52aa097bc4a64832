cd $GRAFT_REPO_ROOT
for args in "--topology static_exponential" "--topology aer --algo accum"; do
  echo "== sweep $args"
  for env in "DG_TMA=0 DG_COOP_MIN_NC=99" "DG_TMA=2" "DG_TMA=0"; do
    echo "-- $env"; SWEEP_ENV="$env" timeout 900 python scripts/sweep.py $args 2>&1
  done
done
