cd $GRAFT_REPO_ROOT
for args in "" "--topology static_exponential" "--topology aer --algo accum"; do
  echo "== sweep $args"; timeout 900 python scripts/sweep.py $args 2>&1 | grep -v waves
done
