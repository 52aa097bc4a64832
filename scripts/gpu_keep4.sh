cd $GRAFT_REPO_ROOT
sed -n '/^one()/,/^}/p' scripts/gpu_pull_cmp.sh > /tmp/one.sh; source /tmp/one.sh
for e in "DG_NONE=1" "DG_P2P_KEEP_NC=4" "DG_P2P_KEEP_NC=8"; do
  one config3 2 4 "$e" --topology static_exponential --bucket-params 350000000
done
for e in "DG_P2P_KEEP_NC=4 DG_COOP_MIN_NC=99" ; do
  one config3 2 4 "$e" --topology static_exponential --bucket-params 350000000
done
