cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|: ok|FAIL" | tail -4
sed -n '/^one()/,/^}/p' scripts/gpu_pull_cmp.sh > /tmp/one.sh; source /tmp/one.sh
for e in "DG_NONE=1" "DG_P2P_SPLIT=1"; do
  one config3 2 4 "$e" --topology static_exponential --bucket-params 350000000
  one config3 4 2 "$e" --topology static_exponential --bucket-params 350000000
  one config4 2 4 "$e" --topology aer --algo accum --bucket-params 1300000000
  one config4 4 2 "$e" --topology aer --algo accum --bucket-params 1300000000
  one config2 4 2 "$e" --topology one_peer_exponential --bucket-params 125000000
done
