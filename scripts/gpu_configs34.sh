cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|: ok|FAIL" | tail -4
sed -n '/^run()/,/^}/p' scripts/gpu_configs.sh > /tmp/run.sh; source /tmp/run.sh
run config3_static_350M 2 4 --topology static_exponential --bucket-params 350000000
run config3_static_350M 4 2 --topology static_exponential --bucket-params 350000000
run config4_aer_1.3B_accum 2 4 --topology aer --algo accum --bucket-params 1300000000
run config4_aer_1.3B_accum 4 2 --topology aer --algo accum --bucket-params 1300000000
run config2_opexp_125M 4 2 --topology one_peer_exponential --bucket-params 125000000
run config5_64x125M 4 16 --topology one_peer_exponential --bucket-params 125000000
