cd $GRAFT_REPO_ROOT
for tr in p2p; do
MP_TRANSPORT=$tr timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/mp_parity_main.py 2>&1 | grep -E "MISMATCH|: ok|FAIL" | tail -3
done
sed -n '/^run()/,/^}/p' scripts/gpu_configs.sh > /tmp/run.sh; source /tmp/run.sh
run config3_static_350M 2 4 --topology static_exponential --bucket-params 350000000
run config4_aer_1.3B_accum 2 4 --topology aer --algo accum --bucket-params 1300000000
