#!/bin/bash
# round 2, 2 GPUs: NVLink evidence for the exchange-round kernels (single-process
# probe, hardware counters via ncu on device 0), and the x-row staging variants
# on P2P exchange rounds / the in-place P2P range step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1"
# in-place P2P with the legacy pair kernel writing the publish copy: parity (+fault), DDP
MP_TRANSPORT=p2p MP_D=100003 MP_CHUNK=16384 timeout 900 $TR --master-port 29641 tests/mp_parity_main.py \
   > gpurun_out/r2c_parity_p2p.log 2>&1; echo "parity p2p rc=$?"; grep -E "MISMATCH|in-place" gpurun_out/r2c_parity_p2p.log | head -6
MP_TRANSPORT=p2p MP_D=100003 DG_FAULT_DELAY_US=5000 DG_FAULT_POISON=1 timeout 900 $TR --master-port 29642 \
   tests/mp_parity_main.py > gpurun_out/r2c_parity_p2p_fault.log 2>&1; echo "parity p2p+fault rc=$?"
timeout 900 $TR --master-port 29643 tests/mp_ddp_main.py > gpurun_out/r2c_ddp.log 2>&1; echo "ddp rc=$?"; grep rank gpurun_out/r2c_ddp.log | head -3
for st in 0 2; do
  timeout 300 build/nvl_probe_st$st 125000000 5 > gpurun_out/r2_nvl_probe_st$st.log 2>&1; echo "probe st$st rc=$?"; cat gpurun_out/r2_nvl_probe_st$st.log
done
timeout 300 build/nvl_probe_st0 125000000 1 > gpurun_out/r2_nvl_probe_plain.log 2>&1 && \
timeout 900 ncu --devices 0 --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/r2_nvl_probe_ncu.csv build/nvl_probe_st0 125000000 1 > gpurun_out/r2_nvl_probe_ncu.log 2>&1
echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2_nvl_probe_ncu.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows:
    print(r[0], r[4][:40], r[-3], r[-1])
PY
for v in default libdg_xs_st1; do
  lib=build/variants/$v.so; [ $v = default ] && lib=paper_2410_11998_b200/libdg.so
  for c in 2 3 4; do
    DG_LIB=$lib DG_XSHARE_REMOTE=1 DG_XSHARE_PAIRS=1 timeout 900 $TR --master-port 29631 bench.py --gpus $N --config $c --no-e2e --steps 20 \
      2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v config $c', 'ms', round(j['ms_per_step'],3), 'kfrac', round(j['roofline']['frac'],3), 'step', round(j['step_roofline']['frac'],3), 'nvl(events)', round((j.get('nvlink') or {}).get('achieved') or 0))
"
  done
  DG_LIB=$lib timeout 300 $TR --master-port 29632 scripts/xchg_bw.py --range --transport p2p --tag "$v" 2>&1 | grep -E "^xchg|rror" | head -2
done
timeout 900 $TR --master-port 29644 scripts/ddp_bench.py > gpurun_out/r2c_ddp_bench.log 2>&1; echo "ddp_bench rc=$?"; grep "^|" gpurun_out/r2c_ddp_bench.log
