#!/bin/bash
# ncu --set full of the known-sync pass (world-1 group, delta = 0, norm_first order) + the plain timing
mkdir -p gpurun_out/kncu
timeout 120 python tools/step_kernel_solo.py norm_first sync > gpurun_out/kncu/plain.log 2>&1; echo "plain rc=$?"; grep order= gpurun_out/kncu/plain.log
SS_KNOWN_SYNC=0 timeout 120 python tools/step_kernel_solo.py norm_first sync > gpurun_out/kncu/plain_off.log 2>&1; echo "plain(off) rc=$?"; grep order= gpurun_out/kncu/plain_off.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/kncu/known_sync \
  python tools/step_kernel_solo.py norm_first sync > gpurun_out/kncu/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py --rep gpurun_out/kncu/known_sync.ncu-rep --out gpurun_out/kncu/summary --P 100000000 --alg-bytes 2800000000 2>&1 | tail -20
