# round 2, one GPU: ncu launch list of the default bench command, ncu --set full of
# K13 (the N = 1 roofline kernel) and of the one-launch step kernel through a
# world-1 group (update-first local step; norm-first known-pass sync step).
# Every ncu command runs only after the same command exited 0 without ncu.
set -x
SMALL="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-replay"
$SMALL > gpurun_out/n_small_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launches.csv $SMALL > gpurun_out/n_ncu_launches.log 2>&1; echo "launches rc=$?"
$SMALL > gpurun_out/n_small_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sgd_kernel -s 4 -c 1 -o gpurun_out/n_prof_k13 $SMALL > gpurun_out/n_ncu_k13.log 2>&1; echo "k13 rc=$?"
S1="python tools/step_kernel_solo.py update_first local"
$S1 > gpurun_out/n_solo_uf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/n_prof_step_uf $S1 > gpurun_out/n_ncu_step_uf.log 2>&1; echo "step uf rc=$?"
S2="python tools/step_kernel_solo.py norm_first sync"
$S2 > gpurun_out/n_solo_nf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/n_prof_step_known $S2 > gpurun_out/n_ncu_step_known.log 2>&1; echo "step known rc=$?"
