#!/bin/bash
# One gpurun call: tests, bench, ncu launch list + full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
SMALL="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/small_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
$SMALL > gpurun_out/small_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sgd_kernel -s 4 -c 2 -o gpurun_out/prof_k13 $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
