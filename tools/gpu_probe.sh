#!/bin/bash
mkdir -p gpurun_out/probe
timeout 240 ./tools/nvlink_probe > gpurun_out/probe/nvlink_probe.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/probe/nvlink_probe.txt
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  tools/overlap_timeline.py 100000000 16384 > gpurun_out/probe/timeline_n2.txt 2>&1; echo "timeline rc=$?"
grep -v -i warn gpurun_out/probe/timeline_n2.txt | tail -40
