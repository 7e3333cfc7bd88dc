#!/bin/bash
mkdir -p gpurun_out/lt
for A in "1000000 1" "1000000 50" "100000000 1" "100000000 20"; do
  set -- $A
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
    tools/local_timeline.py $1 $2 2>&1 | grep -E "rank|skew" | sed "s/^/P=$1 b2b=$2 /"
done
