#!/bin/bash
# VGG-11 (BASELINE config 2) at delta = 0 (every step sync), N = 2, graph mode: known-sync pass on / off
mkdir -p gpurun_out/vgg
for K in 1 0; do
  SS_KNOWN_SYNC=$K timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 2957$K bench.py --gpus 2 --no-e2e --no-cpu-baseline --workload vgg11 --graph --steps 100 --warmup 10 \
    --delta 0 --sel-warmup 1 > gpurun_out/vgg/n2_d0_k$K.json 2> gpurun_out/vgg/n2_d0_k$K.err
  python -c "
import json; d=json.loads(open('gpurun_out/vgg/n2_d0_k$K.json').read().strip().splitlines()[-1]); print('vgg11 N=2 delta=0 known-sync $K:', round(d['value'],1), 'steps/s', round(d['ms_per_step'],4), 'ms/step')" || tail -3 gpurun_out/vgg/n2_d0_k$K.err
done
