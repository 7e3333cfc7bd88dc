#!/bin/bash
# known-sync pass: parity (N=2 + single rank) and bench A/B (SS_KNOWN_SYNC) at N=2
mkdir -p gpurun_out/known
timeout 500 python -m pytest tests/test_multigpu.py -m gpu -q -x \
  -k "((symm-fused or symm-normfirst or symm-adaptive) and not grads) or (large and (norm_first or adaptive or bsp)) or nan" \
  > gpurun_out/known/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -3 gpurun_out/known/pytest_multi.log
timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_bounds_gpu.py -m gpu -q -x -k "symmetric or trace or one_launch or captured or async" \
  > gpurun_out/known/pytest_single.log 2>&1; echo "pytest single rc=$?"; tail -3 gpurun_out/known/pytest_single.log
for K in 1 0; do
  SS_KNOWN_SYNC=$K timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$K \
    bench.py --gpus 2 --steps 200 --warmup 10 --no-e2e > gpurun_out/known/n2_k$K.json 2> gpurun_out/known/n2_k$K.err
  python -c "
import json; d=json.loads(open('gpurun_out/known/n2_k$K.json').read().strip().splitlines()[-1]); m=d['modes']
print('N=2 known-sync $K: mixed', round(d['value']), 'ms', round(d['ms_per_step'],4), 'local', round(m['all_local']['ms_per_step'],4), 'sync(delta=0)', round(m['all_sync']['ms_per_step'],4))" || tail -3 gpurun_out/known/n2_k$K.err
done
