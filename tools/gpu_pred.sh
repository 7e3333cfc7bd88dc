#!/bin/bash
# adaptive-order predictor: parity of the adaptive cases + the default bench at N ranks
N=${1:-2}
mkdir -p gpurun_out/pred
timeout 600 python -m pytest tests/test_multigpu.py tests/test_parity_gpu.py -m gpu -q -x -k "adaptive" > gpurun_out/pred/pytest_n$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pred/pytest_n$N.log
for i in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$i \
    bench.py --gpus $N --steps 200 --warmup 10 --no-e2e > gpurun_out/pred/n${N}_$i.json 2> gpurun_out/pred/n${N}_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/pred/n${N}_$i.json').read().strip().splitlines()[-1]); m=d['modes']
print('N=$N adaptive(2-bit history): mixed', round(d['value']), 'ms', round(d['ms_per_step'],4), 'sync_frac', d['observed_sync_frac'], 'local', round(m['all_local']['ms_per_step'],4), 'sync', round(m['all_sync']['ms_per_step'],4))" || tail -3 gpurun_out/pred/n${N}_$i.err
done
