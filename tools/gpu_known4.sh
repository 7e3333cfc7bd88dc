#!/bin/bash
# known-sync pass at N=4 (NVLS mean): parity subset + default bench
mkdir -p gpurun_out/known4
timeout 400 python -m pytest tests/test_multigpu.py -m gpu -q -x \
  -k "(n4_mixed and (symm-fused or symm-normfirst)) or (large and bsp)" > gpurun_out/known4/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/known4/pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 \
  bench.py --gpus 4 > gpurun_out/known4/n4.json 2> gpurun_out/known4/n4.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/known4/n4.json').read().strip().splitlines()[-1]); m=d['modes']
print('N=4: mixed', round(d['value']), 'ms', round(d['ms_per_step'],4), 'local', round(m['all_local']['ms_per_step'],4), 'sync(delta=0)', round(m['all_sync']['ms_per_step'],4), 'collective', d['config']['collective'], 'e2e', d.get('e2e',{}).get('value'))" || tail -3 gpurun_out/known4/n4.err
