#!/bin/bash
mkdir -p gpurun_out/final2
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 4 > gpurun_out/final2/n4.json 2> gpurun_out/final2/n4.err; echo "bench n4 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/final2/n4.json').read().strip().splitlines()[-1])
m=d.get('modes',{})
print('n4', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'local', m.get('all_local',{}).get('ms_per_step'), 'sync', m.get('all_sync',{}).get('ms_per_step'), 'roof', round(d['roofline']['frac'],3), 'busbw', d.get('exchange',{}).get('nvlink',{}).get('busbw'), 'e2e', d.get('e2e',{}).get('value'), 'clk', d.get('clocks'))
" || tail -5 gpurun_out/final2/n4.err
