#!/bin/bash
# One gpurun --gpus 2 call: GPU tests (incl. N=2 multi-GPU), smoke, bench N=1 and N=2.
mkdir -p gpurun_out/verify
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/verify/nvsmi.txt
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/verify/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/verify/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/verify/smoke.log
timeout 300 python bench.py > gpurun_out/verify/n1.json 2> gpurun_out/verify/n1.err; echo "bench n1 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --gpus 2 > gpurun_out/verify/n2.json 2> gpurun_out/verify/n2.err; echo "bench n2 rc=$?"
for f in n1 n2; do python -c "
import json,sys
d=json.loads(open('gpurun_out/verify/$f.json').read().strip().splitlines()[-1])
m=d.get('modes',{})
print('$f', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'local', m.get('all_local',{}).get('ms_per_step'), 'sync', m.get('all_sync',{}).get('ms_per_step'), 'roof', round(d['roofline']['frac'],3), 'e2e', d.get('e2e',{}).get('value'), 'clk', d.get('clocks'))
" || tail -5 gpurun_out/verify/$f.err; done
