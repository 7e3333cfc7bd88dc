#!/bin/bash
mkdir -p gpurun_out/final1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final1/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final1/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final1/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final1/smoke.log
timeout 300 python bench.py > gpurun_out/final1/n1.json 2> gpurun_out/final1/n1.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/final1/n1.json').read().strip().splitlines()[-1])
print('N=1', round(d['value']), 'roof', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], 'launches', d['gpu_launches'], 'clk', d['clocks'])" || tail -3 gpurun_out/final1/n1.err
