#!/bin/bash
# default bench lines at N = 1, 2, 4 (+ the NCCL back end at N = 4 for comparison)
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/n1.json 2> gpurun_out/final/n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N \
    bench.py --gpus $N > gpurun_out/final/n$N.json 2> gpurun_out/final/n$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29529 \
  bench.py --gpus 4 --collective nccl --no-e2e > gpurun_out/final/n4_nccl.json 2> gpurun_out/final/n4_nccl.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29530 \
  bench.py --gpus 4 --impl reference --steps 20 --warmup 2 > gpurun_out/final/n4_ref.json 2> gpurun_out/final/n4_ref.err
python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/final/n1_ref.json 2> gpurun_out/final/n1_ref.err
python - <<'PY'
import json
for f in ("n1", "n2", "n4", "n4_nccl", "n1_ref", "n4_ref"):
    try:
        d = json.loads(open(f"gpurun_out/final/{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "fail", e); continue
    m = d.get("modes", {})
    ex = d.get("exchange", {}).get("nvlink", {})
    print(f"{f:8s} value {d['value']:10.2f} {d['unit']}  ms/step {d['ms_per_step']:.3f}  "
          f"local {m.get('all_local', {}).get('ms_per_step', float('nan')):.3f}  sync {m.get('all_sync', {}).get('ms_per_step', float('nan')):.3f}  "
          f"roof {d.get('roofline', {}).get('frac', float('nan')):.3f}  busbw {ex.get('busbw', float('nan')):.0f}  "
          f"e2e {d.get('e2e', {}).get('value', float('nan')):.1f}  cpu {d.get('cpu_baseline', {}).get('value', float('nan')):.3f} "
          f"cores {d.get('cpu_baseline', {}).get('cores')}  clocks {d.get('clocks', {}).get('sm_mhz')}")
PY
