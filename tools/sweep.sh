#!/bin/bash
# BASELINE configs[4]: flattened parameter sweep, N = 1 and N = 2 (one box)
mkdir -p gpurun_out/sweep
for P in 1000000 16000000 100000000 1000000000; do
  python bench.py --P $P --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sweep/n1_$P.json 2>/dev/null
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus 2 --P $P --steps 50 --warmup 5 --no-e2e > gpurun_out/sweep/n2_$P.json 2>/dev/null
  python - $P <<'PY'
import json, sys
P = int(sys.argv[1])
for n in (1, 2):
    try:
        d = json.loads(open(f"gpurun_out/sweep/n{n}_{P}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(P, n, "fail", e); continue
    m = d["modes"]
    ex = d.get("exchange", {}).get("nvlink", {})
    print(f"P={P:>11,} N={n}: mixed {d['value']:9.1f} steps/s  local {m['all_local']['ms_per_step']*1e3:8.1f} us  "
          f"sync {m['all_sync']['ms_per_step']*1e3:8.1f} us  K13 {d['roofline']['achieved']:6.0f} GB/s ({d['roofline']['frac']:.3f})  "
          f"C2 busbw {ex.get('busbw', float('nan')):6.0f}")
PY
done
