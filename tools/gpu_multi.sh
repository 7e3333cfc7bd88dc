#!/bin/bash
# multi-GPU checks: tests + bench variants at N ranks
N=${1:-2}
TESTS=${2:-1}
mkdir -p gpurun_out
if [ "$TESTS" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_n$N.log
fi
for C in "symm fused" "symm nccl" "symm p2p" "nccl nccl"; do
  set -- $C
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 100 --warmup 5 --collective $1 --flag-exchange $2 --no-e2e > gpurun_out/bench_n${N}_$1_$2.json 2> gpurun_out/bench_n${N}_$1_$2.err
  echo "bench $1 $2 rc=$?"
  python - "$N" "$1" "$2" <<'PY'
import json, sys
n, c, f = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/bench_n{n}_{c}_{f}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("  no json:", e); sys.exit(0)
m = d["modes"]
ex = d.get("exchange", {})
print(f"  value {d['value']:.1f} steps/s ({d['ms_per_step']:.3f} ms/step, sync_frac {d['observed_sync_frac']:.2f}); "
      f"local {m['all_local']['ms_per_step']:.3f} ms, sync {m['all_sync']['ms_per_step']:.3f} ms; "
      f"roofline {d['roofline']['achieved']:.0f} GB/s ({d['roofline']['frac']:.3f}); "
      f"busbw {ex.get('nvlink', {}).get('busbw', float('nan')):.0f}")
PY
  tail -2 gpurun_out/bench_n${N}_$1_$2.err | grep -v "^$" | grep -iv warn | head -3
done
