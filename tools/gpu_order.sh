#!/bin/bash
# order / tile sweep of the one-launch symmetric step at N ranks
N=${1:-2}
TEST=${2:-0}
mkdir -p gpurun_out
if [ "$TEST" = "1" ]; then
timeout 1200 python -m pytest tests/test_multigpu.py -x -q -k "symm or nan" > gpurun_out/pytest_mg_n$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_mg_n$N.log
fi
# ORDERS: comma-separated "order:tile" pairs
IFS=, read -ra PAIRS <<< "${ORDERS:-update_first:16384,norm_first:8192,norm_first:16384,norm_first:32768,adaptive:16384}"
for OT in "${PAIRS[@]}"; do
  set -- ${OT/:/ }
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 100 --warmup 5 --order $1 --tile $2 --no-e2e > gpurun_out/bench_n${N}_$1_$2.json 2> gpurun_out/bench_n${N}_$1_$2.err
  echo "order $1 tile $2 rc=$?"
  python - "$N" "$1" "$2" <<'PY'
import json, sys
n, o, t = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/bench_n{n}_{o}_{t}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("  no json:", e); sys.exit(0)
m = d["modes"]
print(f"  value {d['value']:.1f} steps/s ({d['ms_per_step']:.3f} ms/step, sync_frac {d['observed_sync_frac']:.2f}); "
      f"local {m['all_local']['ms_per_step']:.3f} ms, sync {m['all_sync']['ms_per_step']:.3f} ms")
PY
  grep -iE "error|Traceback" gpurun_out/bench_n${N}_$1_$2.err | head -3
done
