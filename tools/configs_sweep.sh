#!/bin/bash
# BASELINE configs 1-3 at N ranks: model workloads (CUDA-graph mode) and the
# VGG-11 delta sweep (config 2 is "sync-heavy"); one JSON line per run.
N=${1:-4}
OUT=gpurun_out/configs_n$N
mkdir -p $OUT
run() {  # name, args...
  local name=$1; shift
  if [ "$N" = "1" ]; then
    timeout 600 python bench.py --gpus 1 --no-e2e --no-cpu-baseline "$@" > $OUT/$name.json 2> $OUT/$name.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29515 bench.py --gpus $N --no-e2e --no-cpu-baseline "$@" > $OUT/$name.json 2> $OUT/$name.err
  fi
  echo "$name rc=$?"
  python - "$OUT/$name.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print("  no json:", e); sys.exit(0)
c = d["config"]
print(f"  {d['value']:.1f} steps/s ({d['ms_per_step']:.3f} ms/step) delta={c.get('delta')} "
      f"sync_frac={d.get('observed_sync_frac')} roofline={(d.get('roofline') or {}).get('frac')}")
PY
}
run resnet101_graph --workload resnet101 --graph --steps 100 --warmup 10
run transformer_graph --workload transformer --graph --steps 100 --warmup 10
for D in 0 0.05 0.3 1e9; do
  run vgg11_graph_d$D --workload vgg11 --graph --steps 100 --warmup 10 --delta $D --sel-warmup 1
done
