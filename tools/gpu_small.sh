#!/bin/bash
# small-P latency at N=1: graph-mode bench + ncu launch list (kernel durations)
mkdir -p gpurun_out/small
for P in 1000000 4000000; do
  timeout 200 python bench.py --P $P --graph --steps 400 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/small/b_$P.json 2> gpurun_out/small/b_$P.err; echo "bench $P rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/small/b_$P.json').read().strip().splitlines()[-1]); m=d['modes']
print('$P', round(d['value']), 'local us', round(1e3*m['all_local']['ms_per_step'],2), 'sync us', round(1e3*m['all_sync']['ms_per_step'],2), 'kernel', d['roofline'].get('kernel_ms_mean'))"
done
timeout 200 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/small/launches_1M.csv \
  python bench.py --P 1000000 --graph --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/small/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/small/launches_1M.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(list); grid = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    if r[mi] == "gpu__time_duration.sum": agg[r[ki][:90]].append(float(r[vi].replace(",", "")))
    elif r[mi] == "launch__grid_size": grid[r[ki][:90]] = r[vi]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):5d} x {sum(v)/len(v):10.1f} (min {min(v):.1f})  grid {grid.get(k)}  {k}")
PY
