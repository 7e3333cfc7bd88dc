#!/bin/bash
# BASELINE configs[4]: flattened parameter sweep 1M-1B, forced all-local / all-sync
# and the 50% mix, at N in $NS (default "1 2 4"). P <= 2M replays one CUDA graph
# per step at N = 1 (host-bound there); everything else uses the host launch path
# (prepared step plans + programmatic dependent launch: faster than graph
# replays from 4M up, profiles/r02_plan/, profiles/r02_pdl/).
NS=${NS:-"1 2 4"}
SIZES=${SIZES:-"1000000 4000000 16000000 64000000 100000000 256000000 1000000000"}
mkdir -p gpurun_out/sweep
for P in $SIZES; do
  # graph replay only at N = 1 and P <= 2M: at N > 1 eager cooperative launches
  # measured faster (profiles/r02_small_p/max_blocks_n2.txt)
  G=""; [ "$P" -le 2000000 ] && G="--graph"
  # no per-launch events up to 16M (they cost a few us per step)
  E=""; [ "$P" -le 16000000 ] && E="--no-kernel-events"
  for N in $NS; do
    if [ "$N" = "1" ]; then
      timeout 600 python bench.py --P $P --steps 50 --warmup 5 --no-e2e --no-cpu-baseline ${G:-$E} \
        > gpurun_out/sweep/n1_$P.json 2> gpurun_out/sweep/n1_$P.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 2952$N bench.py --gpus $N --P $P --steps 50 --warmup 5 --no-e2e --no-replay $E \
        > gpurun_out/sweep/n${N}_$P.json 2> gpurun_out/sweep/n${N}_$P.err
    fi
  done
  python - $P "$NS" <<'PY'
import json, sys
P = int(sys.argv[1])
for n in sys.argv[2].split():
    try:
        d = json.loads(open(f"gpurun_out/sweep/n{n}_{P}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(P, n, "fail", e); continue
    m = d["modes"]
    ex = d.get("exchange", {}).get("nvlink", {})
    print(f"P={P:>13,} N={n}: mixed {d['value']:9.1f} steps/s  local {m['all_local']['ms_per_step']*1e3:8.1f} us  "
          f"sync {m['all_sync']['ms_per_step']*1e3:8.1f} us  K13 {d['roofline']['achieved']:6.0f} GB/s ({d['roofline']['frac']:.3f})  "
          f"C2 busbw {ex.get('busbw', float('nan')):6.0f}  {d['config'].get('launch', '')[:9]}")
PY
done
