#!/bin/bash
# small-P N=1: K13 unroll (SS_SGD_VARIANT -> fewer, fatter blocks) at 1M / 4M / 16M, graph mode
for P in 1000000 4000000 16000000; do for V in 0 2 4 0; do
  SS_SGD_VARIANT=$V timeout 200 python bench.py --P $P --graph --steps 400 --warmup 20 --no-cpu-baseline --no-e2e > /tmp/b.json 2>/tmp/b.err
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); m=d['modes']
print('P $P variant $V: local us', round(1e3*m['all_local']['ms_per_step'],2), 'sync us', round(1e3*m['all_sync']['ms_per_step'],2))" || tail -3 /tmp/b.err
done; done
