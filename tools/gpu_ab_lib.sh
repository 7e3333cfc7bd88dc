#!/bin/bash
# same-box A/B of two library builds at N=2 (SS_LIB_PATH): local / sync / mixed
N=${1:-2}
for L in new prev new prev; do
  if [ $L = prev ]; then export SS_LIB_PATH=$PWD/paper_2307_07950_b200/_lib/libselsync_b200_prev.so; else unset SS_LIB_PATH; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 \
    bench.py --gpus $N --steps 200 --warmup 10 --no-e2e > /tmp/ab.json 2> /tmp/ab.err
  python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); m=d['modes']
print('N=$N lib $L: mixed', round(d['value']), 'ms', round(d['ms_per_step'],4), 'local', round(m['all_local']['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms_mean'],4), 'sync', round(m['all_sync']['ms_per_step'],4))" || tail -3 /tmp/ab.err
done
