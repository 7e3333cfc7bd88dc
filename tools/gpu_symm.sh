#!/bin/bash
N=${1:-2}
for U in 0 1 2 4 8; do
  echo "== N=$N SS_SYMM_UNROLL=$U"
  SYMM_ONLY=1 SS_SYMM_UNROLL=$U timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/symm_perf.py 100000000 2>&1 | grep -E "ss_symm_sync|local step"
done
