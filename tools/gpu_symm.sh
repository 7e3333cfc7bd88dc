#!/bin/bash
N=${1:-2}
for G in 0 296 148; do
  echo "== SS_SYMM_GRID=$G"
  SS_SYMM_GRID=$G timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/symm_perf.py 100000000 2>&1 | grep -vE "Warning|warn|OMP_NUM|\*\*\*\*|^$"
done
