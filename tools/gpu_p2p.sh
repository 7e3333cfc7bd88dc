#!/bin/bash
for V in 0 1 2 3; do
  echo "== SS_P2P_VARIANT=$V"
  SYMM_ONLY=1 SS_P2P_VARIANT=$V timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/symm_perf.py 100000000 2>&1 | grep -E "P2P two-shot"
done
