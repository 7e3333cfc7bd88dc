#!/bin/bash
# multi-GPU checks: tests + 2-rank bench variants
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_n$N.log
for C in "symm nccl" "symm p2p" "nccl nccl"; do
  set -- $C
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 100 --warmup 5 --collective $1 --flag-exchange $2 --no-e2e > gpurun_out/bench_n${N}_$1_$2.json 2> gpurun_out/bench_n${N}_$1_$2.err
  echo "bench $1 $2 rc=$?"; tail -c 1500 gpurun_out/bench_n${N}_$1_$2.json; tail -3 gpurun_out/bench_n${N}_$1_$2.err
done
