# round 2 on a 4-GPU box: the real multi-GPU suite (2- and 4-rank cases), the
# NVLink mean vs NCCL / torch symm_mem, local-step vote timeline at small P,
# default bench lines at N = 2 and 4
echo "HEAD $(cat .git_sha)"; nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29511"
$TR --nproc-per-node 4 tools/symm_perf.py 100000000 > gpurun_out/symm_perf_n4.txt 2>&1; echo symm4 rc=$?
NCCL_ALGO=NVLS SYMM_NCCL_ONLY=1 $TR --nproc-per-node 4 tools/symm_perf.py 100000000 > gpurun_out/symm_perf_n4_ncclnvls.txt 2>&1; echo symm4nvls rc=$?
for n in 2 4; do for p in 1000000 4000000; do
  $TR --nproc-per-node $n tools/local_timeline.py $p 1 > gpurun_out/local_tl_n${n}_p${p}.txt 2>&1; echo tl $n $p rc=$?
done; done
$TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2 rc=$?
$TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo bench4 rc=$?
timeout 3000 python -m pytest tests/test_multigpu.py -v -p no:cacheprovider > gpurun_out/pytest_n4.log 2>&1; echo pytest rc=$?
echo "HEAD $(cat .git_sha)" >> gpurun_out/pytest_n4.log
tail -5 gpurun_out/pytest_n4.log
