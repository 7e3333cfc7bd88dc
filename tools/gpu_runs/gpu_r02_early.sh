# exact early vote: parity (colocated on one GPU + real ranks) and A/B timing at N = $1
n=${1:-2}
echo "HEAD $(cat .git_sha) + worktree"; nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29517"
timeout 1500 python -m pytest tests/test_colocated_gpu.py tests/test_parity_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/early_colo.log 2>&1; echo colo rc=$?; tail -3 gpurun_out/early_colo.log
for m in up up-noearly down known; do
  $TR --nproc-per-node $n tools/overlap_timeline.py 100000000 16384 $m 2>&1 | grep -v "OMP_NUM\|^\*\*\*\|^$" > gpurun_out/early_tl_n${n}_$m.txt; echo tl $m rc=$?
done
$TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --no-e2e > gpurun_out/early_bench_n${n}_on.json 2> gpurun_out/early_bench_n${n}_on.err; echo bench on rc=$?
$TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --no-e2e --no-early-vote > gpurun_out/early_bench_n${n}_off.json 2> gpurun_out/early_bench_n${n}_off.err; echo bench off rc=$?
timeout 2000 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "normfirst or adaptive or nansafe or ga or bsp" > gpurun_out/early_multi_n${n}.log 2>&1; echo multi rc=$?; tail -3 gpurun_out/early_multi_n${n}.log
