# 4-GPU box: NVLS mean variants, early-vote A/B (timeline + bench) at N = 2 / 4,
# small-P vote timeline, parity (colocated + real ranks) of the worktree
echo "HEAD $(cat .git_sha) + worktree"; nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29523"
timeout 1500 python -m pytest tests/test_colocated_gpu.py tests/test_parity_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/b_colo.log 2>&1; echo colo rc=$?; tail -2 gpurun_out/b_colo.log
bash tools/gpu_runs/gpu_r02_nvls_ab.sh > gpurun_out/b_nvls_ab.txt 2>&1; echo nvls rc=$?
for n in 2 4; do
  for m in up up-noearly; do
    $TR --nproc-per-node $n tools/overlap_timeline.py 100000000 16384 $m 2>&1 | grep -v "OMP_NUM\|^\*\*\*\|^$" > gpurun_out/b_tl_n${n}_$m.txt; echo tl $n $m rc=$?
  done
  $TR --nproc-per-node $n tools/local_timeline.py 1000000 50 2>&1 | grep -v "OMP_NUM\|^\*\*\*\|^$" > gpurun_out/b_local_n${n}_1m.txt; echo local $n rc=$?
  $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --no-e2e > gpurun_out/b_bench_n${n}_on.json 2> gpurun_out/b_bench_n${n}_on.err; echo bench on rc=$?
  $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --no-e2e --no-early-vote > gpurun_out/b_bench_n${n}_off.json 2> gpurun_out/b_bench_n${n}_off.err; echo bench off rc=$?
done
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "normfirst or adaptive or nansafe or ga or bsp" > gpurun_out/b_multi.log 2>&1; echo multi rc=$?; tail -3 gpurun_out/b_multi.log
