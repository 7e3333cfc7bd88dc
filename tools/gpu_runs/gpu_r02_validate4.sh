# 4-GPU box at HEAD: smoke, the whole GPU suite (single-GPU + real multi-GPU at
# 2 and 4 ranks), default bench lines at N = 1 / 2 / 4, BASELINE configs[4] sweep
echo "HEAD $(cat .git_sha)"; nvidia-smi -L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke rc=$?
timeout 3600 python -m pytest tests -m gpu -v -p no:cacheprovider > gpurun_out/v_pytest_gpu_n4box.log 2>&1; echo pytest rc=$?
echo "HEAD $(cat .git_sha)" >> gpurun_out/v_pytest_gpu_n4box.log; tail -2 gpurun_out/v_pytest_gpu_n4box.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29541"
timeout 600 python bench.py > gpurun_out/v_bench_n1.json 2> gpurun_out/v_bench_n1.err; echo b1 rc=$?
$TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/v_bench_n2.json 2> gpurun_out/v_bench_n2.err; echo b2 rc=$?
$TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/v_bench_n4.json 2> gpurun_out/v_bench_n4.err; echo b4 rc=$?
bash tools/sweep.sh > gpurun_out/v_sweep.txt 2>&1; echo sweep rc=$?
