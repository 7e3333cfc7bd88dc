# round 2, session 3: headline run without per-launch events (back-to-back steps);
# bench at N = 1 and N = 2, single-GPU suite at the final tree
mkdir -p gpurun_out/finalG
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/finalG/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/finalG/pytest_gpu_1.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/finalG/bench_n1.json 2> gpurun_out/finalG/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/finalG/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms_mean'],d['e2e']['value'],d['clocks'],d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 \
  bench.py --gpus 2 > gpurun_out/finalG/bench_n2.json 2> gpurun_out/finalG/bench_n2.err; echo "bench N=2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/finalG/bench_n2.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],{k:round(1e3*v['ms_per_step'],1) for k,v in d['modes'].items()},d['e2e']['value'])"
