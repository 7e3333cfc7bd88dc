# round 2, session 3: final bench lines N = 1 and N = 4 at the final tree
mkdir -p gpurun_out/finalH
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/finalH/bench_n1.json 2> gpurun_out/finalH/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/finalH/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('back_to_back'),d['e2e']['value'],d['clocks'],d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 \
  bench.py --gpus 4 > gpurun_out/finalH/bench_n4.json 2> gpurun_out/finalH/bench_n4.err; echo "bench N=4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/finalH/bench_n4.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],{k:round(1e3*v['ms_per_step'],1) for k,v in d['modes'].items()},d['e2e']['value'],d['clocks'])"
