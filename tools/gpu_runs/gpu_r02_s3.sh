# round 2, session 3: rebuilt tree on one 4-GPU box -- smoke, single-GPU suite,
# default bench line, then the NVLS decomposition probe at N = 4
mkdir -p gpurun_out/s3
echo "HEAD $(cat .git_sha)"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/s3/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/s3/pytest_gpu_1.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/s3/bench_n1.json 2> gpurun_out/s3/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/s3/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr=127.0.0.1 --master-port=29531 \
  tools/nvls_split_probe.py 100000000 > gpurun_out/s3/nvls_split_n4.txt 2>&1; echo probe rc=$?
grep -v Warning gpurun_out/s3/nvls_split_n4.txt | tail -30
