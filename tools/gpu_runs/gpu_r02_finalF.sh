# round 2, session 3: last kernel change (NVLS known pass keeps the base lag): single-GPU
# suite, bench N = 4 and N = 2, the real N = 2/4 NVLS / known-pass / adaptive subset
mkdir -p gpurun_out/finalF
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/finalF/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/finalF/pytest_gpu_1.log
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N \
    bench.py --gpus $N > gpurun_out/finalF/bench_n$N.json 2> gpurun_out/finalF/bench_n$N.err; echo "bench N=$N rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print('N=$N', round(d['value'],1), round(1e3*d['ms_per_step'],1), {k:round(1e3*v.get('ms_per_step'),1) for k,v in m.items()}, round(d['e2e']['value'],1), round(1e3*d.get('exchange',{}).get('mean_ms'),1), d['clocks'])" gpurun_out/finalF/bench_n$N.json
done
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "nvls or bsp or symm-adaptive or symm-fused" > gpurun_out/finalF/pytest_multi.log 2>&1; echo multi rc=$?
tail -1 gpurun_out/finalF/pytest_multi.log
