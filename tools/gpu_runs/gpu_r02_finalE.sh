# round 2, session 3: per-pass mean lag (known pass x3/4, norm-first x3/2) -- parity
# (single-GPU suite incl. colocated W = 2/4/8, real N = 2/4 subset) and the bench at N = 2 / 4
mkdir -p gpurun_out/finalE
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/finalE/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/finalE/pytest_gpu_1.log
for rep in 1 2; do for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N \
    bench.py --gpus $N > gpurun_out/finalE/bench_n${N}_$rep.json 2> gpurun_out/finalE/bench_n${N}_$rep.err; echo "bench N=$N rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print('N=$N', round(d['value'],1), round(1e3*d['ms_per_step'],1), {k:round(1e3*v.get('ms_per_step'),1) for k,v in m.items()}, round(d['e2e']['value'],1), round(1e3*d.get('exchange',{}).get('mean_ms'),1))" gpurun_out/finalE/bench_n${N}_$rep.json
done; done
timeout 1800 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "symm-normfirst or symm-adaptive or symm-nansafe or adaptive or norm_first or bsp or nan_safe" > gpurun_out/finalE/pytest_multi.log 2>&1; echo multi rc=$?
tail -3 gpurun_out/finalE/pytest_multi.log
