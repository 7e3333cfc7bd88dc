# round 2, session 3, final 4-GPU pass at HEAD: the real multi-GPU suite, default
# bench lines at N = 2 / 4, and the configs[4] size sweep (1M-100M, N = 1 / 2 / 4)
mkdir -p gpurun_out/finalB
echo "HEAD $(cat .git_sha)"; nvidia-smi -L
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N \
    bench.py --gpus $N > gpurun_out/finalB/bench_n$N.json 2> gpurun_out/finalB/bench_n$N.err; echo "bench N=$N rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(d['value'], d['ms_per_step'], {k:v.get('ms_per_step') for k,v in m.items()}, d['e2e']['value'], d.get('exchange',{}).get('mean_ms'))" gpurun_out/finalB/bench_n$N.json
done
SIZES="1000000 4000000 16000000 64000000 100000000" bash tools/sweep.sh 2>&1 | grep "P=" > gpurun_out/finalB/sweep.txt
mv gpurun_out/sweep gpurun_out/finalB/ 2>/dev/null
cat gpurun_out/finalB/sweep.txt
timeout 3000 python -m pytest tests/test_multigpu.py -v -p no:cacheprovider > gpurun_out/finalB/pytest_n4.log 2>&1; echo multi rc=$?
echo "HEAD $(cat .git_sha)" >> gpurun_out/finalB/pytest_n4.log
tail -3 gpurun_out/finalB/pytest_n4.log
