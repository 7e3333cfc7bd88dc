# round 2, session 3: prepared step plans (ss_step_plan_*): single-GPU suite, N = 2
# multi-GPU subset, small-P eager steps at N = 1 / 2, the default N = 1 bench line
mkdir -p gpurun_out/plan
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/plan/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/plan/pytest_gpu_1.log
sh1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.2f us'%(1e3*d['ms_per_step']), 'local %.2f'%(1e3*m['all_local']['ms_per_step']), 'sync %.2f'%(1e3*m['all_sync']['ms_per_step']))" "$@"; }
for P in 1000 1000000 4000000 16000000; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --P $P --steps 300 --warmup 20 --no-e2e --no-cpu-baseline --no-replay --no-kernel-events \
    > gpurun_out/plan/n1_${P}.json 2>gpurun_out/plan/n1_${P}.err
  sh1 gpurun_out/plan/n1_${P}.json "N=1 P=$P eager"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
    bench.py --gpus 2 --P $P --steps 300 --warmup 20 --no-e2e --no-replay --no-kernel-events > gpurun_out/plan/n2_${P}.json 2>gpurun_out/plan/n2_${P}.err
  sh1 gpurun_out/plan/n2_${P}.json "N=2 P=$P eager"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/plan/bench_n1.json 2> gpurun_out/plan/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/plan/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "symm-fused or symm-adaptive or update_first or adaptive or bsp or ga or nan" > gpurun_out/plan/pytest_multi.log 2>&1; echo multi rc=$?
tail -3 gpurun_out/plan/pytest_multi.log
