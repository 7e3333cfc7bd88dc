# round 2, session 3: one release fence per multi-peer post (relaxed sys stores after it),
# single-block reductions without the partials round trip, K2 returns the vote
mkdir -p gpurun_out/fence
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/fence/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/fence/pytest_gpu_1.log
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N"
  for P in 1000 1000000; do
    echo "== N=$N P=$P"; timeout 300 $TR tools/local_timeline.py $P 8 2>/dev/null | grep "^rank"
  done
  ORDERS=update_first MAX_BLOCKS=0 timeout 300 $TR tools/small_p_probe.py 1000,1000000,4000000 2>/dev/null | grep "N="
  SYNC=1 ORDERS=update_first MAX_BLOCKS=0 timeout 300 $TR tools/small_p_probe.py 1000,1000000,4000000 2>/dev/null | grep "N=" | sed "s/^/sync /"
done
sh1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.2f us'%(1e3*d['ms_per_step']), 'local %.2f'%(1e3*m['all_local']['ms_per_step']), 'sync %.2f'%(1e3*m['all_sync']['ms_per_step']))" "$@"; }
for P in 1000 1000000; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --P $P --steps 300 --warmup 20 --no-e2e --no-cpu-baseline --no-replay --no-kernel-events \
    > gpurun_out/fence/n1_${P}.json 2>gpurun_out/fence/n1_${P}.err
  sh1 gpurun_out/fence/n1_${P}.json "N=1 P=$P eager"
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --P $P --steps 300 --warmup 20 --no-e2e --no-cpu-baseline --no-replay --graph \
    > gpurun_out/fence/n1g_${P}.json 2>gpurun_out/fence/n1g_${P}.err
  sh1 gpurun_out/fence/n1g_${P}.json "N=1 P=$P graph"
done
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "symm-fused or symm-adaptive or symm-p2p or update_first or adaptive or bsp or ga or nan" > gpurun_out/fence/pytest_multi.log 2>&1; echo multi rc=$?
tail -3 gpurun_out/fence/pytest_multi.log
