# round 2, session 3: programmatic dependent launch (SS_PDL) A/B on one 4-GPU box:
# single-GPU suite with PDL on, small-P steps at N = 1 (graph / eager) and N = 2 / 4,
# the 100M N = 1 bench line, then the N = 2 multi-GPU suite with PDL on
mkdir -p gpurun_out/pdl
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pdl/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pdl/pytest_gpu_1.log
for pdl in 0 1 0 1; do
  for P in 1000000 4000000 16000000; do
    for G in --graph --no-kernel-events; do
      CUDA_VISIBLE_DEVICES=0 SS_PDL=$pdl timeout 300 python bench.py --P $P --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-replay $G \
        > gpurun_out/pdl/n1_${P}_${pdl}${G}.json 2>/dev/null
      python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print('PDL=$pdl N=1 P=$P $G', 'mixed %.2f us'%(1e3*d['ms_per_step']), 'local %.2f'%(1e3*m['all_local']['ms_per_step']), 'sync %.2f'%(1e3*m['all_sync']['ms_per_step']))" gpurun_out/pdl/n1_${P}_${pdl}${G}.json
    done
  done
  for N in 2 4; do
    ORDERS=update_first MAX_BLOCKS=0 SS_PDL=$pdl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
      tools/small_p_probe.py 1000000,4000000 2>/dev/null | grep -v "^\*\|OMP\|NCCL" | sed "s/^/PDL=$pdl N=$N /"
  done
done
for pdl in 0 1; do
  CUDA_VISIBLE_DEVICES=0 SS_PDL=$pdl timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/pdl/n1_100M_${pdl}.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print('PDL=$pdl N=1 P=100M', d['value'], d['roofline']['kernel_ms_mean'])" gpurun_out/pdl/n1_100M_${pdl}.json
done
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "symm-fused or symm-adaptive or update_first or adaptive or bsp or nvls" > gpurun_out/pdl/pytest_multi.log 2>&1; echo multi rc=$?
tail -3 gpurun_out/pdl/pytest_multi.log
