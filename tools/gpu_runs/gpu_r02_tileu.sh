# round 2, session 3: vectors in flight per thread in the per-tile means of the
# overlapped sync step (A/B builds, same box): N = 2 P2P (SS_TILE_U_P2P 2/4/8),
# N = 4 NVLS (SS_TILE_U_NVLS 2/4/8); P = 100M, all-sync (known pass) and the 50% mix
mkdir -p gpurun_out/tileu
echo "HEAD $(cat .git_sha)"
L=$PWD/paper_2307_07950_b200/_lib
one() {  # N variant
  local N=$1 v=$2 lib=""
  [ "$v" != base ] && lib="SS_LIB_PATH=$L/ab/$v.so"
  env $lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N \
    bench.py --gpus $N --steps 100 --warmup 10 --no-e2e --no-replay --no-cpu-baseline > gpurun_out/tileu/n${N}_$v.json 2>gpurun_out/tileu/n${N}_$v.err
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.1f us'%(1e3*d['ms_per_step']), 'local %.1f'%(1e3*m['all_local']['ms_per_step']), 'sync %.1f'%(1e3*m['all_sync']['ms_per_step']), 'C2 %.1f'%(1e3*d.get('exchange',{}).get('mean_ms',0)))" gpurun_out/tileu/n${N}_$v.json "N=$N $v"
}
for rep in 1 2; do
  for v in base p4 p8; do one 2 $v; done
  for v in base n4 n8; do one 4 $v; done
done
