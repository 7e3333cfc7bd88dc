# round 2, session 3: same-box A/B of the per-pass lag: base (known x3/4, sweep x3/2),
# old (x1 / x1), k60 (known x3/5); bench modes at N = 4 and N = 2, P = 100M
mkdir -p gpurun_out/lagE
echo "HEAD $(cat .git_sha)"
L=$PWD/paper_2307_07950_b200/_lib
one() {
  local N=$1 v=$2 lib=""
  [ "$v" != base ] && lib="SS_LIB_PATH=$L/ab/$v.so"
  env $lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N \
    bench.py --gpus $N --steps 100 --warmup 10 --no-e2e --no-replay --no-cpu-baseline > gpurun_out/lagE/n${N}_$v.json 2>gpurun_out/lagE/n${N}_$v.err
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.1f us'%(1e3*d['ms_per_step']), 'local %.1f'%(1e3*m['all_local']['ms_per_step']), 'sync %.1f'%(1e3*m['all_sync']['ms_per_step']), 'C2 %.1f'%(1e3*d.get('exchange',{}).get('mean_ms',0)))" gpurun_out/lagE/n${N}_$v.json "N=$N $v"
}
for rep in 1 2; do for N in 4 2; do for v in base old k60; do one $N $v; done; done; done
