# round 2, session 3: mean lag (A/B builds) and tile size at N = 4 (NVLS) and N = 2,
# P = 100M, after the single-fence posts; all-sync (known pass) and the 50% mix
mkdir -p gpurun_out/lag4
echo "HEAD $(cat .git_sha)"
L=$PWD/paper_2307_07950_b200/_lib
one() {  # N variant [extra args]
  local N=$1 v=$2; shift 2; local lib=""
  case $v in base|t*) ;; *) lib="SS_LIB_PATH=$L/ab/$v.so";; esac
  env $lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N \
    bench.py --gpus $N --steps 100 --warmup 10 --no-e2e --no-replay --no-cpu-baseline "$@" > gpurun_out/lag4/n${N}_$v.json 2>gpurun_out/lag4/n${N}_$v.err
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.1f us'%(1e3*d['ms_per_step']), 'local %.1f'%(1e3*m['all_local']['ms_per_step']), 'sync %.1f'%(1e3*m['all_sync']['ms_per_step']), 'C2 %.1f'%(1e3*d.get('exchange',{}).get('mean_ms',0)))" gpurun_out/lag4/n${N}_$v.json "N=$N $v"
}
for rep in 1 2; do
  for N in 4 2; do
    one $N base; one $N l050; one $N l075; one $N l150; one $N t8k --tile 8192; one $N t32k --tile 32768
  done
done
