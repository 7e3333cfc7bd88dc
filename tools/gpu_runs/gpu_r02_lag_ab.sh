# norm-first / known-pass mean lag and tile size A/B (bench modes) at N = $1
n=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr=127.0.0.1 --master-port=29527"
B="bench.py --gpus $n --no-cpu-baseline --no-e2e --no-replay"
for rep in 1 2; do
for v in ${VARIANTS:-lag1 lag2 lag4 lag0}; do
  for t in ${TILES:-16384 8192}; do
    SS_LIB_PATH=$PWD/paper_2307_07950_b200/_lib/ab/$v.so $TR $B --tile $t 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); m=d['modes']
print('$v tile $t', round(d['value']), 'mixed ms', round(d['ms_per_step'],4), 'local', round(m['all_local']['ms_per_step'],4), 'all_sync', round(m['all_sync']['ms_per_step'],4))"
  done
done
done
