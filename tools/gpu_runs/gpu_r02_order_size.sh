# update-first vs adaptive (norm-first / known pass on sync steps) across P at N = 2 and 4 (bench modes)
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29539"
for n in 2 4; do
for P in 16000000 32000000 48000000 64000000; do
  for order in update_first adaptive; do
    $TR --nproc-per-node $n bench.py --gpus $n --P $P --order $order --no-cpu-baseline --no-e2e --no-replay 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); m=d['modes']
print('N=$n P=$P $order', round(d['value']), 'mixed ms', round(d['ms_per_step'],4), 'local', round(m['all_local']['ms_per_step'],4), 'all_sync', round(m['all_sync']['ms_per_step'],4))"
  done
done
done
