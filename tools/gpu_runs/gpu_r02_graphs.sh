# round 2, session 3: multi-step CUDA graphs (PDL edges inside) vs one-step graphs vs eager at small P
mkdir -p gpurun_out/graphs
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "graph or captured" 2>&1 | tail -2
sh1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);m=d['modes'];print(sys.argv[2], 'mixed %.2f us'%(1e3*d['ms_per_step']), 'local %.2f'%(1e3*m['all_local']['ms_per_step']), 'sync %.2f'%(1e3*m['all_sync']['ms_per_step']), 'launches', d.get('gpu_launches'))" "$@"; }
for P in 1000000 4000000 16000000; do
  for v in "--no-kernel-events" "--graph --graph-steps 1" "--graph --graph-steps 4" "--graph --graph-steps 8"; do
    tag=$(echo "$v" | tr -d ' -')
    CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --P $P --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-replay $v \
      > gpurun_out/graphs/n1_${P}_$tag.json 2>gpurun_out/graphs/n1_${P}_$tag.err
    sh1 gpurun_out/graphs/n1_${P}_$tag.json "N=1 P=$P $v"
  done
  for v in "--no-kernel-events" "--graph --graph-steps 4"; do
    tag=$(echo "$v" | tr -d ' -')
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
      bench.py --gpus 2 --P $P --steps 200 --warmup 10 --no-e2e --no-replay $v > gpurun_out/graphs/n2_${P}_$tag.json 2>gpurun_out/graphs/n2_${P}_$tag.err
    sh1 gpurun_out/graphs/n2_${P}_$tag.json "N=2 P=$P $v"
  done
done
