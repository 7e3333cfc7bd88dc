# round 2, session 3: e2e at N = 4 with the pinned host buffers bound to each GPU's
# NUMA node vs not (same box), and N = 1
echo "HEAD $(cat .git_sha)"
mkdir -p gpurun_out/numa
nvidia-smi topo -m 2>/dev/null | head -8
for v in 1 0 1; do
  SS_BENCH_NUMA=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 \
    bench.py --gpus 4 --steps 50 --no-replay > gpurun_out/numa/n4_$v.json 2> gpurun_out/numa/n4_$v.err; echo "N=4 numa=$v rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);e=d['e2e'];print('  e2e', round(e['value'],1), round(e['h2d_gbs_per_rank'],1), 'GB/s/rank, bound', e.get('host_cpus_bound'), 'value', round(d['value'],1))" gpurun_out/numa/n4_$v.json
done
