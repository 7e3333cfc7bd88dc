# round 2, session 3: last check of the final tree on one GPU (smoke, suite, bench)
mkdir -p gpurun_out/finalD
echo "HEAD $(cat .git_sha)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/finalD/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/finalD/smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/finalD/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/finalD/pytest_gpu_1.log
timeout 600 python bench.py > gpurun_out/finalD/bench_n1.json 2> gpurun_out/finalD/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/finalD/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline'],d['clocks'],d['gpu_launches'])"
