# round 2: smoke + full single-GPU suite + default bench line on one B200
echo "HEAD $(cat .git_sha)"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_1.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench rc=$?
tail -c 2500 gpurun_out/bench_n1.json
