# round 2: full single-GPU suite + default bench line on one B200
git_sha=$(cat .git_sha 2>/dev/null)
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_1.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench_n1.json
