set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests/test_colocated_gpu.py -x -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/colocated.log 2>&1; echo colo rc=$?
tail -5 gpurun_out/colocated.log
