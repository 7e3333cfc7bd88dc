# round 2: the full real multi-GPU suite (torchrun, one process per GPU) at N = $1
n=$1
echo "HEAD $(cat .git_sha)"; nvidia-smi -L
timeout 3000 python -m pytest tests/test_multigpu.py -v -p no:cacheprovider > gpurun_out/pytest_n${n}.log 2>&1; echo rc=$?
echo "HEAD $(cat .git_sha)" >> gpurun_out/pytest_n${n}.log
tail -5 gpurun_out/pytest_n${n}.log
