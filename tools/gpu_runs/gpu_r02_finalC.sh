# round 2, session 3: plan-vs-per-call bit-identity test, then BASELINE configs 1-3
# (model workloads, CUDA-graph mode, VGG-11 delta sweep) at N = 2 and N = 4
echo "HEAD $(cat .git_sha)"
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "plan" 2>&1 | tail -2
for N in 2 4; do bash tools/configs_sweep.sh $N 2>&1 | tail -14; done
mkdir -p gpurun_out/finalC; mv gpurun_out/configs_n2 gpurun_out/configs_n4 gpurun_out/finalC/ 2>/dev/null
