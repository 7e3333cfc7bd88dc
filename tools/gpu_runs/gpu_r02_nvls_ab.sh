# NVLS mean variants (A/B builds from tools/ab_build.sh) at N = 4, P = 100M
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr=127.0.0.1 --master-port=29519"
for v in base u8 u2 weak t256 t1024 base; do
  SS_LIB_PATH=$PWD/paper_2307_07950_b200/_lib/ab/$v.so SYMM_ONLY=1 $TR tools/symm_perf.py 100000000 2>&1 \
    | grep -E "busbw|requested" | sed "s/^/$v: /"
done
