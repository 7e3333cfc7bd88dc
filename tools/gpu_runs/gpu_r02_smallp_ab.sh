# small-P local (and delta = 0 sync) step A/B of library variants (tools/ab_build.sh) at N = $1
n=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr=127.0.0.1 --master-port=29535"
for rep in 1 2; do
for v in ${VARIANTS:-base pt4 pt2 fence}; do
  for sync in 0 1; do
  SYNC=$sync TAG="$v sync=$sync" ORDERS=update_first,adaptive MAX_BLOCKS=0 SS_LIB_PATH=$PWD/paper_2307_07950_b200/_lib/ab/$v.so \
    $TR tools/small_p_probe.py 1000000,4000000,16000000 2>&1 | grep "N="
  done
done
done
