# round 2, session 3: timeline of the overlapped known-pass sync step at N = 2 / 4 (P = 100M)
echo "HEAD $(cat .git_sha)"
for N in 2 4; do
  for mode in known up; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N \
      tools/overlap_timeline.py 100000000 16384 $mode 2>/dev/null | grep -v "^\*\|OMP\|NCCL" | sed "s/^/N=$N $mode: /"
  done
done
