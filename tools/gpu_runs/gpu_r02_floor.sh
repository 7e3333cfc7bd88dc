# round 2, session 3: the N = 2 small-P floor -- device marks of the local step
# (start -> vote posted -> votes in) vs the per-step event time, cooperative
# attribute and PDL on / off
mkdir -p gpurun_out/floor
echo "HEAD $(cat .git_sha)"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571"
for env in "SS_COOP=1 SS_PDL=1" "SS_COOP=0 SS_PDL=1" "SS_COOP=1 SS_PDL=0" "SS_COOP=0 SS_PDL=0"; do
  for P in 1000 1000000; do
    echo "== $env P=$P"
    env $env timeout 300 $TR tools/local_timeline.py $P 8 2>/dev/null | grep rank
  done
  env $env ORDERS=update_first MAX_BLOCKS=0 timeout 300 $TR tools/small_p_probe.py 1000,1000000 2>/dev/null | grep "N=" | sed "s/^/$env /"
done
