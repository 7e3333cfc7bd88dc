# round 2, session 3, final single-GPU pass at HEAD: smoke, single-GPU suite,
# default bench line, BASELINE configs 1-3 at N = 1, ncu (launch list + --set full
# of K13 and of the step kernel through a world-1 group)
mkdir -p gpurun_out/finalA
echo "HEAD $(cat .git_sha)"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/finalA/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/finalA/smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/finalA/pytest_gpu_1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/finalA/pytest_gpu_1.log
timeout 600 python bench.py > gpurun_out/finalA/bench_n1.json 2> gpurun_out/finalA/bench_n1.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/finalA/bench_n1.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['clocks'])"
timeout 300 python bench.py --impl reference > gpurun_out/finalA/bench_ref_n1.json 2> gpurun_out/finalA/bench_ref_n1.err; echo ref rc=$?
tail -c 600 gpurun_out/finalA/bench_ref_n1.json
bash tools/configs_sweep.sh 1 2>&1 | tail -14
mv gpurun_out/configs_n1 gpurun_out/finalA/ 2>/dev/null
set -x
SMALL="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-replay"
$SMALL > gpurun_out/finalA/n_small_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/finalA/launches.csv $SMALL > gpurun_out/finalA/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sgd_kernel -s 4 -c 1 -o gpurun_out/finalA/prof_k13 $SMALL > gpurun_out/finalA/ncu_k13.log 2>&1; echo "k13 rc=$?"
S1="python tools/step_kernel_solo.py update_first local"
$S1 > gpurun_out/finalA/solo_uf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/finalA/prof_step_uf $S1 > gpurun_out/finalA/ncu_step_uf.log 2>&1; echo "step uf rc=$?"
