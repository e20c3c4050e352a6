# usage: bash scripts/gpu_state.sh <tag> -- full GPU suite, smoke, bench (default + reference arm), launch list,
# ncu --set full of k_eval_q, counters, cfg3/cfg4 whole-space sweeps
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --factors unit --no-cpu-baseline > gpurun_out/bench_unit_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
for w in 3 4; do timeout 600 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/full_c${w}_$TAG.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
CMD="python tools/prof_step.py --workload 2 --warmup 0 --steps 1"
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start 0.5 --fraction 0.005 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_c5w.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_q --launch-skip 1 -c 1 -o gpurun_out/prof_eval_$TAG $CMD > gpurun_out/ncu_eval_$TAG.log 2>&1
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_eval_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page details --csv > gpurun_out/prof_eval_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_eval_${TAG}_source.csv 2>/dev/null
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_cfg2.log 2>&1
echo done
