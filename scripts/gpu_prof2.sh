# usage: bash scripts/gpu_prof2.sh <tag> -- bench line, launch list of the bench command, ncu --set full of k_eval_q (cfg2)
cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
CMD="python tools/prof_step.py --workload 2 --warmup 0 --steps 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_q -c 1 -o gpurun_out/prof_eval_$TAG $CMD > gpurun_out/ncu_eval_$TAG.log 2>&1
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page source --csv > gpurun_out/prof_eval_${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_eval_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page details --csv > gpurun_out/prof_eval_${TAG}_details.csv 2>/dev/null
echo done
