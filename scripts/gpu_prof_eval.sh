# usage: bash scripts/gpu_prof_eval.sh <tag> -- one ncu --set full capture of k_eval_q (cfg2 sweep) with source
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python tools/prof_step.py --workload 2 --warmup 0 --steps 1"
timeout 300 $CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_q -c 1 -o gpurun_out/prof_eval_$TAG $CMD > gpurun_out/ncu_eval_$TAG.log 2>&1
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page source --csv > gpurun_out/prof_eval_${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_eval_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_eval_$TAG.ncu-rep --page details --csv > gpurun_out/prof_eval_${TAG}_details.csv 2>/dev/null
echo done
