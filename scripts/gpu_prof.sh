# usage: bash scripts/gpu_prof.sh <tag>   (one GPU; plain run first, then ncu)
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
[ -x tools/fp64_peak ] && timeout 120 tools/fp64_peak > gpurun_out/fp64_peak_$TAG.json 2>&1
CMD="python tools/prof_step.py --workload 2 --warmup 0 --steps 1"
timeout 600 $CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_eval_$TAG $CMD > gpurun_out/ncu_eval_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_radix_scatter -s 2 -c 1 -o gpurun_out/prof_scatter_$TAG $CMD > gpurun_out/ncu_scatter_$TAG.log 2>&1
echo done
