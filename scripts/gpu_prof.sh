# usage: bash scripts/gpu_prof.sh <tag>   (one GPU; plain runs first, then ncu)
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python tools/prof_step.py --workload 2 --warmup 0 --steps 1"
SB="python tools/sort_bench.py --log2n 26 --reps 1"
timeout 600 $CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 300 $SB > gpurun_out/sort_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort_$TAG.csv $SB > gpurun_out/ncu_launch_sort_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_eval_$TAG $CMD > gpurun_out/ncu_eval_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_radix_scatter -s 12 -c 1 -o gpurun_out/prof_scatter_$TAG $SB > gpurun_out/ncu_scatter_$TAG.log 2>&1
echo done
