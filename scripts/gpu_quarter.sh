# usage: bash scripts/gpu_quarter.sh <tag> -- per-rank proxy at N=4: a quarter of cfg2 on one GPU, launch list
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --workload 2 --fraction 0.25 --warmup 3 --steps 5 > gpurun_out/quarter_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_quarter_$TAG.csv python tools/prof_step.py --workload 2 --fraction 0.25 --warmup 0 --steps 1 > /dev/null 2>&1
echo done
