# usage: bash scripts/gpu_seg2.sh <tag> -- bucket vs radix reduction: bench reps and launch lists
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2 3; do
  for r in seg radix; do MIST_REDUCE=$r timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${r}_cfg2_$rep.log 2>&1; done
done
MIST_REDUCE=seg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${TAG}_seg.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
MIST_REDUCE=seg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${TAG}_sortseg.csv python tools/sort_bench.py --log2n 26 --groups 4096 --reps 1 > /dev/null 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
