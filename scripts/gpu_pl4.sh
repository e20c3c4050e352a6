# usage: bash scripts/gpu_pl4.sh <tag> -- cfg2 pilot {3} (default) vs {4}, three reps each
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_pl3_cfg2_$rep.log 2>&1
  MIST_PILOT_LEVELS=4 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_pl4_cfg2_$rep.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --factors unit > gpurun_out/ab_${TAG}_upl3_cfg2_1.log 2>&1
MIST_PILOT_LEVELS=4 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --factors unit > gpurun_out/ab_${TAG}_upl4_cfg2_1.log 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
