# usage: bash scripts/gpu_pilotq.sh <tag> -- pilot sub-grid on the CTA queue kernel vs the lockstep kernel
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do
  for k in queue lockstep; do MIST_PILOT_KERNEL=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${k}_cfg2_$rep.log 2>&1; done
done
for k in queue lockstep; do
  MIST_PILOT_KERNEL=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --factors unit > gpurun_out/ab_${TAG}_u${k}_cfg2_1.log 2>&1
  for w in 3 4; do MIST_PILOT_KERNEL=$k timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${k}_c${w}_1.log 2>&1; done
  for st in 0.4 0.8 0.975; do MIST_PILOT_KERNEL=$k timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${k}_w${st}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
