# usage: bash scripts/gpu_pl3.sh <tag> -- pilot levels re-check with the run-queue pilot
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for pl in def 4 5 3,5 2,4; do
  if [ $pl = def ]; then E=""; else E="MIST_PILOT_LEVELS=$pl"; fi
  env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_pl${pl}_cfg2_1.log 2>&1
  env $E timeout 300 python tools/prof_step.py --workload 4 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_pl${pl}_c4_1.log 2>&1
done
for pl in def 7 4,7 5,9 6,11; do
  if [ $pl = def ]; then E=""; else E="MIST_PILOT_LEVELS=$pl"; fi
  env $E timeout 300 python tools/prof_step.py --workload 3 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_pl${pl}_c3_1.log 2>&1
done
for pl in def 5,9,13 7,13 4,8,16; do
  if [ $pl = def ]; then E=""; else E="MIST_PILOT_LEVELS=$pl"; fi
  for st in 0.4 0.8 0.975; do env $E timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_pl${pl}_w${st}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
