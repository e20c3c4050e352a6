# usage: bash scripts/gpu_pilot.sh <tag> -- pilot-level A/B (MIST_PILOT_LEVELS) on cfg2 and cfg5 windows
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
for lv in default 3,5 4 3,6 5 2,4; do
  for rep in 1 2; do
    if [ $lv = default ]; then E=""; else E="MIST_PILOT_LEVELS=$lv"; fi
    env $E timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_L${lv}_cfg2_$rep.log 2>&1
  done
done
for lv in default 5,9 7,13 4,7 9; do
  for st in 0.4 0.8; do
    if [ $lv = default ]; then E=""; else E="MIST_PILOT_LEVELS=$lv"; fi
    env $E timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_L${lv}_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
