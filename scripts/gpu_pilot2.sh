# usage: bash scripts/gpu_pilot2.sh <tag> -- pilot-level A/B on cfg5 windows, cfg3/cfg4 whole sweeps
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
for lv in default 9 11 5,9 13 5,11; do
  if [ $lv = default ]; then E=""; else E="MIST_PILOT_LEVELS=$lv"; fi
  for st in 0.2 0.6 0.8 0.98; do
    env $E timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_L${lv}_w${st}_1.log 2>&1
  done
done
for lv in default 7 9 4,7; do
  if [ $lv = default ]; then E=""; else E="MIST_PILOT_LEVELS=$lv"; fi
  env $E timeout 300 python tools/prof_step.py --workload 3 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_L${lv}_c3_1.log 2>&1
done
for lv in default 4 5 2,4; do
  if [ $lv = default ]; then E=""; else E="MIST_PILOT_LEVELS=$lv"; fi
  env $E timeout 300 python tools/prof_step.py --workload 4 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_L${lv}_c4_1.log 2>&1
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
