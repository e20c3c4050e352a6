# usage: bash scripts/gpu_r7.sh <tag> -- parity (frontier tests, fp and bench paths), R7 on/off A/B, counters
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for r7 in 1 0; do
    MIST_R7=$r7 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_r7${r7}_cfg2_$rep.log 2>&1
  done
done
for r7 in 1 0; do
  MIST_R7=$r7 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/ab_${TAG}_unit_r7${r7}_cfg2_1.log 2>&1
  for st in 0.4 0.8 0.98; do
    MIST_R7=$r7 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_r7${r7}_w${st}_1.log 2>&1
  done
  MIST_R7=$r7 MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_r7${r7}_cfg2.log 2>&1
  MIST_R7=$r7 MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start 0.8 --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_r7${r7}_w0.8.log 2>&1
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
