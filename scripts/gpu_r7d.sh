# usage: bash scripts/gpu_r7d.sh <tag> -- parity subset, R7 d-bound A/B, pilot levels, counters
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier or sharding" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for L in r7a r7d; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1
  done
done
for pl in 2 4 5 2,4 3,5 3,6; do
  MIST_PILOT_LEVELS=$pl timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_pl${pl}_cfg2_1.log 2>&1
done
for L in r7a r7d; do
  for st in 0.4 0.8 0.98; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_w${st}_1.log 2>&1
  done
done
for pl in 5,11 4,8 7 5,9,13; do
  for st in 0.4 0.8 0.98; do
    MIST_PILOT_LEVELS=$pl timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_pl${pl}_w${st}_1.log 2>&1
  done
done
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_cfg2.log 2>&1
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start 0.8 --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_w0.8.log 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
