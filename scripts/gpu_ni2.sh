# usage: bash scripts/gpu_ni2.sh <tag> -- parity subset with the default build, then code-size A/B
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier or sharding" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
LIBS="def sel ni_pred ni_lb ni_predlb"
for rep in 1 2; do
  for L in $LIBS; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1
  done
done
for L in $LIBS; do
  MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/ab_${TAG}_unit${L}_cfg2_1.log 2>&1
  for st in 0.4 0.8 0.98; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
