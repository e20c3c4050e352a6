# usage: bash scripts/gpu_ab3.sh <tag> <libs...> -- parity subset with the in-tree lib, then cfg2 (3 reps) + cfg5 windows A/B
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2 3; do
for L in "$@"; do
  n=$(basename $L .so)
  MIST_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${n}_cfg2_$rep.log 2>&1
done
done
for L in "$@"; do
  n=$(basename $L .so)
  for st in 0.002 0.4 0.8 0.98; do
    MIST_LIB=$L timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ab_${TAG}_${n}_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
