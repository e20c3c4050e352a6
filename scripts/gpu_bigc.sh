# usage: bash scripts/gpu_bigc.sh <tag> -- 2^28 candidate buffer + rate-based pre-splitting vs HEAD (2^26)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for L in HEAD bigc; do
  MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_1.log 2>&1
  for w in 3 4; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
  MIST_LIB=ab/libmist_$L.so timeout 900 python tools/mgpu_sweep.py --workload 5 > gpurun_out/cfg5_n1_${TAG}_$L.log 2>&1
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
