# usage: bash scripts/gpu_seg4k.sh <tag> -- reduction parity; 4096-record chunks with one sync per level vs 2048 (HEAD)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_seg4k_cfg2_$rep.log 2>&1
  MIST_LIB=ab/libmist_seg2k.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_seg2k_cfg2_$rep.log 2>&1
  MIST_REDUCE=radix timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_radix_cfg2_$rep.log 2>&1
done
for L in seg4k seg2k; do
  LIBV=""; [ $L = seg2k ] && LIBV=ab/libmist_seg2k.so
  for w in 3 4; do MIST_LIB=$LIBV timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
