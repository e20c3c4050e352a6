# usage: bash scripts/gpu_direct.sh <tag> -- frontier straight to the caller's buffers (e2e) vs HEAD; API tests
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sample.py tests/test_gpu_inter.py tests/test_gpu_presets.py -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2 3; do
  for L in HEAD direct; do MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1; done
done
echo done
