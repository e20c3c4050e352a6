# usage: bash scripts/gpu_check.sh <tag> [pytest-args]  -- GPU tests, smoke, bench variants
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --maxfail=8 --timeout=600 -p no:cacheprovider ${@:2} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
for MB in 2 3; do
  MIST_EVAL_MINB=$MB timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_mb$MB.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}_mb$MB.log
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/bench_${TAG}_unit.log 2>&1
echo done
