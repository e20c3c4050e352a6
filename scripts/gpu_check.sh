# usage: bash scripts/gpu_check.sh <tag> [pytest-args]  -- GPU tests, smoke, bench variants
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --maxfail=8 --timeout=600 -p no:cacheprovider ${@:2} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_spec.log 2>&1
MIST_PILOT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_nopilot.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/bench_${TAG}_unit.log 2>&1
echo done
