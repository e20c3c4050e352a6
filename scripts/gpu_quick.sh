# usage: bash scripts/gpu_quick.sh <tag>  -- quick parity subset + bench variants
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "small_spaces or cfg1 or cfg2 or frontier_points or big_configs or sharding" > gpurun_out/pytest_quick_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_q3.log 2>&1
MIST_EVAL_CFG=256x2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_q2.log 2>&1
MIST_EVAL_QUEUE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_lock.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/bench_${TAG}_unit.log 2>&1
echo done
