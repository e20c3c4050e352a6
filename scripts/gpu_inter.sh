# usage: bash scripts/gpu_inter.sh <tag>  -- inter-stage GPU tests + default bench
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "from paper_2503_19050_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_inter.py -q -m gpu --timeout=600 -p no:cacheprovider > gpurun_out/pytest_inter_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_inter_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}.log
echo done
