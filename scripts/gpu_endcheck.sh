# usage: bash scripts/gpu_endcheck.sh <tag> -- every GPU test, smoke, default bench, reference arm
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu --maxfail=8 --timeout=900 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.log 2>&1
echo done
