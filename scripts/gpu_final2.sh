# usage: bash scripts/gpu_final2.sh <tag> -- full GPU suite + smoke + bench at the final state; cfg5 on one GPU
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
timeout 900 python tools/mgpu_sweep.py --workload 5 --plan > gpurun_out/cfg5_n1_$TAG.log 2>&1
echo done
