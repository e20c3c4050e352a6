# usage: bash scripts/gpu_final3.sh <tag> -- full GPU suite, smoke, default bench after the pilot-level change
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --factors unit --no-cpu-baseline > gpurun_out/bench_unit_$TAG.log 2>&1
for w in 3 4; do timeout 600 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/full_c${w}_$TAG.log 2>&1; done
echo done
