# usage: bash scripts/gpu_final.sh <tag> -- every GPU test, smoke, default/unit bench, launch list, ncu capture, cfg5 full-scale parity
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu --maxfail=8 --timeout=900 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.log 2>&1
timeout 600 python bench.py --factors unit --no-cpu-baseline > gpurun_out/bench_${TAG}_unit.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
bash scripts/gpu_prof_eval.sh $TAG
MIST_FULLSCALE=1 timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -m gpu -k "5" --timeout=1400 -p no:cacheprovider > gpurun_out/pytest_fullscale_cfg5_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fullscale_cfg5_$TAG.log
echo done
