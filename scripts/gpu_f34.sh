# usage: bash scripts/gpu_f34.sh <tag> -- interference-model + preset GPU tests, measurements, default bench
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "from paper_2503_19050_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_intf.py -q -m gpu --timeout=600 -p no:cacheprovider > gpurun_out/pytest_intf_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_intf_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_presets.py tests/test_gpu_inter.py -q -m gpu --timeout=900 -p no:cacheprovider > gpurun_out/pytest_presets_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_presets_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python tools/intf_bench.py > gpurun_out/intf_bench_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_intf_$TAG.csv python tools/intf_bench.py --rows 20000000 --fit-rows 1000000 --iters 1 > gpurun_out/ncu_intf_$TAG.log 2>&1
echo done
