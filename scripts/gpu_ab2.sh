# usage: bash scripts/gpu_ab2.sh <tag> <libs...> -- intf tests/bench with the in-tree lib, then cfg2 A/B (3 reps each)
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_intf.py -q -m gpu --timeout=600 -p no:cacheprovider > gpurun_out/pytest_intf_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_intf_$TAG.log
timeout 600 python tools/intf_bench.py > gpurun_out/intf_bench_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_intf_$TAG.csv python tools/intf_bench.py --rows 20000000 --fit-rows 1000000 --iters 1 > gpurun_out/ncu_intf_$TAG.log 2>&1
for rep in 1 2 3; do
for L in "$@"; do
  n=$(basename $L .so)
  MIST_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${n}_cfg2_$rep.log 2>&1
done
done
for L in "$@"; do
  n=$(basename $L .so)
  MIST_LIB=$L timeout 300 python tools/prof_step.py --workload 5 --start 0.8 --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ab_${TAG}_${n}_w0.8_1.log 2>&1
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
