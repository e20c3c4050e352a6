# usage: bash scripts/gpu_sort_ab.sh <tag> -- sort parity tests with the TMA scatter, then plain vs TMA sort bench + ncu launch list
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier_points or frontier_small or cfg1_full or sharding or buffer" > gpurun_out/pytest_sort_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sort_$TAG.log
for rep in 1 2; do
  MIST_SCATTER=plain timeout 300 python tools/sort_bench.py --log2n 26 --reps 3 > gpurun_out/sort_${TAG}_plain_$rep.log 2>&1
  timeout 300 python tools/sort_bench.py --log2n 26 --reps 3 > gpurun_out/sort_${TAG}_tma_$rep.log 2>&1
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort_$TAG.csv python tools/sort_bench.py --log2n 26 --reps 1 > gpurun_out/ncu_sort_$TAG.log 2>&1
MIST_SCATTER=plain timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort_plain_$TAG.csv python tools/sort_bench.py --log2n 26 --reps 1 > gpurun_out/ncu_sort_plain_$TAG.log 2>&1
echo done
