# usage: bash scripts/ab_sort.sh <tag> <lib>...  -- sort_bench per library, then ncu launch lists
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for rep in 1 2; do for L in "$@"; do n=$(basename $L .so)
  MIST_LIB=$L timeout 300 python tools/sort_bench.py --log2n 26 --reps 3 > gpurun_out/abs_${TAG}_${n}_$rep.log 2>&1
done; done
for L in "$@"; do n=$(basename $L .so)
  MIST_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/abs_${TAG}_${n}_launches.csv python tools/sort_bench.py --log2n 26 --reps 1 > /dev/null 2>&1
done
