# usage: bash scripts/gpu_red_ncu.sh <tag> -- DRAM bytes + duration of the reduction kernels (bucket path):
# cfg2 sweep, a cfg5 window with ~30M candidates, and 2^26 random records (sort_bench); radix path for contrast
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K="regex:k_seg_|k_chunk_|k_scan|k_radix|k_fs_|k_gather|k_prepare|k_digit"
timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 3000 --csv --log-file gpurun_out/red_cfg2_$TAG.csv python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 3000 --csv --log-file gpurun_out/red_c5w_$TAG.csv python tools/prof_step.py --workload 5 --start 0.995 --fraction 0.005 --warmup 0 --steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 3000 --csv --log-file gpurun_out/red_sort_$TAG.csv python tools/sort_bench.py --log2n 26 --groups 4096 --reps 0 > /dev/null 2>&1
MIST_REDUCE=radix timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 3000 --csv --log-file gpurun_out/red_sortradix_$TAG.csv python tools/sort_bench.py --log2n 26 --groups 4096 --reps 0 > /dev/null 2>&1
MIST_REDUCE=radix timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 3000 --csv --log-file gpurun_out/red_c5wradix_$TAG.csv python tools/prof_step.py --workload 5 --start 0.995 --fraction 0.005 --warmup 0 --steps 1 > /dev/null 2>&1
echo done
