# usage: bash scripts/gpu_seg1s.sh <tag> -- one-sync-per-level reduction at 2048 / 1024-record chunks vs HEAD
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do
  for L in seg2k seg2k1s seg1k1s; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1
  done
done
for L in seg2k seg2k1s seg1k1s; do
  for w in 3 4; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
