# usage: bash scripts/gpu_ni.sh <tag> -- code-size A/B (noinline knobs) on cfg2, unit factors and cfg5 windows
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do
  for L in def ni_pred ni_lb ni_dlb ni_cut ni_lbdlb; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1
  done
done
for L in def ni_pred ni_lb ni_dlb ni_cut ni_lbdlb; do
  for st in 0.4 0.8 0.98; do
    MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
