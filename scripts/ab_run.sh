# usage: bash scripts/ab_run.sh <tag> <libA> [<libB> ...] -- same-box A/B: cfg2 bench + cfg5 windows per library
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for rep in 1 2; do
for L in "$@"; do
  n=$(basename $L .so)
  MIST_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${n}_cfg2_$rep.log 2>&1
  for st in 0.4 0.8 0.98; do
    MIST_LIB=$L timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ab_${TAG}_${n}_w${st}_$rep.log 2>&1
  done
done
done
