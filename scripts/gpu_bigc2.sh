# usage: bash scripts/gpu_bigc2.sh <tag> -- cfg2 A/B after moving cudaMemGetInfo off the steady-state path
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for rep in 1 2 3; do
  for L in HEAD bigc2; do MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
