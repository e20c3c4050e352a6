# usage: bash scripts/gpu_quick.sh <tag> -- F rows only for units with runs left after a cheap R7 bound, vs HEAD
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
MIST_LIB=ab/libmist_quick16.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier or sharding" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for L in HEAD quick16; do MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1; done
done
for L in HEAD quick16; do
  for w in 3 4; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
  for st in 0.4 0.8 0.975; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_w${st}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
