# usage: bash scripts/gpu_stage.sh <tag> -- coalesced tuple staging in the precompute and zero-pilot kernels vs HEAD
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
MIST_LIB=ab/libmist_stage.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for L in HEAD stage; do MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1; done
done
for L in HEAD stage; do
  for w in 3 4; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
done
MIST_LIB=ab/libmist_stage.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_stage_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
