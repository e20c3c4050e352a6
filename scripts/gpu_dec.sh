# usage: bash scripts/gpu_dec.sh <tag> -- 32-bit unit decode A/B; cfg5 whole space on 1 GPU + both solver schemes
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for L in HEAD dec32; do MIST_LIB=ab/libmist_$L.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_cfg2_$rep.log 2>&1; done
done
for L in HEAD dec32; do
  for w in 3 4; do MIST_LIB=ab/libmist_$L.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${L}_c${w}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
timeout 1500 python tools/mgpu_sweep.py --workload 5 --plan --plan-ab > gpurun_out/cfg5_n1_$TAG.log 2>&1
echo done
