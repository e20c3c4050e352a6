# usage: bash scripts/gpu_pass.sh <tag> -- two unit passes (MIST_PASSES=2) vs one; setup-only diagnostic build
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
MIST_PASSES=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for p in 1 2; do MIST_PASSES=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_p${p}_cfg2_$rep.log 2>&1; done
done
MIST_LIB=ab/libmist_setup.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_setup_cfg2_1.log 2>&1
for p in 1 2; do
  for w in 3 4; do MIST_PASSES=$p timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_p${p}_c${w}_1.log 2>&1; done
  for st in 0.4 0.8 0.9 0.975; do MIST_PASSES=$p timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_p${p}_w${st}_1.log 2>&1; done
done
for w in 3 4; do MIST_LIB=ab/libmist_setup.so timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_setup_c${w}_1.log 2>&1; done
for st in 0.4 0.8 0.9 0.975; do MIST_LIB=ab/libmist_setup.so timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_setup_w${st}_1.log 2>&1; done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
