# usage: bash scripts/gpu_dedup.sh <tag> -- parity subset, L20-twin skip A/B (MIST_DEDUP=0 disables)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py tests/test_gpu_sample.py tests/test_gpu_inter.py -q -m gpu -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for r in 1 0; do MIST_DEDUP=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_dd${r}_cfg2_$rep.log 2>&1; done
done
for r in 1 0; do
  for w in 3 4; do MIST_DEDUP=$r timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_dd${r}_c${w}_1.log 2>&1; done
  for st in 0.4 0.8 0.975 0.99; do MIST_DEDUP=$r timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_dd${r}_w${st}_1.log 2>&1; done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
