# usage: bash scripts/gpu_tcut.sh <tag> -- parity subset, tuple-level R7 cut A/B (MIST_R7=unit disables it)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py tests/test_gpu_fullscale.py -q -m gpu -x --timeout=900 -p no:cacheprovider -k "frontier or sharding or fullscale" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for r in 1 unit; do MIST_R7=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_r7${r}_cfg2_$rep.log 2>&1; done
done
for r in 1 unit; do
  for w in 3 4; do MIST_R7=$r timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_r7${r}_c${w}_1.log 2>&1; done
  for st in 0.4 0.8 0.98; do MIST_R7=$r timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_r7${r}_w${st}_1.log 2>&1; done
done
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_cfg2.log 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
