# usage: bash scripts/gpu_cq.sh <tag> -- parity subset (CTA queue default), then warp queue vs CTA queue A/B
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_cq_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cq_$TAG.log
for rep in 1 2 3; do
 for q in 1 2; do
  for cfg in 256x3 256x2; do
   MIST_EVAL_QUEUE=$q MIST_EVAL_CFG=$cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_q${q}_${cfg}_cfg2_$rep.log 2>&1
  done
 done
done
for q in 1 2; do
  for st in 0.4 0.8; do
   MIST_EVAL_QUEUE=$q timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ab_${TAG}_q${q}_256x3_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
