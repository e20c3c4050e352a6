# usage: bash scripts/gpu_cq2.sh <tag> -- default bench, cfg5 windows 256x2 vs 256x3 (CTA queue), ncu full capture of k_eval_q
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.log 2>&1
for cfg in 256x2 256x3; do
  for st in 0.002 0.4 0.8 0.98; do
   MIST_EVAL_CFG=$cfg timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 0 --steps 1 > gpurun_out/ab_${TAG}_${cfg}_w${st}_1.log 2>&1
  done
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
bash scripts/gpu_prof_eval.sh $TAG
echo done
