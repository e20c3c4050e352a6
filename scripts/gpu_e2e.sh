# usage: bash scripts/gpu_e2e.sh <tag> -- full GPU suite; bench (e2e after the fast enumeration + pinned
# frontier cache); 3-CTA eval A/B
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_def_cfg2_$rep.log 2>&1
  MIST_EVAL_CFG=256x3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_c3_cfg2_$rep.log 2>&1
done
for w in 3 4; do
  timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_def_c${w}_1.log 2>&1
  MIST_EVAL_CFG=256x3 timeout 300 python tools/prof_step.py --workload $w --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_c3_c${w}_1.log 2>&1
done
for st in 0.4 0.8 0.9; do
  timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_def_w${st}_1.log 2>&1
  MIST_EVAL_CFG=256x3 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_c3_w${st}_1.log 2>&1
done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
