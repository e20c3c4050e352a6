# usage: bash scripts/gpu_seg.sh <tag> -- full GPU suite, then A/B of the bucket reduction and the zero-offload pilot
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout=1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
run() { # name env...
  local name=$1; shift
  for rep in 1 2; do env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${name}_cfg2_$rep.log 2>&1; done
  for st in 0.4 0.8 0.98; do env "$@" timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_${name}_w${st}_1.log 2>&1; done
}
run new MIST_REDUCE=seg
run radix MIST_REDUCE=radix
run nozero MIST_PILOT_ZERO=0
run old MIST_REDUCE=radix MIST_PILOT_ZERO=0
for r in seg radix; do MIST_REDUCE=$r timeout 300 python tools/sort_bench.py --log2n 26 --groups 4096 > gpurun_out/sort_${TAG}_$r.log 2>&1; done
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_cfg2.log 2>&1
MIST_COUNTERS=1 MIST_PILOT_ZERO=0 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr_${TAG}_cfg2_nozero.log 2>&1
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
