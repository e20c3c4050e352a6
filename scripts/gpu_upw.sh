# usage: bash scripts/gpu_upw.sh <tag> -- parity subset with MIST_EVAL_UPW=2, then base vs UPW=1 vs UPW=2
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
MIST_EVAL_UPW=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
run() { # name lib upw
  for rep in 1 2 3; do MIST_LIB=$2 MIST_EVAL_UPW=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_$1_cfg2_$rep.log 2>&1; done
  for st in 0.4 0.8 0.98; do MIST_LIB=$2 MIST_EVAL_UPW=$3 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_$1_w${st}_1.log 2>&1; done
}
run base ab/libmist_base2.so 1
run upw1 ab/libmist_upw.so 1
run upw2 ab/libmist_upw.so 2
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
