# usage: bash scripts/gpu_ab4.sh <tag> -- parity subset (in-tree lib), then base vs pc vs pc+tree (256x2, 128x5)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
run() { # name lib cfg
  for rep in 1 2 3; do MIST_LIB=$2 MIST_EVAL_CFG=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_$1_cfg2_$rep.log 2>&1; done
  for st in 0.4 0.8 0.98; do MIST_LIB=$2 MIST_EVAL_CFG=$3 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_$1_w${st}_1.log 2>&1; done
}
run base ab/libmist_base.so 256x2

run wf ab/libmist_wf.so 256x2

python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
