# usage: bash scripts/gpu_ntq.sh <tag> -- parity subset with MIST_EVAL_NTQ=3/4, then cfg2 bench + cfg5 windows for UPW 2/3/4 (same library)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for U in 320 192; do
MIST_EVAL_NTQ=$U timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer" > gpurun_out/pytest_${TAG}_ntq$U.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}_ntq$U.log
done
for rep in 1 2 3; do for U in 256 320 192; do
  MIST_EVAL_NTQ=$U timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_ntq${U}_cfg2_$rep.log 2>&1
done; done
for st in 0.4 0.8 0.98; do for U in 256 320 192; do
  MIST_EVAL_NTQ=$U timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.01 --warmup 1 --steps 1 > gpurun_out/ab_${TAG}_ntq${U}_w${st}_1.log 2>&1
done; done
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
