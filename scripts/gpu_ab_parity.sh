# usage: bash scripts/gpu_ab_parity.sh <tag> <libA> <libB> -- parity subset with the in-tree lib, then same-box A/B
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "small_spaces or cfg1 or frontier_points or big_configs or sharding" > gpurun_out/pytest_quick_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick_$TAG.log
bash scripts/ab_run.sh $TAG "$@"
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
