# usage: bash scripts/gpu_tree.sh <tag> -- parity subset with the in-tree library, then same-box A/B of ab/libmist_base.so vs ab/libmist_tree.so
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_presets.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "frontier or sharding or buffer or eval" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
bash scripts/ab_run.sh $TAG ab/libmist_base.so ab/libmist_tree.so
python scripts/ab_summ.py $TAG > gpurun_out/ab_${TAG}_summary.txt 2>&1
echo done
