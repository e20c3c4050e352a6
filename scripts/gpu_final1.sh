# usage: bash scripts/gpu_final1.sh <tag> -- new parity test + cfg5 whole-space parity test on one GPU
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=500 -p no:cacheprovider -k "prepare_cache or retry or out_of_range" > gpurun_out/pytest_new_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new_$TAG.log
MIST_FULLSCALE=1 timeout 1800 python -m pytest tests/test_gpu_fullscale.py -q -m gpu --timeout=1700 -p no:cacheprovider --durations=0 > gpurun_out/pytest_fullscale_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fullscale_$TAG.log
echo done
