# usage: bash scripts/gpu_cfg5.sh <tag> -- cfg5 whole-space parity test on one GPU
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
MIST_FULLSCALE=1 timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -m gpu -k "5" --timeout=1400 -p no:cacheprovider --durations=0 > gpurun_out/pytest_fullscale_cfg5_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fullscale_cfg5_$TAG.log
echo done
