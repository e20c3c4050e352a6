# usage: bash scripts/gpu_sanitize.sh <tag> <pytest -k expr>
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}; K=${2:-buffer_too_small}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "$K" > gpurun_out/plain_$TAG.log 2>&1; echo "plain rc=$?" >> gpurun_out/plain_$TAG.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "$K" > gpurun_out/sanitize_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$TAG.log
echo done
