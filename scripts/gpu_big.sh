# usage: bash scripts/gpu_big.sh <tag>  -- full-space sweeps of cfg3-5 (parity + timing)
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -m gpu -x --timeout=1400 -p no:cacheprovider --durations=0 > gpurun_out/pytest_full_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full_$TAG.log
for w in 3 4 5; do timeout 900 python tools/mgpu_sweep.py --workload $w > gpurun_out/full_${TAG}_cfg$w.log 2>&1; done
echo done
