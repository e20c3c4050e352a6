# usage: bash scripts/gpu_full.sh <tag> <N>  -- parity tests, multi-GPU test, smoke, bench at 1..N
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}; N=${2:-1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --maxfail=8 --timeout=600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_n1.log 2>&1
MIST_PILOT=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_nopilot.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --factors unit > gpurun_out/bench_${TAG}_unit.log 2>&1
n=2
while [ $n -le $N ]; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_n$n.log 2>&1
  n=$((n*2))
done
echo done
