# usage: bash scripts/gpu_scale.sh <tag> <N>  -- multirank tests, bench at 1..N, full cfg5 sweep at N
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}; N=${2:-4}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$TAG.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_multi_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi_$TAG.log
n=1
while [ $n -le $N ]; do
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_n1.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_n$n.log 2>&1
  fi
  echo "rc=$?" >> gpurun_out/bench_${TAG}_n$n.log
  n=$((n*2))
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/mgpu_sweep.py --workload 5 --plan > gpurun_out/cfg5_${TAG}_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_${TAG}_n$N.log
echo done
