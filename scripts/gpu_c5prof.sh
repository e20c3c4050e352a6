# usage: bash scripts/gpu_c5prof.sh <tag> -- cfg5 cost profile along the tuple range (0.5% windows, counters build)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
for st in 0.0 0.05 0.1 0.15 0.2 0.25 0.3 0.35 0.4 0.45 0.5 0.55 0.6 0.65 0.7 0.75 0.8 0.85 0.9 0.925 0.95 0.975 0.99 0.995; do
  echo "== $st" >> gpurun_out/c5prof_$TAG.log
  MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.005 --warmup 0 --steps 1 >> gpurun_out/c5prof_$TAG.log 2>&1
done
echo done
