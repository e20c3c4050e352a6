cd $GRAFT_REPO_ROOT
for st in 0.0 0.1 0.2 0.3 0.4 0.5 0.6 0.7 0.8 0.9 0.98; do
timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.02 --warmup 0 --steps 1 > gpurun_out/win5_${st}.log 2>&1
done
