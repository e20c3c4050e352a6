cd $GRAFT_REPO_ROOT
for st in 0.1 0.4 0.5 0.8 0.98; do
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.02 --warmup 0 --steps 1 > gpurun_out/ctr5_${st}.log 2>&1
done
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --warmup 0 --steps 1 > gpurun_out/ctr2.log 2>&1
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 2 --factors unit --warmup 0 --steps 1 > gpurun_out/ctr2u.log 2>&1
