cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout=600 -p no:cacheprovider -k "small_spaces or cfg1 or cfg2 or big_configs or sharding" > gpurun_out/pytest_k0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k0.log
for st in 0.4 0.8 0.98; do
MIST_COUNTERS=1 timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.02 --warmup 0 --steps 1 > gpurun_out/k0c5_${st}.log 2>&1
timeout 300 python tools/prof_step.py --workload 5 --start $st --fraction 0.02 --warmup 0 --steps 1 > gpurun_out/k05_${st}.log 2>&1
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_k0.log 2>&1
