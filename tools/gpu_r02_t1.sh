export GP_PARITY_LOG=gpurun_out/parity_counts.jsonl
rm -f $GP_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_t1.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_t1.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_t1.log 2>&1; tail -c 1500 gpurun_out/bench_t1.log
