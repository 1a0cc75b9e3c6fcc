export GP_PARITY_LOG=gpurun_out/parity_counts.jsonl
rm -f $GP_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_engine.py -m gpu -x -q -p no:cacheprovider -k "device_mutation or set_population or teacher or thread" > gpurun_out/pytest_t2a.log 2>&1; echo pytest_a=$?
tail -25 gpurun_out/pytest_t2a.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_t2_c3.log 2>&1; echo bench=$?; tail -c 3000 gpurun_out/bench_t2_c3.log
