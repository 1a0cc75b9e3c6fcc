set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_r01_v17_c3.json
for c in c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_r01_v17_$c.json; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:w4 --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_r01_v17_c5 python bench.py --config c5 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/prof_c5.log 2>&1
