set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_r01_v14_c3.json
