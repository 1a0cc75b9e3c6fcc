set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in c4 c5 c3 c2; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_r01_v18_$c.json; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:w4 --launch-skip 3 --launch-count 1 -f -o gpurun_out/prof_r01_v18_c5 python bench.py --config c5 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/prof_c5.log 2>&1
