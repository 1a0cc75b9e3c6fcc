# Final round-1 GPU pass: parity tests, smoke, bench C3 (full line), reference arm, launch list + ncu of the evaluator.
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_r01_final_c3.json
for c in c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_r01_final_$c.json; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_r01_final_reference.json
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel --launch-skip 10 --launch-count 1 -f -o gpurun_out/prof_r01_final python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof.log 2>&1
