set -x
ncu --set full --clock-control none --import-source on -k regex:eval_kernel --launch-skip 10 --launch-count 2 -f -o gpurun_out/prof_r01_v9 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v9.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launch.log 2>&1
for c in c2 c3 c4 c5; do timeout 600 python bench.py --config $c > gpurun_out/bench_v9_$c.log 2>&1; tail -1 gpurun_out/bench_v9_$c.log > gpurun_out/bench_r01_v9_$c.json; done
