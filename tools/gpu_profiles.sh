# r02 profiles of the current build: per-config DRAM traffic launch lists, ncu --set full of the
# step's evaluator launch (C3 s4, C4 / C5 w4), the C5 population sweep
B="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved --eval-reps 10"
for c in c3 c4 c5; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/traffic_v4_$c.csv python bench.py --config $c $B > gpurun_out/traffic_v4_$c.log 2>&1; echo traffic_$c=$?
done
F="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved --eval-reps 10"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:s4::eval_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_r02_v4_c3step python bench.py --config c3 $F > gpurun_out/ncu_c3step.log 2>&1; echo ncu_c3=$?
for c in c4 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:w4::eval_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_r02_v4_${c}step python bench.py --config $c $F > gpurun_out/ncu_${c}step.log 2>&1; echo ncu_$c=$?
done
for p in 1024 2048 4096 8192 16384 32768 65536; do
  timeout 900 python bench.py --config c5 --pop $p --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved > gpurun_out/c5sweep_$p.log 2>&1; echo sweep_$p=$?
  tail -n 1 gpurun_out/c5sweep_$p.log > gpurun_out/c5sweep_$p.json
done
