set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in c3 c4 c5; do timeout 300 python tools/eval_gen0.py 5 $c > gpurun_out/gen0_$c.log 2>&1; tail -2 gpurun_out/gen0_$c.log; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:s4::eval_kernel --launch-skip 1 --launch-count 1 -f -o gpurun_out/ncu_r02_c3gen0 python tools/eval_gen0.py 2 c3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:w4::eval_kernel --launch-skip 1 --launch-count 1 -f -o gpurun_out/ncu_r02_c4gen0 python tools/eval_gen0.py 2 c4 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c3.log gpurun_out/ncu_c4.log
