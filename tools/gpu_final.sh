# final evidence pass of a build: GPU suite + smoke, bench lines (every config + reference),
# launch list, DRAM traffic per config (caches not flushed), ncu --set full of the step's
# evaluator launches (C3 s4, C4 / C5 w4)
#   bash tools/gpu_final.sh <tag>
T=${1:-v5}
bash tools/gpu_round_pass.sh $T
bash tools/gpu_traffic.sh $T
F="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved --eval-reps 10"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:s4::eval_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_r02_${T}_c3step python bench.py --config c3 $F > gpurun_out/ncu_${T}_c3step.log 2>&1; echo ncu_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:w4::eval_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_r02_${T}_c4step python bench.py --config c4 $F > gpurun_out/ncu_${T}_c4step.log 2>&1; echo ncu_c4=$?
