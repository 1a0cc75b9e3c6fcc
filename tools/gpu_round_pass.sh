# round pass: full GPU suite, smoke, bench lines for every config, reference arm, launch list
#   bash tools/gpu_round_pass.sh <tag>      (outputs gpurun_out/*_<tag>*)
T=${1:-v4}
export GP_PARITY_LOG=gpurun_out/parity_counts_$T.jsonl
rm -f $GP_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$?; tail -n 2 gpurun_out/smoke_$T.log
for c in c3 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${T}_$c.log 2>&1; echo bench_$c=$?
  tail -n 1 gpurun_out/bench_${T}_$c.log > gpurun_out/bench_r02_${T}_$c.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${T}_ref.log 2>&1; echo ref=$?
tail -n 1 gpurun_out/bench_${T}_ref.log > gpurun_out/bench_r02_${T}_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$T.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved --eval-reps 10 > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu=$?
