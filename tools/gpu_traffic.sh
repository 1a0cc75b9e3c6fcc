# per-config DRAM traffic launch lists (ncu dram counters, caches NOT flushed between launches, as in a bench run) + C4 / C5 bench lines
T=${1:-v4b}
B="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved --eval-reps 10"
for c in c3 c4 c5; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/traffic_${T}_$c.csv python bench.py --config $c $B > gpurun_out/traffic_${T}_$c.log 2>&1; echo traffic_$c=$?
done
for c in c4 c5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${T}_$c.log 2>&1; echo bench_$c=$?; tail -n 1 gpurun_out/bench_${T}_$c.log > gpurun_out/bench_r02_${T}_$c.json; done
