# DRAM traffic of every eval-kernel launch of a C3 bench run (cheap metrics, all launches) and the
# final populations of C3/C4/C5 for offline analysis.
set -x
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/traffic.log 2>&1
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --dump-population gpurun_out/pop_$c.npz > gpurun_out/dump_$c.log 2>&1; done
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2e_$c.log 2>&1; done
