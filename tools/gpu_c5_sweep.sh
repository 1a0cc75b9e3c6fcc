# C5 population sweep (BASELINE configs[4]): 1K-64K programs at 1M rows x 90 columns
for p in 1024 2048 4096 8192 16384 32768 65536; do
  timeout 900 python bench.py --config c5 --pop $p --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved > gpurun_out/c5sweep_$p.log 2>&1; echo sweep_$p=$?
  tail -n 1 gpurun_out/c5sweep_$p.log > gpurun_out/c5sweep_$p.json
done
