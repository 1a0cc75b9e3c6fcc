export GP_PARITY_LOG=gpurun_out/parity_counts_wp.jsonl
rm -f $GP_PARITY_LOG
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "wide or global_x or full_size_wide" > gpurun_out/pytest_wp.log 2>&1; echo pytest=$?; tail -n 5 gpurun_out/pytest_wp.log
for c in c5 c4 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved > gpurun_out/wp_$c.log 2>&1; tail -n 1 gpurun_out/wp_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(d["config"]["workload"][:20], round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])'; done
