# quick GPU check: the parity subset plus short bench lines (usage: bash tools/gpu_quick.sh c3 c4 ...)
cfgs=${@:-c3}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomposition.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/pytest_quick.log
for c in $cfgs; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved > gpurun_out/quick_$c.log 2>&1; tail -n 1 gpurun_out/quick_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(d["config"]["workload"][:20], round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])'; done
