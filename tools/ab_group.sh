for g in 0 16 32 64; do
  for c in c4 c5 c3; do
    line=$(GP_PLAN_G=$g timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved 2>/dev/null | tail -1)
    echo "G $g $c | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])')"
  done
done
