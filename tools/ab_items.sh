#!/bin/bash
# Work-item granularity sweep (GP_ITEMS_PER_SLOT, default 128) over configs ($ITEMS, $CONFIGS).
for k in ${ITEMS:-32 64 128 256}; do
  for c in ${CONFIGS:-c3 c5}; do
    line=$(GP_ITEMS_PER_SLOT=$k timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved 2>/dev/null | tail -1)
    echo "$line" > gpurun_out/abi_${k}_$c.json
    echo "items/slot $k $c | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])')"
  done
done
