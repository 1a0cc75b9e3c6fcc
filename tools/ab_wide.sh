#!/bin/bash
# A/B of alternative library builds on the wide-data (global-X) configs C4 / C5.
for lib in paper_2110_11226_b200/libgp_b200.so paper_2110_11226_b200/_exp/libgp_*.so; do
  name=$(basename $lib .so)
  for c in c4 c5; do
    line=$(GP_B200_LIB=$lib timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
    echo "$line" > gpurun_out/abw_${name}_$c.json
    echo "$name $c | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms", "frac", d["roofline"]["frac"], "gen0", d["roofline_gen0"]["frac"])')"
  done
done
