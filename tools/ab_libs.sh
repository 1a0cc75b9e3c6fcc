#!/bin/bash
# A/B benchmark of alternative library builds on one box: the in-tree library first, then every
# paper_2110_11226_b200/_exp/libgp_*.so (tools/exp_variants.py). Quick parity subset + bench.
#   bash tools/ab_libs.sh [config ...]      (default: c3)
cfgs=${@:-c3}
for lib in paper_2110_11226_b200/libgp_b200.so paper_2110_11226_b200/_exp/libgp_*.so; do
  name=$(basename $lib .so)
  ok=$(GP_B200_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fitness_matches_oracle or every_stack_slot or determinism or constant_programs or global_x" 2>&1 | tail -1)
  for c in $cfgs; do
    line=$(GP_B200_LIB=$lib timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved 2>/dev/null | tail -1)
    echo "$line" > gpurun_out/ab_${name}_$c.json
    echo "$name $c | $ok | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])')"
  done
done
