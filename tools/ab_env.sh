#!/bin/bash
# A/B of (library, environment) pairs on one box: quick parity subset + bench per pair.
#   bash tools/ab_env.sh "<name>|<lib or ->|<VAR=V ...>" ... (CONFIGS="c3 c5" selects configs)
# lib "-" = the in-tree library; e.g. "order1|-|GP_ITEM_ORDER=1".
for spec in "$@"; do
  IFS='|' read -r name lib envs <<< "$spec"
  [ "$lib" = "-" ] && lib=paper_2110_11226_b200/libgp_b200.so
  ok=$(env GP_B200_LIB=$lib $envs timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fitness_matches_oracle or every_stack_slot or determinism or constant_programs" 2>&1 | tail -1)
  for c in ${CONFIGS:-c3}; do
    line=$(env GP_B200_LIB=$lib $envs timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved 2>/dev/null | tail -1)
    echo "$line" > gpurun_out/abe_${name}_$c.json
    echo "$name $c | $ok | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["evaluate"]; print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms frac", d["roofline"]["frac"], "| eval", e["median_ms"], "ms frac", e["roofline"]["frac"])')"
  done
done
