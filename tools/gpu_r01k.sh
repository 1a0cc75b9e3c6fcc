set -x
ITEMS="32 64 128" CONFIGS="c3 c5" bash tools/ab_items.sh > gpurun_out/abi2.log 2>&1
for lib in paper_2110_11226_b200/_exp/libgp_hot0.so paper_2110_11226_b200/_exp/libgp_hot1.so paper_2110_11226_b200/_exp/libgp_hot0.so paper_2110_11226_b200/_exp/libgp_hot1.so; do
  name=$(basename $lib .so)
  line=$(GP_ITEMS_PER_SLOT=32 GP_B200_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$name | $(echo $line | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e12,3), "Tnode/s", round(d["ms_per_step"],2), "ms", "frac", d["roofline"]["frac"], "gen0", d["roofline_gen0"]["frac"])')" >> gpurun_out/abhot.log
done
