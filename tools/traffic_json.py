#!/usr/bin/env python
"""profiles/eval_kernel_ncu_<config>.json from a launch list with dram counters (bench.py reads its
dram_bytes_per_launch as roofline.traffic).

    python tools/traffic_json.py gpurun_out/traffic_c3.csv c3 ALGORITHMIC_BYTES
"""
import collections
import csv
import json
import sys

src, cfg, alg = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(src)))
hdr, data = None, collections.defaultdict(dict)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    e = data[int(d["ID"])]
    e["k"] = d["Kernel Name"]
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
per = collections.defaultdict(list)
for _, d in sorted(data.items()):
    if "eval_kernel" in d["k"]:
        per[d["k"].split("(")[0].replace("void ", "")].append(
            d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
n_eval = max(len(v) for v in per.values())
out = {"source": f"{src} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                 "gpu__time_duration.sum --clock-control none --cache-control none, every launch of `python bench.py "
                 "--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-evolved`, config " + cfg + ")",
       "evaluations": n_eval,
       "per_variant_bytes_per_evaluation": {k: sum(v) / n_eval for k, v in per.items()},
       "algorithmic_bytes_per_evaluation": alg,
       "note": "one evaluation = one launch per non-empty stack-need variant; reads of X, y "
               "plus the fp64 partial-sum writes; caches are not flushed between launches (--cache-control none), as in a bench run",
       "dram_bytes_per_launch": sum(sum(v) for v in per.values()) / n_eval}
json.dump(out, open(f"profiles/eval_kernel_ncu_{cfg}.json", "w"), indent=1)
print(json.dumps(out["per_variant_bytes_per_evaluation"]), out["dram_bytes_per_launch"])
