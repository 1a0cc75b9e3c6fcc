#!/usr/bin/env python
"""Summarise an ncu report (or a launch-list CSV) into profiles/: markdown + JSON.

    python tools/ncu_summary.py full gpurun_out/prof_eval.ncu-rep profiles/ncu_eval_rNN
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/launches_rNN
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
]
STALLS = "smsp__average_warps_issue_stalled_"


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        for key in KEYS:
            if key in d:
                k[key] = f"{d[key]} {u[key]}".strip()
        k["stalls_per_issue"] = {h[len(STALLS):].replace("_per_issue_active.ratio", ""): d[h]
                                 for h in hdr if h.startswith(STALLS) and h.endswith(
                                     "_per_issue_active.ratio") and d[h] not in ("", "0")}
        kernels.append((k, d, u))
    def val(d, u, key):
        v, un = float(d[key].replace(",", "")), u[key]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(un, 1)

    def ms(d, u):
        v, un = float(d["gpu__time_duration.sum"].replace(",", "")), u["gpu__time_duration.sum"]
        return v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}.get(un, 1)

    per = []
    for k, d, u in kernels:
        k["dram_bytes"] = val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
        k["ms"] = ms(d, u)
        per.append(k)
    dram = sum(k["dram_bytes"] for k in per)
    # the captured launches are the eval-kernel launches of ONE evaluation (one per non-empty
    # stack-need variant): their summed DRAM traffic is the traffic of one evaluation
    summary = {"report": rep, "kernels": [k["kernel"] for k in per],
               "dram_bytes_per_launch": dram, "traffic_scope": "one evaluation (sum over the "
               "captured eval-kernel launches)", "per_kernel": per}
    json.dump(summary, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu --set full\n\nsource report: `{rep}`\n\n"
                f"DRAM read+write summed over the {len(per)} captured launches: {dram:.4g} B\n\n")
        for k in per:
            f.write(f"## {k['kernel']}\n\n| metric | value |\n|---|---|\n")
            for key in KEYS:
                if key in k:
                    f.write(f"| {key} | {k[key]} |\n")
            f.write(f"| dram bytes (read+write) | {k['dram_bytes']:.4g} B |\n\n"
                    "stall reasons (warps per issue):\n\n")
            for s, v in sorted(k["stalls_per_issue"].items(), key=lambda x: -float(x[1]))[:12]:
                f.write(f"- {s}: {float(v):.3f}\n")
            f.write("\n")
    print(open(out + ".md").read())


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0]
            t[name] += float(d["Metric Value"])
            n[name] += 1
    tot = sum(t.values())
    with open(out + ".md", "w") as f:
        f.write(f"# launch list (ncu gpu__time_duration.sum, --clock-control none)\n\nsource: `{path}`\n\n"
                "| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k in sorted(t, key=lambda k: -t[k]):
            f.write(f"| `{k}` | {n[k]} | {t[k] / 1e6:.3f} | {100 * t[k] / tot:.2f}% |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
