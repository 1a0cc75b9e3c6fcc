#!/usr/bin/env python
"""Benchmark of the B200 hot path of arXiv 2110.11226.

Metric (BASELINE.json): GP node-evals/sec and sec/generation at Pagie 16M rows (config C3:
Pagie-1 on the 4096 x 4096 grid = 16,777,216 rows, population 8192, MSE).

One step = one gp_generation from a FIXED population: the engine is reset to the generation-0
(ramped half-and-half) population and its fitness (gp_engine_set_population, device to device),
then runs tournament selection, mutation (both on the GPU), compile + fused evaluation +
reduction (+ all-reduce at N > 1) + finalize of the children -- every row of SURVEY section 8(a) on
the same workload every step, so the number does not drift with the run length (a free-running
population collapses under parsimony pressure, see the "evolved" field). value = node evaluations
(sum of the children's lengths x dataset rows, all ranks) per second of device time (CUDA events on
the engine stream, max over ranks).

Also reported: "evaluate" (gp_evaluate alone on the generation-0 population, median of >= 10 reps),
"evolved" (sec/generation of consecutive generations from generation 0), the evaluator roofline,
the oracle baseline (1 thread and all cores) and the end-to-end number (dataset streamed from
pinned host memory every step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c3]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, rows sharded)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "GP node-evals/sec and sec/generation at Pagie 16M rows, 1/2/4/8 B200"
CONFIGS = {
    # BASELINE.json configs; c3 is the metric's workload (fits one GPU).
    "c1": dict(workload="Pagie-1 64x64 (4,096 rows x 2), population 256, MSE", data="pagie",
               side=64, pop=256, metric="mse", depth=(2, 6)),
    "c2": dict(workload="Pagie-1 1024x1024 (1,048,576 rows x 2), population 1024, MSE",
               data="pagie", side=1024, pop=1024, metric="mse", depth=(2, 6)),
    "c3": dict(workload="Pagie-1 4096x4096 (16,777,216 rows x 2), population 8192, MSE",
               data="pagie", side=4096, pop=8192, metric="mse", depth=(2, 6)),
    "c4": dict(workload="Higgs-shaped 11,000,000 rows x 28, population 4096, log-loss",
               data="higgs", rows=11_000_000, pop=4096, metric="logloss", depth=(2, 6)),
    "c5": dict(workload="Year-shaped 1,048,576 rows x 90, population 8192, RMSE, depth 2-8",
               data="year", rows=1_048_576, pop=8192, metric="rmse", depth=(2, 8)),
}
# Algorithmic SFU (MUFU) operations per node-row: the transcendental /
# reciprocal evaluations each function needs at the least (tan = one reciprocal after a range
# reduction and a polynomial, 13 FP32 ops; sin / cos one MUFU each). Counted only for nodes whose
# subtree depends on a variable (stats op_count); variable-free subtrees are per-program
# constants, not per-row work.
SFU_COST = {5: 1, 9: 1, 10: 1, 11: 1, 14: 1, 15: 1, 16: 1, 17: 1, 8: 2, 20: 2, 21: 2, 22: 2,
            23: 1, 24: 1, 25: 1}
FP32_COST = {2: 1, 3: 1, 4: 1, 5: 1, 6: 1, 7: 1, 9: 1, 10: 1, 11: 13, 12: 1, 13: 1, 18: 1, 19: 2}
LOSS_FP32 = {"mae": 3, "mse": 3, "rmse": 3, "logloss": 7, "pearson": 5}
LOSS_SFU = {"logloss": 2}
# B200: 148 SMs x 16 MUFU lanes x 1965 MHz (sm_max_mhz); microbenchmarked 4.63e12 MUFU.SIN/s
# (profiles/pipe_peaks_r01.txt). FP32: 148 x 128 lanes x 1965 MHz.
SFU_PEAK = 148 * 16 * 1965e6
FP32_PEAK = 148 * 128 * 1965e6
# L2 read bandwidth, measured: tools/l2_peak.cu (16-byte ld.global.cg loads of an L2-resident
# buffer from every SM; profiles/l2_peak_r02.txt)
L2_PEAK_GBS = 18548.6


def load_dataset(cfg, rank=0, world=1):
    """Synthetic dataset of the config, this rank's contiguous shard,
    plus the global first row (Pearson reference) and global row count."""
    if cfg["data"] == "pagie":
        X, y = synth.pagie_grid(cfg["side"])
    elif cfg["data"] == "higgs":
        X, y = synth.higgs_like(cfg["rows"], seed=2110)
    else:
        X, y = synth.year_like(cfg["rows"], seed=2110)
    m = X.shape[1]
    r0, r1 = synth.shard_rows(m, rank, world)
    return (np.ascontiguousarray(X[:, r0:r1]), np.ascontiguousarray(y[r0:r1]), X[:, 0].copy(),
            float(y[0]), m)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.stop_ev = device, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit()
                else None, "reasons": reasons, "samples": len(self.rows)}


# metrics whose variable-free programs get their fitness from the dataset moments (no per-row
# loss; gp_context_set_const_programs)
CLOSED_FORM_METRICS = ("mse", "rmse", "logloss", "pearson")


def algorithmic_ops(op_count, rows, metric, n_programs, const_programs=0):
    """Per-row algorithmic work of one evaluation: SFU / FP32 ops of the variable-dependent nodes
    plus the loss of every program evaluated per row (constant programs under a closed-form
    metric have no per-row loss)."""
    sfu = sum(SFU_COST.get(op, 0) * c for op, c in enumerate(op_count)) * rows
    fp32 = sum(FP32_COST.get(op, 0) * c for op, c in enumerate(op_count)) * rows
    per_row = n_programs - (const_programs if metric in CLOSED_FORM_METRICS else 0)
    sfu += LOSS_SFU.get(metric, 0) * per_row * rows
    fp32 += LOSS_FP32[metric] * per_row * rows
    return sfu, fp32


def l2_operands(var_nodes, rows, eval_ms):
    """Wide datasets (X read through L1/L2): every variable operand of a
    variable-dependent node is a 4-byte L2 read per row (no shared-memory X tile); achieved rate of
    those reads against the measured L2 read bandwidth (tools/l2_peak.cu)."""
    b = float(var_nodes) * rows * 4
    gbs = b / (eval_ms * 1e-3) / 1e9
    return {"bytes": b, "achieved": round(gbs, 1), "peak": L2_PEAK_GBS, "unit": "GB/s",
            "frac": round(gbs / L2_PEAK_GBS, 4),
            "note": "variable-operand reads (variable nodes x rows x 4 B) / eval time vs the "
                    "measured L2 read bandwidth (profiles/l2_peak_r02.txt)"}


def roofline_of(sfu, fp32, eval_ms, launches, step_ms, traffic=None, l2_var_nodes=None,
                rows=None):
    """Binding ALU pipe of the evaluator for the given algorithmic work: SFU (MUFU) or FP32; for
    wide datasets also the L2 rate of the variable-operand reads (l2_var_nodes x rows)."""
    eval_s = eval_ms * 1e-3
    f_sfu, f_fp32 = sfu / eval_s / SFU_PEAK, fp32 / eval_s / FP32_PEAK
    if f_sfu >= f_fp32:
        r = {"bound": "alu", "pipe": "SFU (MUFU)", "achieved": round(sfu / eval_s / 1e12, 4),
             "peak": round(SFU_PEAK / 1e12, 4), "unit": "Tops/s (MUFU)", "frac": round(f_sfu, 4)}
    else:
        r = {"bound": "alu", "pipe": "FP32", "achieved": round(fp32 / eval_s / 1e12, 4),
             "peak": round(FP32_PEAK / 1e12, 4), "unit": "TFLOP/s (fp32)", "frac": round(f_fp32, 4)}
    tr = ncu_traffic(traffic) if traffic else None
    r.update({"traffic": tr,
              "traffic_scope": (f"DRAM bytes of one evaluation's eval launches of the step "
                                f"(profiles/eval_kernel_ncu_{traffic}.json)") if tr else None,
              "sfu_frac": round(f_sfu, 4), "fp32_frac": round(f_fp32, 4),
              "eval_ms_per_launch": round(eval_ms / max(launches, 1), 3),
              "eval_share_of_step": round(eval_ms / step_ms, 4),
              "peak_note": "SFU: 148 SMs x 16 MUFU/clk x 1965 MHz (measured MUFU.SIN 4.63e12/s); "
                           "FP32: 148 x 128 x 1965 MHz",
              "work_note": "per-row work of variable-dependent nodes only; tan = 1 SFU op (range "
                           "reduction + polynomial + one reciprocal, 13 FP32 ops; r01 counted 3: "
                           "sin, cos, rcp), DESIGN.md section 8"})
    if l2_var_nodes is not None:
        r["l2_operands"] = l2_operands(l2_var_nodes, rows, eval_ms)
    return r


def ncu_traffic(config="c3"):
    """DRAM bytes per evaluation (all variant launches) from the committed launch list with dram
    counters of this config (tools/traffic_json.py), if present."""
    path = os.path.join(ROOT, "profiles", f"eval_kernel_ncu_{config}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")   # per evaluation (all variants)
    except Exception:
        return None


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_chunk(job):
    """Worker of the all-core oracle mode: one contiguous program chunk, single-threaded."""
    import oracle
    nodes, off, X, y, metric = job
    oracle.population_fitness(nodes, off, X, y, None, metric)
    return float(np.diff(off).sum()) * X.shape[1]


def cpu_baseline(nodes, off, X, y, metric, max_seconds=12.0):
    """The oracle (C, double, recursive, as it stands) on a bounded sample: all programs of the
    population on the first rows of this rank's shard; 1 thread, then all host cores (processes
    over program chunks -- the oracle itself is not changed)."""
    import multiprocessing as mp

    import oracle
    oracle.build()
    lens = np.diff(off)
    n_rows = 128
    t0 = time.perf_counter()
    oracle.population_fitness(nodes, off, X[:, :n_rows], y[:n_rows], None, metric)
    dt = time.perf_counter() - t0
    rows = int(min(X.shape[1], max(n_rows, n_rows * (max_seconds * 0.5) / max(dt, 1e-6))))
    Xs, ys = np.ascontiguousarray(X[:, :rows]), np.ascontiguousarray(y[:rows])
    t0 = time.perf_counter()
    oracle.population_fitness(nodes, off, Xs, ys, None, metric)
    dt1 = time.perf_counter() - t0
    one = float(lens.sum()) * rows / dt1
    cores = len(os.sched_getaffinity(0))
    allc = None
    if cores > 1:
        n = len(off) - 1
        bounds = [n * k // cores for k in range(cores + 1)]
        jobs = [(nodes[off[a]:off[b]], off[a:b + 1] - off[a], Xs, ys, metric)
                for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        try:
            with mp.get_context("fork").Pool(cores) as pool:
                t0 = time.perf_counter()
                work = sum(pool.map(_oracle_chunk, jobs))
                dta = time.perf_counter() - t0
            allc = {"value": work / dta, "cores": cores,
                    "sample": f"same sample, programs split over {cores} processes ({dta:.1f} s)"}
        except Exception as ex:                       # no fork / no /dev/shm: report why
            allc = {"value": None, "cores": cores, "error": str(ex)[:200]}
    return {"value": one, "unit": "node-evals/s", "cores": 1, "kind": "oracle",
            "cpu_model": _cpu_model(), "host_cores": cores,
            "sample": f"all {len(lens)} programs of the step's children x first {rows} rows "
                      f"({dt1:.1f} s, C double recursive, 1 thread)",
            "all_cores": allc}


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2110_11226_b200 as gp

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = None
    if world > 1 or args.nccl:
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [gp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.Stream(local)
    ctx = gp.Context(local, stream=stream, unique_id=uid, rank=rank, world_size=world)
    ctx.set_const_programs(not args.no_const_programs)
    by_prog = args.shard == "programs"
    if by_prog:                                   # all rows on every rank
        ctx.set_shard("programs")
    Xh, yh, x0, y0, m_global = load_dataset(cfg, 0 if by_prog else rank, 1 if by_prog else world)
    ctx.set_reference_row(x0, y0)
    X = torch.from_numpy(Xh).cuda(local)
    y = torch.from_numpy(yh).cuda(local)
    torch.cuda.synchronize()
    kw = dict(population_size=cfg["pop"], metric=cfg["metric"], seed=2110,
              init_depth_min=cfg["depth"][0], init_depth_max=cfg["depth"][1],
              device_mutation=0 if args.host_mutation else 1)
    eng = gp.Engine(ctx, X, y, **kw)
    st0 = eng.init_population()
    g0n, g0o, g0f = eng.population_device()        # the fixed starting population (HBM)
    n0_len = int(g0n.shape[0])
    rows_local = X.shape[1] / (world if by_prog else 1)

    def step(e):
        e.set_population(g0n, g0o, g0f, generation=0, stats=False)   # device copies, no sync
        return e.generation()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t]

    for _ in range(args.warmup):
        step(eng)

    # ---- timed region: K steps, inputs resident in HBM ---------------------------------------
    ctx.set_profiling(True)
    ctx.eval_timing(reset=True)
    ctx.kernel_launches(reset=True)
    steps = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            steps.append(step(eng))
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    eval_ms, eval_launches = ctx.eval_timing(reset=True)
    launches = ctx.kernel_launches(reset=True)
    ctx.set_profiling(False)
    ms, eval_ms = max_over_ranks([ms, eval_ms])
    node_evals = sum(s["total_nodes"] for s in steps) * m_global
    value = node_evals / (ms * 1e-3)
    sfu = fp32 = 0
    for s in steps:
        a, b2 = algorithmic_ops(s["op_count"], rows_local, cfg["metric"], cfg["pop"],
                                0 if args.no_const_programs else s["const_programs"])
        sfu, fp32 = sfu + a, fp32 + b2
    wide = cfg["data"] != "pagie"            # X through L1/L2 (no shared-memory X tile)
    roofline = roofline_of(sfu, fp32, eval_ms, eval_launches, ms, traffic=args.config,
                           l2_var_nodes=sum(s["op_count"][0] for s in steps) if wide else None,
                           rows=rows_local)

    # ---- gp_evaluate alone on the fixed generation-0 population (SURVEY D definition) -----------
    fit_buf = torch.empty(cfg["pop"], dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(2):
        ctx.evaluate(g0n, g0o, X, y, metric=cfg["metric"], max_stack=20, fitness_out=fit_buf)
    torch.cuda.synchronize()
    reps = max(10, args.eval_reps)
    times = []
    ctx.set_profiling(True)
    ctx.eval_timing(reset=True)
    for _ in range(reps):
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ctx.evaluate(g0n, g0o, X, y, metric=cfg["metric"], max_stack=20, fitness_out=fit_buf)
        a1.record(stream)
        torch.cuda.synchronize()
        times.append(max_over_ranks([a0.elapsed_time(a1)])[0])
    k_ms, k_l = ctx.eval_timing(reset=True)
    ctx.set_profiling(False)
    t_med = statistics.median(times)
    a0_, b0_ = algorithmic_ops(st0["op_count"], rows_local, cfg["metric"], cfg["pop"],
                               0 if args.no_const_programs else st0["const_programs"])
    roof0 = roofline_of(a0_ * reps, b0_ * reps, k_ms, k_l, k_ms,
                        l2_var_nodes=st0["op_count"][0] * reps if wide else None, rows=rows_local)
    evaluate = {"population": "generation 0 (ramped half-and-half), mean length %.2f"
                              % (n0_len / cfg["pop"]),
                "reps": reps, "median_ms": round(t_med, 3), "min_ms": round(min(times), 3),
                "max_ms": round(max(times), 3),
                "node_evals_per_s": n0_len * m_global / (t_med * 1e-3),
                "row_program_evals_per_s": cfg["pop"] * m_global / (t_med * 1e-3),
                "t_eval_scope": "gp_evaluate call: compile, evaluator, reduction, "
                                "all-reduce (N > 1), finalize (CUDA events, max over ranks)",
                "roofline": roof0}

    # ---- evolved: consecutive generations from generation 0 (the population drifts) -----------
    evolved = None
    if not args.no_evolved:
        eng.set_population(g0n, g0o, g0f, generation=0)
        ev_steps, ev_ms = [], []
        for _ in range(args.evolved_gens):
            barrier()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            ev_steps.append(eng.generation())
            b1.record(stream)
            torch.cuda.synchronize()
            ev_ms.append(max_over_ranks([b0.elapsed_time(b1)])[0])
        tot = sum(ev_ms)
        evolved = {
            "generations": args.evolved_gens,
            "sec_per_generation_median": statistics.median(ev_ms) / 1e3,
            "nominal_node_evals_per_s": sum(s["total_nodes"] for s in ev_steps) * m_global / (tot * 1e-3),
            "var_node_evals_per_s": sum(sum(s["op_count"]) for s in ev_steps) * m_global / (tot * 1e-3),
            "mean_program_length_last": ev_steps[-1]["total_nodes"] / cfg["pop"],
            "const_node_share_last": round(ev_steps[-1]["const_nodes"] / max(1, ev_steps[-1]["total_nodes"]), 4),
            "const_program_share_last": round(ev_steps[-1]["const_programs"] / cfg["pop"], 4),
            "note": "nominal counts every node x row, incl. variable-free subtrees folded at compile "
                    "time and closed-form constant programs; var_node_evals counts only "
                    "variable-dependent nodes"}

    # ---- end-to-end: dataset streamed from pinned host memory every step -----------------------
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(Xh).pin_memory()
        yp = torch.from_numpy(yh).pin_memory()
        for _ in range(2):
            eng.set_dataset(Xp, yp)
            step(eng)
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        e2e_steps = []
        for _ in range(args.steps):
            eng.set_dataset(Xp, yp)
            e2e_steps.append(step(eng))
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms2 = max_over_ranks([f0.elapsed_time(f1)])[0]
        # per step the engine reads back the child node total (8 B), tournament count and error
        # word (4 + 4 B) and the statistics record (op histogram, best, mean); the host mutation
        # path also copies the population and reads fitness + winners
        dev_mut = not args.host_mutation
        d2h = 16 + 280 if dev_mut else int(cfg["pop"] * 4 + 2 * cfg["pop"] * 4)
        h2d_pop = 0 if dev_mut else int(np.mean([s["total_nodes"] for s in e2e_steps]) * 8 + (cfg["pop"] + 1) * 8)
        e2e = {"value": sum(s["total_nodes"] for s in e2e_steps) * m_global / (ms2 * 1e-3),
               "unit": "node-evals/s",
               "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes + h2d_pop),
               "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(ms2 / args.steps, 3)}
        eng.set_dataset(X, y)

    out = None
    if rank == 0:
        nodes, off, _ = eng.population()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            eng.set_population(g0n, g0o, g0f, generation=0)
            eng.generation()                              # the step's children
            nodes, off, _ = eng.population()
            cpu = cpu_baseline(nodes, off, Xh, yh, cfg["metric"])
        mean_len = float(np.mean([s["total_nodes"] for s in steps])) / cfg["pop"]
        out = {
            "metric": METRIC, "value": value, "unit": "node-evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "sec_per_generation": ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, DESIGN.md recipe)",
            "config": {"workload": cfg["workload"], "rows": m_global, "population": cfg["pop"],
                       "metric": cfg["metric"], "mean_program_length": round(mean_len, 3),
                       "step": "gp_generation from the fixed generation-0 population (reset every "
                               "step): GPU selection + mutation, evaluation of the children",
                       "mutation": "host" if args.host_mutation else "device (SURVEY F2)",
                       "parallelism": (f"programs sharded over {world} GPU(s), fitness all-gathered"
                                       if by_prog else f"rows sharded over {world} GPU(s)"),
                       "l2": "inputs larger than L2 (X + y = %.0f MB)" % ((Xh.nbytes + yh.nbytes) * world / 1e6)},
            "roofline": roofline, "evaluate": evaluate, "evolved": evolved,
            "var_node_evals_per_s": sum(sum(s["op_count"]) for s in steps) * m_global / (ms * 1e-3),
            "const_node_share": round(float(np.mean([s["const_nodes"] / max(1, s["total_nodes"]) for s in steps])), 4),
            "const_program_share": round(float(np.mean([s["const_programs"] / cfg["pop"] for s in steps])), 4),
            "const_programs_closed_form": (not args.no_const_programs) and cfg["metric"] in CLOSED_FORM_METRICS,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "phases_ms_per_step": {k: round(1e3 * float(np.mean([s[k] for s in steps])), 3)
                                   for k in ("t_select_s", "t_mutate_s", "t_h2d_s", "t_eval_s")},
        }
    eng.close()
    ctx.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return out


def run_reference(args, cfg):
    """--impl reference: the oracle (C evaluation + Python engine replay) on the host cores, each
    step the same step as the b200 arm -- one generation from the fixed generation-0 population --
    with the children evaluated on a bounded row sample."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return None
    import oracle
    from oracle import engine as oe
    oracle.build()
    Xh, yh, _, _, m = load_dataset(cfg, 0, 1)
    sample = 1024 if cfg["pop"] >= 4096 else 4096
    Xs, ys = np.ascontiguousarray(Xh[:, :sample]), np.ascontiguousarray(yh[:sample])
    ocfg = oe.Config(population_size=cfg["pop"], metric=cfg["metric"], seed=2110,
                     init_depth=cfg["depth"], n_features=Xh.shape[0])
    pop0 = oe.ramped_init(ocfg)
    nodes, off = oe.flatten(pop0)
    fit0, _, _ = oracle.population_fitness(nodes, off, Xs, ys, None, cfg["metric"])
    hb = cfg["metric"] == "pearson"
    total = 0.0
    evals = 0
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rec = oe.next_generation(pop0, fit0.astype(np.float32), ocfg, 1, hb)
        nodes, off = oe.flatten(rec.population)
        oracle.population_fitness(nodes, off, Xs, ys, None, cfg["metric"])
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            total += dt
            evals += int(np.diff(off).sum()) * sample
    value = evals / total
    return {"metric": METRIC, "value": value, "unit": "node-evals/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, DESIGN.md recipe)",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "rows": m, "population": cfg["pop"],
                       "metric": cfg["metric"], "parallelism": "host, 1 thread",
                       "step": "one generation from the fixed generation-0 population"},
            "cpu_baseline": {"value": value, "unit": "node-evals/s", "cores": 1, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"each step: one generation (oracle select + mutate + "
                                       f"evaluate) with evaluation on the first {sample} rows"},
            "e2e": {"value": value, "unit": "node-evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--pop", type=int, default=None, help="population size override (C5 sweep)")
    ap.add_argument("--eval-reps", type=int, default=10)
    ap.add_argument("--evolved-gens", type=int, default=10)
    ap.add_argument("--no-evolved", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--host-mutation", action="store_true",
                    help="mutate on the host (P:237) instead of the GPU (SURVEY F2)")
    ap.add_argument("--shard", default="rows", choices=["rows", "programs"],
                    help="multi-GPU split: row shards + partial-sum all-reduce (default) or "
                         "program chunks + fitness all-gather (SURVEY F3)")
    ap.add_argument("--no-const-programs", action="store_true",
                    help="evaluate variable-free programs per row (no closed-form fitness)")
    ap.add_argument("--nccl", action="store_true",
                    help="use the NCCL communicator path even with one rank (plumbing check)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    cfg = dict(CONFIGS[args.config])
    if args.pop:
        cfg["pop"] = args.pop
        cfg["workload"] = cfg["workload"].replace(f"population {CONFIGS[args.config]['pop']}",
                                                  f"population {args.pop}")
    out = run_reference(args, cfg) if args.impl == "reference" else run_b200(args, cfg)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
