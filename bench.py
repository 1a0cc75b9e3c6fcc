#!/usr/bin/env python
"""Benchmark of the B200 hot path of arXiv 2110.11226.

Metric (BASELINE.json): GP node-evals/sec and sec/generation at Pagie 16M rows (config C3:
Pagie-1 on the 4096 x 4096 grid = 16,777,216 rows, population 8192, MSE). One step = one
gp_generation = the whole hot path of SURVEY section 8(a): tournament selection (GPU), host
mutation, one H2D copy of the flat population, stage + fused evaluate + reduce (+ all-reduce at
N > 1) + finalize. value = node evaluations (sum of program lengths x dataset rows, all ranks)
per second of device time (CUDA events on the engine stream, max over ranks).

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
# reciprocal evaluations the method itself requires, whatever the implementation. Counted only
# for nodes whose subtree depends on a variable (stats op_count); variable-free subtrees are
# per-program constants, not per-row work.
SFU_COST = {5: 1, 9: 1, 10: 1, 11: 3, 14: 1, 15: 1, 16: 1, 17: 1, 8: 2, 20: 2, 21: 2, 22: 2,
            23: 1, 24: 1, 25: 1}
FP32_COST = {2: 1, 3: 1, 4: 1, 5: 1, 6: 1, 7: 1, 9: 1, 10: 1, 11: 2, 12: 1, 13: 1, 18: 1, 19: 2}
LOSS_FP32 = {"mae": 3, "mse": 3, "rmse": 3, "logloss": 7, "pearson": 5}
LOSS_SFU = {"logloss": 2}
# B200: 148 SMs x 16 MUFU lanes x 1965 MHz (sm_max_mhz); microbenchmarked 4.63e12 MUFU.SIN/s
# (profiles/pipe_peaks_r01.txt). FP32: 148 x 128 lanes x 1965 MHz.
SFU_PEAK = 148 * 16 * 1965e6
FP32_PEAK = 148 * 128 * 1965e6


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


def roofline_of(sfu, fp32, eval_ms, launches, step_ms, traffic=True):
    """Binding ALU pipe of the evaluator for the given algorithmic work: SFU (MUFU) or FP32."""
    eval_s = eval_ms * 1e-3
    f_sfu, f_fp32 = sfu / eval_s / SFU_PEAK, fp32 / eval_s / FP32_PEAK
    if f_sfu >= f_fp32:
        r = {"bound": "alu", "pipe": "SFU (MUFU)", "achieved": round(sfu / eval_s / 1e12, 4),
             "peak": round(SFU_PEAK / 1e12, 4), "unit": "Tops/s (MUFU)", "frac": round(f_sfu, 4)}
    else:
        r = {"bound": "alu", "pipe": "FP32", "achieved": round(fp32 / eval_s / 1e12, 4),
             "peak": round(FP32_PEAK / 1e12, 4), "unit": "TFLOP/s (fp32)", "frac": round(f_fp32, 4)}
    r.update({"traffic": ncu_traffic() if traffic else None,
              "traffic_scope": "DRAM bytes of one C3 evaluation's eval launches "
                               "(profiles/eval_kernel_ncu.json)" if traffic else "measured for C3 only", "sfu_frac": round(f_sfu, 4), "fp32_frac": round(f_fp32, 4),
              "eval_ms_per_launch": round(eval_ms / max(launches, 1), 3),
              "eval_share_of_step": round(eval_ms / step_ms, 4),
              "peak_note": "SFU: 148 SMs x 16 MUFU/clk x 1965 MHz (measured MUFU.SIN 4.63e12/s); "
                           "FP32: 148 x 128 x 1965 MHz"})
    return r


def ncu_traffic():
    """dram bytes per eval launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "eval_kernel_ncu.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")   # per evaluation (all variants)
    except Exception:
        return None


def cpu_baseline(nodes, off, X, y, metric, max_seconds=20.0):
    """The oracle (C, double, recursive, single-threaded, as it stands) on a bounded sample:
    all programs of the final population on the first rows of this rank's shard."""
    import oracle
    oracle.build()
    lens = np.diff(off)
    n_rows = 256
    t0 = time.perf_counter()
    oracle.population_fitness(nodes, off, X[:, :n_rows], y[:n_rows], None, metric)
    dt = time.perf_counter() - t0
    rows = int(min(X.shape[1], max(n_rows, n_rows * (max_seconds * 0.5) / max(dt, 1e-6))))
    t0 = time.perf_counter()
    oracle.population_fitness(nodes, off, X[:, :rows], y[:rows], None, metric)
    dt = time.perf_counter() - t0
    return {"value": float(lens.sum()) * rows / dt, "unit": "node-evals/s", "cores": 1,
            "kind": "oracle", "sample": f"all {len(lens)} programs of the final population x "
                                        f"first {rows} rows ({dt:.1f} s, C double recursive)"}


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
              init_depth_min=cfg["depth"][0], init_depth_max=cfg["depth"][1])
    eng = gp.Engine(ctx, X, y, **kw)
    st0 = eng.init_population()
    n0, o0, _ = eng.population()
    gen0 = (n0, o0, st0["op_count"], st0["const_programs"])
    for _ in range(args.warmup):
        eng.generation()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    # ---- timed region: K generations, inputs resident in HBM -----------------------------------
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
            steps.append(eng.generation())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    eval_ms, eval_launches = ctx.eval_timing(reset=True)
    launches = ctx.kernel_launches(reset=True)
    ctx.set_profiling(False)
    node_evals = sum(s["total_nodes"] for s in steps) * m_global
    t = torch.tensor([ms, eval_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, eval_ms_max = float(t[0]), float(t[1])
    value = node_evals / (ms * 1e-3)

    # roofline of the dominant kernel (the fused evaluator), this rank's launches: algorithmic
    # per-row work = variable-dependent nodes only (variable-free subtrees are constants)
    # this rank's share of the per-row work: its row shard, or (program sharding) all rows x about
    # 1 / world of the programs
    rows_local = X.shape[1] / (world if by_prog else 1)
    sfu = fp32 = 0
    for s in steps:
        a, b2 = algorithmic_ops(s["op_count"], rows_local, cfg["metric"], cfg["pop"],
                                0 if args.no_const_programs else s["const_programs"])
        sfu, fp32 = sfu + a, fp32 + b2
    roofline = roofline_of(sfu, fp32, eval_ms, eval_launches, ms, traffic=args.config == "c3")
    var_nodes = sum(sum(s["op_count"]) for s in steps) * m_global
    const_share = float(np.mean([s["const_nodes"] / max(1, s["total_nodes"]) for s in steps]))

    # the same kernel on the generation-0 (ramped half-and-half) population, which carries far
    # more per-row transcendental work than evolved populations: a capability point
    roof0 = None
    if gen0 is not None:
        n0, o0, ops0, cp0 = gen0
        nd, of = torch.from_numpy(n0).cuda(local), torch.from_numpy(o0).cuda(local)
        fit_buf = torch.empty(len(o0) - 1, dtype=torch.float32, device=f"cuda:{local}")
        for _ in range(2):
            ctx.evaluate(nd, of, X, y, metric=cfg["metric"], max_stack=20, fitness_out=fit_buf)
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        ctx.eval_timing(reset=True)
        reps = 5
        for _ in range(reps):
            ctx.evaluate(nd, of, X, y, metric=cfg["metric"], max_stack=20, fitness_out=fit_buf)
        torch.cuda.synchronize()
        ms0, l0 = ctx.eval_timing(reset=True)
        ctx.set_profiling(False)
        a0, b0 = algorithmic_ops(ops0, rows_local, cfg["metric"], cfg["pop"],
                                 0 if args.no_const_programs else cp0)
        roof0 = roofline_of(a0 * reps, b0 * reps, ms0, l0, ms0, traffic=args.config == "c3")
        roof0["node_evals_per_s"] = float(len(n0)) * rows_local * reps / (ms0 * 1e-3)
        roof0["population"] = "generation 0 (ramped half-and-half), mean length %.2f" % (
            len(n0) / (len(o0) - 1))

    # ---- end-to-end: dataset streamed from pinned host memory every step ------------------------
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(Xh).pin_memory()
        yp = torch.from_numpy(yh).pin_memory()
        pop_bytes = 0
        # a fresh engine with the same seed replays the SAME generations as the timed region
        # (the engine is deterministic), so value and e2e price identical populations
        eng = gp.Engine(ctx, X, y, **kw)
        eng.init_population()
        for _ in range(args.warmup):
            eng.generation()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        e2e_steps = []
        for _ in range(args.steps):
            eng.set_dataset(Xp, yp)
            e2e_steps.append(eng.generation())
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms2 = f0.elapsed_time(f1)
        t2 = torch.tensor([ms2], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ms2 = float(t2[0])
        pop_bytes = sum(s["total_nodes"] * 8 + (cfg["pop"] + 1) * 8 for s in e2e_steps) / len(e2e_steps)
        e2e = {"value": sum(s["total_nodes"] for s in e2e_steps) * m_global / (ms2 * 1e-3),
               "unit": "node-evals/s",
               "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes + pop_bytes),
               "d2h_bytes_per_step": int(cfg["pop"] * 4 + np.mean([s["n_tournaments"] for s in e2e_steps]) * 4),
               "ms_per_step": round(ms2 / args.steps, 3)}

    out = None
    if rank == 0:
        nodes, off, _ = eng.population()
        if args.dump_population:
            np.savez_compressed(args.dump_population, nodes=nodes, off=off)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(nodes, off, Xh, yh, cfg["metric"])
        mean_len = float(np.mean([s["total_nodes"] for s in steps])) / cfg["pop"]
        out = {
            "metric": METRIC, "value": value, "unit": "node-evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "sec_per_generation": ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, DESIGN.md recipe)",
            "config": {"workload": cfg["workload"], "rows": m_global, "population": cfg["pop"],
                       "metric": cfg["metric"], "mean_program_length": round(mean_len, 3),
                       "parallelism": (f"programs sharded over {world} GPU(s), fitness all-gathered"
                                       if by_prog else f"rows sharded over {world} GPU(s)"),
                       "l2": "inputs larger than L2 (X + y = %.0f MB)" % ((Xh.nbytes + yh.nbytes) * world / 1e6)},
            "roofline": roofline, "roofline_gen0": roof0,
            "var_node_evals_per_s": var_nodes / (ms * 1e-3), "const_node_share": round(const_share, 4),
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
    """--impl reference: the oracle (C evaluation + Python engine replay) on the host cores,
    each step one generation of the same workload on a bounded row sample."""
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
    pop = oe.ramped_init(ocfg)
    nodes, off = oe.flatten(pop)
    fit, _, _ = oracle.population_fitness(nodes, off, Xs, ys, None, cfg["metric"])
    hb = cfg["metric"] == "pearson"
    total = 0.0
    evals = 0
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rec = oe.next_generation(pop, fit.astype(np.float32), ocfg, step + 1, hb)
        pop = rec.population
        nodes, off = oe.flatten(pop)
        fit, _, _ = oracle.population_fitness(nodes, off, Xs, ys, None, cfg["metric"])
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            total += dt
            evals += int(np.diff(off).sum()) * sample
    value = evals / total
    return {"metric": METRIC, "value": value, "unit": "node-evals/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, DESIGN.md recipe)",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "rows": m, "population": cfg["pop"],
                       "metric": cfg["metric"], "parallelism": "host, 1 thread"},
            "cpu_baseline": {"value": value, "unit": "node-evals/s", "cores": 1, "kind": "oracle",
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
    ap.add_argument("--weak", action="store_true", help="per-GPU rows fixed (default: strong)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="rows", choices=["rows", "programs"],
                    help="multi-GPU split: row shards + partial-sum all-reduce (default) or "
                         "program chunks + fitness all-gather (SURVEY F3)")
    ap.add_argument("--no-const-programs", action="store_true",
                    help="evaluate variable-free programs per row (no closed-form fitness)")
    ap.add_argument("--dump-population", default=None,
                    help="save the final population (nodes, offsets) to this .npz (analysis)")
    ap.add_argument("--nccl", action="store_true",
                    help="use the NCCL communicator path even with one rank (plumbing check)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    cfg = CONFIGS[args.config]
    out = run_reference(args, cfg) if args.impl == "reference" else run_b200(args, cfg)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
