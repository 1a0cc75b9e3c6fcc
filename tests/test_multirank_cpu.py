"""World-size-2 CPU (gloo) tests of the N > 1 host path of bench.py / DESIGN.md section 10:
contiguous row sharding, the global reference row, the NCCL-id broadcast, max-over-ranks timing,
and that per-rank partial sums combined by a SUM all-reduce give the full-dataset fitness.
The per-rank "kernel" here is the oracle (no GPU on this box)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        import oracle
        import synth
        cfg = dict(bench.CONFIGS["c1"])
        X, y, x0, y0, m = bench.load_dataset(cfg, rank, world)
        Xf, yf = synth.pagie_grid(cfg["side"])
        r0, r1 = synth.shard_rows(m, rank, world)
        # contiguous shard of the global data, same global reference row on every rank
        assert np.array_equal(X, Xf[:, r0:r1]) and np.array_equal(y, yf[r0:r1])
        assert np.array_equal(x0, Xf[:, 0]) and y0 == yf[0]
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([r1 - r0]))
        assert sum(int(s) for s in sizes) == m
        # the unique-id broadcast of bench.run_b200
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        # per-rank partial sums -> one SUM all-reduce -> finalize == full-data fitness
        nodes, off = synth.random_population(12, seed=4, depth=(1, 5))
        w = synth.weights(m, seed=1)[r0:r1].astype(np.float64)
        parts = []
        for p in range(len(off) - 1):
            prog = nodes[off[p]:off[p + 1]]
            v, _, _ = oracle.eval_program(prog, X)
            K = oracle.eval_program(prog, x0.reshape(-1, 1))[0][0]     # shift about global row 0
            d, yc = v - K, y.astype(float) - y0
            live = w != 0
            parts += [np.sum(w[live] * (v[live] - y[live]) ** 2), np.sum(w[live] * d[live]),
                      np.sum(w[live] * d[live] ** 2), np.sum(w[live] * d[live] * yc[live])]
        parts += [np.sum(w), np.sum(w * (y - y0)), np.sum(w * (y.astype(float) - y0) ** 2)]
        t = torch.tensor(parts, dtype=torch.float64)
        dist.all_reduce(t)
        t = t.numpy()
        W, Sy, Syy = t[-3:]
        wf = synth.weights(m, seed=1)
        for p in range(len(off) - 1):
            s_mse, Sd, Sdd, Sdy = t[4 * p:4 * p + 4]
            vf, _, _ = oracle.eval_program(nodes[off[p]:off[p + 1]], Xf)
            mse_ref = oracle.fitness("mse", vf, yf, wf)[0]
            assert abs(s_mse / W - mse_ref) <= 1e-12 * max(1.0, mse_ref)
            r_ref, und = oracle.fitness("pearson", vf, yf, wf)
            vd, vy = Sdd - Sd * Sd / W, Syy - Sy * Sy / W
            if not und and vd > 0:
                r = (Sdy - Sd * Sy / W) / np.sqrt(vd * vy)
                assert abs(r - r_ref) <= 1e-9
        # max-over-ranks timing reduction
        tm = torch.tensor([10.0 + rank], dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        assert float(tm) == 10.0 + world - 1
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


def test_two_rank_sharded_fitness_gloo():
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


def _program_chunk(n, rank, world):
    """The program range of one rank under GP_SHARD_PROGRAMS (include/gp.h, api.cpp
    gp_evaluate): equal-count chunks c = ceil(n / world), rank r owns [min(n, r c), min(n, r c + c))."""
    c = (n + world - 1) // world
    lo = min(n, rank * c)
    return c, lo, min(n, lo + c)


def _worker_programs(rank, world, port, errq, n_programs):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        import oracle
        import synth
        cfg = dict(bench.CONFIGS["c1"])
        X, y, _, _, m = bench.load_dataset(cfg, 0, 1)            # every rank holds all rows
        nodes, off = synth.random_population(n_programs, seed=9, depth=(1, 5))
        c, lo, hi = _program_chunk(n_programs, rank, world)
        # this rank's chunk in a padded world x c buffer, combined by an all-gather
        mine = torch.full((c,), float("nan"), dtype=torch.float64)
        for p in range(lo, hi):
            v, _, _ = oracle.eval_program(nodes[off[p]:off[p + 1]], X)
            mine[p - lo] = oracle.fitness("mse", v, y, None)[0]
        parts = [torch.empty(c, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        fit = torch.cat(parts)[:n_programs].numpy()
        for p in range(n_programs):
            v, _, _ = oracle.eval_program(nodes[off[p]:off[p + 1]], X)
            assert fit[p] == oracle.fitness("mse", v, y, None)[0], p
        # every program owned by exactly one rank
        owned = torch.zeros(n_programs, dtype=torch.int64)
        owned[lo:hi] = 1
        dist.all_reduce(owned)
        assert bool((owned == 1).all())
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,n_programs", [(2, 13), (3, 2)])
def test_program_sharded_fitness_gloo(world, n_programs):
    """SURVEY F3 host logic: program chunks (ragged last chunk; an empty chunk when world > n)
    evaluated per rank and all-gathered give the whole population's fitness on every rank."""
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_programs, args=(r, world, port, errq, n_programs))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
