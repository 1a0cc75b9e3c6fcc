"""GPU engine (gp_generation) against the oracle's replay of Alg. 1, and full-size sampled parity.

Teacher forcing: each generation the oracle selects and mutates from the SAME fp32 fitness the GPU
produced, so kinds, tournament winners and children must be bit-identical; the GPU fitness of the
children is checked against the oracle's evaluation within the tolerance model."""
import math

import numpy as np
import pytest

import synth
from tests.test_gpu_parity import check_fitness, dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_11226_b200 as gp
    return gp


@pytest.fixture(scope="module")
def ctx(gp):
    c = gp.Context(0)
    yield c
    c.close()


# Evolved populations (Pearson especially) select fp32-indeterminate constructs -- cos / sin of a
# quotient whose denominator nearly cancels -- so up to a quarter of the programs carry rows whose
# fp32 value the error bound cannot pin to 1e-2 (measured on the oracle replay: <= 35 / 256).
# They are still compared at their bound and counted.
ILL_EVOLVED = 0.25


def _oracle_cfg(oe, **kw):
    return oe.Config(**kw)


@pytest.mark.parametrize("metric", ["mse", "pearson"])
def test_engine_teacher_forced_replay_c1(gp, ctx, orc, metric):
    """C1 (BASELINE configs[0]): Pagie 64x64, population 256, 10 generations (incl. gen 0)."""
    from oracle import engine as oe
    X, y = synth.pagie_grid(64)
    e = gp.Engine(ctx, dev(X), dev(y), population_size=256, metric=metric, seed=2110)
    ocfg = oe.Config(population_size=256, metric=metric, seed=2110)
    e.init_population()
    nodes, off, fit = e.population()
    opop = oe.ramped_init(ocfg)
    on, oo = oe.flatten(opop)
    assert np.array_equal(nodes, on) and np.array_equal(off, oo)
    ref, sens, flags = orc.population_fitness(nodes, off, X, y, None, metric)
    check_fitness(fit, ref, sens, flags, metric, max_ill=ILL_EVOLVED, label=f"c1 gen0 {metric}")
    hb = metric == "pearson"
    for g in range(1, 10):
        st = e.generation()
        kinds, winners = e.last_selection()
        rec = oe.next_generation(opop, fit, ocfg, g, hb)
        assert kinds.tolist() == rec.kinds
        assert np.array_equal(winners, rec.winners)
        nodes, off, fit = e.population()
        on, oo = oe.flatten(rec.population)
        assert np.array_equal(off, oo) and np.array_equal(nodes, on), f"generation {g}"
        ref, sens, flags = orc.population_fitness(nodes, off, X, y, None, metric)
        check_fitness(fit, ref, sens, flags, metric, max_ill=ILL_EVOLVED, label=f"c1 gen{g} {metric}")
        assert st["generation"] == g and st["n_tournaments"] == len(winners)
        opop = rec.population


def test_engine_thread_count_independent(gp, ctx):
    X, y = synth.pagie_grid(32)
    outs = []
    for threads in (1, 7):
        e = gp.Engine(ctx, dev(X), dev(y), population_size=300, metric="mae", seed=5,
                      n_threads=threads)
        e.init_population()
        for _ in range(3):
            e.generation()
        outs.append(e.population())
        e.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_full_size_c3_sampled(gp, ctx, orc):
    """C3 at full size in the bench launch configuration (16,777,216 rows x 8192 programs):
    sampled programs' fitness against the oracle over ALL rows."""
    X, y = synth.pagie_grid(4096)
    e = gp.Engine(ctx, dev(X), dev(y), population_size=8192, metric="mse", seed=2110)
    e.init_population()
    e.generation()
    nodes, off, fit = e.population()
    rng = np.random.default_rng(0)
    lens = np.diff(off)
    sample = list(rng.choice(np.where(lens > 5)[0], 11, replace=False)) + [int(np.argmax(lens))]
    sub_nodes = np.concatenate([nodes[off[p]:off[p + 1]] for p in sample])
    sub_off = np.zeros(len(sample) + 1, np.int64)
    sub_off[1:] = np.cumsum([lens[p] for p in sample])
    ref, sens, flags = orc.population_fitness(sub_nodes, sub_off, X, y, None, "mse")
    check_fitness(fit[sample], ref, sens, flags, "mse", max_excluded=1.0, max_ill=1.0)


def test_full_size_c3_decomposition_invariant(gp, ctx):
    """Every program of the C3 population at full size (bench launch configuration: groups of 512
    programs whose code streams span several shared-memory windows, 16-program reduction blocks)
    against the same programs evaluated 8 at a time (groups of 8, one window): the work
    decomposition only changes the fp32 / fp64 summation order. Constant programs are compared
    between the closed form and the per-row path as well."""
    X, y = synth.pagie_grid(4096)
    Xd, yd = dev(X), dev(y)
    e = gp.Engine(ctx, Xd, yd, population_size=8192, metric="mse", seed=2110)
    e.init_population()
    e.generation()
    nodes, off, fit = e.population()
    e.close()
    nd, of = dev(nodes), dev(off)
    full, _ = ctx.evaluate(nd, of, Xd, yd, metric="mse", max_stack=20)
    ctx.set_const_programs(False)
    try:
        rows, _ = ctx.evaluate(nd, of, Xd, yd, metric="mse", max_stack=20)
    finally:
        ctx.set_const_programs(True)
    full, rows = full.cpu().numpy(), rows.cpu().numpy()
    assert np.array_equal(full, fit)                  # the engine's own evaluation
    fin = np.isfinite(full)
    assert np.array_equal(fin, np.isfinite(rows))
    assert np.all(np.abs(full[fin] - rows[fin]) <= 1e-5 * np.maximum(np.abs(full[fin]), 1e-6))
    part = np.empty_like(full)
    for p0 in range(0, len(off) - 1, 8):
        sub = nodes[off[p0]:off[min(p0 + 8, len(off) - 1)]]
        so = off[p0:min(p0 + 8, len(off) - 1) + 1] - off[p0]
        f, _ = ctx.evaluate(dev(sub), dev(so), Xd, yd, metric="mse", max_stack=20)
        part[p0:p0 + len(so) - 1] = f.cpu().numpy()
    assert np.array_equal(np.isfinite(part), fin)
    assert np.all(np.abs(full[fin] - part[fin]) <= 1e-5 * np.maximum(np.abs(full[fin]), 1e-6))


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_size_wide_configs_sampled(gp, ctx, orc, cfg):
    """C4 (Higgs-shaped 11M x 28, log-loss, population 4096) and C5 (Year-shaped 1M x 90, RMSE,
    depth 2-8) at full size through the engine (wide datasets -> global-X evaluator path); sampled
    programs' fitness against the oracle over ALL rows."""
    import bench
    c = bench.CONFIGS[cfg]
    X, y, _, _, m = bench.load_dataset(c)
    e = gp.Engine(ctx, dev(X), dev(y), population_size=c["pop"], metric=c["metric"], seed=2110,
                  init_depth_min=c["depth"][0], init_depth_max=c["depth"][1])
    e.init_population()
    e.generation()
    nodes, off, fit = e.population()
    lens = np.diff(off)
    rng = np.random.default_rng(1)
    sample = list(rng.choice(np.where(lens > 4)[0], 3, replace=False)) + [int(np.argmax(lens))]
    sub_nodes = np.concatenate([nodes[off[p]:off[p + 1]] for p in sample])
    sub_off = np.zeros(len(sample) + 1, np.int64)
    sub_off[1:] = np.cumsum([lens[p] for p in sample])
    ref, sens, flags = orc.population_fitness(sub_nodes, sub_off, X, y, None, c["metric"])
    check_fitness(fit[sample], ref, sens, flags, c["metric"], max_excluded=1.0, max_ill=1.0)
    e.close()


# ---- GPU-side mutation ------------------------------------------------------------------
@pytest.mark.parametrize("kw", [
    dict(metric="mse"),
    dict(metric="pearson"),
    dict(metric="mae", p_crossover=0.2, p_subtree=0.3, p_hoist=0.2, p_point=0.25,
         p_point_replace=0.3, function_set=list(range(2, 26)), stack_capacity=7,
         init_depth_min=2, init_depth_max=6),
    dict(metric="rmse", init_depth_min=2, init_depth_max=8, p_subtree=0.4, p_crossover=0.4,
         p_hoist=0.1, p_point=0.05, const_lo=-5.0, const_hi=3.0),
])
def test_device_mutation_matches_host_mutation(gp, ctx, kw):
    """The device path (mutate.cu) and the host path (engine.cpp) of gp_generation produce
    bit-identical populations, selections and statistics over 8 generations -- crossover with
    re-hoisting (small stack_capacity), subtree mutation with generated donors (init depth up to
    8), hoist, point mutation over the whole catalog, reproduction."""
    X, y = synth.pagie_grid(24)
    X5 = np.ascontiguousarray(np.concatenate([X, X[::-1] * 0.5, X[:1] + 1.0]))  # 5 features
    Xd, yd = dev(X5), dev(y)
    engines = [gp.Engine(ctx, Xd, yd, population_size=300, seed=77, device_mutation=dm, **kw)
               for dm in (1, 0)]
    stats = [e.init_population() for e in engines]
    keys = ("total_nodes", "best_index", "best_len", "best_depth", "max_stack_need",
            "const_nodes", "const_programs", "op_count", "n_tournaments", "generation")
    for g in range(8):
        stats = [e.generation() for e in engines]
        (n0, o0, f0), (n1, o1, f1) = engines[0].population(), engines[1].population()
        assert np.array_equal(o0, o1) and np.array_equal(n0, n1), f"generation {g + 1}"
        assert np.array_equal(f0, f1)
        k0, w0 = engines[0].last_selection()
        k1, w1 = engines[1].last_selection()
        assert np.array_equal(k0, k1) and np.array_equal(w0, w1)
        for k in keys:
            assert stats[0][k] == stats[1][k], (g, k, stats[0][k], stats[1][k])
        assert stats[0]["best_raw"] == stats[1]["best_raw"] or (
            math.isnan(stats[0]["best_raw"]) and math.isnan(stats[1]["best_raw"]))
        assert abs(stats[0]["mean_raw"] - stats[1]["mean_raw"]) <= 1e-9 * abs(stats[1]["mean_raw"])
    for e in engines:
        e.close()


def test_device_mutation_depth_bound(gp, ctx, orc):
    """Hoisted crossover keeps every child within depth stack_capacity - 1 on the device
    path; the oracle's depth is the judge."""
    X, y = synth.pagie_grid(16)
    e = gp.Engine(ctx, dev(X), dev(y), population_size=400, seed=3, stack_capacity=5,
                  init_depth_min=2, init_depth_max=4, p_crossover=0.9, p_subtree=0.1,
                  p_hoist=0.0, p_point=0.0)
    e.init_population()
    for _ in range(6):
        e.generation()
        nodes, off, _ = e.population()
        for p in range(len(off) - 1):
            prog = nodes[off[p]:off[p + 1]]
            assert orc.validate(prog) == 0 and orc.depth(prog) <= 4


def test_set_population_and_reset(gp, ctx, orc):
    """gp_engine_set_population: a host population is validated and evaluated (fitness == the
    oracle's); re-seeding the device population with its fitness and generation reproduces the
    same next generation (what bench.py does every step)."""
    X, y = synth.pagie_grid(32)
    Xd, yd = dev(X), dev(y)
    e = gp.Engine(ctx, Xd, yd, population_size=200, metric="mse", seed=9)
    nodes, off = synth.random_population(200, seed=4, depth=(1, 5))
    st = e.set_population(nodes, off)
    n2, o2, f2 = e.population()
    assert np.array_equal(n2, nodes) and np.array_equal(o2, off)
    ref, sens, flags = orc.population_fitness(nodes, off, X, y, None, "mse")
    check_fitness(f2, ref, sens, flags, "mse", label="set_population")
    assert st["total_nodes"] == len(nodes)
    dn, do, df = e.population_device()
    a = e.generation()
    pa = e.population()
    e.set_population(dn, do, df, generation=0)
    b = e.generation()
    pb = e.population()
    assert all(np.array_equal(u, v) for u, v in zip(pa, pb))
    assert a["total_nodes"] == b["total_nodes"] and a["best_index"] == b["best_index"]
    bad = nodes.copy()
    bad[0] = (99, 0)                                # not an opcode
    with pytest.raises(gp.GPError):
        e.set_population(bad, off)
    e.close()
