"""Pins for the oracle's Philox, tournament selection and host-engine replay
(S:68-97). CPU only."""
import math

import numpy as np
import pytest

import synth


# ---- Philox4x32-10: Random123 known-answer vectors (Salmon et al. 2011, cited at P:202) ---------
@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_kat(orc, ctr, key, want):
    assert tuple(int(x) for x in orc.philox4x32_10(ctr, key)) == want


# ---- Eqs. 1-2, S:260-262 ---------------------------------------------------------------
def test_parsimony_examples(orc):
    # raw 2.0, len 5, c 0.01 -> 2.05 (fp32 2.0499999523); 0.8, len 10 -> 0.70.
    f32 = np.float32
    assert f32(f32(2.0) + f32(f32(0.01) * f32(5))) == f32(2.049999952316284)
    assert f32(f32(0.8) - f32(f32(0.01) * f32(10))) == f32(0.7000000476837158)
    # Eq. 2 is evaluated in fp32 (C10): program 0 (raw 2.0, len 5) and program 1
    # (raw fp32(2.05), len 0) tie in fp32 -> smallest index 0 wins; in double 1 would win.
    fit = np.array([2.0, 2.05], np.float32)
    w = orc.tournament(fit, np.array([5, 0], np.int32), 32, 16, 0.01, False, 1, 1)
    assert set(w.tolist()) == {0}
    fit = np.array([0.8, 0.7000000476837158], np.float32)   # higher-better mirror
    w = orc.tournament(fit, np.array([10, 0], np.int32), 32, 16, 0.01, True, 1, 1)
    assert set(w.tolist()) == {0}


def _draws(orc, seed, gen, t, n, k):
    key = (seed & 0xFFFFFFFF, seed >> 32)
    out = []
    for i in range(k):
        words = orc.philox4x32_10((t, gen, i // 4, 0), key)
        out.append((int(words[i % 4]) * n) >> 32)
    return out


def test_tournament_worked_example(orc):
    # DESIGN.md C10 layout: seed 0, generation 0, n = 35, k = 4 (Table 6: P:483-484)
    assert _draws(orc, 0, 0, 0, 35, 4) == [13, 30, 25, 21]
    assert _draws(orc, 0, 0, 1, 35, 4) == [34, 12, 24, 1]
    lens = np.ones(35, np.int32)
    up = np.arange(35, dtype=np.float32)
    assert orc.tournament(up, lens, 2, 4, 0.0, False, 0, 0).tolist() == [13, 1]
    assert orc.tournament(up, lens, 2, 4, 0.0, True, 0, 0).tolist() == [30, 34]


def test_tournament_brute_force(orc):
    fit = np.array([3.0, 1.0, 2.0], np.float32)
    lens = np.ones(3, np.int32)
    assert set(orc.tournament(fit, lens, 20, 60, 0.0, False, 9, 3).tolist()) == {1}
    assert orc.tournament(fit, lens, 5, 1, 0.0, False, 4, 2).tolist() == \
        [_draws(orc, 4, 2, t, 3, 1)[0] for t in range(5)]       # S:269 k = 1
    # exhaustive: winner is the best drawn, ties -> smallest index, NaN worst
    rng = np.random.default_rng(0)
    for trial in range(300):
        n = int(rng.integers(1, 9))
        k = int(rng.integers(1, 9))
        fit = rng.integers(0, 4, n).astype(np.float32)
        fit[rng.random(n) < 0.2] = np.nan
        lens = rng.integers(1, 20, n).astype(np.int32)
        c = float(rng.choice([0.0, 0.01, 0.5]))
        hb = bool(rng.integers(2))
        got = orc.tournament(fit, lens, 4, k, c, hb, trial, 7)
        for t in range(4):
            d = _draws(orc, trial, 7, t, n, k)
            pen = np.float32(c) * lens[d].astype(np.float32)
            adj = fit[d] - pen if hb else fit[d] + pen
            adj = np.where(np.isnan(adj), -np.inf if hb else np.inf, adj)
            best = adj.max() if hb else adj.min()
            want = min(i for i, a in zip(d, adj) if a == best)
            assert got[t] == want


def test_tournament_win_law_chi_square(orc):
    # With replacement, distinct fitness: P(rank r wins) = ((n-r+1)^k - (n-r)^k) / n^k.
    n, k, T = 3, 2, 90000
    fit = np.array([0.5, 0.1, 0.9], np.float32)       # ranks: 1 -> idx1, 2 -> idx0, 3 -> idx2
    w = orc.tournament(fit, np.ones(3, np.int32), T, k, 0.0, False, 123, 5)
    cnt = np.bincount(w, minlength=3)
    expect = T * np.array([3 / 9, 5 / 9, 1 / 9])
    chi2 = ((cnt - expect) ** 2 / expect).sum()
    assert chi2 < 13.8                                  # p > 0.001 at 2 dof


def test_parsimony_monotone_win_rate(orc):
    # uniform fitness, c > 0 -> shorter programs win more often.
    n = 20
    lens = np.arange(1, n + 1, dtype=np.int32)
    w = orc.tournament(np.zeros(n, np.float32), lens, 10000, 4, 0.01, False, 5, 1)
    cnt = np.bincount(w, minlength=n)
    assert all(cnt[i] >= cnt[i + 1] for i in range(n - 1))


# ---- host engine replay: SPEC examples and properties ---------------------------------------------
@pytest.fixture(scope="module")
def eng(orc):
    from oracle import engine
    return engine


def test_random_program_full_and_grow(orc, eng):
    cfg = eng.Config(function_set=(2,), n_features=2)
    for i in range(50):
        p = eng.random_program(eng.Stream(1, i, 0, 3), eng.FULL, 1, cfg)
        assert len(p) == 3 and p[0] == (2, 0) and all(orc.arity(op) == 0 for op, _ in p[1:])
    cfg = eng.Config()
    for i in range(1000):
        md = 1 + i % 6
        p = eng.random_program(eng.Stream(2, i, 0, 3), eng.GROW, md, cfg)
        a = eng._arr(p)
        assert orc.validate(a) == 0 and orc.depth(a) <= md
        q = eng.random_program(eng.Stream(3, i, 0, 3), eng.FULL, md, cfg)
        assert _leaf_depths(q) == {md}


def _leaf_depths(p):
    out = set()

    def rec(i, d):
        a = synth._arity(p[i][0])
        if a == 0:
            out.add(d)
            return i + 1
        j = i + 1
        for _ in range(a):
            j = rec(j, d + 1)
        return j
    rec(0, 0)
    return out


def test_ramped_init_split(orc, eng):
    for n, full in ((50, 25), (35, 17), (1, 0)):
        cfg = eng.Config(population_size=n)
        pop = eng.ramped_init(cfg)
        assert len(pop) == n
        n_full = sum(1 for i, p in enumerate(pop) if i < n // 2)
        assert n_full == full
        for i, p in enumerate(pop):
            md = 2 + i % 5
            assert orc.validate(eng._arr(p)) == 0 and orc.depth(eng._arr(p)) <= md
            if i < n // 2:
                assert _leaf_depths(p) == {md}


def test_mutation_kind_frequencies(eng):
    # SPEC acceptance 7: within +-0.01 of (0.7, 0.1, 0.1, 0.05, 0.05) over 1e5 draws.
    cfg = eng.Config(population_size=100000)
    kinds = np.array(eng.choose_kinds(cfg, 1))
    freq = np.bincount(kinds, minlength=5) / len(kinds)
    want = [0.7, 0.1, 0.05, 0.1, 0.05]      # crossover, subtree, hoist, point, reproduction
    assert np.all(np.abs(freq - want) < 0.01)
    z = eng.Config(population_size=100, p_crossover=0, p_subtree=0, p_hoist=0, p_point=0)
    assert set(eng.choose_kinds(z, 1)) == {eng.REPRODUCTION}
    one = eng.Config(population_size=100, p_crossover=1.0)
    assert set(eng.choose_kinds(one, 1)) == {eng.CROSSOVER}


def test_point_mutation(orc, eng):
    parent = [(2, 0), (0, 0), (0, 1)]
    cfg = eng.Config(p_point_replace=0.0)
    assert eng.point_mutation(eng.Stream(1, 0, 1, 2), parent, cfg) == parent
    cfg = eng.Config(p_point_replace=1.0, function_set=(2, 3))
    for i in range(50):
        c = eng.point_mutation(eng.Stream(1, i, 1, 2), parent, cfg)
        assert c[0][0] in (2, 3) and len(c) == 3 and orc.depth(eng._arr(c)) == 1
    cfg = eng.Config(p_point_replace=0.3)
    pop = eng.ramped_init(eng.Config(population_size=200))
    for i, p in enumerate(pop):
        c = eng.point_mutation(eng.Stream(5, i, 1, 2), p, cfg)
        assert len(c) == len(p) and orc.depth(eng._arr(c)) == orc.depth(eng._arr(p))


def test_hoist_and_crossover(orc, eng):
    assert eng.hoist_mutation(eng.Stream(1, 0, 1, 2), [(0, 0)]) == [(0, 0)]
    cfg = eng.Config()
    assert eng.hoisted_crossover(eng.Stream(1, 0, 1, 2), [(0, 0)], [(0, 1)], cfg) == [(0, 1)]
    pop = eng.ramped_init(eng.Config(population_size=300, init_depth=(2, 8)))
    for i in range(300):
        p, d = pop[i], pop[(7 * i + 3) % 300]
        h = eng.hoist_mutation(eng.Stream(9, i, 1, 2), p)
        assert orc.validate(eng._arr(h)) == 0 and len(h) <= len(p)
        assert orc.depth(eng._arr(h)) <= orc.depth(eng._arr(p))
        c = eng.hoisted_crossover(eng.Stream(9, i, 2, 2), p, d, cfg)
        assert orc.validate(eng._arr(c)) == 0 and orc.depth(eng._arr(c)) <= 19
    small = eng.Config(stack_capacity=4)
    shallow = [p for p in pop if orc.depth(eng._arr(p)) <= 3]
    for i in range(200):
        p = shallow[i % len(shallow)]
        d = pop[(5 * i + 1) % 300]
        c = eng.hoisted_crossover(eng.Stream(4, i, 1, 2), p, d, small)
        assert orc.validate(eng._arr(c)) == 0 and orc.depth(eng._arr(c)) <= 3
        s = eng.subtree_mutation(eng.Stream(4, i, 2, 2), p, small)
        assert orc.validate(eng._arr(s)) == 0 and orc.depth(eng._arr(s)) <= 3


def test_pick_subtree_weights(eng):
    # 90% of the mass on function nodes, 10% on terminals.
    prog = [(2, 0), (0, 0), (3, 0), (0, 1), (1, 0)]    # 2 functions, 3 terminals
    cnt = np.zeros(5)
    for i in range(20000):
        cnt[eng.pick_subtree(eng.Stream(3, i, 1, 2), prog)[0]] += 1
    p = cnt / cnt.sum()
    want = np.array([9, 1, 9, 1, 1]) / 21
    assert np.all(np.abs(p - want) < 0.012)


def test_generation_tournament_count_and_gp_run(orc, eng):
    """Alg. 1 loop on a 64x64 Pagie grid: tournament count = 2 #cx + #others,
    every program valid with depth <= capacity - 1, best raw fitness improves (S:613b)."""
    X, y = synth.pagie_grid(32)
    cfg = eng.Config(population_size=50, metric="rmse", seed=17)
    pop = eng.ramped_init(cfg)
    best = []
    for g in range(0, 12):
        if g > 0:
            rec = eng.next_generation(pop, fit32, cfg, g, False)
            assert len(rec.winners) == sum(2 if k == eng.CROSSOVER else 1 for k in rec.kinds)
            pop = rec.population
        nodes, off = eng.flatten(pop)
        for i in range(len(pop)):
            a = nodes[off[i]:off[i + 1]]
            assert orc.validate(a) == 0 and orc.depth(a) <= cfg.stack_capacity - 1
        fit, _, _ = orc.population_fitness(nodes, off, X, y, None, "rmse")
        fit32 = fit.astype(np.float32)
        best.append(np.nanmin(fit))
    assert min(best[1:]) <= best[0]
    assert math.isfinite(best[-1])
