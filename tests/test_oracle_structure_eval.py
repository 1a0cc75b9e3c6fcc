"""Pins for the oracle's structure helpers and evaluator (CPU only).

Each expected value comes from PAPER.md / SPEC.md examples, a closed form, or brute force that is
independent of the oracle's own code path. Citations: P:L = PAPER.md line, S:L = SPEC.md line.
"""
import math

import numpy as np
import pytest

import synth

E = math.e


def P(orc, *t):
    return orc.program(*t)


# ---- validate_prefix / depth / subtree_span: SPEC examples S:47-67 ------------------------------
def test_validate_spec_examples(orc):
    assert orc.validate(P(orc, "add", ("var", 0), ("var", 1))) == 0
    assert orc.validate(P(orc, "add", ("var", 0))) == 3                          # S:48 Dangling
    p = P(orc, "sin", "add", ("var", 0), ("const", 2.0))
    assert orc.validate(p) == 0 and len(p) == 4
    assert orc.validate(P(orc, ("var", 0), ("var", 1))) == 2                     # Underflow
    assert orc.validate(np.zeros((0, 2), np.int32)) == 1
    assert orc.validate(np.array([[99, 0]], np.int32)) == 4
    assert orc.validate(P(orc, ("var", 2)), n_cols=2) == 5


def test_depth_spec_examples(orc):
    assert orc.depth(P(orc, ("var", 0))) == 0
    assert orc.depth(P(orc, "add", ("var", 0), ("var", 1))) == 1
    assert orc.depth(P(orc, "add", "sin", ("var", 0), ("const", 1.0))) == 2


def test_subtree_span_spec_examples(orc):
    p = P(orc, "add", ("var", 0), ("var", 1))
    assert orc.subtree_end(p, 1) == 2
    assert orc.subtree_end(p, 0) == 3
    q = P(orc, "add", "sin", ("var", 0), ("var", 1))
    assert orc.subtree_end(q, 1) == 3


def test_stack_need_left_and_right_deep(orc):
    # depth m-1 needs a stack of m; a left-deep depth-4 tree reaches it, right-deep does not
    x = ("var", 0)
    left = P(orc, "add", "add", "add", "add", x, x, x, x, x)
    right = P(orc, "add", x, "add", x, "add", x, "add", x, x)
    assert orc.depth(left) == 4 and orc.stack_need(left) == 5
    assert orc.depth(right) == 4 and orc.stack_need(right) == 2


def _need_rec(prog, i=0):
    """Independent recursive definition of reverse-prefix stack need: for [op, A, B] the
    second operand B is evaluated first and stays on the stack while A is evaluated."""
    op = prog[i][0]
    a = synth._arity(op)
    if a == 0:
        return 1, i + 1
    na, j = _need_rec(prog, i + 1)
    if a == 1:
        return na, j
    nb, k = _need_rec(prog, j)
    return max(nb, 1 + na), k


def _depth_rec(prog, i=0):
    op = prog[i][0]
    a = synth._arity(op)
    j, d = i + 1, 0
    for _ in range(a):
        dc, j = _depth_rec(prog, j)
        d = max(d, dc + 1)
    return d, j


def test_structure_brute_force_random(orc):
    nodes, off = synth.random_population(400, seed=3, depth=(0, 9), funcs=synth.ALL_FUNCS)
    for i in range(len(off) - 1):
        p = nodes[off[i]:off[i + 1]]
        pl = [tuple(t) for t in p]
        assert orc.validate(p) == 0
        d, end = _depth_rec(pl)
        assert end == len(pl) and orc.depth(p) == d
        need, _ = _need_rec(pl)
        assert orc.stack_need(p) == need <= d + 1                   # P:243 bound
        for s in range(len(p)):                                      # S:91 every span validates
            e = orc.subtree_end(p, s)
            assert orc.validate(p[s:e]) == 0
            assert e - s == _span_len(pl, s)


def _span_len(pl, s):
    need, i = 1, s
    while need:
        need += synth._arity(pl[i][0]) - 1
        i += 1
    return i - s


# ---- catalog semantics: closed forms (S:132 protected rules, C2) ------------------------
CLOSED = [
    ("add", 2.0, 3.0, 5.0), ("sub", 2.0, 3.0, -1.0), ("mul", -2.5, 4.0, -10.0),
    ("div", 1.0, 4.0, 0.25), ("div", 1.0, 0.0, 1.0), ("div", 1.0, 0.000999, 1.0),
    ("div", 1.0, 0.002, 500.0), ("div", 3.0, -0.0005, 1.0), ("min", 2.0, -3.0, -3.0),
    ("max", 2.0, -3.0, 2.0), ("pow", 2.0, 10.0, 1024.0), ("pow", -2.0, 3.0, 8.0),
    ("pow", 0.0, -1.0, 1e30), ("pow", 0.0, 2.0, 0.0), ("pow", 5.0, 0.0, 1.0),
    ("pow", 0.5, -200.0, 1e30), ("pow", 9.0, 0.5, 3.0),
    ("sin", math.pi / 6, 0, 0.5), ("cos", math.pi / 3, 0, 0.5), ("tan", math.pi / 4, 0, 1.0),
    ("abs", -7.0, 0, 7.0), ("neg", 7.0, 0, -7.0), ("sqrt", -9.0, 0, 3.0), ("sqrt", 16.0, 0, 4.0),
    ("log", E, 0, 1.0), ("log", -E * E, 0, 2.0), ("log", 0.0005, 0, 0.0), ("log", -0.000999, 0, 0.0),
    ("exp", 1.0, 0, E), ("exp", 100.0, 0, 1e30), ("exp", 0.0, 0, 1.0),
    ("inv", 4.0, 0, 0.25), ("inv", 0.0, 0, 1.0), ("inv", -0.0005, 0, 1.0), ("inv", -0.5, 0, -2.0),
    ("square", -3.0, 0, 9.0), ("cube", -2.0, 0, -8.0),
    ("tanh", math.log(2), 0, 0.6), ("sinh", math.log(2), 0, 0.75), ("cosh", math.log(2), 0, 1.25),
    ("sinh", 100.0, 0, 1e30), ("sinh", -100.0, 0, -1e30), ("cosh", -100.0, 0, 1e30),
    ("asin", 0.5, 0, math.pi / 6), ("asin", 2.0, 0, math.pi / 2), ("acos", 0.5, 0, math.pi / 3),
    ("acos", -3.0, 0, math.pi), ("atan", 1.0, 0, math.pi / 4),
]


@pytest.mark.parametrize("name,a,b,want", CLOSED)
def test_catalog_closed_forms(orc, name, a, b, want):
    got = orc.apply(orc.NAMES.index(name), a, b)
    assert got == pytest.approx(want, rel=1e-14, abs=1e-15)


def test_catalog_threshold_is_strict(orc):
    # S:132 "|b| < 1e-3" strict: b = 1e-3 itself divides.
    assert orc.apply(orc.DIV, 1.0, 1e-3) == pytest.approx(1000.0)
    assert orc.apply(orc.LOG, 1e-3, 0) == pytest.approx(math.log(1e-3))
    assert orc.apply(orc.INV, 1e-3, 0) == pytest.approx(1000.0)


# ---- hand-derived programs ---------------------------
def _ev(orc, prog, *row):
    X = np.array(row, dtype=np.float32).reshape(-1, 1)
    v, e, f = orc.eval_program(prog, X)
    return v[0]


def test_hand_programs(orc):
    x0, x1 = ("var", 0), ("var", 1)
    assert _ev(orc, P(orc, "add", x0, x1), 2, 3) == 5.0
    assert _ev(orc, P(orc, "sub", x0, x1), 2, 3) == -1.0                       # S:166 operand order
    assert _ev(orc, P(orc, ("const", 7.5)), 0) == 7.5
    assert _ev(orc, P(orc, "div", x0, ("const", 0.0)), 2) == 1.0
    assert _ev(orc, P(orc, "div", ("const", 1.0), ("const", 0.0005)), 0) == 1.0
    assert _ev(orc, P(orc, "div", ("const", 1.0), ("const", 0.002)), 0) == pytest.approx(500.0,
                                                                                         rel=1e-7)
    assert _ev(orc, P(orc, "log", ("const", 0.0005)), 0) == 0.0
    assert _ev(orc, P(orc, "log", ("const", -E)), 0) == pytest.approx(1.0, abs=1e-7)
    assert _ev(orc, P(orc, "sqrt", ("const", -4.0)), 0) == 2.0
    assert _ev(orc, P(orc, "inv", ("const", 0.0)), 0) == 1.0
    assert _ev(orc, P(orc, "inv", ("const", 4.0)), 0) == 0.25
    assert _ev(orc, P(orc, "sin", "add", x0, ("const", 1.0)), -1) == 0.0
    assert _ev(orc, P(orc, "exp", ("const", 100.0)), 0) == 1e30
    assert _ev(orc, P(orc, "div", "sin", x0, "cos", x0), 1) == pytest.approx(1.557407724654902,
                                                                             rel=1e-15)
    assert _ev(orc, P(orc, "mul", "sub", x0, x1, "add", x0, x1), 3, 2) == 5.0  # (3-2)(3+2)


def pagie_program(orc):
    """Eq. 3 as a 35-node prefix program over {add, mul, div}: add, T(x0), T(x1) with
    T(v) = div, P4(v), add, P4(v), 1 and P4(v) = mul, mul, v, v, mul, v, v."""
    def p4(v):
        return ["mul", "mul", v, v, "mul", v, v]

    def T(v):
        return ["div"] + p4(v) + ["add"] + p4(v) + [("const", 1.0)]
    return P(orc, *(["add"] + T(("var", 0)) + T(("var", 1))))


def test_pagie_program_closed_form(orc):
    p = pagie_program(orc)
    assert len(p) == 35 and orc.stack_need(p) == 5 and orc.depth(p) == 5
    assert _ev(orc, p, 1, 1) == pytest.approx(1.0, rel=1e-15)
    assert _ev(orc, p, -5, -5) == pytest.approx(1.996805111821086, rel=1e-15)  # 2 * 625/626
    assert _ev(orc, p, 0.5, 2) == pytest.approx(1.0, rel=1e-15)                # x*y = 1
    assert 2 * 625 / 626 == pytest.approx(1.996805111821086, rel=1e-15)


def test_pagie_generator_matches_eq3(orc):
    X, y = synth.pagie_grid(64)
    assert X.shape == (2, 4096)                                                # Table 3
    idx = np.random.default_rng(0).integers(0, 4096, 200)
    for r in idx:
        assert np.float32(orc.pagie(X[0, r], X[1, r])) == y[r]
    assert orc.pagie(1, 1) == 1.0 and orc.pagie(0, 1) == 0.5
    assert orc.pagie(-5, -5) == pytest.approx(2 * 625 / 626, rel=1e-15)
    X2, y2 = synth.pagie_grid(2)
    assert np.allclose(y2, 1.996805111821086) and y.min() > 0 and y.max() < 2
    assert synth.pagie_grid(128)[1].shape[0] == 4 * 4096                       # S:530 doubling


def _stack_walk(orc, prog, row):
    """Independent reverse-prefix stack evaluation: first pop = first operand."""
    st = []
    for op, pl in reversed([tuple(t) for t in prog]):
        if op == 0:
            st.append(float(row[pl]))
        elif op == 1:
            st.append(orc.bits_f32(pl))
        elif orc.arity(op) == 1:
            st.append(orc.apply(op, st.pop()))
        else:
            a = st.pop()
            b = st.pop()
            st.append(orc.apply(op, a, b))
    assert len(st) == 1
    return st[0]


def test_recursive_equals_stack_walk(orc):
    # SPEC acceptance 1: >= 1e4 (program, row) pairs, recursive == stack walk.
    nodes, off = synth.random_population(250, seed=11, depth=(0, 10), funcs=synth.ALL_FUNCS)
    rng = np.random.default_rng(5)
    X = rng.uniform(-4, 4, (2, 48)).astype(np.float32)
    pairs = 0
    for i in range(len(off) - 1):
        p = nodes[off[i]:off[i + 1]]
        v, _, _ = orc.eval_program(p, X)
        for r in range(X.shape[1]):
            w = _stack_walk(orc, p, X[:, r])
            assert (v[r] == w) or (math.isnan(v[r]) and math.isnan(w))
            pairs += 1
    assert pairs >= 10_000


# ---- the error bound E: an fp32 evaluation with IEEE-accurate ops must land within E ------------
_F = np.float32
_FLT_MIN = float(np.finfo(np.float32).tiny)


def _ftz(x, on):
    """Flush-to-zero of an fp32 value (the GPU build's -ftz=true): subnormals become signed 0."""
    return _F(0.0) * np.sign(x) if on and abs(x) < _FLT_MIN else x


def _f32_op(op, a, b):
    """One catalog function in fp32 (S:117-122, S:132 protected rules; C2): the IEEE
    ops correctly rounded by numpy float32, the others as the double libm value rounded to fp32
    (within an ulp of the exact value -- the evaluator's budgets are wider)."""
    T, BIG = _F(1e-3), _F(1e30)
    d = lambda v: _F(v)                                      # noqa: E731 (round double -> fp32)
    A, B = float(a), float(b)
    with np.errstate(all="ignore"):
        if op == 2: return a + b
        if op == 3: return a - b
        if op == 4: return a * b
        if op == 5: return _F(1) if abs(b) < T else a / b
        if op == 6: return np.fmin(a, b)
        if op == 7: return np.fmax(a, b)
        if op == 8:
            if b == 0: return _F(1)
            if a == 0: return _F(0) if b > 0 else BIG
            lg = B * math.log(abs(A))
            return min(d(math.exp(lg)) if lg < 89.0 else _F(np.inf), BIG)
        if op == 9: return d(math.sin(A))
        if op == 10: return d(math.cos(A))
        if op == 11: return d(math.tan(A))
        if op == 12: return abs(a)
        if op == 13: return -a
        if op == 14: return d(math.sqrt(abs(A)))
        if op == 15: return _F(0) if abs(a) < T else d(math.log(abs(A)))
        if op == 16: return min(d(math.exp(A)) if A < 89 else _F(np.inf), BIG)
        if op == 17: return _F(1) if abs(a) < T else _F(1) / a
        if op == 18: return a * a
        if op == 19: return (a * a) * a
        if op == 20: return d(math.tanh(A))
        if op == 21: return max(min(d(math.sinh(A)) if abs(A) < 89 else _F(math.copysign(np.inf, A)), BIG), -BIG)
        if op == 22: return min(d(math.cosh(A)) if abs(A) < 89 else _F(np.inf), BIG)
        if op == 23: return d(math.asin(min(max(A, -1.0), 1.0)))
        if op == 24: return d(math.acos(min(max(A, -1.0), 1.0)))
        if op == 25: return d(math.atan(A))
    raise ValueError(op)


def _f32_eval(orc, prog, row, ftz=False):
    """fp32 emulation of a program by a reverse-prefix stack walk (an independent evaluation
    order from the oracle's recursion), optionally flushing subnormals like the GPU build."""
    st = []
    for op, pl in reversed([tuple(t) for t in prog]):
        if op == 0:
            st.append(_ftz(_F(row[pl]), ftz))
            continue
        if op == 1:
            st.append(_ftz(_F(orc.bits_f32(pl)), ftz))
            continue
        a = st.pop()
        b = st.pop() if orc.arity(op) == 2 else _F(0)
        st.append(_ftz(_F(_f32_op(op, a, b)), ftz))
    return st[0]


def _bound_rows(n=48, seed=5):
    """Rows for the E pins: the Pagie grid plus values over many magnitudes (1e-20 .. 1e3, both
    signs), so underflow (cube, pow, mul of tiny values), overflow and the protected thresholds
    are all reached."""
    Xg, _ = synth.pagie_grid(6)
    rng = np.random.default_rng(seed)
    mag = 10.0 ** rng.uniform(-20, 3, (2, n))
    Xr = (mag * rng.choice([-1.0, 1.0], (2, n))).astype(np.float32)
    return np.ascontiguousarray(np.concatenate([Xg, Xr], axis=1))


@pytest.mark.parametrize("funcs,seed", [(synth.TABLE2_SET, 21), (synth.ALL_FUNCS, 22),
                                        (synth.ALL_FUNCS, 23)])
def test_error_bound_covers_fp32_evaluation(orc, funcs, seed):
    """SURVEY "exact result within the error bound": for every one of the 24 catalog functions an
    fp32 evaluation (IEEE with gradual underflow, and flush-to-zero as on the GPU) lies within the
    oracle's E of the exact (double) value on every row the oracle does not flag."""
    nodes, off = synth.random_population(260, seed=seed, depth=(1, 6), funcs=funcs)
    X = _bound_rows()
    checked = 0
    used = set()
    for i in range(len(off) - 1):
        p = nodes[off[i]:off[i + 1]]
        v, e, fl = orc.eval_program(p, X)
        for r in range(X.shape[1]):
            if fl[r] or not math.isfinite(e[r]):
                continue
            for ftz in (False, True):
                g = float(_f32_eval(orc, p, X[:, r], ftz))
                assert abs(g - v[r]) <= e[r], (i, r, ftz, g, v[r], e[r], p.tolist())
            checked += 1
        used.update(int(o) for o in p[:, 0] if o > 1)
    assert checked > 10_000
    assert used == set(funcs)


def test_error_bound_underflow_cases(orc):
    """Results below FLT_MIN: fp32 gives a subnormal or (FTZ) zero where double keeps 1e-60; E must
    cover the difference (the round-1 review found cube / pow rows violating E without an
    underflow term)."""
    x = ("var", 0)
    X = np.array([[1e-20, -3e-13, 2e-30]], np.float32)
    for prog in (P(orc, "cube", x), P(orc, "mul", x, x), P(orc, "square", x),
                 P(orc, "pow", x, ("const", 3.0)), P(orc, "mul", "cube", x, ("const", 0.5))):
        v, e, fl = orc.eval_program(prog, X)
        for r in range(X.shape[1]):
            assert not fl[r]
            for ftz in (False, True):
                g = float(_f32_eval(orc, prog, X[:, r], ftz))
                assert abs(g - v[r]) <= e[r], (prog.tolist(), r, g, v[r], e[r])
        assert (e >= np.abs(v)).all() or (np.abs(v) >= _FLT_MIN).any()


@pytest.mark.parametrize("metric", ["mae", "mse", "rmse", "logloss", "pearson"])
def test_fitness_sensitivity_covers_fp32_fitness(orc, metric):
    """orc_fitness_sensitivity pin (SURVEY acceptance rule per program): the fitness of the fp32
    predictions (each within E of the exact one) lies within the sensitivity of the exact fitness
    -- brute force over random programs, with the fitness itself from the oracle's metric on the
    fp32 values. Also: predictions perturbed by +-E on every row (signs random) stay within
    the bound to first order (factor 2 slack for the second-order term)."""
    X = _bound_rows(n=24, seed=9)[:, :60]
    if metric == "logloss":
        y = (X[0] > 0).astype(np.float32)
    else:
        y = np.asarray([orc.pagie(float(a), float(b)) for a, b in X.T], np.float32)
    w = synth.weights(X.shape[1], seed=3)
    nodes, off = synth.random_population(120, seed=31, depth=(1, 5), funcs=synth.ALL_FUNCS)
    rng = np.random.default_rng(4)
    checked = 0
    for i in range(len(off) - 1):
        p = nodes[off[i]:off[i + 1]]
        v, e, fl = orc.eval_program(p, X)
        live = w != 0
        if fl[live].any() or not np.isfinite(e[live]).all() or np.ptp(v[live]) == 0:
            continue
        F = orc.fitness(metric, v, y, w)[0]
        s = orc.fitness_sensitivity(metric, v, e, y, w)
        if not math.isfinite(s) or not math.isfinite(F):
            continue
        g = np.array([float(_f32_eval(orc, p, X[:, r], True)) for r in range(X.shape[1])])
        Fg = orc.fitness(metric, g, y, w)[0]
        # (+ double rounding of the metric's own sums, ~1e-16 relative)
        assert abs(Fg - F) <= s * (1 + 1e-9) + 1e-12 * abs(F) + 1e-15, (i, metric, Fg, F, s)
        for _ in range(3):
            vp = v + e * rng.choice([-1.0, 1.0], v.shape)
            Fp = orc.fitness(metric, vp, y, w)[0]
            assert abs(Fp - F) <= 2 * s + 1e-12 * abs(F), (i, metric, Fp, F, s)
        checked += 1
    assert checked >= 40
