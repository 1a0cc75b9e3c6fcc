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
def _f32_eval(orc, prog, row):
    """fp32 emulation (numpy float32, correctly rounded +-*/; float32 libm for the rest)."""
    f = np.float32
    st = []
    T = f(1e-3)
    for op, pl in reversed([tuple(t) for t in prog]):
        if op == 0:
            st.append(f(row[pl]))
            continue
        if op == 1:
            st.append(f(orc.bits_f32(pl)))
            continue
        a = st.pop()
        b = st.pop() if orc.arity(op) == 2 else f(0)
        with np.errstate(all="ignore"):
            r = {2: lambda: a + b, 3: lambda: a - b, 4: lambda: a * b,
                 5: lambda: f(1) if abs(b) < T else a / b, 9: lambda: np.sin(a),
                 10: lambda: np.cos(a), 11: lambda: np.tan(a)}[op]()
        st.append(f(r))
    return st[0]


def test_error_bound_covers_fp32_evaluation(orc):
    nodes, off = synth.random_population(300, seed=21, depth=(1, 7))
    X, _ = synth.pagie_grid(8)
    checked = 0
    for i in range(len(off) - 1):
        p = nodes[off[i]:off[i + 1]]
        v, e, fl = orc.eval_program(p, X)
        for r in range(X.shape[1]):
            if fl[r]:
                continue
            g = float(_f32_eval(orc, p, X[:, r]))
            assert abs(g - v[r]) <= e[r] + 1e-300, (i, r, g, v[r], e[r])
            checked += 1
    assert checked > 10_000
