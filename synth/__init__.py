"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no evaluation, no fitness, no selection, no
mutation). It only produces inputs: datasets with the shapes of the paper's workloads and random
prefix programs, all from explicit seeds. Recipes are stated in DESIGN.md "Input recipe".

Datasets are returned column-major: ``X`` has shape ``(n_cols, n_rows)`` float32.
Programs are flat: ``nodes`` (N, 2) int32 -- column 0 opcode, column 1 var index or float32 bits of
the constant -- and ``offsets`` (n+1,) int64.
"""
from __future__ import annotations

import numpy as np

# Public opcode numbering; inputs only need to name opcodes.
VAR, CONST = 0, 1
BINARY = (2, 3, 4, 5, 6, 7, 8)          # add sub mul div min max pow
UNARY = tuple(range(9, 26))             # sin cos tan abs neg sqrt log exp inv square cube tanh
#                                         sinh cosh asin acos atan
TABLE2_SET = (2, 3, 4, 5, 9, 10, 11)    # {+,-,*,/,sin,cos,tan}, P:369 / P:493
ALL_FUNCS = BINARY + UNARY


def _arity(op: int) -> int:
    return 0 if op in (VAR, CONST) else (2 if op in BINARY else 1)


# ---- datasets -------------------------------------------------------------------------------------
def pagie_grid(side: int):
    """Pagie-1 data set (Eq. 3) on the inclusive uniform side x side grid over
    [-5, 5]^2 (SPEC S:502 reading, C14): g_i = -5 + 10 i / (side - 1) in double, stored
    fp32; row r = i * side + j holds (g_i, g_j); target in double from the fp32 coordinates, stored
    fp32. Returns (X (2, side^2) float32, y (side^2,) float32)."""
    assert side >= 2
    g = (-5.0 + 10.0 * np.arange(side, dtype=np.float64) / (side - 1)).astype(np.float32)
    x0 = np.repeat(g, side)
    x1 = np.tile(g, side)
    X = np.stack([x0, x1])
    xd, yd = x0.astype(np.float64), x1.astype(np.float64)
    with np.errstate(divide="ignore"):
        t0 = np.where(xd == 0.0, 0.0, 1.0 / (1.0 + xd ** -4.0))
        t1 = np.where(yd == 0.0, 0.0, 1.0 / (1.0 + yd ** -4.0))
    return X, (t0 + t1).astype(np.float32)


def higgs_like(n_rows: int, seed: int = 2110, n_cols: int = 28):
    """Higgs-shaped binary classification (Table 5: 11M x 28): features iid N(0,1) fp32,
    labels 1[sum_j a_j x_j + 0.5 x0 x1 + 0.5 eps > 0] with a, eps ~ N(0,1) from the seed."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_cols, n_rows), dtype=np.float32)
    a = rng.standard_normal(n_cols).astype(np.float32)
    eps = rng.standard_normal(n_rows, dtype=np.float32)
    s = a @ X + 0.5 * X[0] * X[1] + 0.5 * eps
    return X, (s > 0).astype(np.float32)


def year_like(n_rows: int, seed: int = 2110, n_cols: int = 90):
    """YearPredictionMSD-shaped regression (Table 5: 515K x 90): features iid N(0,1) fp32,
    y = 1998 + 10.9 * clip(sum_j b_j x_j / sqrt(90) + 0.3 x0 x1, -3, 3)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_cols, n_rows), dtype=np.float32)
    b = rng.standard_normal(n_cols).astype(np.float32)
    s = (b @ X) / np.float32(np.sqrt(n_cols)) + np.float32(0.3) * X[0] * X[1]
    return X, (np.float32(1998.0) + np.float32(10.9) * np.clip(s, -3, 3)).astype(np.float32)


def weights(n_rows: int, seed: int = 7, zero_fraction: float = 0.1):
    """Non-uniform sample weights in [0, 2) with a fraction of exact zeros (w >= 0)."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.0, 2.0, n_rows).astype(np.float32)
    w[rng.random(n_rows) < zero_fraction] = 0.0
    return w


# ---- programs -------------------------------------------------------------------------------------
def random_population(n: int, seed: int = 1, depth=(1, 6), funcs=TABLE2_SET, n_features: int = 2,
                      const_range=(-1.0, 1.0), p_terminal: float = 0.3, max_stack: int | None = None):
    """Random valid prefix programs for parity tests (NOT the engine's ramped init): each node at
    depth < max_depth is a terminal with probability p_terminal, else a uniformly chosen function;
    terminals are a variable or a constant with equal probability. Programs whose reverse-prefix
    stack need exceeds max_stack are redrawn. Returns (nodes (N,2) int32, offsets (n+1,) int64)."""
    rng = np.random.default_rng(seed)
    progs = []
    while len(progs) < n:
        md = int(rng.integers(depth[0], depth[1] + 1))
        out = []

        def rec(d):
            if d < md and rng.random() >= p_terminal:
                f = int(funcs[rng.integers(len(funcs))])
                out.append((f, 0))
                for _ in range(_arity(f)):
                    rec(d + 1)
            elif rng.random() < 0.5:
                out.append((VAR, int(rng.integers(n_features))))
            else:
                v = np.float32(rng.uniform(*const_range))
                out.append((CONST, int(np.array([v]).view(np.int32)[0])))

        rec(0)
        if max_stack is not None and stack_occupancy(out) > max_stack:
            continue
        progs.append(out)
    return flatten(progs)


def deep_population(n: int, seed: int = 1, need=(9, 20), funcs=(2, 3, 4, 9, 10),
                    n_features: int = 2, const_range=(-1.0, 1.0)):
    """Left-deep programs with a prescribed reverse-prefix stack need in [need[0], need[1]]: each
    binary node's FIRST operand carries the deep chain (the second operand is evaluated first and
    stays on the stack), so a chain of d binary nodes needs d + 1 slots. Sides are terminals or
    unary-wrapped terminals; sin/cos in the default op mix keep values bounded (well-conditioned
    programs for exercising every stack slot of the 12- and 20-slot kernels)."""
    rng = np.random.default_rng(seed)
    binary = [f for f in funcs if f in BINARY]
    unary = [f for f in funcs if f in UNARY]

    def term():
        if rng.random() < 0.5:
            return [(VAR, int(rng.integers(n_features)))]
        v = np.float32(rng.uniform(*const_range))
        return [(CONST, int(np.array([v]).view(np.int32)[0]))]

    progs = []
    for _ in range(n):
        d = int(rng.integers(need[0], need[1] + 1)) - 1
        out = []
        for _ in range(d):
            if unary and rng.random() < 0.3:
                out.append((int(rng.choice(unary)), 0))
            out.append((int(rng.choice(binary)), 0))
        out += term()
        # prefix = b_1 [u] b_2 [u] ... b_d t0 s_d ... s_1: the second operand s_i of b_i follows
        # b_i's first-operand chain; each s_i is a terminal or a unary of a terminal
        seconds = []
        for op, _ in out:
            if op in BINARY:
                s = term()
                if unary and rng.random() < 0.5:
                    s = [(int(rng.choice(unary)), 0)] + s
                seconds.append(s)
        prog = list(out)
        for s in reversed(seconds):
            prog += s
        progs.append(prog)
    return flatten(progs)


def stack_occupancy(prog) -> int:
    """Maximum occupancy of a reverse-prefix stack walk (counter only; for input filtering)."""
    sp = need = 0
    for op, _ in reversed(prog):
        sp += 1 - _arity(op)
        need = max(need, sp)
    return need


def flatten(progs):
    off = np.zeros(len(progs) + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in progs])
    nodes = np.array([t for p in progs for t in p], dtype=np.int32).reshape(-1, 2)
    return nodes, off


def shard_rows(n_rows: int, rank: int, world: int):
    """Contiguous, even row shard of rank: [r*m//P, (r+1)*m//P)."""
    return (rank * n_rows) // world, ((rank + 1) * n_rows) // world
