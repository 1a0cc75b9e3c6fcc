"""CPU oracle for arXiv 2110.11226's data-parallel hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this package. The product package ``paper_2110_11226_b200`` never imports it, and
the two share no code (see ``gp_oracle.c`` header and DESIGN.md "Oracle").

This module is argument marshalling over ``libgp_oracle.so`` (plain C, double precision) plus the
pure-Python replay of the host engine in :mod:`oracle.engine`.

Node arrays are numpy ``int32`` arrays of shape ``(len, 2)``: column 0 the opcode, column 1 the
variable index or the float32 bits of the constant (the C-ABI's 8-byte node).

Parity pinned: every function here is pinned by ``tests/test_oracle_*.py`` (values from PAPER.md /
SPEC.md, closed forms, identities, brute force). None is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gp_oracle.c")
_LIB = os.path.join(_HERE, "libgp_oracle.so")

# Opcodes (the public interface numbering, retyped -- DESIGN.md "Function catalog").
VAR, CONST = 0, 1
ADD, SUB, MUL, DIV, MIN, MAX, POW = 2, 3, 4, 5, 6, 7, 8
SIN, COS, TAN, ABS, NEG, SQRT, LOG, EXP, INV = 9, 10, 11, 12, 13, 14, 15, 16, 17
SQUARE, CUBE, TANH, SINH, COSH, ASIN, ACOS, ATAN = 18, 19, 20, 21, 22, 23, 24, 25
N_OPS = 26
NAMES = ["var", "const", "add", "sub", "mul", "div", "min", "max", "pow", "sin", "cos", "tan",
         "abs", "neg", "sqrt", "log", "exp", "inv", "square", "cube", "tanh", "sinh", "cosh",
         "asin", "acos", "atan"]
METRICS = {"mae": 0, "mse": 1, "rmse": 2, "logloss": 3, "pearson": 4, "spearman": 5}
# Program flags returned by population_fitness.
F_OVERFLOW, F_AMBIGUOUS, F_INVALID, F_UNDEFINED = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11",
                               "-D_DEFAULT_SOURCE", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u32, u64, f32, dbl = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                        ctypes.c_uint64, ctypes.c_float, ctypes.c_double)
        L.orc_arity.argtypes, L.orc_arity.restype = [ctypes.c_int], ctypes.c_int
        L.orc_validate.argtypes, L.orc_validate.restype = [P, i64, ctypes.c_int], ctypes.c_int
        L.orc_subtree_end.argtypes, L.orc_subtree_end.restype = [P, i64, i64], i64
        L.orc_depth.argtypes, L.orc_depth.restype = [P, i64], ctypes.c_int
        L.orc_stack_need.argtypes, L.orc_stack_need.restype = [P, i64], ctypes.c_int
        L.orc_apply.argtypes, L.orc_apply.restype = [ctypes.c_int, dbl, dbl], dbl
        L.orc_eval_program.argtypes = [P, i64, P, i64, i64, P, P, P]
        L.orc_eval_program.restype = None
        L.orc_eval_row.argtypes, L.orc_eval_row.restype = [P, P, i64, i64], dbl
        L.orc_fitness.argtypes, L.orc_fitness.restype = [ctypes.c_int, P, P, P, i64, P], dbl
        L.orc_rank_vector.argtypes, L.orc_rank_vector.restype = [P, i64, P], None
        L.orc_fitness_sensitivity.argtypes = [ctypes.c_int, P, P, P, P, i64]
        L.orc_fitness_sensitivity.restype = dbl
        L.orc_philox4x32_10.argtypes, L.orc_philox4x32_10.restype = [P, P, P], None
        L.orc_tournament_one.argtypes = [P, P, i32, i32, i32, f32, ctypes.c_int, u64, u32]
        L.orc_tournament_one.restype = i32
        L.orc_tournament.argtypes = [P, P, i32, i32, i32, f32, ctypes.c_int, u64, u32, P]
        L.orc_tournament.restype = None
        L.orc_pagie.argtypes, L.orc_pagie.restype = [dbl, dbl], dbl
        L.orc_population_fitness.argtypes = [P, P, i32, P, i64, P, P, i64, i32, ctypes.c_int,
                                             P, P, P]
        L.orc_population_fitness.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _nodes(nodes) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(nodes, dtype=np.int32))
    assert a.ndim == 2 and a.shape[1] == 2, "nodes must be (len, 2) int32"
    return a


def _colmajor(X) -> tuple[np.ndarray, int, int]:
    """X given as (n_cols, n_rows) float32 (column-major storage)."""
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
    if X.ndim == 1:
        X = X[None, :]
    return X, X.shape[1], X.shape[0]


# ---- node helpers -------------------------------------------------------------------------------
def f32_bits(v: float) -> int:
    return int(np.array([v], dtype=np.float32).view(np.int32)[0])


def bits_f32(b: int) -> float:
    return float(np.array([b], dtype=np.int32).view(np.float32)[0])


def node(op, payload=0):
    """Build one node: node('add'), node('var', 1), node('const', 2.5)."""
    if isinstance(op, str):
        op = NAMES.index(op)
    if op == CONST:
        return (CONST, f32_bits(payload))
    return (op, int(payload))


def program(*tokens) -> np.ndarray:
    """program('add', ('var', 0), ('const', 1.0)) -> (len, 2) int32 node array."""
    out = []
    for t in tokens:
        out.append(node(*t) if isinstance(t, tuple) else node(t))
    return np.array(out, dtype=np.int32).reshape(-1, 2)


def arity(op: int) -> int:
    return lib().orc_arity(int(op))


# ---- structure ----------------------------------------------------------------------------------
def validate(nodes, n_cols: int = 1 << 30) -> int:
    a = _nodes(nodes)
    return lib().orc_validate(_p(a), len(a), n_cols)


def depth(nodes) -> int:
    a = _nodes(nodes)
    return lib().orc_depth(_p(a), len(a))


def stack_need(nodes) -> int:
    a = _nodes(nodes)
    return lib().orc_stack_need(_p(a), len(a))


def subtree_end(nodes, start: int) -> int:
    a = _nodes(nodes)
    return int(lib().orc_subtree_end(_p(a), len(a), start))


def apply(op: int, a: float, b: float = 0.0) -> float:
    return lib().orc_apply(int(op), float(a), float(b))


# ---- evaluation ---------------------------------------------------------------------------------
def eval_program(nodes, X):
    """Recursive evaluation over all rows: returns (value float64[n], err_bound float64[n],
    flags uint8[n])."""
    a = _nodes(nodes)
    Xc, ld, _ = _colmajor(X)
    n = ld
    v = np.empty(n, np.float64)
    e = np.empty(n, np.float64)
    f = np.empty(n, np.uint8)
    lib().orc_eval_program(_p(a), len(a), _p(Xc), ld, n, _p(v), _p(e), _p(f))
    return v, e, f


def fitness(metric, yhat, y, w=None):
    """Weighted metric. Returns (fitness, undefined_flag)."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    yh = np.ascontiguousarray(yhat, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    ww = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    und = ctypes.c_int(0)
    f = lib().orc_fitness(m, _p(yh), _p(yy), _p(ww), len(yh), ctypes.byref(und))
    return f, bool(und.value)


def rank_vector(values):
    """ranks 1..n, ties averaged."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(len(v), np.float64)
    lib().orc_rank_vector(_p(v), len(v), _p(out))
    return out


def fitness_sensitivity(metric, yhat, err, y, w=None) -> float:
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    yh = np.ascontiguousarray(yhat, dtype=np.float64)
    ee = np.ascontiguousarray(err, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    ww = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    return lib().orc_fitness_sensitivity(m, _p(yh), _p(ee), _p(yy), _p(ww), len(yh))


def population_fitness(nodes, offsets, X, y, w, metric):
    """All programs of a flat population: returns (fitness f64[n], sensitivity f64[n],
    flags i32[n])."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    a = _nodes(nodes)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    Xc, ld, n_cols = _colmajor(X)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    ww = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    n = len(off) - 1
    fit = np.empty(n, np.float64)
    sens = np.empty(n, np.float64)
    flags = np.empty(n, np.int32)
    lib().orc_population_fitness(_p(a), _p(off), n, _p(Xc), ld, _p(yy), _p(ww), ld, n_cols, m,
                                 _p(fit), _p(sens), _p(flags))
    return fit, sens, flags


# ---- RNG / selection ----------------------------------------------------------------------------
def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32).reshape(4))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32).reshape(2))
    o = np.empty(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def tournament(fitness_f32, lens, n_tournaments, k, parsimony, higher_better, seed, generation):
    f = np.ascontiguousarray(fitness_f32, dtype=np.float32)
    L = np.ascontiguousarray(lens, dtype=np.int32)
    out = np.empty(n_tournaments, np.int32)
    lib().orc_tournament(_p(f), _p(L), len(f), n_tournaments, k, np.float32(parsimony),
                         int(bool(higher_better)), seed, generation, _p(out))
    return out


def pagie(x: float, y: float) -> float:
    """Eq. 3."""
    return lib().orc_pagie(float(x), float(y))
