"""Oracle replay of the host side of the generational GP loop -- TEST INFRASTRUCTURE ONLY.

Pure-Python, step-by-step implementation of Alg. 1 as the paper's implementation runs it
(P:212-245): mutation kinds are decided first, tournaments are run, mutations
are applied on the host, including the hoisted crossover. Initialization is
ramped half-and-half. Where the paper is silent the SPEC readings apply (S:68-97,
S:317-390) and the exact random-draw order is DESIGN.md "Host RNG draw order"; the product's C++
engine implements the same readings independently, and tests compare the two bit-exactly
(teacher-forced: both sides are fed the same fp32 fitness every generation).

Uses only ``oracle`` (Philox, structure helpers, tournament); never imports the product.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (CONST, VAR, arity, depth, f32_bits, philox4x32_10, subtree_end, tournament)

FULL, GROW = 0, 1
# Mutation kinds, in the cumulative order of DESIGN.md C11 (crossover, subtree, hoist, point,
# residual reproduction).
CROSSOVER, SUBTREE, HOIST, POINT, REPRODUCTION = 0, 1, 2, 3, 4
# Philox counter word 3 ("purpose") per stream family.
P_TOURNAMENT, P_KIND, P_MUTATE, P_INIT = 0, 1, 2, 3


class Stream:
    """Sequential 32-bit words from Philox4x32-10 with key = seed and counter =
    (index, generation, block, purpose); block counts up from 0, words 0..3 used in order."""

    def __init__(self, seed: int, index: int, generation: int, purpose: int):
        self.key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
        self.index, self.generation, self.purpose = index, generation, purpose
        self.block, self.buf = 0, []

    def u32(self) -> int:
        if not self.buf:
            out = philox4x32_10((self.index, self.generation, self.block, self.purpose), self.key)
            self.buf = [int(x) for x in out]
            self.block += 1
        return self.buf.pop(0)

    def randint(self, n: int) -> int:
        """Uniform integer in [0, n): multiply-shift (C10)."""
        return (self.u32() * n) >> 32

    def uniform(self) -> float:
        """Uniform double in [0, 1) with 24 random bits: (word >> 8) * 2^-24."""
        return (self.u32() >> 8) * (1.0 / 16777216.0)


@dataclass
class Config:
    """EngineConfig, S:406-409 (Tables 2 and 6, P:354-374 / P:474-498)."""
    population_size: int = 256
    n_generations: int = 10
    tournament_size: int = 4
    parsimony: float = 0.01
    metric: str = "mse"
    p_crossover: float = 0.7
    p_subtree: float = 0.1
    p_hoist: float = 0.05
    p_point: float = 0.1
    p_point_replace: float = 0.05
    init_depth: tuple = (2, 6)
    const_range: tuple = (-1.0, 1.0)
    function_set: tuple = (2, 3, 4, 5, 9, 10, 11)   # {+,-,*,/,sin,cos,tan}
    n_features: int = 2
    stack_capacity: int = 20
    seed: int = 2110


def _terminal(st: Stream, cfg: Config):
    """Terminal draw: uniform over the n_features variables and one constant slot;
    a constant is lo + (hi - lo) * u rounded to fp32."""
    t = st.randint(cfg.n_features + 1)
    if t < cfg.n_features:
        return (VAR, t)
    lo, hi = cfg.const_range
    v = np.float32(lo + (hi - lo) * st.uniform())
    return (CONST, f32_bits(float(v)))


def random_program(st: Stream, method: int, max_depth: int, cfg: Config):
    """Full / Grow generation in prefix order."""
    fset = cfg.function_set
    out = []

    def rec(d):
        if d < max_depth:
            if method == FULL:
                f = fset[st.randint(len(fset))]
                out.append((f, 0))
                for _ in range(arity(f)):
                    rec(d + 1)
                return
            r = st.randint(len(fset) + cfg.n_features + 1)
            if r < len(fset):
                f = fset[r]
                out.append((f, 0))
                for _ in range(arity(f)):
                    rec(d + 1)
                return
        out.append(_terminal(st, cfg))

    rec(0)
    return out


def ramped_init(cfg: Config):
    """Ramped half-and-half: program i is Full if i < n//2 else Grow, with
    max depth d_min + (i mod (d_max - d_min + 1)); stream (i, 0, *, P_INIT)."""
    n = cfg.population_size
    dmin, dmax = cfg.init_depth
    pop = []
    for i in range(n):
        st = Stream(cfg.seed, i, 0, P_INIT)
        method = FULL if i < n // 2 else GROW
        pop.append(random_program(st, method, dmin + i % (dmax - dmin + 1), cfg))
    return pop


def choose_kinds(cfg: Config, generation: int):
    """Mutation kind per child, decided before selection."""
    kinds = []
    for i in range(cfg.population_size):
        u = Stream(cfg.seed, i, generation, P_KIND).uniform()
        c = 0.0
        kind = REPRODUCTION
        for kk, p in ((CROSSOVER, cfg.p_crossover), (SUBTREE, cfg.p_subtree),
                      (HOIST, cfg.p_hoist), (POINT, cfg.p_point)):
            c += p
            if u < c:
                kind = kk
                break
        kinds.append(kind)
    return kinds


def _arr(prog):
    return np.array(prog, dtype=np.int32).reshape(-1, 2)


def pick_subtree(st: Stream, prog):
    """Random subtree root: weight 9 for function nodes, 1 for terminals (90% / 10%),
    drawn as an integer in [0, total) and located by a linear cumulative scan."""
    weights = [9 if arity(op) > 0 else 1 for op, _ in prog]
    r = st.randint(sum(weights))
    c = 0
    for i, wgt in enumerate(weights):
        c += wgt
        if r < c:
            start = i
            break
    return start, subtree_end(_arr(prog), start)


def point_mutation(st: Stream, parent, cfg: Config):
    """each node replaced with probability p_point_replace; terminals by a random
    terminal, functions by a random same-arity function from the set."""
    child = list(parent)
    for i, (op, pl) in enumerate(child):
        if st.uniform() < cfg.p_point_replace:
            a = arity(op)
            if a == 0:
                child[i] = _terminal(st, cfg)
            else:
                cands = [f for f in cfg.function_set if arity(f) == a]
                if cands:
                    child[i] = (cands[st.randint(len(cands))], 0)
    return child


def hoist_mutation(st: Stream, parent):
    """S:343-351 / P:100: subtree S of the parent, subtree S' of S, S replaced by S'."""
    s, e = pick_subtree(st, parent)
    sub = parent[s:e]
    s2, e2 = pick_subtree(st, sub)
    return parent[:s] + sub[s2:e2] + parent[e:]


def hoisted_crossover(st: Stream, parent, donor, cfg: Config):
    """Crossover with the paper's re-hoist loop: while the child is
    deeper than stack_capacity - 1, the inserted donor subtree is replaced by a uniformly chosen
    proper subtree of itself."""
    s, e = pick_subtree(st, parent)
    ds, de = pick_subtree(st, donor)
    ins = donor[ds:de]
    child = parent[:s] + ins + parent[e:]
    while depth(_arr(child)) > cfg.stack_capacity - 1 and len(ins) > 1:
        r = 1 + st.randint(len(ins) - 1)
        ins = ins[r:subtree_end(_arr(ins), r)]
        child = parent[:s] + ins + parent[e:]
    return child


def subtree_mutation(st: Stream, parent, cfg: Config):
    """P:123 / S:370-377: hoisted crossover with a fresh Grow donor (init depth range)."""
    dmin, dmax = cfg.init_depth
    md = dmin + st.randint(dmax - dmin + 1)
    donor = random_program(st, GROW, md, cfg)
    return hoisted_crossover(st, parent, donor, cfg)


def make_children(pop, kinds, winners, cfg: Config, generation: int):
    """Apply the mutations for one generation given tournament winners."""
    children = []
    t = 0
    for i, kind in enumerate(kinds):
        st = Stream(cfg.seed, i, generation, P_MUTATE)
        parent = pop[winners[t]]
        t += 1
        if kind == CROSSOVER:
            donor = pop[winners[t]]
            t += 1
            children.append(hoisted_crossover(st, parent, donor, cfg))
        elif kind == SUBTREE:
            children.append(subtree_mutation(st, parent, cfg))
        elif kind == HOIST:
            children.append(hoist_mutation(st, parent))
        elif kind == POINT:
            children.append(point_mutation(st, parent, cfg))
        else:
            children.append(list(parent))
    return children


def flatten(pop):
    """Population -> (nodes (N,2) int32, offsets (n+1,) int64)."""
    lens = [len(p) for p in pop]
    off = np.zeros(len(pop) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    nodes = np.array([t for p in pop for t in p], dtype=np.int32).reshape(-1, 2)
    return nodes, off


def unflatten(nodes, offsets):
    nodes = np.asarray(nodes)
    return [[(int(a), int(b)) for a, b in nodes[offsets[i]:offsets[i + 1]]]
            for i in range(len(offsets) - 1)]


@dataclass
class GenerationRecord:
    generation: int
    kinds: list
    winners: np.ndarray
    population: list = field(default_factory=list)


def next_generation(pop, fitness_f32, cfg: Config, generation: int, higher_better: bool):
    """One iteration of Alg. 1's loop body minus evaluation: kinds, tournaments
    (2 per crossover, 1 otherwise: P:214), mutations."""
    kinds = choose_kinds(cfg, generation)
    n_t = sum(2 if k == CROSSOVER else 1 for k in kinds)
    lens = np.array([len(p) for p in pop], np.int32)
    winners = tournament(np.asarray(fitness_f32, np.float32), lens, n_t, cfg.tournament_size,
                         cfg.parsimony, higher_better, cfg.seed, generation)
    children = make_children(pop, kinds, winners, cfg, generation)
    return GenerationRecord(generation, kinds, winners, children)
