"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck): every evaluator kernel
(s4 / s8 / s12 / s20 with the shared-memory X tile, w4 / w8 with global X), all five streaming
metrics weighted and unweighted, Spearman, gp_predict, the partial / finalize split, tournament
selection and the engine with device mutation -- at C1-like sizes so the tools finish in minutes.

    compute-sanitizer --tool memcheck python tools/sanitize_drive.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_11226_b200 as gp  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


ctx = gp.Context(0)
X, y = synth.pagie_grid(48)                               # 2304 rows: a tile + a ragged tail
Xw, yw = synth.higgs_like(2048 + 300, seed=3)             # 28 columns: global-X kernels
w = synth.weights(X.shape[1], seed=1)
nodes, off = synth.random_population(150, seed=2, depth=(0, 6), funcs=synth.ALL_FUNCS, max_stack=8)
deep, doff = synth.deep_population(60, seed=4, need=(2, 20))
for metric in ("mae", "mse", "rmse", "logloss", "pearson", "spearman"):
    for ww in (None, dev(w)):
        yy = y if metric != "logloss" else (y > 1).astype(np.float32)
        ctx.evaluate(dev(nodes), dev(off), dev(X), dev(yy), ww, metric=metric, max_stack=8)
    ctx.evaluate(dev(nodes), dev(off), dev(Xw), dev(yw), None, metric=metric, max_stack=8)
ctx.set_eval_order(False)
for metric in ("mse", "pearson"):
    ctx.evaluate(dev(deep), dev(doff), dev(X), dev(y), metric=metric, max_stack=20)
ctx.predict(dev(deep), dev(doff), dev(X), max_stack=20)
ctx.set_eval_order(True)
ctx.predict(dev(nodes), dev(off), dev(Xw), max_stack=8)
ctx.set_plan(128, 1)
ctx.evaluate(dev(nodes), dev(off), dev(X), dev(y), dev(w), metric="mse", max_stack=8)
ctx.set_plan(0, 0)
s = ctx.evaluate_partial(dev(nodes), dev(off), dev(X), dev(y), metric="pearson", max_stack=8)
ctx.finalize_sums(dev(nodes), dev(off), s, X.shape[0], metric="pearson", max_stack=8)
fit, _ = ctx.evaluate(dev(nodes), dev(off), dev(X), dev(y), metric="mse", max_stack=8)
ctx.tournament_select(fit, dev(off), 300, 4, 0.01, False, seed=1, generation=1)
for cfg in (dict(metric="mse"), dict(metric="pearson", init_depth_max=8, stack_capacity=10)):
    e = gp.Engine(ctx, dev(X), dev(y), population_size=128, seed=5, **cfg)
    e.init_population()
    for _ in range(3):
        e.generation()
    e.population()
    e.close()
torch.cuda.synchronize()
ctx.close()
print("sanitize drive done")
