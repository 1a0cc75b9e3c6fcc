"""Evaluate a fixed generation-0 (ramped half-and-half) C3 population repeatedly: a profiling
harness for the evaluator on SFU-heavy programs (python tools/eval_gen0.py [reps] [config])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2110_11226_b200 as gp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3"]
X, y, _, _, _ = bench.load_dataset(cfg)
X, y = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
ctx = gp.Context(0)
e = gp.Engine(ctx, X, y, population_size=cfg["pop"], metric=cfg["metric"], seed=2110,
              init_depth_min=cfg["depth"][0], init_depth_max=cfg["depth"][1])
e.init_population()
n, o, _ = e.population()
nd, of = torch.from_numpy(n).cuda(), torch.from_numpy(o).cuda()
ctx.set_profiling(True)
for _ in range(reps):
    ctx.evaluate(nd, of, X, y, metric=cfg["metric"], max_stack=20)
torch.cuda.synchronize()
ms, launches = ctx.eval_timing()
print(f"gen0: {len(o) - 1} programs, {len(n)} nodes, {ms / reps:.2f} ms per evaluation, "
      f"{len(n) * X.shape[1] * reps / (ms * 1e-3) / 1e12:.3f} Tnode-evals/s")
