#!/usr/bin/env python
"""Builds alternative evaluator shapes for an A/B on one GPU box (tools/ab_libs.sh).

    python tools/exp_variants.py s4 name=NT,R,SUB,MINB,RED_ROWS[,MACRO:VALUE...] [name=...]

Each experiment recompiles the kernels of ONE shape (the shape_<v>.h macros replaced; one
translation unit per (PREDICT, XSMEM) as in build.py) and links them with the in-tree objects of
everything else into paper_2110_11226_b200/_exp/libgp_<name>.so (GP_B200_LIB selects it at run
time). The shape must keep its tile NT * R * SUB (8192 for s4..s20, 2048 for w4 / w8) and the SUB
of its s/w partner.
"""
import concurrent.futures as cf
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2110_11226_b200")
sys.path.insert(0, ROOT)
from paper_2110_11226_b200 import build as B  # noqa: E402


def one(var, name, shape):
    nt, r, sub, minb, rr, *extra = shape.split(",")
    base = open(os.path.join(PKG, "csrc", f"shape_{var}.h")).read()
    keep = [ln for ln in base.splitlines()
            if ln.startswith("#define") and not re.match(
                r"#define GP_(R|SUB|NT|MINB|RED_ROWS|MINB_GLOBAL)\b", ln)]
    defs = "\n".join(keep) + (f"\n#define GP_R {r}\n#define GP_SUB {sub}\n#define GP_NT {nt}\n"
                              f"#define GP_MINB {minb}\n#define GP_RED_ROWS {rr}\n")
    if var.startswith("w"):
        defs += f"#define GP_MINB_GLOBAL {minb}\n"
    defs += "".join(f"#define {kv.split(':')[0]} {kv.split(':')[1]}\n" for kv in extra)
    exp = os.path.join(PKG, "_exp")
    os.makedirs(exp, exist_ok=True)
    m = B.SHAPES[var]                     # the shape's build modes (build.py)
    modes = ([(0, 0), (1, 0)] if m == "P" else [(0, 1), (1, 1)] if m == "S"
             else [(0, 0), (0, 1), (1, 0), (1, 1)])
    objs = []
    impl = os.path.join(PKG, "csrc", "eval_impl.cuh")

    def comp(m):
        kp, kxs = m
        src = os.path.join(exp, f"eval_{var}_{name}_{kp}{kxs}.cu")
        text = defs + f"#define GP_KP {kp}\n#define GP_KXS {kxs}\n#include \"{impl}\"\n"
        obj = src + ".o"
        if (os.path.exists(obj) and open(src).read() == text
                and os.path.getmtime(obj) > os.path.getmtime(impl)):
            return obj
        with open(src, "w") as f:
            f.write(text)
        r_ = subprocess.run([B.NVCC] + B.NVCC_FLAGS + ["-I", os.path.join(PKG, "csrc"), "-c", src,
                                                       "-o", obj], capture_output=True, text=True)
        if r_.returncode:
            raise RuntimeError(r_.stderr)
        with open(src + ".ptxas.log", "w") as f:
            f.write(r_.stderr)
        return obj

    with cf.ThreadPoolExecutor(len(modes)) as ex:
        objs = list(ex.map(comp, modes))
    main = [os.path.join(B.OBJ, f) for f in sorted(os.listdir(B.OBJ))
            if f.endswith(".o") and not f.startswith(f"eval_{var}_")
            and not re.match(r"eval_(s4|s8|s12|s20|w4|w8)\.cu\.o$", f)]
    lib = os.path.join(exp, f"libgp_{name}.so")
    r_ = subprocess.run([B.NVCC, "-shared", "-o", lib] + main + objs +
                        ["-cudart", "static", "-ldl", "-lpthread", "-lrt"], capture_output=True,
                        text=True)
    if r_.returncode:
        raise RuntimeError(r_.stderr)
    return lib


if __name__ == "__main__":
    var = sys.argv[1]
    jobs = [a.split("=") for a in sys.argv[2:]]
    with cf.ThreadPoolExecutor(len(jobs)) as ex:
        for lib in ex.map(lambda j: one(var, j[0], j[1]), jobs):
            print(lib)
