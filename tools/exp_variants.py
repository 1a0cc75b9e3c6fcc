#!/usr/bin/env python
"""Builds alternative evaluator shapes for an A/B on one GPU box (tools/ab_libs.sh).

    python tools/exp_variants.py s4 name=NT,R,SUB,MINB,RED_ROWS[,Y_REGS[,MACRO:VALUE...]] [name=...]

Each experiment recompiles ONE variant translation unit (eval_<v>.cu's shape macros replaced)
and links it with the in-tree objects of everything else into
paper_2110_11226_b200/_exp/libgp_<name>.so (GP_B200_LIB selects it at run time).
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2110_11226_b200")
sys.path.insert(0, ROOT)
from paper_2110_11226_b200 import build as B  # noqa: E402

STACK = {"s4": 4, "s8": 8, "s12": 12, "s20": 20}


def one(var, name, shape):
    nt, r, sub, minb, rr, *extra = shape.split(",")
    yregs = extra[0] if extra else "0"
    defs = "".join(f"#define {kv.split(':')[0]} {kv.split(':')[1]}\n" for kv in extra[1:])
    exp = os.path.join(PKG, "_exp")
    os.makedirs(exp, exist_ok=True)
    src = os.path.join(exp, f"eval_{var}_{name}.cu")
    with open(src, "w") as f:
        f.write(f"#define GP_STACK {STACK[var]}\n#define GP_R {r}\n#define GP_SUB {sub}\n"
                f"#define GP_NT {nt}\n#define GP_MINB {minb}\n#define GP_RED_ROWS {rr}\n"
                f"#define GP_Y_REGS {yregs}\n" + defs +
                f'#include "{os.path.join(PKG, "csrc", "eval_impl.cuh")}"\n')
    obj = src + ".o"
    impl = os.path.join(PKG, "csrc", "eval_impl.cuh")
    if os.path.exists(obj) and os.path.getmtime(obj) > os.path.getmtime(impl):
        r_ = None                                   # up to date (rerun = relink only)
    else:
        r_ = subprocess.run([B.NVCC] + B.NVCC_FLAGS + ["-I", os.path.join(PKG, "csrc"), "-c", src,
                                                       "-o", obj], capture_output=True, text=True)
    if r_ is not None and r_.returncode:
        raise RuntimeError(r_.stderr)
    objs = [os.path.join(B.OBJ, f) for f in sorted(os.listdir(B.OBJ))
            if f.endswith(".o") and f != f"eval_{var}.cu.o"] + [obj]
    lib = os.path.join(exp, f"libgp_{name}.so")
    r_ = subprocess.run([B.NVCC, "-shared", "-o", lib] + objs +
                        ["-cudart", "static", "-ldl", "-lpthread", "-lrt"], capture_output=True, text=True)
    if r_.returncode:
        raise RuntimeError(r_.stderr)
    return lib, r_.stderr


if __name__ == "__main__":
    var = sys.argv[1]
    jobs = [a.split("=") for a in sys.argv[2:]]
    with cf.ThreadPoolExecutor(len(jobs)) as ex:
        for lib, _ in ex.map(lambda j: one(var, j[0], j[1]), jobs):
            print(lib)
