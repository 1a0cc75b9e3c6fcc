#!/usr/bin/env python
"""Coefficients and accuracy of the evaluator's tan (device_ops.cuh tan_poly, GP_TAN_POLY = 1).

1. Fits P(z), z = r^2, with tan r = r + r z P(z) on |r| <= pi/4: degree-5 polynomial, minimax on
   the relative error of tan by Lawson's iteratively reweighted least squares (Chebyshev nodes).
2. Emulates the kernel's fp32 FFMA sequence in numpy (an fp32 FMA = the exact double product-sum
   rounded once to fp32; the reciprocal correctly rounded -- MUFU.RCP is within 1 ulp of it) and
   reports, per argument range, the max relative error and the max error as a fraction of the
   oracle's tan budget (oracle/gp_oracle.c eval_rec O_TAN, for an exact input: es = SFU_ABS +
   |a| 2 U32, (es + |tan a| es) / (|cos a| - es) + 2 U32 |tan a|).

    python tools/tan_fit.py
"""
import numpy as np

f32 = np.float32


def fit(deg=5, n=20000, iters=200):
    lim = np.pi / 4
    t = np.cos(np.pi * (np.arange(n) + 0.5) / n)
    z = (t + 1) / 2 * lim * lim
    r = np.sqrt(z)
    target = (np.tan(r) / r - 1) / z
    w = r * z / np.tan(r)                     # P error -> relative error of tan
    A = np.vander(z, deg + 1, increasing=True) * w[:, None]
    u = np.ones(n)
    for _ in range(iters):
        sw = np.sqrt(u)
        c = np.linalg.lstsq(A * sw[:, None], target * w * sw, rcond=None)[0]
        e = np.abs(A @ c - target * w)
        u = u * e
        u /= u.sum()
    return c.astype(f32), float(np.max(np.abs(A @ c - target * w)))


def fma(a, b, c):
    return (np.float64(a) * np.float64(b) + np.float64(c)).astype(f32)


def tan_poly(x, c):
    """The FFMA sequence of device_ops.cuh tan_poly, in fp32."""
    magic, two_over_pi = f32(12582912.0), f32(2 / np.pi)
    c1 = f32(np.pi / 2)
    c2 = f32(np.pi / 2 - float(c1))
    c3 = f32(np.pi / 2 - float(c1) - float(c2))
    j = fma(x, two_over_pi, magic)
    k = (j - magic).astype(f32)
    odd = (j.view(np.int32) & 1) == 1
    r = fma(k, -c1, x)
    r = fma(k, -c2, r)
    r = fma(k, -c3, r)
    z = (r * r).astype(f32)
    p = fma(f32(c[5]), z, f32(c[4]))
    for i in (3, 2, 1, 0):
        p = fma(p, z, f32(c[i]))
    t = fma((r * z).astype(f32), p, r)
    return np.where(odd, (f32(-1) / t).astype(f32), t), (c1, c2, c3)


def main():
    c, err = fit()
    print("P coefficients (fp32):", ", ".join(repr(float(v)) for v in c), f"; fit rel err {err:.3g}")
    u32, sfu_abs = 2.0 ** -24, 2.0 ** -21.41
    rng = np.random.default_rng(0)
    for lo, hi in [(-np.pi, np.pi), (-10, 10), (-1e3, 1e3), (-1e5, 1e5), (-3e6, 3e6)]:
        x = rng.uniform(lo, hi, 2_000_000).astype(f32)
        g, consts = tan_poly(x, c)
        g = g.astype(np.float64)
        a = x.astype(np.float64)
        e = np.tan(a)
        es = sfu_abs + np.abs(a) * 2 * u32
        cc = np.abs(np.cos(a))
        budget = np.where(cc > es, (es + np.abs(e) * es) / np.maximum(cc - es, 1e-300)
                          + 2 * u32 * np.abs(e), np.inf)
        rel = np.abs(g - e) / np.maximum(np.abs(e), 1e-30)
        print(f"|x| <= {hi:g}: max rel err {rel.max():.3g} ({rel.max() / u32:.1f} ulp), "
              f"max err / oracle budget {np.max(np.abs(g - e) / budget):.3f}")
    print("pi/2 split:", ", ".join(repr(float(v)) for v in consts))


if __name__ == "__main__":
    main()
