"""CPU check of the evaluator's polynomial tan (device_ops.cuh tan_poly, DESIGN.md section 8 item 9).

The constants are parsed from device_ops.cuh itself and the kernel's FFMA sequence is emulated in
numpy fp32 (tools/tan_fit.py: an fp32 FMA = the exact double product-sum rounded once); the result
must stay inside the oracle's tan error budget (oracle/gp_oracle.c eval_rec O_TAN for an exact
input) with margin, and match a fresh minimax fit of the polynomial. A typo in a coefficient or in
the pi/2 split fails here before any GPU run.
"""
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import tan_fit  # noqa: E402

F32 = np.float32
SRC = os.path.join(ROOT, "paper_2110_11226_b200", "csrc", "device_ops.cuh")


def _consts():
    text = open(SRC).read()
    vals = {}
    for name, val in re.findall(r"\b(k(?:TanP\d|Pio2[ABC]|TanMagic|TwoOverPi))\s*=\s*([-0-9.eE+]+)f", text):
        vals[name] = F32(float(val))
    return vals


def test_constants_present():
    c = _consts()
    for k in ["kTanP0", "kTanP1", "kTanP2", "kTanP3", "kTanP4", "kTanP5", "kPio2A", "kPio2B",
              "kPio2C", "kTanMagic", "kTwoOverPi"]:
        assert k in c, k
    # the three-constant split sums to pi/2 (to double precision of the split) and the magic
    # number is 1.5 * 2^23 (bit 0 of the sum = the parity of k)
    assert abs(float(c["kPio2A"]) + float(c["kPio2B"]) + float(c["kPio2C"]) - np.pi / 2) < 1e-15
    assert float(c["kTanMagic"]) == 1.5 * 2 ** 23
    assert c["kTwoOverPi"] == F32(2 / np.pi)


def _emulate(x, c):
    fma = tan_fit.fma
    j = fma(x, c["kTwoOverPi"], c["kTanMagic"])
    k = (j - c["kTanMagic"]).astype(F32)
    odd = (j.view(np.int32) & 1) == 1
    r = fma(k, -c["kPio2A"], x)
    r = fma(k, -c["kPio2B"], r)
    r = fma(k, -c["kPio2C"], r)
    z = (r * r).astype(F32)
    p = fma(c["kTanP5"], z, c["kTanP4"])
    for i in (3, 2, 1, 0):
        p = fma(p, z, c[f"kTanP{i}"])
    t = fma((r * z).astype(F32), p, r)
    return np.where(odd, (F32(-1) / t).astype(F32), t)


def test_device_tan_within_oracle_budget():
    c = _consts()
    u32, sfu_abs = 2.0 ** -24, 2.0 ** -21.41          # oracle/gp_oracle.c U32, SFU_ABS
    rng = np.random.default_rng(3)
    for lo, hi, max_ulp in [(-np.pi, np.pi, 4), (-10, 10, 4), (-1e3, 1e3, 4), (-1e5, 1e5, None)]:
        x = rng.uniform(lo, hi, 400_000).astype(F32)
        g = _emulate(x, c).astype(np.float64)
        a = x.astype(np.float64)
        e = np.tan(a)
        es = sfu_abs + np.abs(a) * 2 * u32
        cc = np.abs(np.cos(a))
        ok = cc > es
        budget = (es + np.abs(e) * es) / (cc - es) + 2 * u32 * np.abs(e)
        assert np.all(np.abs(g - e)[ok] <= 0.25 * budget[ok]), (lo, hi)
        if max_ulp:
            rel = np.abs(g - e) / np.maximum(np.abs(e), 1e-30)
            assert rel.max() <= max_ulp * u32, (lo, hi, rel.max() / u32)


def test_coefficients_match_a_fresh_fit():
    c = _consts()
    fitted, err = tan_fit.fit(iters=60)
    assert err < 3e-8
    for i in range(6):
        assert abs(float(c[f"kTanP{i}"]) - float(fitted[i])) <= 1e-5 * max(1.0, abs(float(fitted[i]))) + 2e-6, i
