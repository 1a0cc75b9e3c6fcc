// device_ops.cuh -- fp32 function semantics of the GP catalog on sm_100a.
//
// Semantics: SPEC's protected catalog as read in DESIGN.md C2 / include/gp.h.
// Transcendentals use the SFU (MUFU) approximations: __sinf/__cosf (MUFU.SIN/COS after an
// FMUL.RZ range scaling), __expf (MUFU.EX2), __logf (MUFU.LG2), rcp.approx (MUFU.RCP); compiled
// with -ftz=true. Every body is branch-free (selects only).
// Their error budgets are what the oracle's tolerance model assumes.
// min/max/clamps follow the oracle's C semantics: fmin/fmax drop a NaN operand, comparison
// clamps (sinh, asin, acos) propagate it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/gp.h"
#include "common.h"

namespace gpb {

constexpr float kProt = 1e-3f;   // S:132 protection threshold, strict "<" (no float in [1e-3, 1e-3f))
constexpr float kBig = 1e30f;    // S:132 exp clamp; reused for sinh / cosh / pow (C2)

// MUFU.SQRT (no IEEE slow-path call inside the dispatch switch).
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// MUFU.RCP, branch-free (the protected ops select afterwards so no case body contains a branch).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Reciprocal on the FMA pipe instead of MUFU.RCP (GP_RCP_FMA = 1; default 0 = MUFU.RCP). A third
// of the MUFU work of the paper's function set is the reciprocal of div and tan and the FMA pipe
// has 8x the XU's throughput, but the r02 A/B (profiles/ab_r02_rcp.log) measured C3 134 -> 242 ms
// per step and C5 / C4 slower too: the evaluator is bound by issue and latency around the SFU, and
// 12 more instructions per row pair (plus register pressure: spills at the 128-register budget)
// cost more than the XU time they free. Kept as a documented option. Seed: the magic-constant estimate
// of 1/|b| (5 % relative error), then three Newton steps r += r (1 - |b| r) -- <= 0.59 ulp over
// every normal |b| (numpy emulation of the FFMA sequence over 2^-126..2^126), i.e. as accurate as
// rcp.approx (the oracle's budget for div / inv is 3 u). |b| > 2^126
// -> 0 (the flushed result); 0 -> inf; NaN propagates. Branch-free. The _x2 form runs two rows
// through FFMA2 with the same roundings (bit-identical to two scalar calls).
#ifndef GP_RCP_FMA
#define GP_RCP_FMA 0
#endif
constexpr int kRcpMagic = 0x7EF311C7;
constexpr float kRcpHuge = 8.50705917e37f;   // 2^126
__device__ __forceinline__ float rcp_fast(float b) {
#if GP_RCP_FMA
  const float ab = fabsf(b);
  float r = __int_as_float(kRcpMagic - __float_as_int(ab)), e;
  e = fmaf(-ab, r, 1.0f); r = fmaf(r, e, r);
  e = fmaf(-ab, r, 1.0f); r = fmaf(r, e, r);
  e = fmaf(-ab, r, 1.0f); r = fmaf(r, e, r);
  return copysignf(ab > kRcpHuge ? 0.0f : r, b);
#else
  return rcp_approx(b);
#endif
}

// a = first operand (first popped), b = second operand.
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Branch-free bodies for the extended catalog (libdevice versions branch internally, which makes
// ptxas insert register copies in front of the dispatch for EVERY node). Polynomials: Taylor
// series where stated, Cephes single-precision minimax coefficients for asin / atan.
__device__ __forceinline__ float tanh_bf(float a) {
  const float t = 1.0f - 2.0f * rcp_approx(__expf(2.0f * a) + 1.0f);
  const float a2 = a * a;
  const float p = a * (1.0f + a2 * (-1.0f / 3.0f + a2 * (2.0f / 15.0f + a2 * (-17.0f / 315.0f))));
  return fabsf(a) < 0.125f ? p : t;
}
__device__ __forceinline__ float sinh_bf(float a) {
  const float e = __expf(a), s = 0.5f * (e - rcp_approx(e));
  const float a2 = a * a;
  const float p = a * (1.0f + a2 * (1.0f / 6.0f + a2 * (1.0f / 120.0f + a2 * (1.0f / 5040.0f +
                                                                               a2 / 362880.0f))));
  const float r = fabsf(a) < 0.5f ? p : s;
  return r > kBig ? kBig : (r < -kBig ? -kBig : r);
}
// asin on [0, 1] given z and s (Cephes asinf): |x| <= 0.5: s = |x|, z = x^2;
// |x| > 0.5: z = (1 - |x|) / 2, s = sqrt(z), asin|x| = pi/2 - 2 * core.
__device__ __forceinline__ float asin_core(float s, float z) {
  const float p = (((4.2163199048e-2f * z + 2.4181311049e-2f) * z + 4.5470025998e-2f) * z +
                   7.4953002686e-2f) * z + 1.6666752422e-1f;
  return s + s * z * p;
}
__device__ __forceinline__ float asin_bf(float x) {
  x = x < -1.0f ? -1.0f : (x > 1.0f ? 1.0f : x);
  const float ax = fabsf(x);
  const bool big = ax > 0.5f;
  const float z = big ? 0.5f * (1.0f - ax) : ax * ax;
  const float c = asin_core(big ? sqrt_approx(z) : ax, z);
  return copysignf(big ? 1.57079632679489662f - 2.0f * c : c, x);
}
__device__ __forceinline__ float acos_bf(float x) {
  x = x < -1.0f ? -1.0f : (x > 1.0f ? 1.0f : x);
  const float ax = fabsf(x);
  const bool big = ax > 0.5f;
  const float z = big ? 0.5f * (1.0f - ax) : ax * ax;
  const float c = asin_core(big ? sqrt_approx(z) : ax, z);
  const float small_r = 1.57079632679489662f - copysignf(c, x);
  const float big_r = x > 0.0f ? 2.0f * c : 3.14159265358979324f - 2.0f * c;
  return big ? big_r : small_r;
}
__device__ __forceinline__ float atan_bf(float x) {
  const float ax = fabsf(x);
  const bool c1 = ax > 2.414213562373095f, c2 = ax > 0.4142135623730950f;  // tan(3pi/8), tan(pi/8)
  const float xr = c1 ? -rcp_approx(ax) : (c2 ? (ax - 1.0f) * rcp_approx(ax + 1.0f) : ax);
  const float y0 = c1 ? 1.57079632679489662f : (c2 ? 0.78539816339744831f : 0.0f);
  const float z = xr * xr;
  const float r = y0 + ((((8.05374449538e-2f * z - 1.38776856032e-1f) * z + 1.99777106478e-1f) * z -
                         3.33329491539e-1f) * z * xr + xr);
  return copysignf(r, x);
}

// a = first operand (first popped), b = second operand.
template <int OP>
__device__ __forceinline__ float apply2(float a, float b) {
  if constexpr (OP == GP_OP_ADD) return a + b;
  else if constexpr (OP == GP_OP_SUB) return a - b;
  else if constexpr (OP == GP_OP_MUL) return a * b;
  else if constexpr (OP == GP_OP_DIV) { const float q = a * rcp_fast(b); return fabsf(b) < kProt ? 1.0f : q; }
  else if constexpr (OP == GP_OP_MIN) return fminf(a, b);
  else if constexpr (OP == GP_OP_MAX) return fmaxf(a, b);
  else {  // GP_OP_POW: |a|^b = 2^(b * log2|a|), clamped; 0^b and b == 0 by selects
    const float r = fminf(ex2_approx(b * lg2_approx(fabsf(a))), kBig);
    const float r0 = a == 0.0f ? (b > 0.0f ? 0.0f : kBig) : r;
    return b == 0.0f ? 1.0f : r0;
  }
}

// tan on the FMA pipe plus ONE MUFU.RCP (GP_TAN_POLY = 1, default) instead of sin, cos and rcp
// (3 MUFU): x = k pi/2 + r with k = rint(2x/pi) (the 1.5 * 2^23 magic addition; bit 0 of the sum
// is k's parity) and r by a three-constant FMA Cody-Waite reduction (|r| <= pi/4); tan r =
// r + r z P(z), z = r^2, P the degree-5 minimax fit of (tan r / r - 1) / z on [0, (pi/4)^2]
// (tools/tan_fit.py: 1.8e-8 relative; the coefficients agree with Cephes tanf); tan x = tan r for
// even k, -1 / tan r for odd k. numpy emulation of this FFMA sequence (tools/tan_fit.py): <= 3 ulp
// for |x| < 1e3 and <= 0.12 of the oracle's tan budget for |x| up
// to 3e6; beyond 2^22 pi/2 the magic rounding fails and the budget is infinite (excluded).
#ifndef GP_TAN_POLY
#define GP_TAN_POLY 1
#endif
constexpr float kTanMagic = 12582912.0f, kTwoOverPi = 0.636619772f;
constexpr float kPio2A = 1.5707964f, kPio2B = -4.371139e-08f, kPio2C = -1.7763568e-15f;
constexpr float kTanP0 = 0.33333156f, kTanP1 = 0.133388f, kTanP2 = 0.053411208f,
                kTanP3 = 0.024430392f, kTanP4 = 0.0031195127f, kTanP5 = 0.009385642f;
__device__ __forceinline__ float tan_poly(float x) {
  const float j = fmaf(x, kTwoOverPi, kTanMagic);
  const float k = j - kTanMagic;
  float r = fmaf(k, -kPio2A, x);
  r = fmaf(k, -kPio2B, r);
  r = fmaf(k, -kPio2C, r);
  const float z = r * r;
  float p = fmaf(kTanP5, z, kTanP4);
  p = fmaf(p, z, kTanP3);
  p = fmaf(p, z, kTanP2);
  p = fmaf(p, z, kTanP1);
  p = fmaf(p, z, kTanP0);
  const float t = fmaf(r * z, p, r);
  const float u = rcp_approx(-t);
  return (__float_as_int(j) & 1) ? u : t;
}
template <int OP>
__device__ __forceinline__ float apply1(float a) {
  if constexpr (OP == GP_OP_SIN) return __sinf(a);
  else if constexpr (OP == GP_OP_COS) return __cosf(a);
  else if constexpr (OP == GP_OP_TAN) {
#if GP_TAN_POLY
    return tan_poly(a);
#else
    return __sinf(a) * rcp_fast(__cosf(a));
#endif
  }
  else if constexpr (OP == GP_OP_ABS) return fabsf(a);
  else if constexpr (OP == GP_OP_NEG) return -a;
  else if constexpr (OP == GP_OP_SQRT) return sqrt_approx(fabsf(a));
  else if constexpr (OP == GP_OP_LOG) { const float l = __logf(fabsf(a)); return fabsf(a) < kProt ? 0.0f : l; }
  else if constexpr (OP == GP_OP_EXP) return fminf(__expf(a), kBig);
  else if constexpr (OP == GP_OP_INV) { const float r = rcp_fast(a); return fabsf(a) < kProt ? 1.0f : r; }
  else if constexpr (OP == GP_OP_SQUARE) return a * a;
  else if constexpr (OP == GP_OP_CUBE) return a * a * a;
  else if constexpr (OP == GP_OP_TANH) return tanh_bf(a);
  else if constexpr (OP == GP_OP_SINH) return sinh_bf(a);
  else if constexpr (OP == GP_OP_COSH) { const float e = __expf(fabsf(a)); return fminf(0.5f * (e + rcp_approx(e)), kBig); }
  else if constexpr (OP == GP_OP_ASIN) return asin_bf(a);
  else if constexpr (OP == GP_OP_ACOS) return acos_bf(a);
  else return atan_bf(a);  // GP_OP_ATAN
}

// ---- row pairs: Blackwell's packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2) ---------------------------
// Two rows per instruction for the ops whose scalar form is one correctly rounded add / mul / fma:
// bit-identical to the scalar path (same rounding, same -ftz), half the issue slots. ptxas keeps
// the row pairs of the register stack in aligned register pairs, so no packing moves are emitted.
#define GPB_X2(OPC, d0, d1, a0, a1, b0, b1)                                                      \
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2,%3};\n\tmov.b64 b, {%4,%5};\n\t" OPC               \
      " d, a, b;\n\tmov.b64 {%0,%1}, d;}"                                                        \
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1))
__device__ __forceinline__ void add_x2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  GPB_X2("add.rn.ftz.f32x2", d0, d1, a0, a1, b0, b1);
}
__device__ __forceinline__ void sub_x2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  GPB_X2("sub.rn.ftz.f32x2", d0, d1, a0, a1, b0, b1);
}
__device__ __forceinline__ void mul_x2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  GPB_X2("mul.rn.ftz.f32x2", d0, d1, a0, a1, b0, b1);
}
// d = a * b + c on both lanes (one rounding, as fmaf)
__device__ __forceinline__ void fma_x2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                       float c0, float c1) {
  asm("{.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2,%3};\n\tmov.b64 b, {%4,%5};\n\t"
      "mov.b64 c, {%6,%7};\n\tfma.rn.ftz.f32x2 d, a, b, c;\n\tmov.b64 {%0,%1}, d;}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
#undef GPB_X2

// rcp_fast on two rows (FFMA2), bit-identical to two rcp_fast calls
__device__ __forceinline__ void rcp_fast_x2(float& r0, float& r1, float b0, float b1) {
#if GP_RCP_FMA
  const float a0 = fabsf(b0), a1 = fabsf(b1);
  float x0 = __int_as_float(kRcpMagic - __float_as_int(a0));
  float x1 = __int_as_float(kRcpMagic - __float_as_int(a1));
  float e0, e1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    fma_x2(e0, e1, -a0, -a1, x0, x1, 1.0f, 1.0f);
    fma_x2(x0, x1, x0, x1, e0, e1, x0, x1);
  }
  r0 = copysignf(a0 > kRcpHuge ? 0.0f : x0, b0);
  r1 = copysignf(a1 > kRcpHuge ? 0.0f : x1, b1);
#else
  r0 = rcp_approx(b0);
  r1 = rcp_approx(b1);
#endif
}

// tan_poly on two rows (FFMA2 / FMUL2 / FADD2), bit-identical to two tan_poly calls
__device__ __forceinline__ void tan_poly_x2(float& d0, float& d1, float x0, float x1) {
  float j0, j1, k0, k1, r0, r1, z0, z1, p0, p1, q0, q1;
  fma_x2(j0, j1, x0, x1, kTwoOverPi, kTwoOverPi, kTanMagic, kTanMagic);
  sub_x2(k0, k1, j0, j1, kTanMagic, kTanMagic);
  fma_x2(r0, r1, k0, k1, -kPio2A, -kPio2A, x0, x1);
  fma_x2(r0, r1, k0, k1, -kPio2B, -kPio2B, r0, r1);
  fma_x2(r0, r1, k0, k1, -kPio2C, -kPio2C, r0, r1);
  mul_x2(z0, z1, r0, r1, r0, r1);
  fma_x2(p0, p1, kTanP5, kTanP5, z0, z1, kTanP4, kTanP4);
  fma_x2(p0, p1, p0, p1, z0, z1, kTanP3, kTanP3);
  fma_x2(p0, p1, p0, p1, z0, z1, kTanP2, kTanP2);
  fma_x2(p0, p1, p0, p1, z0, z1, kTanP1, kTanP1);
  fma_x2(p0, p1, p0, p1, z0, z1, kTanP0, kTanP0);
  mul_x2(q0, q1, r0, r1, z0, z1);
  fma_x2(q0, q1, q0, q1, p0, p1, r0, r1);
  const float u0 = rcp_approx(-q0), u1 = rcp_approx(-q1);
  d0 = (__float_as_int(j0) & 1) ? u0 : q0;
  d1 = (__float_as_int(j1) & 1) ? u1 : q1;
}

// apply2 on two rows: (d0, d1) = (a0 OP b0, a1 OP b1), bit-identical to two apply2 calls.
template <int OP>
__device__ __forceinline__ void apply2_x2(float& d0, float& d1, float a0, float a1, float b0,
                                          float b1) {
  if constexpr (OP == GP_OP_ADD) add_x2(d0, d1, a0, a1, b0, b1);
  else if constexpr (OP == GP_OP_SUB) sub_x2(d0, d1, a0, a1, b0, b1);
  else if constexpr (OP == GP_OP_MUL) mul_x2(d0, d1, a0, a1, b0, b1);
  else if constexpr (OP == GP_OP_DIV) {
    float q0, q1, i0, i1;
    rcp_fast_x2(i0, i1, b0, b1);
    mul_x2(q0, q1, a0, a1, i0, i1);
    d0 = fabsf(b0) < kProt ? 1.0f : q0;
    d1 = fabsf(b1) < kProt ? 1.0f : q1;
  } else {
    const float r0 = apply2<OP>(a0, b0), r1 = apply2<OP>(a1, b1);
    d0 = r0;
    d1 = r1;
  }
}
// apply1 on two rows, bit-identical to two apply1 calls.
template <int OP>
__device__ __forceinline__ void apply1_x2(float& d0, float& d1, float a0, float a1) {
  if constexpr (OP == GP_OP_SQUARE) mul_x2(d0, d1, a0, a1, a0, a1);
  else if constexpr (OP == GP_OP_CUBE) {
    float s0, s1;
    mul_x2(s0, s1, a0, a1, a0, a1);
    mul_x2(d0, d1, s0, s1, a0, a1);
  } else if constexpr (OP == GP_OP_TAN) {
#if GP_TAN_POLY
    tan_poly_x2(d0, d1, a0, a1);
#else
    float i0, i1;
    rcp_fast_x2(i0, i1, __cosf(a0), __cosf(a1));
    mul_x2(d0, d1, __sinf(a0), __sinf(a1), i0, i1);
#endif
  } else if constexpr (OP == GP_OP_INV) {
    float i0, i1;
    rcp_fast_x2(i0, i1, a0, a1);
    d0 = fabsf(a0) < kProt ? 1.0f : i0;
    d1 = fabsf(a1) < kProt ? 1.0f : i1;
  } else {
    const float r0 = apply1<OP>(a0), r1 = apply1<OP>(a1);
    d0 = r0;
    d1 = r1;
  }
}

// Runtime-dispatched scalar version (used by the Pearson shift kernel: one row per program).
__device__ __forceinline__ float apply_rt(int op, float a, float b) {
  switch (op) {
    case GP_OP_ADD: return apply2<GP_OP_ADD>(a, b);
    case GP_OP_SUB: return apply2<GP_OP_SUB>(a, b);
    case GP_OP_MUL: return apply2<GP_OP_MUL>(a, b);
    case GP_OP_DIV: return apply2<GP_OP_DIV>(a, b);
    case GP_OP_MIN: return apply2<GP_OP_MIN>(a, b);
    case GP_OP_MAX: return apply2<GP_OP_MAX>(a, b);
    case GP_OP_POW: return apply2<GP_OP_POW>(a, b);
    case GP_OP_SIN: return apply1<GP_OP_SIN>(a);
    case GP_OP_COS: return apply1<GP_OP_COS>(a);
    case GP_OP_TAN: return apply1<GP_OP_TAN>(a);
    case GP_OP_ABS: return apply1<GP_OP_ABS>(a);
    case GP_OP_NEG: return apply1<GP_OP_NEG>(a);
    case GP_OP_SQRT: return apply1<GP_OP_SQRT>(a);
    case GP_OP_LOG: return apply1<GP_OP_LOG>(a);
    case GP_OP_EXP: return apply1<GP_OP_EXP>(a);
    case GP_OP_INV: return apply1<GP_OP_INV>(a);
    case GP_OP_SQUARE: return apply1<GP_OP_SQUARE>(a);
    case GP_OP_CUBE: return apply1<GP_OP_CUBE>(a);
    case GP_OP_TANH: return apply1<GP_OP_TANH>(a);
    case GP_OP_SINH: return apply1<GP_OP_SINH>(a);
    case GP_OP_COSH: return apply1<GP_OP_COSH>(a);
    case GP_OP_ASIN: return apply1<GP_OP_ASIN>(a);
    case GP_OP_ACOS: return apply1<GP_OP_ACOS>(a);
    case GP_OP_ATAN: return apply1<GP_OP_ATAN>(a);
  }
  return __int_as_float(0x7fc00000);
}

// ---- compiled program code (written by the stage kernel, read by the evaluator) ---------------
// One uint4 per EMITTED node, in evaluation order (reverse prefix). Terminals are not
// emitted on their own: each terminal operand is folded into its parent function's code word
// ("superinstruction"), so only function nodes are dispatched (a lone-terminal program emits one
// push). Word layout:
//   .x = case id * 4 (byte offset into the dispatch jump table), case id = opv * STACK + slot
//   .y = payload of the first operand a  (variable index, or fp32 constant bits)
//   .z = payload of the second operand b (variable index, or fp32 constant bits)
// opv enumerates (op, operand-source variant) pairs:
//   0 push var, 1 push const;
//   binary op o (2..8): 2 + (o-2)*10 + v, v = SS, SV, SC, VS, CS, VV, VC, CV, CC, SSR
//       (S = stack, V = variable, C = constant; first letter = operand a, second = operand b;
//        SSR = both on the stack with a evaluated FIRST -- Sethi-Ullman order)
//   unary op o (9..25): 72 + (o-9)*3 + u, u = S, V, C
// slot = destination stack slot (static: occupancy depends only on the tree shape):
//   SS -> a = st[slot+1], b = st[slot];  SSR -> a = st[slot], b = st[slot+1];
//   one S -> that operand is st[slot];  no S -> new slot.
enum { OPV_PUSH_V = 0, OPV_PUSH_C = 1, OPV_BIN0 = 2, OPV_UN0 = 72, OPV_COUNT = 123 };
enum { BV_SS = 0, BV_SV, BV_SC, BV_VS, BV_CS, BV_VV, BV_VC, BV_CV, BV_CC, BV_SSR };
enum { UV_S = 0, UV_V, UV_C };
__host__ __device__ constexpr int opv_bin(int op, int v) { return OPV_BIN0 + (op - GP_OP_ADD) * 10 + v; }
__host__ __device__ constexpr int opv_un(int op, int u) { return OPV_UN0 + (op - GP_OP_SIN) * 3 + u; }

// Dispatch numbering of the evaluator (pack_kernel rewrites the stage kernel's case ids into it):
// case = opv_rank(opv) * STACK + slot with the variant's own slot count (not kCaseStride), and
// the paper's function set first -- push, add / sub / mul / div (all operand variants), sin / cos /
// tan -- so the jump table the hot loop indexes is small and dense (s4: 204 hot entries in 816 B
// instead of ~1 in 5 entries used over 9.8 KB): the ncu SASS profile of r02 put 9 % of all stall
// samples on the jump-table constant load (profiles/ncu_eval_r02_c3gen0_base.md).
__host__ __device__ constexpr int opv_rank(int opv) {
  if (opv < OPV_BIN0) return opv;                                   // push var / const: 0, 1
  if (opv < OPV_UN0) {
    const int o = GP_OP_ADD + (opv - OPV_BIN0) / 10, v = (opv - OPV_BIN0) % 10;
    return o <= GP_OP_DIV ? 2 + (o - GP_OP_ADD) * 10 + v            // 2 .. 41
                          : 51 + (o - GP_OP_MIN) * 10 + v;          // 51 .. 80
  }
  const int o = GP_OP_SIN + (opv - OPV_UN0) / 3, u = (opv - OPV_UN0) % 3;
  return o <= GP_OP_TAN ? 42 + (o - GP_OP_SIN) * 3 + u              // 42 .. 50
                        : 81 + (o - GP_OP_ABS) * 3 + u;             // 81 .. 122
}

}  // namespace gpb
