// eval_impl.cuh -- the fused population evaluator, sm_100a.
//
// Included by eval_s{8,12,20}.cu with GP_STACK (register-stack capacity), GP_R (rows per thread
// per pass), GP_SUB (passes per program per tile) and GP_NT (threads per CTA) defined, so every
// (op, slot) case of the dispatch switch is generated for exactly GP_STACK slots.
//
// What one CTA does (work item = row chunk q x program group g; grid = (n_chunks, n_groups)):
//   for each tile of TILE = NT*R*SUB rows of the chunk:
//     stage y, w (and X when n_cols is small) into shared memory, coalesced, zero-padded  [A2]
//     for each program p of the group:                     -- warp-uniform: no divergence
//       for each of SUB passes: run the compiled program on R rows per thread with the stack in
//         REGISTERS: the stack slot of every node is static (stage kernel), so the dispatch is one
//         switch on (op, slot) and no stack index is ever computed at run time  [A3]
//       fused weighted loss of those rows (no m x n prediction matrix)             [A4]
//       warp shuffle reduction, lane 0 accumulates into a per-(warp, program) fp64 smem slot   [A5]
//   per-(program) sums over warps in fixed order -> partial[q][p] (no atomics, deterministic)
//
// The paper's design is one thread per row and a (ceil(m/256), n) grid; here each thread
// owns R*SUB rows and loops over programs, so X is read from HBM once per program GROUP rather
// than once per program, and node dispatch is amortised over R rows.
#include <cfloat>
#include "device_ops.cuh"
#include "kernels.h"

#ifndef GP_STACK
#error "define GP_STACK"
#endif

#define GP_CAT2(a, b) a##b
#define GP_CAT(a, b) GP_CAT2(a, b)
#define GP_NS GP_CAT(s, GP_STACK)

namespace gpb {
namespace GP_NS {

constexpr int STACK = GP_STACK, R = GP_R, SUB = GP_SUB, NT = GP_NT;
constexpr int TILE = NT * R * SUB, NW = NT / 32, R4 = R / 4;
static_assert(R % 4 == 0 && NT % 32 == 0, "R must be a multiple of 4");
static_assert(GP_OP_COUNT * STACK <= (1 << kCaseBits), "case id must fit kCaseBits");

constexpr float kLogLossLo = 1.0000000000000005e-15f;  // -ln(1 - 1e-15), S:191 clamp (C7)
constexpr float kLogLossHi = 34.538776394910684f;      // -ln(1e-15)

// Shared-memory layout (bytes); G programs per group, S accumulators per program.
__host__ __device__ inline size_t smem_acc_bytes(int G, int S) {
  return (((size_t)NW * G * S + NW * 3) * sizeof(double) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t smem_bytes(int G, int S, int n_cols, bool xsmem) {
  return smem_acc_bytes(G, S) + 2 * TILE * sizeof(float) +
         (xsmem ? (size_t)n_cols * TILE * sizeof(float) : 0);
}

#define LBL(OP, s) ((OP) * STACK + (s))

// -- dispatch cases -------------------------------------------------------------------------------
// Variable push: from shared memory (xsmem: LDS.128 per 4 rows) or from global memory via L1.
#define GP_LOAD_VAR(s)                                                                         \
  {                                                                                            \
    const int var = (int)(cw.x >> kCaseBits);                                                  \
    if constexpr (XSMEM) {                                                                     \
      const float4* xv = reinterpret_cast<const float4*>(xs + var * TILE + ebase);             \
      _Pragma("unroll") for (int k = 0; k < R4; ++k) {                                         \
        const float4 v = xv[k * NT];                                                           \
        st[s][4 * k] = v.x; st[s][4 * k + 1] = v.y; st[s][4 * k + 2] = v.z;                    \
        st[s][4 * k + 3] = v.w;                                                                \
      }                                                                                        \
    } else {                                                                                   \
      const float* xv = a.X + (int64_t)var * a.ldx + t0;                                       \
      _Pragma("unroll") for (int r = 0; r < R; ++r) {                                          \
        const int e = min(ebase + (r >> 2) * NT * 4 + (r & 3), nvalid - 1);                    \
        st[s][r] = __ldg(xv + e);                                                              \
      }                                                                                        \
    }                                                                                          \
  }
#define GP_TERM(s)                                                                             \
  case LBL(GP_OP_VAR, s): GP_LOAD_VAR(s) break;                                                \
  case LBL(GP_OP_CONST, s): {                                                                  \
    const float c = __uint_as_float(cw.y);                                                     \
    _Pragma("unroll") for (int r = 0; r < R; ++r) st[s][r] = c;                                \
  } break;
#define GP_UN(OP, s)                                                                           \
  case LBL(OP, s): {                                                                           \
    _Pragma("unroll") for (int r = 0; r < R; ++r) st[s][r] = apply1<OP>(st[s][r]);             \
  } break;
#define GP_BIN(OP, s)                                                                          \
  case LBL(OP, s): {                                                                           \
    _Pragma("unroll") for (int r = 0; r < R; ++r) st[s][r] = apply2<OP>(st[(s) + 1][r], st[s][r]); \
  } break;
#define GP_SLOT_TU(s)                                                                          \
  GP_TERM(s) GP_UN(GP_OP_SIN, s) GP_UN(GP_OP_COS, s) GP_UN(GP_OP_TAN, s) GP_UN(GP_OP_ABS, s)   \
  GP_UN(GP_OP_NEG, s) GP_UN(GP_OP_SQRT, s) GP_UN(GP_OP_LOG, s) GP_UN(GP_OP_EXP, s)             \
  GP_UN(GP_OP_INV, s) GP_UN(GP_OP_SQUARE, s) GP_UN(GP_OP_CUBE, s) GP_UN(GP_OP_TANH, s)         \
  GP_UN(GP_OP_SINH, s) GP_UN(GP_OP_COSH, s) GP_UN(GP_OP_ASIN, s) GP_UN(GP_OP_ACOS, s)          \
  GP_UN(GP_OP_ATAN, s)
#define GP_SLOT_B(s)                                                                           \
  GP_BIN(GP_OP_ADD, s) GP_BIN(GP_OP_SUB, s) GP_BIN(GP_OP_MUL, s) GP_BIN(GP_OP_DIV, s)          \
  GP_BIN(GP_OP_MIN, s) GP_BIN(GP_OP_MAX, s) GP_BIN(GP_OP_POW, s)

#define GP_FOR_0_6(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6)
#define GP_FOR_8_10(M) M(8) M(9) M(10)
#define GP_FOR_12_18(M) M(12) M(13) M(14) M(15) M(16) M(17) M(18)
#if GP_STACK == 8
#define GP_ALL_CASES GP_FOR_0_6(GP_SLOT_TU) GP_SLOT_TU(7) GP_FOR_0_6(GP_SLOT_B)
#elif GP_STACK == 12
#define GP_ALL_CASES                                                                           \
  GP_FOR_0_6(GP_SLOT_TU) GP_SLOT_TU(7) GP_FOR_8_10(GP_SLOT_TU) GP_SLOT_TU(11)                  \
  GP_FOR_0_6(GP_SLOT_B) GP_SLOT_B(7) GP_FOR_8_10(GP_SLOT_B)
#elif GP_STACK == 20
#define GP_ALL_CASES                                                                           \
  GP_FOR_0_6(GP_SLOT_TU) GP_SLOT_TU(7) GP_FOR_8_10(GP_SLOT_TU) GP_SLOT_TU(11)                  \
  GP_FOR_12_18(GP_SLOT_TU) GP_SLOT_TU(19)                                                      \
  GP_FOR_0_6(GP_SLOT_B) GP_SLOT_B(7) GP_FOR_8_10(GP_SLOT_B) GP_SLOT_B(11) GP_FOR_12_18(GP_SLOT_B)
#else
#error "GP_STACK must be 8, 12 or 20"
#endif

template <int M> struct MTag { static constexpr int value = M; };

__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool PREDICT, bool XSMEM>
__global__ void __launch_bounds__(NT) eval_kernel(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int S = (a.metric == GP_PEARSON) ? 3 : 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x, g = blockIdx.y;
  const int p0 = g * a.G;
  const int np = min(a.G, a.n_programs - p0);
  double* acc = reinterpret_cast<double*>(smem);                 // [NW][G][S]
  double* cacc = acc + (size_t)NW * a.G * S;                     // [NW][3] dataset constants
  float* ys = reinterpret_cast<float*>(smem + (PREDICT ? 0 : smem_acc_bytes(a.G, S)));
  float* ws = ys + TILE;
  float* xs = ws + TILE;                                         // [n_cols][TILE] if XSMEM
  const bool do_consts = !PREDICT && g == 0;

  if constexpr (!PREDICT) {
    for (int i = tid; i < NW * a.G * S + NW * 3; i += NT) acc[i] = 0.0;
  }
  const float Ky = (!PREDICT && S == 3) ? *a.y_shift : 0.0f;

  const int64_t r_begin = (int64_t)q * a.rows_per_chunk;
  const int64_t r_end = min(r_begin + a.rows_per_chunk, a.n_rows);

  for (int64_t t0 = r_begin; t0 < r_end; t0 += TILE) {
    const int nvalid = (int)min((int64_t)TILE, r_end - t0);
    __syncthreads();  // previous tile's smem reads are done
    // ---- A2: stage the tile (coalesced; padded rows get w = 0 -> skipped) -------------------
    for (int i = tid; i < TILE; i += NT) {
      const bool in = i < nvalid;
      const int64_t row = t0 + i;
      if constexpr (!PREDICT) {
        ys[i] = in ? a.y[row] : 0.0f;
        ws[i] = in ? (a.w ? a.w[row] : 1.0f) : 0.0f;
      }
      if constexpr (XSMEM) {
        for (int c = 0; c < a.n_cols; ++c) xs[c * TILE + i] = in ? a.X[(int64_t)c * a.ldx + row] : 0.0f;
      }
    }
    __syncthreads();

    // ---- dataset constants W, S_y, S_yy (program independent; group 0 only) ----------------
    if (do_consts) {
      float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
      for (int sub = 0; sub < SUB; ++sub) {
        const int ebase = sub * NT * R + tid * 4;
#pragma unroll
        for (int k = 0; k < R4; ++k) {
          const float4 yv = *reinterpret_cast<const float4*>(ys + ebase + k * NT * 4);
          const float4 wv = *reinterpret_cast<const float4*>(ws + ebase + k * NT * 4);
          const float yy[4] = {yv.x, yv.y, yv.z, yv.w}, ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float yc = yy[j] - Ky;
            if (ww[j] != 0.0f) { c0 += ww[j]; c1 += ww[j] * yc; c2 += ww[j] * yc * yc; }
          }
        }
      }
      const double d0 = warp_sum_f64(c0), d1 = warp_sum_f64(c1), d2 = warp_sum_f64(c2);
      if (lane == 0) { cacc[warp * 3] += d0; cacc[warp * 3 + 1] += d1; cacc[warp * 3 + 2] += d2; }
    }

    // ---- A3 + A4 + A5 per program ----------------------------------------------------------
    for (int pl = 0; pl < np; ++pl) {
      const int p = p0 + pl;
      const int len = a.code_len[p];
      if (len == 0) continue;                       // invalid program (stage flags say why)
      const uint2* __restrict__ pc = a.code + a.code_off[p];
      const float Kp = (!PREDICT && S == 3) ? a.shift[p] : 0.0f;
      float l0 = 0.f, l1 = 0.f, l2 = 0.f;
#pragma unroll 1
      for (int sub = 0; sub < SUB; ++sub) {
        const int ebase = sub * NT * R + tid * 4;   // element e(r) = ebase + (r/4)*NT*4 + r%4
        float st[STACK][R];
        // two-deep software prefetch of the (warp-uniform) code words
        uint2 nxt = __ldg(pc), nxt2 = __ldg(pc + 1);
#pragma unroll 1
        for (int kk = 0; kk < len; ++kk) {
          const uint2 cw = nxt;
          nxt = nxt2;
          nxt2 = __ldg(pc + kk + 2);                // code buffer carries two pad words
          switch (cw.x & kCaseMask) {
            GP_ALL_CASES
            default: __builtin_unreachable();  // stage kernel guarantees a valid (op, slot)
          }
        }
        if constexpr (PREDICT) {
          float* o = a.out + (int64_t)p * a.ld_out + t0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int e = ebase + (r >> 2) * NT * 4 + (r & 3);
            if (e < nvalid) o[e] = st[0][r];
          }
        } else {
          // fused weighted loss, one uniform metric branch per pass (A4)
          auto loss = [&](auto tag) {
            constexpr int M = decltype(tag)::value;
#pragma unroll
            for (int k = 0; k < R4; ++k) {
              const float4 yv = *reinterpret_cast<const float4*>(ys + ebase + k * NT * 4);
              const float4 wv = *reinterpret_cast<const float4*>(ws + ebase + k * NT * 4);
              const float yy[4] = {yv.x, yv.y, yv.z, yv.w}, ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float yh = st[0][4 * k + j];
                const bool live = ww[j] != 0.0f;    // w = 0 rows are skipped, never multiplied
                if constexpr (M == GP_MSE) {
                  const float d = yh - yy[j];
                  l0 += live ? ww[j] * d * d : 0.0f;
                } else if constexpr (M == GP_MAE) {
                  l0 += live ? ww[j] * fabsf(yh - yy[j]) : 0.0f;
                } else if constexpr (M == GP_LOGLOSS) {
                  // -[y ln p + (1-y) ln(1-p)], p = sigmoid(yh), y in {0,1}: softplus(-+yh),
                  // clamped to the p-clamp's range (C7)
                  const float z = yy[j] > 0.5f ? -yh : yh;
                  float l = fmaxf(z, 0.0f) + __logf(1.0f + __expf(-fabsf(z)));
                  l = l < kLogLossLo ? kLogLossLo : (l > kLogLossHi ? kLogLossHi : l);
                  l0 += live ? ww[j] * l : 0.0f;
                } else {  // Pearson: shifted sums (C9)
                  const float d = yh - Kp, yc = yy[j] - Ky, wd = ww[j] * d;
                  l0 += live ? wd : 0.0f;
                  l1 += live ? wd * d : 0.0f;
                  l2 += live ? wd * yc : 0.0f;
                }
              }
            }
          };
          switch (a.metric) {
            case GP_MAE: loss(MTag<GP_MAE>{}); break;
            case GP_MSE: case GP_RMSE: loss(MTag<GP_MSE>{}); break;
            case GP_LOGLOSS: loss(MTag<GP_LOGLOSS>{}); break;
            default: loss(MTag<GP_PEARSON>{}); break;
          }
        }
      }
      if constexpr (!PREDICT) {
        double* slot = acc + ((size_t)warp * a.G + pl) * S;
        if (S == 1) {
          const float v = warp_sum_f32(l0);
          if (lane == 0) slot[0] += (double)v;
        } else {
          const double v0 = warp_sum_f64(l0), v1 = warp_sum_f64(l1), v2 = warp_sum_f64(l2);
          if (lane == 0) { slot[0] += v0; slot[1] += v1; slot[2] += v2; }
        }
      }
    }
  }

  if constexpr (!PREDICT) {
    __syncthreads();
    double* prow = a.partial + (int64_t)q * a.ld_part;
    for (int j = tid; j < np * S; j += NT) {
      const int pl = j / S, k = j - pl * S;
      double s = 0.0;
      for (int wv = 0; wv < NW; ++wv) s += acc[((size_t)wv * a.G + pl) * S + k];
      prow[(int64_t)(p0 + pl) * S + k] = s;
    }
    if (g == 0 && tid < 3) {
      double s = 0.0;
      for (int wv = 0; wv < NW; ++wv) s += cacc[wv * 3 + tid];
      prow[(int64_t)a.n_programs * S + tid] = s;
    }
  }
}

template <bool P, bool XS>
static cudaError_t launch_t(const EvalArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(eval_kernel<P, XS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  eval_kernel<P, XS><<<grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

static cudaError_t launch(const EvalArgs& a, bool predict, bool xsmem, dim3 grid, size_t smem,
                          cudaStream_t s) {
  if (predict) return xsmem ? launch_t<true, true>(a, grid, smem, s) : launch_t<true, false>(a, grid, smem, s);
  return xsmem ? launch_t<false, true>(a, grid, smem, s) : launch_t<false, false>(a, grid, smem, s);
}

template <bool P, bool XS>
static int occ_t(size_t smem) {
  int n = 0;
  cudaFuncSetAttribute(eval_kernel<P, XS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, eval_kernel<P, XS>, NT, smem);
  return n;
}
static int occupancy(bool predict, bool xsmem, size_t smem) {
  if (predict) return xsmem ? occ_t<true, true>(smem) : occ_t<true, false>(smem);
  return xsmem ? occ_t<false, true>(smem) : occ_t<false, false>(smem);
}

}  // namespace GP_NS

const EvalVariant& GP_CAT(eval_variant_, GP_NS)() {
  static const EvalVariant v = {EvalShape{GP_NS::STACK, GP_NS::R, GP_NS::SUB, GP_NS::NT},
                                &GP_NS::launch, &GP_NS::occupancy};
  return v;
}

}  // namespace gpb
