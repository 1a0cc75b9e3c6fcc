// eval_impl.cuh -- the fused population evaluator, sm_100a.
//
// Included by the translation units build.py generates from shape_<name>.h, which defines GP_STACK
// (register-stack capacity), GP_R (rows per thread per pass), GP_SUB (passes per program per tile),
// GP_NT (threads per CTA) and GP_MINB (resident CTAs per SM the register budget must allow), so
// every (op, operand variant, slot) case of the dispatch switch is generated for exactly GP_STACK
// slots. Shared-memory-X shapes run one 512-thread CTA per SM (the warps of an SM sub-partition
// share the instruction cache while they walk the same code stream).
//
// Persistent CTAs pull work items (program group g x row chunk q) from a queue. Per item:
//   for each tile of TILE = NT*R*SUB rows of the chunk (8192; wide shapes 4096 / 2048):
//     stage the tile into shared memory: X (when the layout fits) by TMA bulk copies on an
//     mbarrier, y / w by the threads, coalesced, zero-padded                            [A2]
//     walk the group's packed code stream (aux.cu pack_kernel): for each program of the group
//     (programs of this variant's stack-need bucket), SUB copies of its code, one per row pass,
//     the last word of each pass flagged so the loss / reduction follows its case -- one
//     contiguous stream, so the 2-deep code prefetch never restarts at a program boundary:
//       -- warp-uniform control flow: all lanes run the same program, no divergence
//       for each of SUB passes: run the compiled code on R rows per thread with the stack in
//         REGISTERS: the destination slot of every code word is static (stage kernel) and terminal
//         operands are folded into their parent's word, so one jump-table branch per function
//         node dispatches an (op, operand-source, slot) case; no stack index is ever computed at
//         run time (the paper's unrolled slot loop, costs O(capacity) per push) [A3]
//       fused weighted loss of those rows (no m x n prediction matrix)             [A4]
//       per-lane fp32 sums -> the warp's 16-program shared-memory reduction block -> fp64
//       per-(warp, program) accumulators (Pearson: warp shuffles)                            [A5]
//   per-program sums over warps in fixed order -> partial[q][bucket position] (no atomics on data:
//   the sums do not depend on which CTA ran which item)
//
// The paper's design is one thread per row and a (ceil(m/256), n) grid; here each thread
// owns R*SUB rows and loops over programs, so X is read from HBM about once (program groups are
// the fastest-varying work-item index, co-resident CTAs share row chunks through L2) and the
// dispatch is amortised over R rows.
#include <cfloat>
#include "device_ops.cuh"
#include "kernels.h"

#ifndef GP_STACK
#error "define GP_STACK"
#endif
#ifndef GP_MINB
#define GP_MINB 1   // minimum resident CTAs per SM (register budget = 64K / (GP_MINB * NT))
#endif
#ifndef GP_RED_ROWS
#define GP_RED_ROWS 16  // programs per warp reduction block (32 / GP_RED_ROWS lanes per program)
#endif

#define GP_CAT2(a, b) a##b
#define GP_CAT(a, b) GP_CAT2(a, b)
// GP_GLOBAL_X_ONLY: a translation unit holding only the global-memory-X instantiations (wide
// datasets), with its own shape; its variant is eval_variant_w<STACK> (namespace w<STACK>).
#ifdef GP_GLOBAL_X_ONLY
#define GP_NS GP_CAT(w, GP_STACK)
#else
#define GP_NS GP_CAT(s, GP_STACK)
#endif
#ifndef GP_MINB_GLOBAL
#define GP_MINB_GLOBAL (GP_MINB > 1 ? GP_MINB - 1 : 1)  // global-X path: more live addresses
#endif

namespace gpb {
namespace GP_NS {

constexpr int STACK = GP_STACK, R = GP_R, SUB = GP_SUB, NT = GP_NT;
constexpr int TILE = NT * R * SUB;
#ifdef GP_GLOBAL_X_ONLY
static_assert(kTileGlobal % TILE == 0, "a wide-dataset shape's tile divides the plan tile");
#else
static_assert(kTileSmem % TILE == 0, "a shared-memory-X shape's tile divides the plan tile");
#endif
constexpr int NW = NT / 32, R4 = R / 4;
constexpr int RR = GP_RED_ROWS, LPR = 32 / RR, RED_BYTES = NW * RR * kRedStride * 4;
static_assert(RR == 8 || RR == 16, "reduction block: 8 or 16 programs");
static_assert(R % 4 == 0 && NT % 32 == 0, "R must be a multiple of 4");
static_assert(STACK <= kCaseStride, "slot must fit the case stride");
static_assert(opv_rank(OPV_COUNT - 1) < OPV_COUNT, "opv_rank is a permutation of 0..OPV_COUNT-1");

static_assert(kStreamWin % 4 == 0, "stream window");

constexpr float kLogLossLo = 1.0000000000000005e-15f;  // -ln(1 - 1e-15), S:191 clamp (C7)
constexpr float kLogLossHi = 34.538776394910684f;      // -ln(1e-15)
constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;

// Shared-memory layout (bytes): fp64 accumulators [NW][G][S] | reduction blocks [NW][kRedRows]
// [kRedStride] fp32 | ys[TILE] | ws[TILE] (weighted only) | xs[n_cols][TILE] (small n_cols only)
// | code-stream window [kStreamWin + 2] uint4
// (the reduction blocks serve the single-sum metrics only: Pearson reduces by warp shuffles)
__host__ __device__ inline size_t smem_fp64_bytes(int G, int S) {
  return ((size_t)NW * G * S * sizeof(double) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t smem_acc_bytes(int G, int S) {
  return smem_fp64_bytes(G, S) + (S == 1 ? RED_BYTES : 0);
}
// Dynamic shared memory of one launch of this shape.
inline size_t smem_total(int G, int S, int n_cols, bool weighted, bool xsmem, bool predict) {
  const size_t yw = predict ? 0 : (weighted ? 2 : 1) * (size_t)TILE * sizeof(float);
  return (predict ? 0 : smem_acc_bytes(G, S)) + yw +
         (xsmem ? (size_t)n_cols * TILE * sizeof(float) : 0) + (size_t)(kStreamWin + 2) * 16;
}

#define LBL(OPV, s) (opv_rank(OPV) * STACK + (s))   // pack_kernel's numbering
// End of a case. GP_CASE_CONTINUE = 1 (default): an unflagged word (the common case) continues
// with the next dispatch straight from the case (one taken branch per word instead of two: case ->
// shared tail -> loop head); C3 step 123.2 -> 121.2 ms (profiles/ab_r02_dispatch.log). The
// compiled loop head then also rotates the two prefetched case ids without waiting on the LDS.
// (GP_PREFETCH = 1, a one-deep id prefetch, measured slower without the per-case continue,
// 125.5 ms, and slightly faster with it on the final build: shape_s4.h sets it.)
#ifndef GP_CASE_CONTINUE
#define GP_CASE_CONTINUE 1
#endif
#if GP_CASE_CONTINUE
#define GP_BRK if (cw.w == 0u) continue; break;
#else
#define GP_BRK break;
#endif

// -- dispatch cases -------------------------------------------------------------------------------
// Cases work on 4-row chunks (one LDS.128 of a variable per chunk), so a fused variable operand
// needs 4 temporary registers, not R: register pressure sets the occupancy of this latency-bound
// kernel. GP_VAR4(v, var, k) loads rows 4k..4k+3 of variable `var` into float4 v: from the
// shared-memory tile, or (wide datasets) from global memory through L1/L2 with rows clamped into
// the tile.
#define GP_VAR4(v, var, k)                                                                     \
  float4 v;                                                                                    \
  GP_CHECK((int)(var) >= 0 && (int)(var) < a.n_cols);                                          \
  if constexpr (XSMEM) {                                                                       \
    v = reinterpret_cast<const float4*>(xs + (int)(var) * TILE + ebase)[(k) * NT];             \
  } else {                                                                                     \
    const float* xv_ = a.X + (int64_t)(var) * a.ldx + t0;                                      \
    const int e_ = ebase + (k) * NT * 4;                                                       \
    if (x_vec && nvalid == TILE) {                   /* full, 16-byte aligned tile: LDG.128 */ \
      v = __ldg(reinterpret_cast<const float4*>(xv_ + e_));                                    \
    } else {                                                                                   \
      v.x = __ldg(xv_ + min(e_, nvalid - 1));                                                  \
      v.y = __ldg(xv_ + min(e_ + 1, nvalid - 1));                                              \
      v.z = __ldg(xv_ + min(e_ + 2, nvalid - 1));                                              \
      v.w = __ldg(xv_ + min(e_ + 3, nvalid - 1));                                              \
    }                                                                                          \
  }
#define GP_CONST(w) __uint_as_float(w)
#define GP_ROWS(stmt) _Pragma("unroll") for (int r = 0; r < R; ++r) { stmt; }
// for each 4-row chunk k: stmt4(j) applied to rows r = 4k + j
#define GP_CHUNKS(pre, stmt)                                                                   \
  _Pragma("unroll") for (int k = 0; k < R4; ++k) {                                             \
    pre;                                                                                       \
    { const int r = 4 * k;     const int j_ = 0; (void)j_; stmt; }                             \
    { const int r = 4 * k + 1; const int j_ = 1; (void)j_; stmt; }                             \
    { const int r = 4 * k + 2; const int j_ = 2; (void)j_; stmt; }                             \
    { const int r = 4 * k + 3; const int j_ = 3; (void)j_; stmt; }                             \
  }
#define GP_F4(v) (j_ == 0 ? v.x : j_ == 1 ? v.y : j_ == 2 ? v.z : v.w)
// row pairs (r, r + 1): the FP32x2 forms of device_ops.cuh (apply2_x2 / apply1_x2)
#define GP_PAIRS(stmt) _Pragma("unroll") for (int r = 0; r < R; r += 2) { stmt; }
// for each 4-row chunk k: stmt on the pairs (4k, 4k+1) <- (v.x, v.y) and (4k+2, 4k+3) <- (v.z, v.w)
#define GP_CHUNKS2(pre, stmt)                                                                  \
  _Pragma("unroll") for (int k = 0; k < R4; ++k) {                                             \
    pre;                                                                                       \
    { const int r = 4 * k;     const int j_ = 0; (void)j_; stmt; }                             \
    { const int r = 4 * k + 2; const int j_ = 1; (void)j_; stmt; }                             \
  }
#define GP_LO(v) (j_ == 0 ? v.x : v.z)
#define GP_HI(v) (j_ == 0 ? v.y : v.w)
#define GP_ST2(s) st[s][r], st[s][r + 1]

#define GP_PUSH(s)                                                                             \
  case LBL(OPV_PUSH_V, s): { GP_CHUNKS(GP_VAR4(t, cw.y, k), st[s][r] = GP_F4(t)) } GP_BRK      \
  case LBL(OPV_PUSH_C, s): { const float c = GP_CONST(cw.y); GP_ROWS(st[s][r] = c) } GP_BRK

// binary op OP at destination slot s; a = first operand, b = second operand
#define GP_BIN_SS(OP, s)                                                                       \
  case LBL(opv_bin(OP, BV_SS), s): {                                                           \
    GP_PAIRS(apply2_x2<OP>(GP_ST2(s), GP_ST2((s) + 1), GP_ST2(s))) } GP_BRK                    \
  case LBL(opv_bin(OP, BV_SSR), s): {                                                          \
    GP_PAIRS(apply2_x2<OP>(GP_ST2(s), GP_ST2(s), GP_ST2((s) + 1))) } GP_BRK
#define GP_BIN_T(OP, s)                                                                        \
  case LBL(opv_bin(OP, BV_SV), s): {                                                           \
    GP_CHUNKS2(GP_VAR4(t, cw.z, k), apply2_x2<OP>(GP_ST2(s), GP_ST2(s), GP_LO(t), GP_HI(t))) } GP_BRK \
  case LBL(opv_bin(OP, BV_SC), s): { const float c = GP_CONST(cw.z);                           \
    GP_PAIRS(apply2_x2<OP>(GP_ST2(s), GP_ST2(s), c, c)) } GP_BRK                               \
  case LBL(opv_bin(OP, BV_VS), s): {                                                           \
    GP_CHUNKS2(GP_VAR4(t, cw.y, k), apply2_x2<OP>(GP_ST2(s), GP_LO(t), GP_HI(t), GP_ST2(s))) } GP_BRK \
  case LBL(opv_bin(OP, BV_CS), s): { const float c = GP_CONST(cw.y);                           \
    GP_PAIRS(apply2_x2<OP>(GP_ST2(s), c, c, GP_ST2(s))) } GP_BRK                               \
  case LBL(opv_bin(OP, BV_VV), s): {                                                           \
    GP_CHUNKS2(GP_VAR4(t, cw.y, k) GP_VAR4(u, cw.z, k),                                        \
               apply2_x2<OP>(GP_ST2(s), GP_LO(t), GP_HI(t), GP_LO(u), GP_HI(u))) } GP_BRK      \
  case LBL(opv_bin(OP, BV_VC), s): { const float c = GP_CONST(cw.z);                           \
    GP_CHUNKS2(GP_VAR4(t, cw.y, k), apply2_x2<OP>(GP_ST2(s), GP_LO(t), GP_HI(t), c, c)) } GP_BRK \
  case LBL(opv_bin(OP, BV_CV), s): { const float c = GP_CONST(cw.y);                           \
    GP_CHUNKS2(GP_VAR4(u, cw.z, k), apply2_x2<OP>(GP_ST2(s), c, c, GP_LO(u), GP_HI(u))) } GP_BRK \
  case LBL(opv_bin(OP, BV_CC), s): {                                                           \
    const float v = apply2<OP>(GP_CONST(cw.y), GP_CONST(cw.z)); GP_ROWS(st[s][r] = v) } GP_BRK
#define GP_UN(OP, s)                                                                           \
  case LBL(opv_un(OP, UV_S), s): { GP_PAIRS(apply1_x2<OP>(GP_ST2(s), GP_ST2(s))) } GP_BRK      \
  case LBL(opv_un(OP, UV_V), s): {                                                             \
    GP_CHUNKS2(GP_VAR4(t, cw.y, k), apply1_x2<OP>(GP_ST2(s), GP_LO(t), GP_HI(t))) } GP_BRK     \
  case LBL(opv_un(OP, UV_C), s): { const float v = apply1<OP>(GP_CONST(cw.y));                 \
    GP_ROWS(st[s][r] = v) } GP_BRK

// Every case whose destination slot is s (SS needs slot s + 1 as well), listed as the paper's
// function set (Table 2 / 6: add, sub, mul, div, sin, cos, tan) and the rest of the
// catalog. (Emitting the paper-set cases of all slots first, as one contiguous code block, was
// measured: no difference.)
#define GP_HOT_BIN(M, s) M(GP_OP_ADD, s) M(GP_OP_SUB, s) M(GP_OP_MUL, s) M(GP_OP_DIV, s)
#define GP_COLD_BIN(M, s) M(GP_OP_MIN, s) M(GP_OP_MAX, s) M(GP_OP_POW, s)
#define GP_HOT_UN(M, s) M(GP_OP_SIN, s) M(GP_OP_COS, s) M(GP_OP_TAN, s)
#define GP_COLD_UN(M, s)                                                                       \
  M(GP_OP_ABS, s) M(GP_OP_NEG, s) M(GP_OP_SQRT, s) M(GP_OP_LOG, s) M(GP_OP_EXP, s)              \
  M(GP_OP_INV, s) M(GP_OP_SQUARE, s) M(GP_OP_CUBE, s) M(GP_OP_TANH, s) M(GP_OP_SINH, s)         \
  M(GP_OP_COSH, s) M(GP_OP_ASIN, s) M(GP_OP_ACOS, s) M(GP_OP_ATAN, s)
#define GP_SLOT_TU_HOT(s) GP_PUSH(s) GP_HOT_BIN(GP_BIN_T, s) GP_HOT_UN(GP_UN, s)
#define GP_SLOT_TU_COLD(s) GP_COLD_BIN(GP_BIN_T, s) GP_COLD_UN(GP_UN, s)
#define GP_SLOT_B_HOT(s) GP_HOT_BIN(GP_BIN_SS, s)    // SS and SSR
#define GP_SLOT_B_COLD(s) GP_COLD_BIN(GP_BIN_SS, s)
#define GP_SLOT_TU(s) GP_SLOT_TU_HOT(s) GP_SLOT_TU_COLD(s)
#define GP_SLOT_B(s) GP_SLOT_B_HOT(s) GP_SLOT_B_COLD(s)

#define GP_FOR_0_2(M) M(0) M(1) M(2)
#define GP_FOR_0_6(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6)
#define GP_FOR_8_10(M) M(8) M(9) M(10)
#define GP_FOR_12_18(M) M(12) M(13) M(14) M(15) M(16) M(17) M(18)
// GP_CASES(TU, B): the TU cases of every slot, then the SS / SSR cases of every slot below the top
#if GP_STACK == 4
#define GP_CASES(TU, B) GP_FOR_0_2(TU) TU(3) GP_FOR_0_2(B)
#elif GP_STACK == 8
#define GP_CASES(TU, B) GP_FOR_0_6(TU) TU(7) GP_FOR_0_6(B)
#elif GP_STACK == 12
#define GP_CASES(TU, B)                                                                        \
  GP_FOR_0_6(TU) TU(7) GP_FOR_8_10(TU) TU(11) GP_FOR_0_6(B) B(7) GP_FOR_8_10(B)
#elif GP_STACK == 20
#define GP_CASES(TU, B)                                                                        \
  GP_FOR_0_6(TU) TU(7) GP_FOR_8_10(TU) TU(11) GP_FOR_12_18(TU) TU(19)                          \
  GP_FOR_0_6(B) B(7) GP_FOR_8_10(B) B(11) GP_FOR_12_18(B)
#else
#error "GP_STACK must be 4, 8, 12 or 20"
#endif
#define GP_ALL_CASES GP_CASES(GP_SLOT_TU, GP_SLOT_B)

template <int M> struct MTag { static constexpr int value = M; };

// GP_DEBUG_BOUNDS (build.py GP_BUILD_DEBUG=1): every index into the code stream, the shared-memory
// tiles, the accumulators and the partial buffer is checked; a violation traps (the launch fails
// with an error). Off in the product build.
#ifndef GP_DEBUG_BOUNDS
#define GP_DEBUG_BOUNDS 0
#endif
#if GP_DEBUG_BOUNDS
#define GP_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define GP_CHECK(cond) do { } while (0)
#endif

// TMA bulk copies (non-tensor) into shared memory, completion tracked by an mbarrier
#ifndef GP_TMA_X
#define GP_TMA_X 1
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n"
               "GP_WAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra GP_WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void tma_bulk_g2s(float* dst, const float* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

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
// the global-X instantiation holds more live addresses: one resident CTA less
__global__ void __launch_bounds__(NT, XSMEM ? GP_MINB : GP_MINB_GLOBAL)
    eval_kernel(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_item;
  // shared-memory X tiles arrive by TMA bulk copies (cp.async.bulk) signalled on this mbarrier
  __shared__ __align__(8) uint64_t s_xbar;
  __shared__ uint32_t s_xphase;     // the mbarrier's current phase (thread 0 only)
  const int S = (a.metric == GP_PEARSON) ? 3 : 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int count = *a.prog_count;                 // programs in this variant's bucket
  // this bucket's group size (<= a.G; bucket_kernel), read once through shared memory
  __shared__ int s_gv;
  if (threadIdx.x == 0) {
    s_gv = *a.group_size;
    if constexpr (XSMEM && GP_TMA_X) {
      mbar_init(&s_xbar, 1);
      s_xphase = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const int Gv = s_gv;
  const int n_groups = (count + Gv - 1) / Gv;
  const int64_t n_items = (int64_t)n_groups * a.n_chunks;
  double* acc = reinterpret_cast<double*>(smem);                 // [NW][G][S]
  // this warp's transposed reduction block [RR][kRedStride] (single-sum metrics)
  float* rbw = reinterpret_cast<float*>(smem + (PREDICT ? 0 : smem_fp64_bytes(a.G, S))) +
               warp * (RR * kRedStride);
  const bool has_w = a.w != nullptr;
  // global-X path: 16-byte vector loads when every column start is 16-byte aligned
  const bool x_vec = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && ((a.ldx & 3) == 0);
  float* ys = reinterpret_cast<float*>(smem + (PREDICT ? 0 : smem_acc_bytes(a.G, S)));
  float* ws = ys + (PREDICT ? 0 : TILE);
  float* xs = ws + (has_w ? TILE : 0);                           // [n_cols][TILE] if XSMEM
  uint4* sw = reinterpret_cast<uint4*>(xs + (XSMEM ? a.n_cols * TILE : 0));  // stream window
  const float Ky = (!PREDICT && S == 3) ? *a.y_shift : 0.0f;

  // Persistent CTAs pull work items (program group g fastest, then row chunk q) from a queue;
  // each item's results go to fixed partial slots, so the sums do not depend on scheduling.
  for (;;) {
    __syncthreads();                               // previous item fully done with smem / s_item
    if (tid == 0) s_item = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= n_items) break;
    const int g = a.item_order ? (int)(item / a.n_chunks) : (int)(item % n_groups);
    const int64_t q0 = a.item_order ? item % a.n_chunks : item / n_groups;
    const int64_t q = a.chunk_reverse ? a.n_chunks - 1 - q0 : q0;
    GP_CHECK(g >= 0 && g < n_groups && q >= 0 && q < a.n_chunks);
    const int np = min(Gv, count - g * Gv);
    const int32_t* __restrict__ gids = a.prog_ids + (int64_t)g * Gv;    // group's program ids
    const int64_t s_begin = a.gstart[g], s_len = a.gstart[g + 1] - s_begin;
    if constexpr (!PREDICT) {
      for (int i = tid; i < NW * a.G * S; i += NT) acc[i] = 0.0;
    }
    const int64_t r_begin = q * a.rows_per_chunk;
    const int64_t r_end = min(r_begin + a.rows_per_chunk, a.n_rows);

    for (int64_t t0 = r_begin; t0 < r_end; t0 += TILE) {
      const int nvalid = (int)min((int64_t)TILE, r_end - t0);
      __syncthreads();  // previous tile's smem reads are done
      // ---- A2: stage the tile (coalesced; padded rows get w = 0 -> skipped) -----------------
      // X columns: one elected thread issues a TMA bulk copy per column (16-byte aligned
      // columns, whole 16-byte rows; padded rows keep stale values: every use of a padded row is
      // masked by w = 0 / the nvalid predicate); otherwise the threads copy, zero-padded
      const bool tma_x = XSMEM && GP_TMA_X && x_vec && (nvalid & 3) == 0;
      if constexpr (XSMEM && GP_TMA_X) {
        GP_CHECK(!tma_x || (int64_t)a.n_cols * nvalid * 4 < (1 << 20));   // mbarrier tx count
        if (tma_x && tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads -> async writes
          mbar_expect_tx(&s_xbar, (uint32_t)(a.n_cols * nvalid * 4));
          for (int c = 0; c < a.n_cols; ++c)
            tma_bulk_g2s(xs + c * TILE, a.X + (int64_t)c * a.ldx + t0, (uint32_t)(nvalid * 4),
                         &s_xbar);
        }
      }
      for (int i = tid; i < TILE; i += NT) {
        const bool in = i < nvalid;
        const int64_t row = t0 + i;
        if constexpr (!PREDICT) {
          // LogLoss stages the sign s = -1 (y > 1/2) / +1 instead of y: the per-row loss is then
          // softplus(s yhat) (one multiply instead of a compare and a select)
          const float yv = in ? a.y[row] : 0.0f;
          ys[i] = a.metric == GP_LOGLOSS ? (in ? (yv > 0.5f ? -1.0f : 1.0f) : 0.0f) : yv;
          if (has_w) ws[i] = in ? a.w[row] : 0.0f;
        }
        if constexpr (XSMEM) {
          if (!tma_x)
            for (int c = 0; c < a.n_cols; ++c)
              xs[c * TILE + i] = in ? a.X[(int64_t)c * a.ldx + row] : 0.0f;
        }
      }
      if constexpr (XSMEM && GP_TMA_X) {
        // thread 0 waits for the X bytes, the barrier releases everyone (no phase register is
        // kept live through the hot loop below)
        if (tma_x && tid == 0) {
          mbar_wait_parity(&s_xbar, s_xphase);
          s_xphase ^= 1u;
        }
      }
      __syncthreads();

      // ---- A3 + A4 + A5: walk the group's code stream --------------------------------------
      int ebase = tid * 4;                           // element e(r) = ebase + (r/4)*NT*4 + r%4
      float l0 = 0.f, l1 = 0.f, l2 = 0.f;
      // unweighted MSE / RMSE over a full tile: the FFMA-only loss, chosen once per tile
      const bool fast_mse = !PREDICT && (a.metric == GP_MSE || a.metric == GP_RMSE) && !has_w &&
                            nvalid == TILE;
      const bool fast_ll = !PREDICT && a.metric == GP_LOGLOSS && !has_w && nvalid == TILE;
      // Single-sum metrics (A5): each lane stores its fp32 sum of a finished program into row
      // (slot % RR) of the warp's block; every RR programs the warp reduces the block at once --
      // LPR lanes per row each sum 32 / LPR values (LDS.128, conflict-free with the padded
      // stride), log2(LPR) shuffles join them, and the row's first lane adds the program sum into
      // its fp64 accumulator. Fixed order -> deterministic. (Replaces one shuffle butterfly per
      // program.)
      auto flush = [&](int p0, int n) {
        __syncwarp();
        const int row = lane / LPR, part = lane % LPR;
        const float4* src =
            reinterpret_cast<const float4*>(rbw + row * kRedStride + part * (32 / LPR));
        float m = 0.0f;
#pragma unroll
        for (int k = 0; k < 8 / LPR; k += 2) {
          const float4 u = src[k], v = src[k + 1];
          m += ((u.x + u.y) + (u.z + u.w)) + ((v.x + v.y) + (v.z + v.w));
        }
#pragma unroll
        for (int o = 1; o < LPR; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
        GP_CHECK(p0 >= 0 && p0 + n <= a.G && n <= RR);
        if (part == 0 && row < n) acc[(size_t)warp * a.G + p0 + row] += (double)m;
        __syncwarp();
      };
      float st[STACK][R];
      // fused weighted loss of the current pass's rows (A4)
      // unweighted full tile: every row is live, w = 1 (FP32x2 sub + FFMA2 only)
      auto loss_fast_mse = [&]() {
#pragma unroll
        for (int k = 0; k < R4; ++k) {
          const float4 yv = *reinterpret_cast<const float4*>(ys + ebase + k * NT * 4);
          float d0, d1, d2, d3;
          sub_x2(d0, d1, st[0][4 * k], st[0][4 * k + 1], yv.x, yv.y);
          sub_x2(d2, d3, st[0][4 * k + 2], st[0][4 * k + 3], yv.z, yv.w);
          fma_x2(l0, l1, d0, d1, d0, d1, l0, l1);  // even / odd rows: l1 joins l0 at the end
          fma_x2(l0, l1, d2, d3, d2, d3, l0, l1);
        }
      };
      // unweighted LogLoss over a full tile: every row is live, ys holds the signs; row pairs
      // on the FP32x2 pipe (the FMNMX clamps stay scalar), even / odd rows into l0 / l1
      auto loss_fast_ll = [&]() {
#pragma unroll
        for (int k = 0; k < R4; ++k) {
          const float4 sv = *reinterpret_cast<const float4*>(ys + ebase + k * NT * 4);
          float z[4], a[4], e[4], g[4], l[4];
          mul_x2(z[0], z[1], st[0][4 * k], st[0][4 * k + 1], sv.x, sv.y);
          mul_x2(z[2], z[3], st[0][4 * k + 2], st[0][4 * k + 3], sv.z, sv.w);
          // softplus(z) = max(z, 0) + ln(1 + 2^(-|z| log2 e)), clamped to the S:191 range
#pragma unroll
          for (int j = 0; j < 4; j += 2) {
            mul_x2(a[j], a[j + 1], fabsf(z[j]), fabsf(z[j + 1]), -kLog2e, -kLog2e);
            e[j] = ex2_approx(a[j]);
            e[j + 1] = ex2_approx(a[j + 1]);
            add_x2(e[j], e[j + 1], e[j], e[j + 1], 1.0f, 1.0f);
            g[j] = lg2_approx(e[j]);
            g[j + 1] = lg2_approx(e[j + 1]);
            fma_x2(l[j], l[j + 1], g[j], g[j + 1], kLn2, kLn2, fmaxf(z[j], 0.0f),
                   fmaxf(z[j + 1], 0.0f));
            l[j] = fminf(fmaxf(l[j], kLogLossLo), kLogLossHi);
            l[j + 1] = fminf(fmaxf(l[j + 1], kLogLossLo), kLogLossHi);
            add_x2(l0, l1, l0, l1, l[j], l[j + 1]);
          }
        }
      };
      auto loss = [&](auto tag, float Kp) {
        constexpr int M = decltype(tag)::value;
#pragma unroll
        for (int k = 0; k < R4; ++k) {
          const float4 yv = *reinterpret_cast<const float4*>(ys + ebase + k * NT * 4);
          float4 wv;
          if (has_w) {
            wv = *reinterpret_cast<const float4*>(ws + ebase + k * NT * 4);
          } else {  // unweighted: w = 1 on rows of the tile, 0 on padding
            const int e = ebase + k * NT * 4;
            wv = make_float4(e < nvalid, e + 1 < nvalid, e + 2 < nvalid, e + 3 < nvalid);
          }
          const float yy[4] = {yv.x, yv.y, yv.z, yv.w}, ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float yh = st[0][4 * k + j];
            const bool live = ww[j] != 0.0f;         // w = 0 rows are skipped, never multiplied
            if constexpr (M == GP_MSE) {
              const float d = yh - yy[j];
              l0 += live ? ww[j] * d * d : 0.0f;
            } else if constexpr (M == GP_MAE) {
              l0 += live ? ww[j] * fabsf(yh - yy[j]) : 0.0f;
            } else if constexpr (M == GP_LOGLOSS) {
              // -[y ln p + (1-y) ln(1-p)], p = sigmoid(yh), y in {0,1}: softplus(-+yh),
              // clamped to the p-clamp's range (C7); yy = the staged sign
              const float z = yy[j] * yh;
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
      // end of one row pass of the program in group slot `pslot`: prediction store or loss
      int pslot = 0;
      auto end_pass = [&]() {
        // one pass per program: the loss starts from zero here (folds into the first FFMA2)
        // instead of being reset after the reduction
        if constexpr (SUB == 1) { l0 = l1 = l2 = 0.f; }
        if constexpr (PREDICT) {
          float* o = a.out + (int64_t)gids[pslot] * a.ld_out + t0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int e = ebase + (r >> 2) * NT * 4 + (r & 3);
            if (e < nvalid) o[e] = st[0][r];
          }
#ifdef GP_GLOBAL_X_ONLY
        } else if (fast_ll) {                        // wide shapes (C4's log-loss): before the MSE
          loss_fast_ll();                            // test, whose short body would otherwise be
        } else if (fast_mse) {                       // issued predicated off on every pass
          loss_fast_mse();
#else
        } else if (fast_mse) {                       // (C3: LogLoss first measured 2 % slower)
          loss_fast_mse();
        } else if (fast_ll) {
          loss_fast_ll();
#endif
        } else {
          switch (a.metric) {
            case GP_MAE: loss(MTag<GP_MAE>{}, 0.0f); break;
            case GP_MSE: case GP_RMSE: loss(MTag<GP_MSE>{}, 0.0f); break;
            case GP_LOGLOSS: loss(MTag<GP_LOGLOSS>{}, 0.0f); break;
            default: loss(MTag<GP_PEARSON>{}, __ldg(a.shift + gids[pslot])); break;
          }
        }
      };
      // The stream is read from a shared-memory window (copied by the whole CTA: once per item
      // when the group's stream fits, else window by window per tile); each warp walks it with a
      // two-deep prefetch that runs uninterrupted across program boundaries.
      for (int64_t w0 = 0; w0 < s_len; w0 += kStreamWin) {
        const int wn = (int)min((int64_t)kStreamWin, s_len - w0);
        if (s_len > kStreamWin || t0 == r_begin) {
          __syncthreads();                           // every warp is done with the old window
          GP_CHECK(wn > 0 && wn <= kStreamWin);
          for (int i = tid; i < wn + 2; i += NT) sw[i] = __ldg(a.stream + s_begin + w0 + i);
          __syncthreads();
        }
        // prefetch only the case ids (2 registers); the payload word is read from the window
        // at the top of each iteration (its LDS latency overlaps the dispatch branch). The loop
        // has no trip counter: the window's last word carries kEndWin (pack_kernel).
        const uint4* wp = sw;
#ifndef GP_PREFETCH
#define GP_PREFETCH 2
#endif
#if GP_PREFETCH == 2
        uint32_t c_n = wp[0].x, c_n2 = wp[1].x;
#else
        uint32_t c_n = wp[0].x;
#endif
#pragma unroll 1
        for (;;) {
          const uint32_t cid = c_n;
#if GP_PREFETCH == 2
          c_n = c_n2;
          c_n2 = wp[2].x;                            // window carries two look-ahead words
#else
          c_n = wp[1].x;                             // loaded into the register the next dispatch
                                                     // reads: no rotation move before the BRX
#endif
          const uint4 cw = *wp;
          ++wp;
          GP_CHECK(wp <= sw + kStreamWin);             // never past the window's last word
          switch (cid) {                             // one jump table (BRX) over every case
            GP_ALL_CASES
            default: __builtin_unreachable();        // stage / pack guarantee a valid case
          }
          if (cw.w) {                                // last word of a row pass or of the window
            if (cw.w & (kEndPass | kEndProgram)) {
              end_pass();
              if (SUB > 1 && (cw.w & kEndPass)) {    // next row pass of the same program
                ebase = (int)(cw.w >> 8) * NT * R + tid * 4;
              } else {                               // program done (A5)
                if constexpr (!PREDICT) {
                  const int j = (int)(cw.w >> 8);    // == pslot
                  GP_CHECK(j == pslot && j < np && j < a.G);
                  if (S == 1) {
                    rbw[(j % RR) * kRedStride + lane] = l0 + l1;  // l1: odd rows (MSE)
                    if (j % RR == RR - 1) flush(j - (RR - 1), RR);
                  } else {
                    double* slot = acc + ((size_t)warp * a.G + j) * S;
                    const double v0 = warp_sum_f64(l0), v1 = warp_sum_f64(l1),
                                 v2 = warp_sum_f64(l2);
                    if (lane == 0) { slot[0] += v0; slot[1] += v1; slot[2] += v2; }
                  }
                  if constexpr (SUB > 1) { l0 = l1 = l2 = 0.f; }
                }
                if constexpr (SUB > 1) ebase = tid * 4;
                ++pslot;
              }
            }
            if (cw.w & kEndWin) break;
          }
        }
      }
      if (!PREDICT && S == 1 && np % RR != 0)        // last partial block of the tile
        flush(np - np % RR, np % RR);
    }

    if constexpr (!PREDICT) {
      __syncthreads();
      // compact layout: the program in bucket slot j of this variant owns partial column
      // kConstCols + (part_base + j) * S (part_base = programs of the lower-capacity buckets), so
      // only programs that were evaluated per row are written and tile-reduced
      double* prow = a.partial + q * a.ld_part + kConstCols +
                     ((int64_t)*a.part_base + (int64_t)g * Gv) * S;
      GP_CHECK(np >= 0 && np <= Gv && Gv <= a.G &&
               kConstCols + ((int64_t)*a.part_base + (int64_t)g * Gv + np) * S <= a.ld_part);
      for (int j = tid; j < np * S; j += NT) {
        const int pl = j / S, k = j - pl * S;
        double sum = 0.0;
        for (int wv = 0; wv < NW; ++wv) sum += acc[((size_t)wv * a.G + pl) * S + k];
        prow[j] = sum;
      }
    }
  }
}

// ---- exports of this translation unit: ONE (PREDICT, XSMEM) instantiation ------------------------
// build.py generates one translation unit per (shape, PREDICT, XSMEM) (GP_KP, GP_KXS) so the
// heavy dispatch switch of each kernel compiles in parallel; eval_registry.cpp assembles the
// EvalVariant of each shape from these functions.
#if !defined(GP_KP) || !defined(GP_KXS)
#error "define GP_KP and GP_KXS (generated translation units, build.py)"
#endif
#define GP_KTAG GP_CAT(GP_KP, GP_KXS)
#define GP_KERNEL eval_kernel<GP_KP, GP_KXS>

cudaError_t GP_CAT(launch_k, GP_KTAG)(const EvalArgs& a, int n_ctas, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(GP_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxDynSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GP_KERNEL<<<n_ctas, NT, smem, s>>>(a);
  return cudaGetLastError();
}

// resident CTAs per SM for a dynamic shared-memory size (memoised: the size rarely changes)
int GP_CAT(occ_k, GP_KTAG)(size_t smem) {
  thread_local size_t last_smem = ~(size_t)0;
  thread_local int last_n = 0;
  if (smem == last_smem) return last_n;
  int n = 0;
  cudaFuncSetAttribute(GP_KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, GP_KERNEL, NT, smem);
  last_smem = smem;
  last_n = n;
  return n;
}

#if GP_KP == 0 && ((defined(GP_GLOBAL_X_ONLY) && GP_KXS == 0) || (!defined(GP_GLOBAL_X_ONLY) && GP_KXS == 1))
// the shape's static description (exported once per shape)
EvalShape shape_info() { return EvalShape{STACK, R, SUB, NT}; }
size_t smem_bytes(int G, int S, int n_cols, int weighted, int xsmem, int predict) {
  return smem_total(G, S, n_cols, weighted != 0, xsmem != 0, predict != 0);
}
#endif

}  // namespace GP_NS
}  // namespace gpb
