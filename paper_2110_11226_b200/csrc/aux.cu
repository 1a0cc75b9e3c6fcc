// aux.cu -- the small kernels around the fused evaluator:
//   stage      (A1) validate + compile the flat population into evaluation-order code words
//   shift      (A4) Pearson shift K_p = f_p(reference row), one thread per program
//   tile_reduce(A5) fixed-order fp64 sum of per-work-item partials
//   finalize   (A7) sums -> fp32 raw fitness + status bits
//   select     (A8) Philox tournament selection with parsimony
#include <cfloat>
#include "device_ops.cuh"
#include "kernels.h"

namespace gpb {

// ---------------------------------------------------------------------------------------------
// Stage / compile. One thread per program (programs are short; this is a few µs).
//  - prefix validation with the needed-counter scan, opcode and variable-range checks
//  - reverse (evaluation-order) emission with the static stack slot of every node
//  - stack need = max occupancy; > capacity -> GP_FLAG_STACK_OVERFLOW
// Invalid programs get code_len = 0 and are skipped by every later kernel.
// ---------------------------------------------------------------------------------------------
__global__ void stage_kernel(const gp_node* __restrict__ nodes, const int64_t* __restrict__ off,
                             int32_t n_programs, int64_t n_nodes, int32_t n_cols, int32_t cap,
                             uint2* __restrict__ code, int64_t* __restrict__ code_off,
                             int32_t* __restrict__ code_len, uint32_t* __restrict__ status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) code[n_nodes] = code[n_nodes + 1] = make_uint2(0u, 0u);  // prefetch pad words
  if (p >= n_programs) return;
  const int64_t b = off[p], e = off[p + 1];
  uint32_t flags = 0;
  if (b < 0 || e > n_nodes || e <= b) {
    flags |= GP_FLAG_INVALID_PREFIX;
  } else {
    int64_t needed = 1;
    for (int64_t i = b; i < e; ++i) {
      if (needed == 0) { flags |= GP_FLAG_INVALID_PREFIX; break; }
      const gp_node nd = nodes[i];
      const int a = op_arity(nd.op);
      if (a < 0 || nd.op < 0) { flags |= GP_FLAG_BAD_OPCODE; break; }
      if (nd.op == GP_OP_VAR && (nd.var < 0 || nd.var >= n_cols)) flags |= GP_FLAG_VAR_RANGE;
      needed += a - 1;
    }
    if (!(flags & GP_FLAG_BAD_OPCODE) && needed != 0) flags |= GP_FLAG_INVALID_PREFIX;
  }
  if (!flags) {
    const int64_t len = e - b;
    int sp = 0, need = 0;
    for (int64_t k = 0; k < len; ++k) {
      const gp_node nd = nodes[e - 1 - k];
      const int a = op_arity(nd.op);
      const int slot = a == 0 ? sp : sp - a;  // terminal pushes at sp; f writes over its operands
      sp += 1 - a;
      need = need > sp ? need : sp;
      if (need > cap) break;
      const uint32_t payload = nd.op == GP_OP_VAR ? ((uint32_t)nd.var << kCaseBits) : 0u;
      code[b + k] = make_uint2((uint32_t)(nd.op * cap + slot) | payload, __float_as_uint(nd.value));
    }
    if (need > cap) flags |= GP_FLAG_STACK_OVERFLOW;
  }
  code_off[p] = b;
  code_len[p] = flags ? 0 : (int32_t)(e - b);
  status[p] = flags;
}

cudaError_t launch_stage(const gp_node* nodes, const int64_t* offsets, int32_t n_programs,
                         int64_t n_nodes, int32_t n_cols, int32_t stack_cap, uint2* code,
                         int64_t* code_off, int32_t* code_len, uint32_t* status, cudaStream_t s) {
  const int nt = 128;
  stage_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(nodes, offsets, n_programs, n_nodes,
                                                          n_cols, stack_cap, code, code_off,
                                                          code_len, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Pearson shift (C9): K_p = f_p(x_ref), evaluated with the SAME fp32 op code as the
// register-stack evaluator so a constant program gives d = yhat - K_p = 0 exactly on every row.
// ---------------------------------------------------------------------------------------------
__global__ void shift_kernel(const uint2* __restrict__ code, const int64_t* __restrict__ code_off,
                             const int32_t* __restrict__ code_len, int32_t n_programs, int32_t cap,
                             const float* __restrict__ xref, int64_t stride,
                             float* __restrict__ shift) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_programs) return;
  const int len = code_len[p];
  if (len == 0) { shift[p] = 0.0f; return; }
  float stk[GP_MAX_STACK + 1];
  const uint2* pc = code + code_off[p];
  for (int k = 0; k < len; ++k) {
    const uint2 cw = pc[k];
    const int id = (int)(cw.x & kCaseMask), kind = id / cap, slot = id - kind * cap;
    if (kind == GP_OP_VAR) stk[slot] = xref[(int64_t)(cw.x >> kCaseBits) * stride];
    else if (kind == GP_OP_CONST) stk[slot] = __uint_as_float(cw.y);
    else if (op_arity(kind) == 1) stk[slot] = apply_rt(kind, stk[slot], 0.0f);
    else stk[slot] = apply_rt(kind, stk[slot + 1], stk[slot]);
  }
  shift[p] = stk[0];
}

cudaError_t launch_shift(const uint2* code, const int64_t* code_off, const int32_t* code_len,
                         int32_t n_programs, int32_t stack_cap, const float* xref,
                         int64_t xref_stride, float* shift_out, cudaStream_t s) {
  const int nt = 128;
  shift_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(code, code_off, code_len, n_programs,
                                                          stack_cap, xref, xref_stride, shift_out);
  return cudaGetLastError();
}

__global__ void copy_scalar_kernel(const float* src, float* dst) { *dst = *src; }
cudaError_t launch_copy_scalar(const float* src, float* dst, cudaStream_t s) {
  copy_scalar_kernel<<<1, 1, 0, s>>>(src, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Cross-work-item reduction: sums[j] = sum_{q < n_chunks} partial[q][j], in fixed q
// order -> run-to-run deterministic.
// ---------------------------------------------------------------------------------------------
__global__ void tile_reduce_kernel(const double* __restrict__ partial, int64_t n_chunks,
                                   int64_t ld, double* __restrict__ sums) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ld) return;
  double s = 0.0;
  for (int64_t q = 0; q < n_chunks; ++q) s += partial[q * ld + j];
  sums[j] = s;
}

cudaError_t launch_tile_reduce(const double* partial, int64_t n_chunks, int64_t ld_part,
                               double* sums, cudaStream_t s) {
  const int nt = 256;
  tile_reduce_kernel<<<(unsigned)((ld_part + nt - 1) / nt), nt, 0, s>>>(partial, n_chunks,
                                                                          ld_part, sums);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Finalize: per-program sums (+ dataset constants W, S_y, S_yy at the end) ->
// raw fitness ("vector containing final raw fitness values"), S:201 normalisation.
// ---------------------------------------------------------------------------------------------
__global__ void finalize_kernel(const double* __restrict__ sums, int32_t n_programs,
                                int32_t metric, const int32_t* __restrict__ code_len,
                                float* __restrict__ fitness, uint32_t* __restrict__ status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_programs) return;
  const int S = metric == GP_PEARSON ? 3 : 1;
  const int64_t nS = (int64_t)n_programs * S;
  const double W = sums[nS], Sy = sums[nS + 1], Syy = sums[nS + 2];
  uint32_t fl = status[p];
  float out;
  if (code_len[p] == 0) {
    out = metric == GP_PEARSON ? -INFINITY : INFINITY;
  } else if (metric != GP_PEARSON) {
    double f = sums[p] / W;
    if (metric == GP_RMSE) f = sqrt(f);
    if (!isfinite(f) || f > (double)FLT_MAX) { f = INFINITY; fl |= GP_FLAG_NONFINITE; }
    out = (float)f;
  } else {
    const double Sd = sums[3 * (int64_t)p], Sdd = sums[3 * (int64_t)p + 1],
                 Sdy = sums[3 * (int64_t)p + 2];
    const double cov = Sdy - Sd * Sy / W, vd = Sdd - Sd * Sd / W, vy = Syy - Sy * Sy / W;
    double r = cov / sqrt(vd * vy);
    if (!(vd > 0.0) || !(vy > 0.0) || !isfinite(r)) { r = 0.0; fl |= GP_FLAG_UNDEFINED_CORR; }
    r = r > 1.0 ? 1.0 : (r < -1.0 ? -1.0 : r);
    out = (float)r;
  }
  fitness[p] = out;
  status[p] = fl;
}

cudaError_t launch_finalize(const double* sums, int32_t n_programs, int32_t metric,
                            const int32_t* code_len, float* fitness, uint32_t* status,
                            cudaStream_t s) {
  const int nt = 128;
  finalize_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(sums, n_programs, metric, code_len,
                                                             fitness, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Tournament selection (Eqs. 1-2). One thread per tournament.
// Layout (C10): draw i of tournament t = word i%4 of Philox4x32-10 with
// counter (t, generation, i/4, 0) and key (seed lo, seed hi); index = (u64(word) * n) >> 32.
// Adjusted fitness with explicit fp32 roundings (no FMA contraction); NaN = worst; ties ->
// smallest index.
// ---------------------------------------------------------------------------------------------
__global__ void select_kernel(const float* __restrict__ fitness, const int64_t* __restrict__ off,
                              int32_t n, int32_t n_tournaments, int32_t k, float c, int32_t higher,
                              uint32_t k0, uint32_t k1, uint32_t generation,
                              int32_t* __restrict__ winners) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tournaments) return;
  int32_t best = -1;
  float best_adj = 0.0f;
  u32x4 words = {0, 0, 0, 0};
  for (int i = 0; i < k; ++i) {
    if ((i & 3) == 0) words = philox4x32_10(u32x4{(uint32_t)t, generation, (uint32_t)(i >> 2), 0u},
                                            k0, k1);
    const uint32_t wd = (i & 3) == 0 ? words.x : (i & 3) == 1 ? words.y : (i & 3) == 2 ? words.z
                                                                                        : words.w;
    const int32_t idx = (int32_t)(((uint64_t)wd * (uint64_t)n) >> 32);
    const float pen = __fmul_rn(c, (float)(off[idx + 1] - off[idx]));   // Eq. 1
    float adj = higher ? __fsub_rn(fitness[idx], pen) : __fadd_rn(fitness[idx], pen);  // Eq. 2
    if (adj != adj) adj = higher ? -INFINITY : INFINITY;
    bool better;
    if (best < 0) better = true;
    else if (higher) better = adj > best_adj || (adj == best_adj && idx < best);
    else better = adj < best_adj || (adj == best_adj && idx < best);
    if (better) { best = idx; best_adj = adj; }
  }
  winners[t] = best;
}

cudaError_t launch_select(const float* fitness, const int64_t* offsets, int32_t n_programs,
                          int32_t n_tournaments, int32_t k, float parsimony, int32_t higher,
                          uint64_t seed, uint32_t generation, int32_t* winners, cudaStream_t s) {
  const int nt = 128;
  select_kernel<<<(n_tournaments + nt - 1) / nt, nt, 0, s>>>(
      fitness, offsets, n_programs, n_tournaments, k, parsimony, higher, (uint32_t)seed,
      (uint32_t)(seed >> 32), generation, winners);
  return cudaGetLastError();
}

}  // namespace gpb
