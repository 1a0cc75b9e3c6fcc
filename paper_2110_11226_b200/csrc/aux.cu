// aux.cu -- the small kernels around the fused evaluator:
//   stage      (A1) validate + compile the flat population into evaluation-order code words
//   shift      (A4) Pearson shift K_p = f_p(reference row), one thread per program
//   tile_reduce(A5) fixed-order fp64 sum of per-work-item partials
//   finalize   (A7) sums -> fp32 raw fitness + status bits
//   select     (A8) Philox tournament selection with parsimony
#include <cfloat>
#include "device_ops.cuh"
#include "aux.h"

namespace gpb {

// ---------------------------------------------------------------------------------------------
// Stage / compile. One thread per program (programs are short; a few µs total).
//  - prefix validation with the needed-counter scan, opcode and variable-range checks
//  - a bottom-up pass folds variable-free subtrees into constants (evaluated once, with the
//    evaluator's fp32 op functions) and computes every subtree's stack need with terminals folded
//    into their parent's code word and the Sethi-Ullman order (evaluate the child needing more slots first;
//    the classic reverse-prefix order of P:194 is the default, swapped only when it needs more);
//    a post-order emission then writes one code word per function node with its static
//    destination slot (device_ops.cuh "compiled program code"); stack need > capacity ->
//    GP_FLAG_STACK_OVERFLOW. Depth > 127 is also reported as overflow.
// Invalid programs get code_len = 0 and are skipped by every later kernel. Variable-free programs
// (the whole tree folds to one constant) get need = 0.
// ---------------------------------------------------------------------------------------------
__global__ void stage_kernel(const gp_node* __restrict__ nodes, const int64_t* __restrict__ off,
                             int32_t n_programs, int64_t n_nodes, int32_t n_cols, int32_t cap,
                             uint4* __restrict__ code, int64_t* __restrict__ code_off,
                             int32_t* __restrict__ code_len, int32_t* __restrict__ need_out,
                             uint32_t* __restrict__ status, int32_t* __restrict__ scratch,
                             int32_t sethi_ullman) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) code[n_nodes] = code[n_nodes + 1] = make_uint4(0u, 0u, 0u, 0u);  // prefetch pads
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
      if (a < 0) { flags |= GP_FLAG_BAD_OPCODE; break; }
      if (nd.op == GP_OP_VAR && (nd.var < 0 || nd.var >= n_cols)) flags |= GP_FLAG_VAR_RANGE;
      needed += a - 1;
    }
    if (!(flags & GP_FLAG_BAD_OPCODE) && needed != 0) flags |= GP_FLAG_INVALID_PREFIX;
  }
  int64_t emitted = 0;
  int need_root = 0;
  if (!flags) {
    // (1) bottom-up (reverse prefix) pass over the nodes: subtree end, constant folding and stack
    // need. A variable-free subtree is evaluated ONCE here, with the same fp32 op functions the
    // evaluator uses, and becomes a constant operand of its parent (per-program constant, not
    // per-row work). Terminal and constant operands are folded into their parent's code word
    // (need 0); binary nodes whose operands are both computed values use the Sethi-Ullman order
    // (evaluate the child needing more slots first) unless the classic order is requested.
    int32_t* nd_need = scratch + b;               // per node
    int32_t* nd_end = scratch + n_nodes + b;      // per node (relative to b)
    int32_t* nd_cst = scratch + 2 * n_nodes + b;  // 1: variable-free subtree
    uint32_t* nd_val = reinterpret_cast<uint32_t*>(scratch + 3 * n_nodes + b);  // its fp32 value
    const int64_t len = e - b;
    for (int64_t i = len - 1; i >= 0; --i) {
      const gp_node nd = nodes[b + i];
      const int a = op_arity(nd.op);
      if (a == 0) {
        nd_need[i] = 0;
        nd_end[i] = (int32_t)(i + 1);
        nd_cst[i] = nd.op == GP_OP_CONST;
        nd_val[i] = __float_as_uint(nd.value);
        continue;
      }
      const int64_t A = i + 1;
      if (a == 1) {
        nd_end[i] = nd_end[A];
        nd_cst[i] = nd_cst[A];
        if (nd_cst[A]) {
          nd_val[i] = __float_as_uint(apply_rt(nd.op, __uint_as_float(nd_val[A]), 0.0f));
          nd_need[i] = 0;
        } else {
          nd_need[i] = nd_need[A] > 0 ? nd_need[A] : 1;
        }
        continue;
      }
      const int64_t B = nd_end[A];
      nd_end[i] = nd_end[B];
      nd_cst[i] = nd_cst[A] && nd_cst[B];
      if (nd_cst[i]) {
        nd_val[i] = __float_as_uint(apply_rt(nd.op, __uint_as_float(nd_val[A]),
                                             __uint_as_float(nd_val[B])));
        nd_need[i] = 0;
        continue;
      }
      const int nA = nd_need[A], nB = nd_need[B];
      int n;
      if (nA == 0 || nB == 0) n = max(max(nA, nB), 1);
      else n = sethi_ullman ? min(max(nB, 1 + nA), max(nA, 1 + nB)) : max(nB, 1 + nA);
      nd_need[i] = n;
    }
    need_root = (len == 1 || nd_cst[0]) ? 1 : nd_need[0];
    if (need_root > cap) flags |= GP_FLAG_STACK_OVERFLOW;
    // a variable-free program is ONE constant c (its single PUSH_C word carries c): need 0 marks
    // it, so its loss can come from the dataset moments (finalize_kernel) instead of per row
    if (nd_cst[0]) need_root = 0;
  }
  if (!flags) {
    // (2) post-order emission with the chosen child order; terminal and folded-constant operands
    // go into the parent's word
    const int32_t* nd_need = scratch + b;
    const int32_t* nd_end = scratch + n_nodes + b;
    const int32_t* nd_cst = scratch + 2 * n_nodes + b;
    const uint32_t* nd_val = reinterpret_cast<const uint32_t*>(scratch + 3 * n_nodes + b);
    auto src = [&](int64_t i, uint32_t* pl) -> int {  // 0 stack, 1 variable, 2 constant
      const gp_node nd = nodes[b + i];
      if (nd.op == GP_OP_VAR) { *pl = (uint32_t)nd.var; return 1; }
      if (nd_cst[i]) { *pl = nd_val[i]; return 2; }
      *pl = 0u;
      return 0;
    };
    auto emit = [&](int opv, int slot, uint32_t pa, uint32_t pb) {
      code[b + emitted++] = make_uint4((uint32_t)(opv * kCaseStride + slot), pa, pb, 0u);
    };
    if (e - b == 1 || nd_cst[0]) {
      uint32_t pl;
      const int k = src(0, &pl);
      emit(k == 1 ? OPV_PUSH_V : OPV_PUSH_C, 0, pl, 0u);
    } else {
      constexpr int kMaxDepth = 128;
      int64_t stk_i[kMaxDepth];
      int stk_ph[kMaxDepth];
      int top = 0, sp = 0;
      stk_i[0] = 0;
      stk_ph[0] = 0;
      while (top >= 0) {
        const int64_t i = stk_i[top];
        const int ph = stk_ph[top];
        const int ar = op_arity(nodes[b + i].op);
        const int64_t A = i + 1, B = ar == 2 ? nd_end[A] : -1;
        uint32_t pa, pb = 0u;
        const int sa = src(A, &pa), sb = ar == 2 ? src(B, &pb) : -1;
        // both operands on the stack: default order evaluates B first (reverse prefix);
        // Sethi-Ullman swaps when that needs fewer slots
        const bool both = ar == 2 && sa == 0 && sb == 0;
        const bool a_first = both && sethi_ullman &&
                             max(nd_need[A], 1 + nd_need[B]) < max(nd_need[B], 1 + nd_need[A]);
        int64_t child = -1;
        if (ph == 0) {
          if (ar == 1) child = sa == 0 ? A : -1;
          else if (both) child = a_first ? A : B;
          else if (sa == 0) child = A;
          else if (sb == 0) child = B;
        } else if (ph == 1 && both) {
          child = a_first ? B : A;
        }
        if (child >= 0) {
          stk_ph[top] = ph + 1;
          if (top + 1 >= kMaxDepth) { flags |= GP_FLAG_STACK_OVERFLOW; break; }
          ++top;
          stk_i[top] = child;
          stk_ph[top] = 0;
          continue;
        }
        // all stack operands are evaluated: emit this node
        const int op = nodes[b + i].op;
        if (ar == 1) {
          if (sa == 0) { emit(opv_un(op, UV_S), sp - 1, 0u, 0u); }
          else { emit(opv_un(op, sa == 1 ? UV_V : UV_C), sp, pa, 0u); ++sp; }
        } else if (both) {
          sp -= 1;
          emit(opv_bin(op, a_first ? BV_SSR : BV_SS), sp - 1, 0u, 0u);
        } else if (sa == 0) {
          emit(opv_bin(op, sb == 1 ? BV_SV : BV_SC), sp - 1, pa, pb);
        } else if (sb == 0) {
          emit(opv_bin(op, sa == 1 ? BV_VS : BV_CS), sp - 1, pa, pb);
        } else {
          const int v = sa == 1 ? (sb == 1 ? BV_VV : BV_VC) : (sb == 1 ? BV_CV : BV_CC);
          emit(opv_bin(op, v), sp, pa, pb);
          ++sp;
        }
        --top;
      }
    }
  }
  need_out[p] = need_root;
  code_off[p] = b;
  code_len[p] = flags ? 0 : (int32_t)emitted;
  status[p] = flags;
}

cudaError_t launch_stage(const gp_node* nodes, const int64_t* offsets, int32_t n_programs,
                         int64_t n_nodes, int32_t n_cols, int32_t max_stack, uint4* code,
                         int64_t* code_off, int32_t* code_len, int32_t* need, uint32_t* status,
                         int32_t* scratch, int32_t sethi_ullman, cudaStream_t s) {
  const int nt = 128;
  stage_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(nodes, offsets, n_programs, n_nodes,
                                                          n_cols, max_stack, code, code_off,
                                                          code_len, need, status, scratch,
                                                          sethi_ullman);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Bucketing by stack need + code-stream layout (one CTA of 1024 threads). Program p goes to the
// first variant whose register stack holds its need; each bucket list keeps ascending program
// order (deterministic). Each variant's stream holds, per program, SUB_b copies of its code words;
// pos / gstart are absolute stream offsets (group g of bucket b starts at gstart[b][g]).
// ---------------------------------------------------------------------------------------------
namespace {
// Block-wide exclusive scan of one int64 per thread (1024 threads); returns the block total.
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* out, int64_t* warp_tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t t = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  *out = (warp ? warp_tot[warp - 1] : 0) + x - v;
  const int64_t total = warp_tot[31];
  __syncthreads();
  return total;
}
}  // namespace

__global__ void __launch_bounds__(1024) bucket_kernel(const int32_t* __restrict__ need,
                                                      const int32_t* __restrict__ code_len,
                                                      int32_t n, int32_t G,
                                                      int32_t* __restrict__ lists,
                                                      int64_t* __restrict__ pos,
                                                      int64_t* __restrict__ gstart,
                                                      int32_t* __restrict__ counts,
                                                      int64_t* __restrict__ base, int4 sub4,
                                                      int32_t skip_const, int32_t p_lo,
                                                      int32_t p_hi, int32_t* __restrict__ inv) {
  __shared__ int warp_cnt[kNumVariants][32];
  __shared__ int cnt[kNumVariants];
  __shared__ int64_t warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int caps[kNumVariants] = {4, 8, 12, 20};   // kVariantStack
  const int subs[kNumVariants] = {sub4.x, sub4.y, sub4.z, sub4.w};  // row passes per variant
  if (tid < kNumVariants) { cnt[tid] = 0; counts[kNumVariants + tid] = 0; }  // work counters
  __syncthreads();
  // phase 1: stable partition by stack need
  for (int c0 = 0; c0 < n; c0 += 1024) {
    const int p = c0 + tid;
    int b = -1;
    if (p >= p_lo && p < p_hi && code_len[p] > 0 && !(skip_const && need[p] == 0)) {
      b = kNumVariants - 1;
      for (int v = kNumVariants - 1; v >= 0; --v)
        if (need[p] <= caps[v]) b = v;
    }
    int rank[kNumVariants];
    for (int v = 0; v < kNumVariants; ++v) {
      const unsigned m = __ballot_sync(0xffffffffu, b == v);
      rank[v] = __popc(m & ((1u << lane) - 1u));
      if (lane == 0) warp_cnt[v][warp] = __popc(m);
    }
    __syncthreads();
    if (b >= 0) {
      int off = cnt[b] + rank[b];
      for (int w2 = 0; w2 < warp; ++w2) off += warp_cnt[b][w2];
      lists[(int64_t)b * n + off] = p;
    }
    __syncthreads();
    if (tid < kNumVariants) {
      int t = 0;
      for (int w2 = 0; w2 < 32; ++w2) t += warp_cnt[tid][w2];
      cnt[tid] += t;
    }
    __syncthreads();
  }
  // per-bucket group size: as many groups as the plan gives the whole population (ceil(n / G)),
  // so a small bucket (deep programs) is still spread over enough groups that the CTAs working on
  // it share row chunks (a few large groups would keep ~CTAs / groups chunks of X in flight and
  // spill L2: C5 generation 0's 8-slot launch re-read X from DRAM ~50 times)
  // (only buckets that would get fewer than half the plan's groups are re-cut; the large ones
  // keep G -- smaller groups there cost staging and measured slower on C3 / C4)
  __shared__ int gsz_s[kNumVariants];
  if (tid < kNumVariants) {
    const int ng = (n + G - 1) / G;
    const int groups_at_G = (cnt[tid] + G - 1) / G;
    gsz_s[tid] = 2 * groups_at_G >= ng ? G : min(G, max(1, (cnt[tid] + ng - 1) / ng));
    inv[n + kNumVariants + 1 + tid] = gsz_s[tid];
  }
  __syncthreads();
  // phase 2: stream offsets per bucket (words = SUB x (len + 1) per program)
  int64_t running = 0;
  for (int b = 0; b < kNumVariants; ++b) {
    const int cb = cnt[b];
    const int Gb = gsz_s[b];
    if (tid == 0) base[b] = running;
    for (int c0 = 0; c0 < cb; c0 += 1024) {
      const int j = c0 + tid;
      const int64_t words = j < cb ? (int64_t)subs[b] * code_len[lists[(int64_t)b * n + j]] : 0;
      int64_t ex;
      const int64_t tot = block_exclusive_scan(words, &ex, warp_tot);
      if (j < cb) {
        pos[(int64_t)b * n + j] = running + ex;
        if (j % Gb == 0) gstart[(int64_t)b * (n + 1) + j / Gb] = running + ex;
      }
      running += tot;
    }
    if (tid == 0) gstart[(int64_t)b * (n + 1) + (cb + Gb - 1) / Gb] = running;
    __syncthreads();
  }
  if (tid == 0) base[kNumVariants] = running;
  if (tid < kNumVariants) counts[tid] = cnt[tid];
  // phase 3: compact partial-sum positions (kernels.h kConstCols): bucket b's programs follow
  // those of buckets < b; inv[p] = position or -1 (not evaluated); inv[n + b] = first position of
  // bucket b, inv[n + kNumVariants] = evaluated programs in total
  for (int p = tid; p < n; p += 1024) inv[p] = -1;
  __syncthreads();
  int pb = 0;
  for (int b = 0; b < kNumVariants; ++b) {
    if (tid == 0) inv[n + b] = pb;
    for (int j = tid; j < cnt[b]; j += 1024) inv[lists[(int64_t)b * n + j]] = pb + j;
    pb += cnt[b];
  }
  if (tid == 0) inv[n + kNumVariants] = pb;
}

cudaError_t launch_bucket(const int32_t* need, const int32_t* code_len, int32_t n_programs,
                          int32_t G, const int* subs, int32_t* lists, int64_t* pos,
                          int64_t* gstart, int32_t* counts, int64_t* base, int32_t skip_const,
                          int32_t p_lo, int32_t p_hi, int32_t* inv, cudaStream_t s) {
  bucket_kernel<<<1, 1024, 0, s>>>(need, code_len, n_programs, G, lists, pos, gstart, counts,
                                   base, make_int4(subs[0], subs[1], subs[2], subs[3]), skip_const,
                                   p_lo, p_hi, inv);
  return cudaGetLastError();
}

// One thread per (bucket, list entry): SUB copies of the program's code, one per row pass. The
// last word of each pass carries the pass flags in .w (kernels.h kEndPass / kEndProgram): the next
// pass index, or the program's slot in its group at the end of the last pass.
__global__ void pack_kernel(const uint4* __restrict__ code, const int64_t* __restrict__ code_off,
                            const int32_t* __restrict__ code_len, const int32_t* __restrict__ lists,
                            const int64_t* __restrict__ pos, const int32_t* __restrict__ counts,
                            const int64_t* __restrict__ base, const int64_t* __restrict__ gstart,
                            int32_t n, int4 sub4, const int32_t* __restrict__ inv,
                            uint4* __restrict__ stream) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) stream[base[kNumVariants]] = stream[base[kNumVariants] + 1] = make_uint4(0, 0, 0, 0);
  if (i >= (int64_t)kNumVariants * n) return;
  const int b = (int)(i / n), j = (int)(i % n);
  if (j >= counts[b]) return;
  const int subs[kNumVariants] = {sub4.x, sub4.y, sub4.z, sub4.w};
  const int p = lists[i];
  const int len = code_len[p];
  const uint4* src = code + code_off[p];
  uint4* dst = stream + pos[i];
  const int caps[kNumVariants] = {4, 8, 12, 20};   // kVariantStack
  const int vstack = caps[b];            // the variant's dispatch numbering (device_ops opv_rank)
  // the group's stream [gs, ge): words at window ends get kEndWin
  const int Gb = inv[n + kNumVariants + 1 + b];   // the bucket's group size (bucket_kernel)
  const int64_t gs = gstart[(int64_t)b * (n + 1) + j / Gb], ge = gstart[(int64_t)b * (n + 1) + j / Gb + 1];
  for (int pass = 0; pass < subs[b]; ++pass) {
    for (int k = 0; k < len; ++k) {
      uint4 w = src[k];
      const int opv = (int)w.x / kCaseStride, slot = (int)w.x - opv * kCaseStride;
      w.x = (uint32_t)(opv_rank(opv) * vstack + slot);
      *dst++ = w;
    }
    const bool last = pass == subs[b] - 1;
    dst[-1].w = last ? (kEndProgram | ((uint32_t)(j % Gb) << 8))
                     : (kEndPass | ((uint32_t)(pass + 1) << 8));
  }
  for (int64_t t = pos[i] - gs; t < pos[i] - gs + (int64_t)subs[b] * len; ++t)
    if ((t + 1) % kStreamWin == 0 || gs + t + 1 == ge) stream[gs + t].w |= kEndWin;
}

cudaError_t launch_pack(const uint4* code, const int64_t* code_off, const int32_t* code_len,
                        const int32_t* lists, const int64_t* pos, const int32_t* counts,
                        const int64_t* base, const int64_t* gstart, int32_t n_programs,
                        const int* subs, const int32_t* inv, uint4* stream, cudaStream_t s) {
  const int nt = 256;
  const int64_t total = (int64_t)kNumVariants * n_programs;
  pack_kernel<<<(unsigned)((total + nt - 1) / nt), nt, 0, s>>>(code, code_off, code_len, lists,
                                                               pos, counts, base, gstart,
                                                               n_programs,
                                                               make_int4(subs[0], subs[1], subs[2],
                                                                         subs[3]),
                                                               inv, stream);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Dataset constants per row chunk (program independent): W = sum w, S_y = sum w (y - K_y),
// S_yy = sum w (y - K_y)^2 over live rows (w != 0), fp64, fixed order. For LogLoss S_y is instead
// W_1 = sum of w over rows with y > 1/2 (the rows the per-row loss scores as positives).
// ---------------------------------------------------------------------------------------------
__global__ void consts_kernel(const float* __restrict__ y, const float* __restrict__ w,
                              int64_t n_rows, int64_t rows_per_chunk, const float* y_shift,
                              double* __restrict__ partial, int64_t ld_part, int64_t col0,
                              int32_t logloss) {
  __shared__ double red[3][256];
  const int q = blockIdx.x, tid = threadIdx.x;
  const int64_t r0 = (int64_t)q * rows_per_chunk, r1 = min(r0 + rows_per_chunk, n_rows);
  const float Ky = y_shift ? *y_shift : 0.0f;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  for (int64_t i = r0 + tid; i < r1; i += 256) {
    const double wi = w ? (double)w[i] : 1.0;
    if (wi != 0.0) {
      const double yc = (double)(y[i] - Ky);
      c0 += wi;
      c1 += logloss ? (y[i] > 0.5f ? wi : 0.0) : wi * yc;
      c2 += wi * yc * yc;
    }
  }
  red[0][tid] = c0; red[1][tid] = c1; red[2][tid] = c2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) for (int k = 0; k < 3; ++k) red[k][tid] += red[k][tid + o];
    __syncthreads();
  }
  if (tid < 3) partial[(int64_t)q * ld_part + col0 + tid] = red[tid][0];
}

cudaError_t launch_consts(const float* y, const float* w, int64_t n_rows, int64_t rows_per_chunk,
                          int64_t n_chunks, const float* y_shift, double* partial, int64_t ld_part,
                          int64_t col0, int32_t logloss, cudaStream_t s) {
  consts_kernel<<<(unsigned)n_chunks, 256, 0, s>>>(y, w, n_rows, rows_per_chunk, y_shift, partial,
                                                    ld_part, col0, logloss);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Pearson shift (C9): K_p = f_p(x_ref), evaluated with the SAME fp32 op code as the
// register-stack evaluator so a constant program gives d = yhat - K_p = 0 exactly on every row.
// ---------------------------------------------------------------------------------------------
__global__ void shift_kernel(const uint4* __restrict__ code, const int64_t* __restrict__ code_off,
                             const int32_t* __restrict__ code_len, int32_t n_programs,
                             const float* __restrict__ xref, int64_t stride,
                             float* __restrict__ shift) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_programs) return;
  const int len = code_len[p];
  if (len == 0) { shift[p] = 0.0f; return; }
  float stk[GP_MAX_STACK + 1];
  const uint4* pc = code + code_off[p];
  auto term = [&](int src, uint32_t pl) {   // 1 variable, 2 constant
    return src == 1 ? xref[(int64_t)pl * stride] : __uint_as_float(pl);
  };
  for (int k = 0; k < len; ++k) {
    const uint4 cw = pc[k];
    const int id = (int)cw.x, opv = id / kCaseStride, slot = id - opv * kCaseStride;
    if (opv < OPV_BIN0) {
      stk[slot] = term(opv == OPV_PUSH_V ? 1 : 2, cw.y);
    } else if (opv < OPV_UN0) {
      const int op = GP_OP_ADD + (opv - OPV_BIN0) / 10, v = (opv - OPV_BIN0) % 10;
      float a, bb;
      switch (v) {
        case BV_SS: a = stk[slot + 1]; bb = stk[slot]; break;
        case BV_SSR: a = stk[slot]; bb = stk[slot + 1]; break;
        case BV_SV: case BV_SC: a = stk[slot]; bb = term(v == BV_SV ? 1 : 2, cw.z); break;
        case BV_VS: case BV_CS: a = term(v == BV_VS ? 1 : 2, cw.y); bb = stk[slot]; break;
        default:
          a = term(v == BV_VV || v == BV_VC ? 1 : 2, cw.y);
          bb = term(v == BV_VV || v == BV_CV ? 1 : 2, cw.z);
      }
      stk[slot] = apply_rt(op, a, bb);
    } else {
      const int op = GP_OP_SIN + (opv - OPV_UN0) / 3, u = (opv - OPV_UN0) % 3;
      const float a = u == UV_S ? stk[slot] : term(u == UV_V ? 1 : 2, cw.y);
      stk[slot] = apply_rt(op, a, 0.0f);
    }
  }
  shift[p] = stk[0];
}

cudaError_t launch_shift(const uint4* code, const int64_t* code_off, const int32_t* code_len,
                         int32_t n_programs, int32_t stack_cap, const float* xref,
                         int64_t xref_stride, float* shift_out, cudaStream_t s) {
  const int nt = 128;
  (void)stack_cap;
  shift_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(code, code_off, code_len, n_programs,
                                                          xref, xref_stride, shift_out);
  return cudaGetLastError();
}

__global__ void copy_scalar_kernel(const float* src, float* dst) { *dst = *src; }
cudaError_t launch_copy_scalar(const float* src, float* dst, cudaStream_t s) {
  copy_scalar_kernel<<<1, 1, 0, s>>>(src, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Cross-work-item reduction: sums[j] = sum over the n_chunks row chunks of
// partial[q][j] for the live columns j < kConstCols + S * (evaluated programs) (count read on the
// device: inv[n + kNumVariants]). CTA = 32 columns x 8 chunk slices: thread (x, y) sums the
// chunks of slice y in ascending q, the 8 slice sums are then added in ascending y. The order is
// fixed for a given n_chunks -> run-to-run deterministic; 32 consecutive columns per warp
// -> 256-byte coalesced rows; 8 independent load streams per column.
// ---------------------------------------------------------------------------------------------
constexpr int kTrCols = 32, kTrSlices = 8;
__global__ void __launch_bounds__(kTrCols * kTrSlices)
    tile_reduce_kernel(const double* __restrict__ partial, int64_t n_chunks, int64_t ld,
                       const int32_t* __restrict__ live, int32_t S, double* __restrict__ sums) {
  __shared__ double part[kTrSlices][kTrCols];
  const int64_t n_live = kConstCols + (int64_t)S * (*live);
  const int64_t j = (int64_t)blockIdx.x * kTrCols + threadIdx.x;
  if ((int64_t)blockIdx.x * kTrCols >= n_live) return;      // whole CTA past the live columns
  const int y = threadIdx.y;
  const int64_t per = (n_chunks + kTrSlices - 1) / kTrSlices;
  const int64_t q0 = y * per, q1 = min(n_chunks, q0 + per);
  double a0 = 0.0, a1 = 0.0;                                   // even / odd chunks of the slice
  if (j < n_live) {
    int64_t q = q0;
    for (; q + 1 < q1; q += 2) {
      a0 += partial[q * ld + j];
      a1 += partial[(q + 1) * ld + j];
    }
    if (q < q1) a0 += partial[q * ld + j];
  }
  part[y][threadIdx.x] = a0 + a1;
  __syncthreads();
  if (y == 0 && j < n_live) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kTrSlices; ++k) t += part[k][threadIdx.x];
    sums[j] = t;
  }
}

cudaError_t launch_tile_reduce(const double* partial, int64_t n_chunks, int64_t ld_part,
                               const int32_t* live, int32_t S, double* sums, cudaStream_t s) {
  const dim3 blk(kTrCols, kTrSlices);
  tile_reduce_kernel<<<(unsigned)((ld_part + kTrCols - 1) / kTrCols), blk, 0, s>>>(
      partial, n_chunks, ld_part, live, S, sums);
  return cudaGetLastError();
}

// Compact (bucket-order) sums -> program order: out[p S + k] = sums of p or 0 if p was not
// evaluated per row; out[n S + c] = dataset constant c. (gp_evaluate_partial's output layout.)
__global__ void expand_sums_kernel(const double* __restrict__ sums, const int32_t* __restrict__ inv,
                                   int32_t n, int32_t S, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nS = (int64_t)n * S;
  if (i < nS) {
    const int p = (int)(i / S), k = (int)(i - (int64_t)p * S);
    const int c = inv[p];
    out[i] = c >= 0 ? sums[kConstCols + (int64_t)c * S + k] : 0.0;
  } else if (i < nS + kConstCols) {
    out[i] = sums[i - nS];
  }
}

cudaError_t launch_expand_sums(const double* sums, const int32_t* inv, int32_t n, int32_t S,
                               double* out, cudaStream_t s) {
  const int64_t total = (int64_t)n * S + kConstCols;
  expand_sums_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(sums, inv, n, S, out);
  return cudaGetLastError();
}

// Row 0 of this rank's shard (X[c * ldx], y[0]) -> dst[0..n_cols] (the Pearson reference row that
// rank 0 broadcasts when the caller did not set one).
__global__ void gather_row_kernel(const float* __restrict__ X, int64_t ldx, int32_t n_cols,
                                  const float* __restrict__ y, float* __restrict__ dst) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_cols) dst[c] = X[(int64_t)c * ldx];
  if (c == n_cols) dst[c] = y[0];
}

cudaError_t launch_gather_row(const float* X, int64_t ldx, int32_t n_cols, const float* y,
                              float* dst, cudaStream_t s) {
  gather_row_kernel<<<(n_cols + 1 + 127) / 128, 128, 0, s>>>(X, ldx, n_cols, y, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Finalize: per-program sums (+ dataset constants W, S_y, S_yy at the end) ->
// raw fitness ("vector containing final raw fitness values"), S:201 normalisation.
// ---------------------------------------------------------------------------------------------
__global__ void finalize_kernel(const double* __restrict__ consts, const double* __restrict__ psums,
                                const int32_t* __restrict__ idx, int32_t n_programs,
                                int32_t metric, const int32_t* __restrict__ code_len,
                                const int32_t* __restrict__ need, const uint4* __restrict__ code,
                                const int64_t* __restrict__ code_off, int32_t closed_const,
                                float* __restrict__ fitness, uint32_t* __restrict__ status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_programs) return;
  const int S = metric == GP_PEARSON ? 3 : 1;
  const double W = consts[0], Sy = consts[1], Syy = consts[2];
  // this program's S sums: compact position idx[p] (-1: not evaluated per row -> zeros), or
  // program order when idx is null
  const int64_t pos = idx ? (int64_t)idx[p] : (int64_t)p;
  const double zero3[3] = {0.0, 0.0, 0.0};
  const double* sums = pos >= 0 ? psums + pos * S : zero3;
  uint32_t fl = status[p];
  float out;
  // closed_const: variable-free programs (need 0) were not evaluated per row; their sums follow
  // from the dataset moments (consts_kernel, K_y = 0 for MSE): sum w (c - y)^2 =
  // W c^2 - 2 c S_y + S_yy, and a constant prediction has an undefined Pearson correlation
  const bool cst = closed_const && code_len[p] > 0 && need[p] == 0;
  if (code_len[p] == 0) {
    out = metric == GP_PEARSON ? -INFINITY : INFINITY;
  } else if (metric != GP_PEARSON) {
    double f;
    if (cst && metric == GP_LOGLOSS) {
      // the per-row loss of a constant prediction c is one of two values: softplus(-c) on rows
      // with y > 1/2 (total weight W_1 = Sy here), softplus(c) on the others, each clamped to
      // the p-clamp's range (C7)
      const double c = (double)__uint_as_float(code[code_off[p]].y);
      auto sp = [](double z) {
        const double l = fmax(z, 0.0) + log1p(exp(-fabs(z)));
        return l < 1.0000000000000005e-15 ? 1.0000000000000005e-15
                                          : (l > 34.538776394910684 ? 34.538776394910684 : l);
      };
      f = isnan(c) ? c : (Sy * sp(-c) + (W - Sy) * sp(c)) / W;
    } else if (cst) {
      const double c = (double)__uint_as_float(code[code_off[p]].y);
      f = (W * c * c - 2.0 * c * Sy + Syy) / W;
      if (f < 0.0) f = 0.0;                        // rounding; NaN / inf pass through
    } else {
      f = sums[0] / W;
    }
    if (metric == GP_RMSE) f = sqrt(f);
    if (!isfinite(f) || f > (double)FLT_MAX) { f = INFINITY; fl |= GP_FLAG_NONFINITE; }
    out = (float)f;
  } else {
    const double Sd = cst ? 0.0 : sums[0], Sdd = cst ? 0.0 : sums[1], Sdy = cst ? 0.0 : sums[2];
    const double cov = Sdy - Sd * Sy / W, vd = Sdd - Sd * Sd / W, vy = Syy - Sy * Sy / W;
    double r = cov / sqrt(vd * vy);
    if (!(vd > 0.0) || !(vy > 0.0) || !isfinite(r)) { r = 0.0; fl |= GP_FLAG_UNDEFINED_CORR; }
    r = r > 1.0 ? 1.0 : (r < -1.0 ? -1.0 : r);
    out = (float)r;
  }
  fitness[p] = out;
  status[p] = fl;
}

cudaError_t launch_finalize(const double* consts, const double* psums, const int32_t* idx,
                            int32_t n_programs, int32_t metric,
                            const int32_t* code_len, const int32_t* need, const uint4* code,
                            const int64_t* code_off, int32_t closed_const, float* fitness,
                            uint32_t* status, cudaStream_t s) {
  const int nt = 128;
  finalize_kernel<<<(n_programs + nt - 1) / nt, nt, 0, s>>>(consts, psums, idx, n_programs, metric, code_len,
                                                             need, code, code_off, closed_const,
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
