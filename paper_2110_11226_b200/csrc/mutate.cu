// mutate.cu -- the host step of gp_generation moved onto the GPU (P:237 keeps mutation
// on the CPU because of warp divergence, P:302-306 / P:586 name the transfer cost of that choice).
//
// One generation's variation, with the population resident in HBM as a flat CSR (gp_node[] +
// int64 offsets), no host round trip:
//   kinds    one thread per child: mutation kind from the child's Philox stream (purpose 1)
//   scan     tournament offsets (exclusive prefix sum of 1 / 2 tournaments per child)
//   select   aux.cu select_kernel (2 n tournaments: tournament t depends on t only, so launching
//            the upper bound and using the first T is identical to launching T)
//   plan     one thread per child: runs the mutation's random decisions (subtree picks, re-hoists,
//            the donor of a subtree mutation) and records the child as a recipe -- a prefix of the
//            parent, a range of a donor, a suffix of the parent -- and its length
//   scan     child offsets (int64)
//   emit     one thread per child: writes the child's nodes (point mutation and generated donors
//            replay the same Philox stream)
//   stats    per program of the new population: opcode histogram of variable-dependent nodes,
//            variable-free nodes / programs, stack need, depth
//   fitstats after the evaluation: best program (ties to the smallest index), mean finite fitness
//
// The random decisions are the host engine's (engine.cpp) in the same order, on the same streams
// (DESIGN.md "Host RNG draw order"): Philox4x32-10, key = seed, counter = (child, generation,
// block, purpose), words in order; randint(n) = (u64(w) n) >> 32; uniform() = (w >> 8) 2^-24 in
// double. Double arithmetic uses explicit round-to-nearest intrinsics so no FMA contraction can
// change a constant or a kind decision: the populations are bit-identical to the host engine's
// and to the oracle's replay (tests/test_gpu_engine.py).
//
// One thread per child: the work per child is a few dozen node reads / writes and is latency
// bound; 8192 children are 64 CTAs -- microseconds, not a throughput concern.
#include <cstdint>
#include "common.h"
#include "mutate.h"

namespace gpb {

namespace {

enum { FULL = 0, GROW = 1 };
enum { K_CROSSOVER = 0, K_SUBTREE = 1, K_HOIST = 2, K_POINT = 3, K_REPRODUCTION = 4 };

struct DevRng {
  uint32_t k0, k1, idx, gen, purpose, block = 0;
  u32x4 buf{};
  int pos = 4;
  __device__ DevRng(uint32_t key0, uint32_t key1, uint32_t index, uint32_t generation,
                    uint32_t purp)
      : k0(key0), k1(key1), idx(index), gen(generation), purpose(purp) {}
  __device__ uint32_t u32() {
    if (pos == 4) {
      buf = philox4x32_10(u32x4{idx, gen, block++, purpose}, k0, k1);
      pos = 0;
    }
    const uint32_t w = pos == 0 ? buf.x : pos == 1 ? buf.y : pos == 2 ? buf.z : buf.w;
    ++pos;
    return w;
  }
  __device__ uint32_t randint(uint32_t n) { return (uint32_t)(((uint64_t)u32() * n) >> 32); }
  __device__ double uniform() { return __dmul_rn((double)(u32() >> 8), 1.0 / 16777216.0); }
};

__device__ __forceinline__ gp_node make_node(int op, int32_t var) {
  gp_node n;
  n.op = op;
  n.var = var;
  return n;
}

// terminal: one draw over n_features + 1 outcomes, then one uniform for a constant
__device__ gp_node terminal(DevRng& r, const MutConfig& c) {
  const uint32_t t = r.randint((uint32_t)c.n_features + 1);
  if ((int)t < c.n_features) return make_node(GP_OP_VAR, (int32_t)t);
  const double lo = (double)c.const_lo, hi = (double)c.const_hi;
  gp_node n;
  n.op = GP_OP_CONST;
  n.value = __double2float_rn(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), r.uniform())));
  return n;
}

// Full / Grow in prefix order, one draw per decision -- the iterative form
// of engine.cpp random_program_rec: rem[d] = children still to generate at depth d.
template <class Emit>
__device__ int gen_program(DevRng& r, int method, int max_depth, const MutConfig& c, Emit emit) {
  int rem[kMaxDepth + 2];
  int level = 0, k = 0;
  rem[0] = 1;
  while (level >= 0) {
    if (rem[level] == 0) { --level; continue; }
    --rem[level];
    int f = -1;
    if (level < max_depth) {
      if (method == FULL) {
        f = c.function_set[r.randint((uint32_t)c.n_functions)];
      } else {
        const uint32_t x = r.randint((uint32_t)(c.n_functions + c.n_features + 1));
        if ((int)x < c.n_functions) f = c.function_set[x];
      }
    }
    if (f >= 0) {
      emit(k++, make_node(f, 0));
      ++level;
      rem[level] = op_arity(f);
    } else {
      emit(k++, terminal(r, c));
    }
  }
  return k;
}

// Arity access to a program held as gp_node[] (population) or as an arity byte array (generated
// donor of a subtree mutation).
struct NodeAcc {
  const gp_node* p;
  __device__ int ar(int64_t k) const { return op_arity(p[k].op); }
};
struct ArityAcc {
  const uint8_t* a;
  __device__ int ar(int64_t k) const { return a[k]; }
};

template <class A>
__device__ int64_t subtree_end(const A& p, int64_t len, int64_t start) {
  int64_t needed = 1, i = start;
  while (needed > 0 && i < len) { needed += p.ar(i) - 1; ++i; }
  return i;
}

// Subtree root: weight 9 for functions, 1 for terminals, integer draw + linear scan.
template <class A>
__device__ void pick_subtree(DevRng& r, const A& p, int64_t base, int64_t len, int64_t* s,
                             int64_t* e) {
  int64_t total = 0;
  for (int64_t i = 0; i < len; ++i) total += p.ar(base + i) > 0 ? 9 : 1;
  const uint32_t x = r.randint((uint32_t)total);
  int64_t c = 0, start = 0;
  for (int64_t i = 0; i < len; ++i) {
    c += p.ar(base + i) > 0 ? 9 : 1;
    if ((int64_t)x < c) { start = i; break; }
  }
  *s = start;
  // end of the subtree at base + start, relative to base
  int64_t needed = 1, i = start;
  while (needed > 0 && i < len) { needed += p.ar(base + i) - 1; ++i; }
  *e = i;
}

// Depth of the tree p[a, b) (a lone terminal has depth 0); *ok = 0 if deeper than
// kMaxDepth (cannot happen for engine populations: depth <= stack_capacity - 1).
template <class A>
__device__ int range_depth(const A& p, int64_t a, int64_t b, int* ok) {
  int open[kMaxDepth + 2];
  int top = 0, depth = 0;
  for (int64_t k = a; k < b; ++k) {
    depth = max(depth, top);
    const int ar = p.ar(k);
    if (ar > 0) {
      if (top > kMaxDepth) { *ok = 0; return depth; }
      open[top++] = ar;
    } else {
      while (top > 0 && --open[top - 1] == 0) --top;
    }
  }
  return depth;
}

// For a splice of the parent at [s, e): the depth of node s and the largest depth of the parent
// nodes outside [s, e) (-1 if none). depth(child) = max(outside, d_s + depth(inserted)).
__device__ void splice_depths(const NodeAcc& p, int64_t len, int64_t s, int64_t e, int* d_s,
                              int* outside, int* ok) {
  int open[kMaxDepth + 2];
  int top = 0, out = -1, ds = 0;
  for (int64_t k = 0; k < len; ++k) {
    if (k == s) ds = top;
    if (k < s || k >= e) out = max(out, top);
    const int ar = p.ar(k);
    if (ar > 0) {
      if (top > kMaxDepth) { *ok = 0; break; }
      open[top++] = ar;
    } else {
      while (top > 0 && --open[top - 1] == 0) --top;
    }
  }
  *d_s = ds;
  *outside = out;
}

// Hoisted crossover: parent subtree [s, e) replaced by the donor subtree [a, b),
// re-hoisted (a random proper subtree of the inserted one) while depth > capacity - 1.
template <class A>
__device__ void hoisted_crossover(DevRng& r, const NodeAcc& par, int64_t plen, const A& don,
                                  int64_t dlen, const MutConfig& c, Recipe* rc, int* ok) {
  int64_t s, e, a, b;
  pick_subtree(r, par, 0, plen, &s, &e);
  pick_subtree(r, don, 0, dlen, &a, &b);
  int d_s, outside;
  splice_depths(par, plen, s, e, &d_s, &outside, ok);
  for (;;) {
    const int depth = max(outside, d_s + range_depth(don, a, b, ok));
    if (!(depth > c.stack_capacity - 1 && b - a > 1)) break;
    const int64_t x = 1 + (int64_t)r.randint((uint32_t)(b - a - 1));
    int64_t needed = 1, i = a + x;                       // end of the subtree at a + x
    while (needed > 0 && i < b) { needed += don.ar(i) - 1; ++i; }
    b = i;
    a = a + x;
  }
  rc->s = (int32_t)s;
  rc->e = (int32_t)e;
  rc->a = (int32_t)a;
  rc->b = (int32_t)b;
  rc->len = (int32_t)(plen - (e - s) + (b - a));
}

}  // namespace

// ---- kinds: mutation kind of each child, cumulative order crossover, subtree, hoist,
// point, else reproduction (C11) ------------------------------------------------------
__global__ void kinds_kernel(int32_t n, uint32_t generation, MutConfig c, int32_t* __restrict__ kinds,
                             int32_t* __restrict__ tcount) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  DevRng r(c.k0, c.k1, (uint32_t)i, generation, 1u);
  const double u = r.uniform();
  double cum = 0.0;
  int kind = K_REPRODUCTION;
  for (int k = 0; k < 4; ++k) {
    cum = __dadd_rn(cum, c.p[k]);
    if (u < cum) { kind = k; break; }
  }
  kinds[i] = kind;
  tcount[i] = kind == K_CROSSOVER ? 2 : 1;
}

// ---- single-CTA exclusive scan (n values -> out[0..n], out[n] = total) -------------------------
template <class In, class Out>
__global__ void __launch_bounds__(1024) scan_kernel(const In* __restrict__ in, int32_t n,
                                                    Out* __restrict__ out) {
  __shared__ Out warp_tot[32];
  __shared__ Out carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += 1024) {
    const int i = c0 + tid;
    const Out v = i < n ? (Out)in[i] : (Out)0;
    Out x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Out y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      Out t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Out y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const Out carry = carry_s;
    if (i < n) out[i] = carry + (warp ? warp_tot[warp - 1] : (Out)0) + x - v;
    __syncthreads();
    if (tid == 0) carry_s = carry + warp_tot[31];
    __syncthreads();
  }
  if (tid == 0) out[n] = carry_s;
}

// ---- plan: the child's recipe and length ------------------------------------------------------
__global__ void plan_kernel(const gp_node* __restrict__ nodes, const int64_t* __restrict__ off,
                            int32_t n, uint32_t generation, MutConfig c,
                            const int32_t* __restrict__ kinds, const int32_t* __restrict__ toff,
                            const int32_t* __restrict__ winners, Recipe* __restrict__ recipes,
                            int32_t* __restrict__ lens, int32_t* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Recipe rc{};
  rc.kind = kinds[i];
  rc.parent = winners[toff[i]];
  rc.donor = rc.kind == K_CROSSOVER ? winners[toff[i] + 1] : -1;
  const int64_t pb = off[rc.parent], plen = off[rc.parent + 1] - pb;
  const NodeAcc par{nodes + pb};
  DevRng r(c.k0, c.k1, (uint32_t)i, generation, 2u);
  int ok = 1;
  rc.len = (int32_t)plen;                      // reproduction, point mutation
  if (rc.kind == K_HOIST) {
    int64_t s, e, s2, e2;
    pick_subtree(r, par, 0, plen, &s, &e);
    pick_subtree(r, par, s, e - s, &s2, &e2);
    rc.s = (int32_t)s;
    rc.e = (int32_t)e;
    rc.a = (int32_t)(s + s2);
    rc.b = (int32_t)(s + e2);
    rc.len = (int32_t)(plen - (e - s) + (e2 - s2));
  } else if (rc.kind == K_CROSSOVER) {
    const int64_t db = off[rc.donor], dlen = off[rc.donor + 1] - db;
    hoisted_crossover(r, par, plen, NodeAcc{nodes + db}, dlen, c, &rc, &ok);
  } else if (rc.kind == K_SUBTREE) {
    // donor: Grow with the init depth range, generated here as arities only; the emit
    // kernel regenerates its nodes from the same stream
    const int md = c.init_depth_min +
                   (int)r.randint((uint32_t)(c.init_depth_max - c.init_depth_min + 1));
    uint8_t ar[kMaxDonorNodes];
    const int dlen = gen_program(r, GROW, md, c, [&](int k, gp_node nd) {
      if (k < kMaxDonorNodes) ar[k] = (uint8_t)op_arity(nd.op);
    });
    if (dlen > kMaxDonorNodes) ok = 0;
    else hoisted_crossover(r, par, plen, ArityAcc{ar}, dlen, c, &rc, &ok);
  }
  if (!ok) atomicOr(err, 1);
  recipes[i] = rc;
  lens[i] = rc.len;
}

// ---- emit: the child's nodes at out + out_off[i] ------------------------------------------------
__global__ void emit_kernel(const gp_node* __restrict__ nodes, const int64_t* __restrict__ off,
                            int32_t n, uint32_t generation, MutConfig c,
                            const Recipe* __restrict__ recipes, const int64_t* __restrict__ out_off,
                            gp_node* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Recipe rc = recipes[i];
  const gp_node* P = nodes + off[rc.parent];
  const int64_t plen = off[rc.parent + 1] - off[rc.parent];
  gp_node* o = out + out_off[i];
  if (rc.kind == K_REPRODUCTION) {
    for (int64_t k = 0; k < plen; ++k) o[k] = P[k];
  } else if (rc.kind == K_POINT) {
    // one uniform per node; replacement: a fresh terminal, or a same-arity function in
    // function-set order (engine.cpp point_mutation)
    DevRng r(c.k0, c.k1, (uint32_t)i, generation, 2u);
    for (int64_t k = 0; k < plen; ++k) {
      gp_node nd = P[k];
      if (r.uniform() < c.p_point_replace) {
        const int a = op_arity(nd.op);
        if (a == 0) {
          nd = terminal(r, c);
        } else {
          int nc = 0;
          for (int q = 0; q < c.n_functions; ++q) nc += op_arity(c.function_set[q]) == a;
          if (nc) {
            int pick = (int)r.randint((uint32_t)nc);
            for (int q = 0; q < c.n_functions; ++q) {
              if (op_arity(c.function_set[q]) != a) continue;
              if (pick-- == 0) { nd = make_node(c.function_set[q], 0); break; }
            }
          }
        }
      }
      o[k] = nd;
    }
  } else {
    // prefix [0, s) + inserted range + suffix [e, plen)
    int64_t w = 0;
    for (int64_t k = 0; k < rc.s; ++k) o[w++] = P[k];
    if (rc.kind == K_HOIST) {
      for (int64_t k = rc.a; k < rc.b; ++k) o[w++] = P[k];
    } else if (rc.kind == K_CROSSOVER) {
      const gp_node* D = nodes + off[rc.donor];
      for (int64_t k = rc.a; k < rc.b; ++k) o[w++] = D[k];
    } else {                                   // K_SUBTREE: regenerate the donor's range
      DevRng r(c.k0, c.k1, (uint32_t)i, generation, 2u);
      const int md = c.init_depth_min +
                     (int)r.randint((uint32_t)(c.init_depth_max - c.init_depth_min + 1));
      gp_node* ins = o + w;
      const int a = rc.a, b = rc.b;
      gen_program(r, GROW, md, c, [&](int k, gp_node nd) {
        if (k >= a && k < b) ins[k - a] = nd;
      });
      w += b - a;
    }
    for (int64_t k = rc.e; k < plen; ++k) o[w++] = P[k];
  }
}

// ---- initial population: ramped half-and-half ------------------
// Program i: Full iff i < n / 2, max depth d_min + i mod (d_max - d_min + 1), its own Philox stream
// (purpose 3, generation 0). Two passes over the same stream: the length, then the nodes.
__global__ void init_len_kernel(int32_t n, MutConfig c, int32_t* __restrict__ lens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  DevRng r(c.k0, c.k1, (uint32_t)i, 0u, 3u);
  const int method = i < n / 2 ? FULL : GROW;
  const int md = c.init_depth_min + i % (c.init_depth_max - c.init_depth_min + 1);
  lens[i] = gen_program(r, method, md, c, [](int, gp_node) {});
}

__global__ void init_emit_kernel(int32_t n, MutConfig c, const int64_t* __restrict__ off,
                                 gp_node* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  DevRng r(c.k0, c.k1, (uint32_t)i, 0u, 3u);
  const int method = i < n / 2 ? FULL : GROW;
  const int md = c.init_depth_min + i % (c.init_depth_max - c.init_depth_min + 1);
  gp_node* o = out + off[i];
  gen_program(r, method, md, c, [&](int k, gp_node nd) { o[k] = nd; });
}

// ---- stats of a population (engine.cpp evaluate(): histogram of variable-dependent nodes) -------
__global__ void pop_stats_kernel(const gp_node* __restrict__ nodes, const int64_t* __restrict__ off,
                                 int32_t n, int32_t* __restrict__ depth_out, DevGenStats* st) {
  __shared__ unsigned long long h[GP_OP_COUNT + 2];
  __shared__ int s_need;
  const int tid = threadIdx.x;
  for (int k = tid; k < GP_OP_COUNT + 2; k += blockDim.x) h[k] = 0ull;
  if (tid == 0) s_need = 0;
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + tid;
  if (p < n) {
    const int64_t b = off[p], len = off[p + 1] - b;
    // reverse-prefix walk: a bit stack of "variable-free" flags; occupancy = stack need
    uint64_t cst = 0;                 // bit j = flag of stack entry j (entry 0 at the bottom)
    int sp = 0, need = 0;
    bool ok = true;
    for (int64_t k = len - 1; k >= 0; --k) {
      const int op = nodes[b + k].op;
      const int a = op_arity(op);
      bool c = op == GP_OP_CONST;
      if (a > 0) {
        c = true;
        for (int j = 0; j < a && sp > 0; ++j) { --sp; c = c && ((cst >> sp) & 1ull); }
      }
      if (sp >= 64) { ok = false; break; }
      cst = (cst & ~(1ull << sp)) | ((uint64_t)c << sp);
      ++sp;
      need = max(need, sp);
      if (c) atomicAdd(&h[GP_OP_COUNT], 1ull);
      else if (op >= 0 && op < GP_OP_COUNT) atomicAdd(&h[op], 1ull);
    }
    if (ok && len > 0 && (cst & 1ull)) atomicAdd(&h[GP_OP_COUNT + 1], 1ull);
    atomicMax(&s_need, need);
    int okd = 1;
    depth_out[p] = range_depth(NodeAcc{nodes + b}, 0, len, &okd);
  }
  __syncthreads();
  for (int k = tid; k < GP_OP_COUNT; k += blockDim.x)
    if (h[k]) atomicAdd((unsigned long long*)&st->op_count[k], h[k]);
  if (tid == 0) {
    if (h[GP_OP_COUNT]) atomicAdd((unsigned long long*)&st->const_nodes, h[GP_OP_COUNT]);
    if (h[GP_OP_COUNT + 1]) atomicAdd((unsigned long long*)&st->const_programs, h[GP_OP_COUNT + 1]);
    atomicMax(&st->max_need, s_need);
  }
}

// ---- fitness stats (engine.cpp fill_stats): best (first index among equals, NaN skipped), mean
// of the finite values in a fixed order ----------------------------------------------------------
__global__ void __launch_bounds__(1024) fit_stats_kernel(const float* __restrict__ fit, int32_t n,
                                                         int32_t higher,
                                                         const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ depth,
                                                         DevGenStats* st) {
  __shared__ double ssum[1024];
  __shared__ int scnt[1024], sbest[1024];
  const int tid = threadIdx.x;
  double sum = 0.0;
  int cnt = 0, best = -1;
  const int per = (n + 1023) / 1024;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  for (int i = lo; i < hi; ++i) {
    const float f = fit[i];
    if (isfinite(f)) { sum += (double)f; ++cnt; }
    if (isnan(f)) continue;
    if (best < 0 || (higher ? f > fit[best] : f < fit[best])) best = i;
  }
  ssum[tid] = sum;
  scnt[tid] = cnt;
  sbest[tid] = best;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) {
      ssum[tid] += ssum[tid + o];
      scnt[tid] += scnt[tid + o];
      // strided partners: the ranges interleave, so equal values go to the smaller index
      const int a = sbest[tid], b = sbest[tid + o];
      if (a < 0 || (b >= 0 && ((higher ? fit[b] > fit[a] : fit[b] < fit[a]) ||
                               (fit[b] == fit[a] && b < a))))
        sbest[tid] = b;
    }
    __syncthreads();
  }
  if (tid == 0) {
    st->mean = scnt[0] ? ssum[0] / scnt[0] : __longlong_as_double(0x7ff8000000000000ll);
    st->best = sbest[0];
    st->best_raw = sbest[0] >= 0 ? fit[sbest[0]] : __int_as_float(0x7fc00000);
    st->best_len = sbest[0] >= 0 ? (int32_t)(off[sbest[0] + 1] - off[sbest[0]]) : 0;
    st->best_depth = sbest[0] >= 0 ? depth[sbest[0]] : 0;
  }
}

// ---- launchers ---------------------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_kinds(int32_t n, uint32_t generation, const MutConfig& c, int32_t* kinds,
                         int32_t* tcount, int32_t* toff, cudaStream_t s) {
  kinds_kernel<<<nblk(n, 128), 128, 0, s>>>(n, generation, c, kinds, tcount);
  scan_kernel<int32_t, int32_t><<<1, 1024, 0, s>>>(tcount, n, toff);
  return cudaGetLastError();
}

cudaError_t launch_plan(const gp_node* nodes, const int64_t* off, int32_t n, uint32_t generation,
                        const MutConfig& c, const int32_t* kinds, const int32_t* toff,
                        const int32_t* winners, Recipe* recipes, int32_t* lens, int64_t* out_off,
                        int32_t* err, cudaStream_t s) {
  plan_kernel<<<nblk(n, 64), 64, 0, s>>>(nodes, off, n, generation, c, kinds, toff, winners,
                                         recipes, lens, err);
  scan_kernel<int32_t, int64_t><<<1, 1024, 0, s>>>(lens, n, out_off);
  return cudaGetLastError();
}

cudaError_t launch_emit(const gp_node* nodes, const int64_t* off, int32_t n, uint32_t generation,
                        const MutConfig& c, const Recipe* recipes, const int64_t* out_off,
                        gp_node* out, cudaStream_t s) {
  emit_kernel<<<nblk(n, 64), 64, 0, s>>>(nodes, off, n, generation, c, recipes, out_off, out);
  return cudaGetLastError();
}

cudaError_t launch_init_lengths(int32_t n, const MutConfig& c, int32_t* lens, int64_t* off,
                                cudaStream_t s) {
  init_len_kernel<<<nblk(n, 64), 64, 0, s>>>(n, c, lens);
  scan_kernel<int32_t, int64_t><<<1, 1024, 0, s>>>(lens, n, off);
  return cudaGetLastError();
}

cudaError_t launch_init_emit(int32_t n, const MutConfig& c, const int64_t* off, gp_node* out,
                             cudaStream_t s) {
  init_emit_kernel<<<nblk(n, 64), 64, 0, s>>>(n, c, off, out);
  return cudaGetLastError();
}

cudaError_t launch_pop_stats(const gp_node* nodes, const int64_t* off, int32_t n, int32_t* depth,
                             DevGenStats* st, cudaStream_t s) {
  pop_stats_kernel<<<nblk(n, 128), 128, 0, s>>>(nodes, off, n, depth, st);
  return cudaGetLastError();
}

cudaError_t launch_fit_stats(const float* fit, int32_t n, int32_t higher, const int64_t* off,
                             const int32_t* depth, DevGenStats* st, cudaStream_t s) {
  fit_stats_kernel<<<1, 1024, 0, s>>>(fit, n, higher, off, depth, st);
  return cudaGetLastError();
}

}  // namespace gpb
