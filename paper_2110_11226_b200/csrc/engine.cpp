// engine.cpp -- host engine of the generational GP loop (Alg. 1).
//
// Selection and evaluation run on the GPU (gp_tournament_select / gp_evaluate); mutation runs on
// the host, parallel over children with one counter-based Philox stream per child,
// so the result is independent of the thread count. The population lives as one flat CSR
// (gp_node[] + int64 offsets) in pinned host memory and is copied to HBM with ONE copy per
// generation (the paper's future work, instead of per-program copies).
//
// Random draw order, identical on every rank:
//   stream(index, generation, purpose) = Philox4x32-10, key = seed, counter = (index, generation,
//   block, purpose), block = 0, 1, 2, ..., words used in order;
//   randint(n) = (u64(word) * n) >> 32;  uniform() = (word >> 8) * 2^-24.
//   purpose 1: mutation kind of child i;  purpose 2: mutation internals of child i;
//   purpose 3: initial program i;  purpose 0: tournaments (device kernel).
#include <algorithm>
#include <array>
#include <chrono>
#include <mutex>
#include <memory>
#include <functional>
#include <condition_variable>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "common.h"
#include "gp_internal.h"
#include "mutate.h"

using namespace gpb;

namespace {

using Prog = std::vector<gp_node>;
enum { FULL = 0, GROW = 1 };
enum { K_CROSSOVER = 0, K_SUBTREE = 1, K_HOIST = 2, K_POINT = 3, K_REPRODUCTION = 4 };

struct Rng {
  uint32_t k0, k1, idx, gen, purpose, block = 0;
  u32x4 buf{};
  int pos = 4;
  Rng(uint64_t seed, uint32_t index, uint32_t generation, uint32_t purp)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), idx(index), gen(generation), purpose(purp) {}
  uint32_t u32() {
    if (pos == 4) {
      buf = philox4x32_10(u32x4{idx, gen, block++, purpose}, k0, k1);
      pos = 0;
    }
    const uint32_t w[4] = {buf.x, buf.y, buf.z, buf.w};
    return w[pos++];
  }
  uint32_t randint(uint32_t n) { return (uint32_t)(((uint64_t)u32() * n) >> 32); }
  double uniform() { return (double)(u32() >> 8) * (1.0 / 16777216.0); }
};

inline int arity(int op) { return op_arity(op); }

int64_t subtree_end(const gp_node* p, int64_t len, int64_t start) {
  int64_t needed = 1, i = start;
  while (needed > 0 && i < len) { needed += arity(p[i].op) - 1; ++i; }
  return i;
}

// depth and stack need (max occupancy of the reverse-prefix walk) in one pass
void shape(const Prog& p, int* depth_out, int* need_out) {
  // depth: explicit stack of (remaining children) per open function
  int depth = 0;
  std::vector<int> open;  // remaining operands per open node
  open.reserve(32);
  for (const gp_node& n : p) {
    const int d = (int)open.size();
    depth = std::max(depth, d);
    const int a = arity(n.op);
    if (a > 0) {
      open.push_back(a);
    } else {
      while (!open.empty() && --open.back() == 0) open.pop_back();
    }
  }
  int sp = 0, need = 0;
  for (auto it = p.rbegin(); it != p.rend(); ++it) {
    sp += 1 - arity(it->op);
    need = std::max(need, sp);
  }
  *depth_out = depth;
  *need_out = need;
}
int depth_of(const Prog& p) {
  int d, n;
  shape(p, &d, &n);
  return d;
}

gp_node make_node(int op, int var) {
  gp_node n;
  n.op = op;
  n.var = var;
  return n;
}

gp_node terminal(Rng& st, const gp_config& c, int n_features) {
  const uint32_t t = st.randint((uint32_t)n_features + 1);
  if ((int)t < n_features) return make_node(GP_OP_VAR, (int)t);
  gp_node n;
  n.op = GP_OP_CONST;
  n.value = (float)((double)c.const_lo + ((double)c.const_hi - (double)c.const_lo) * st.uniform());
  return n;
}

// Full / Grow, prefix order, one draw per decision.
void random_program_rec(Rng& st, int method, int max_depth, int d, const gp_config& c,
                        int n_features, Prog& out) {
  const int nF = c.n_functions;
  if (d < max_depth) {
    int f = -1;
    if (method == FULL) {
      f = c.function_set[st.randint((uint32_t)nF)];
    } else {
      const uint32_t r = st.randint((uint32_t)(nF + n_features + 1));
      if ((int)r < nF) f = c.function_set[r];
    }
    if (f >= 0) {
      out.push_back(make_node(f, 0));
      for (int k = 0; k < arity(f); ++k) random_program_rec(st, method, max_depth, d + 1, c, n_features, out);
      return;
    }
  }
  out.push_back(terminal(st, c, n_features));
}
Prog random_program(Rng& st, int method, int max_depth, const gp_config& c, int n_features) {
  Prog p;
  random_program_rec(st, method, max_depth, 0, c, n_features, p);
  return p;
}

// Subtree root: weight 9 for functions, 1 for terminals, integer draw + linear scan.
std::pair<int64_t, int64_t> pick_subtree(Rng& st, const gp_node* p, int64_t len) {
  int64_t total = 0;
  for (int64_t i = 0; i < len; ++i) total += arity(p[i].op) > 0 ? 9 : 1;
  const uint32_t r = st.randint((uint32_t)total);
  int64_t c = 0, start = 0;
  for (int64_t i = 0; i < len; ++i) {
    c += arity(p[i].op) > 0 ? 9 : 1;
    if ((int64_t)r < c) { start = i; break; }
  }
  return {start, subtree_end(p, len, start)};
}

Prog splice(const Prog& parent, int64_t s, int64_t e, const gp_node* ins, int64_t ins_len) {
  Prog child;
  child.reserve(parent.size() - (e - s) + ins_len);
  child.insert(child.end(), parent.begin(), parent.begin() + s);
  child.insert(child.end(), ins, ins + ins_len);
  child.insert(child.end(), parent.begin() + e, parent.end());
  return child;
}

Prog point_mutation(Rng& st, const Prog& parent, const gp_config& c, int n_features) {
  Prog child = parent;
  for (gp_node& n : child) {
    if (st.uniform() < c.p_point_replace) {
      const int a = arity(n.op);
      if (a == 0) {
        n = terminal(st, c, n_features);
      } else {
        int cands[32], nc = 0;
        for (int k = 0; k < c.n_functions; ++k)
          if (arity(c.function_set[k]) == a) cands[nc++] = c.function_set[k];
        if (nc) n = make_node(cands[st.randint((uint32_t)nc)], 0);
      }
    }
  }
  return child;
}

Prog hoist_mutation(Rng& st, const Prog& parent) {
  auto [s, e] = pick_subtree(st, parent.data(), (int64_t)parent.size());
  auto [s2, e2] = pick_subtree(st, parent.data() + s, e - s);
  return splice(parent, s, e, parent.data() + s + s2, e2 - s2);
}

// Hoisted crossover: re-hoist the inserted donor subtree until depth <= cap - 1.
Prog hoisted_crossover(Rng& st, const Prog& parent, const Prog& donor, const gp_config& c) {
  auto [s, e] = pick_subtree(st, parent.data(), (int64_t)parent.size());
  auto [ds, de] = pick_subtree(st, donor.data(), (int64_t)donor.size());
  Prog ins(donor.begin() + ds, donor.begin() + de);
  Prog child = splice(parent, s, e, ins.data(), (int64_t)ins.size());
  while (depth_of(child) > c.stack_capacity - 1 && ins.size() > 1) {
    const int64_t r = 1 + (int64_t)st.randint((uint32_t)(ins.size() - 1));
    const int64_t re = subtree_end(ins.data(), (int64_t)ins.size(), r);
    ins = Prog(ins.begin() + r, ins.begin() + re);
    child = splice(parent, s, e, ins.data(), (int64_t)ins.size());
  }
  return child;
}

Prog subtree_mutation(Rng& st, const Prog& parent, const gp_config& c, int n_features) {
  const int md = c.init_depth_min + (int)st.randint((uint32_t)(c.init_depth_max - c.init_depth_min + 1));
  Prog donor = random_program(st, GROW, md, c, n_features);
  return hoisted_crossover(st, parent, donor, c);
}

// Persistent worker pool for the host steps of a generation (kinds, mutations, flattening): the
// workers are created once per engine, so a generation pays a wake-up, not thread creation.
// Work split is static (contiguous index ranges), so results never depend on scheduling.
class Pool {
 public:
  explicit Pool(int n) {
    for (int t = 1; t < n; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++epoch_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return (int)workers_.size() + 1; }
  // runs body(t) for t in [0, parts) on the caller + workers, returns when all are done
  void run(int parts, const std::function<void(int)>& body) {
    {
      std::lock_guard<std::mutex> g(m_);
      body_ = &body;
      parts_ = parts;
      pending_ = (int)workers_.size();
      ++epoch_;
    }
    cv_.notify_all();
    if (parts > 0) body(0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* body;
      int parts;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return epoch_ != seen; });
        seen = epoch_;
        if (stop_) return;
        body = body_;
        parts = parts_;
      }
      if (t < parts) (*body)(t);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* body_ = nullptr;
  int parts_ = 0, pending_ = 0;
  uint64_t epoch_ = 0;
  bool stop_ = false;
};

template <class F>
void parallel_for(Pool* pool, int n, F&& f) {
  const int threads = pool ? std::min(pool->size(), (n + 31) / 32) : 1;
  if (threads <= 1 || n < 64) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  pool->run(threads, [&](int t) {
    const int b = (int)((int64_t)n * t / threads), e = (int)((int64_t)n * (t + 1) / threads);
    for (int i = b; i < e; ++i) f(i);
  });
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct gp_engine {
  gp_context* ctx = nullptr;
  gp_config cfg{};
  bool higher = false;
  int threads = 1;
  std::unique_ptr<Pool> pool;    // host worker pool (threads - 1 workers + the caller)
  // dataset (device views; owned copies when the caller passed host memory)
  const float *X = nullptr, *y = nullptr, *w = nullptr;
  int64_t ldx = 0, n_rows = 0;
  int32_t n_cols = 0;
  void *own_X = nullptr, *own_y = nullptr, *own_w = nullptr;
  size_t own_X_bytes = 0, own_rows = 0;
  // population
  std::vector<Prog> pop;
  std::vector<float> fit;
  int generation = -1;
  int max_need = 1;
  int64_t op_count[GP_OP_COUNT] = {};
  int64_t const_nodes = 0;
  int64_t const_programs = 0;
  // flat CSR (pinned host) and its device copy
  gp_node* h_nodes = nullptr;
  int64_t* h_off = nullptr;
  size_t h_nodes_cap = 0, h_off_cap = 0;
  StageBuf d_nodes, d_off, d_fit, d_win, d_status;
  int64_t n_nodes = 0;
  std::vector<int32_t> kinds, winners;
  // device mutation (mutate.cu): the population lives in d_nodes / d_off; the next
  // generation is built in d_nodes2 / d_off2 and swapped in
  bool dev_mut = false;
  bool host_view_valid = true;   // h_nodes / h_off / fit mirror the current population
  int32_t last_T = 0;            // tournaments of the last generation (device path)
  bool sel_valid = false;        // d_kinds / d_win hold the last generation's selection
  StageBuf d_nodes2, d_off2, d_kinds, d_tcnt, d_toff, d_recipe, d_len, d_depth, d_stats;
  DevGenStats* h_stats = nullptr;  // pinned
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  ~gp_engine() {
    if (h_nodes) cudaFreeHost(h_nodes);
    if (h_off) cudaFreeHost(h_off);
    if (h_stats) cudaFreeHost(h_stats);
    for (cudaEvent_t x : ev)
      if (x) cudaEventDestroy(x);
    for (StageBuf* b : {&d_nodes, &d_off, &d_fit, &d_win, &d_status, &d_nodes2, &d_off2, &d_kinds,
                        &d_tcnt, &d_toff, &d_recipe, &d_len, &d_depth, &d_stats})
      if (b->p) cudaFree(b->p);
    if (own_X) cudaFree(own_X);
    if (own_y) cudaFree(own_y);
    if (own_w) cudaFree(own_w);
  }

  gp_status set_dataset(const float* X_, int64_t ldx_, const float* y_, const float* w_,
                        int64_t n_rows_, int32_t n_cols_) {
    if (!X_ || !y_ || n_rows_ < 1 || n_cols_ < 1 || ldx_ < n_rows_)
      return ctx->fail(GP_ERR_ARG, "engine dataset: invalid arguments");
    n_rows = n_rows_;
    n_cols = n_cols_;
    cudaStream_t s = ctx->stream;
    gp_status st;
    if (is_host_pointer(X_)) {
      const size_t bytes = (size_t)n_rows * n_cols * sizeof(float);
      if (own_X_bytes != bytes) {
        if (own_X) cudaFree(own_X);
        own_X = nullptr;
        if ((st = ctx->cuda(cudaMalloc(&own_X, bytes), "engine X"))) return st;
        own_X_bytes = bytes;
      }
      if ((st = ctx->cuda(cudaMemcpy2DAsync(own_X, (size_t)n_rows * sizeof(float), X_, (size_t)ldx_ * sizeof(float),
                                            (size_t)n_rows * sizeof(float), (size_t)n_cols,
                                            cudaMemcpyHostToDevice, s), "engine X H2D"))) return st;
      X = (const float*)own_X;
      ldx = n_rows;
    } else {
      X = X_;
      ldx = ldx_;
    }
    auto vec = [&](const float* src, void** own, const float** dst) -> gp_status {
      if (!src) { *dst = nullptr; return GP_OK; }
      if (!is_host_pointer(src)) { *dst = src; return GP_OK; }
      if (!*own || own_rows != (size_t)n_rows) {
        if (*own) cudaFree(*own);
        *own = nullptr;
        gp_status e = ctx->cuda(cudaMalloc(own, (size_t)n_rows * sizeof(float)), "engine vec");
        if (e) return e;
      }
      *dst = (const float*)*own;
      return ctx->cuda(cudaMemcpyAsync(*own, src, (size_t)n_rows * sizeof(float),
                                       cudaMemcpyHostToDevice, s), "engine vec H2D");
    };
    if ((st = vec(y_, &own_y, &y))) return st;
    if ((st = vec(w_, &own_w, &w))) return st;
    own_rows = (size_t)n_rows;
    return GP_OK;
  }

  // Flatten pop into pinned CSR, copy to HBM (one copy each for nodes and offsets), evaluate,
  // read back fitness.
  gp_status evaluate(gp_generation_stats* stats, const float* given_fitness = nullptr) {
    const int n = (int)pop.size();
    double t0 = now_s();
    int64_t total = 0;
    std::vector<int> needs(n);
    for (int i = 0; i < n; ++i) total += (int64_t)pop[i].size();
    if ((size_t)total > h_nodes_cap) {
      if (h_nodes) cudaFreeHost(h_nodes);
      h_nodes_cap = (size_t)total + total / 2 + 1024;
      if (cudaMallocHost(&h_nodes, h_nodes_cap * sizeof(gp_node)) != cudaSuccess) return ctx->fail(GP_ERR_OOM, "pinned nodes");
    }
    if ((size_t)n + 1 > h_off_cap) {
      if (h_off) cudaFreeHost(h_off);
      h_off_cap = (size_t)n + 1;
      if (cudaMallocHost(&h_off, h_off_cap * sizeof(int64_t)) != cudaSuccess) return ctx->fail(GP_ERR_OOM, "pinned offsets");
    }
    h_off[0] = 0;
    for (int i = 0; i < n; ++i) h_off[i + 1] = h_off[i] + (int64_t)pop[i].size();
    // per program (parallel): flatten into the pinned CSR, stack need, and the opcode histogram of
    // variable-dependent nodes (per-row work; variable-free subtrees are per-program constants)
    std::vector<std::array<int32_t, GP_OP_COUNT + 2>> hist(n);  // [ops..., const nodes, const prog]
    parallel_for(pool.get(), n, [&](int i) {
      const Prog& pr = pop[i];
      std::memcpy(h_nodes + h_off[i], pr.data(), pr.size() * sizeof(gp_node));
      int d;
      shape(pr, &d, &needs[i]);
      auto& h = hist[i];
      h.fill(0);
      std::vector<char> is_const(pr.size(), 0);
      std::vector<int64_t> kids;  // reverse-prefix stack of child indices
      kids.reserve(pr.size());
      for (int64_t k = (int64_t)pr.size() - 1; k >= 0; --k) {
        const int op = pr[k].op;
        const int ar = arity(op);
        bool c = op == GP_OP_CONST;
        if (ar > 0) {
          c = true;
          for (int j = 0; j < ar; ++j) { c = c && is_const[kids.back()]; kids.pop_back(); }
        }
        is_const[k] = c;
        kids.push_back(k);
        if (c) ++h[GP_OP_COUNT];
        else if (op >= 0 && op < GP_OP_COUNT) ++h[op];
      }
      h[GP_OP_COUNT + 1] = !pr.empty() && is_const[0];
    });
    max_need = 1;
    for (int v : needs) max_need = std::max(max_need, v);
    std::fill(op_count, op_count + GP_OP_COUNT, (int64_t)0);
    const_nodes = 0;
    const_programs = 0;
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < GP_OP_COUNT; ++k) op_count[k] += hist[i][k];
      const_nodes += hist[i][GP_OP_COUNT];
      const_programs += hist[i][GP_OP_COUNT + 1];
    }
    n_nodes = total;
    gp_status s;
    if ((s = ctx->grow(&d_nodes.p, &d_nodes.cap, (size_t)total * sizeof(gp_node), "d_nodes"))) return s;
    if ((s = ctx->grow(&d_off.p, &d_off.cap, (size_t)(n + 1) * sizeof(int64_t), "d_off"))) return s;
    if ((s = ctx->grow(&d_fit.p, &d_fit.cap, (size_t)n * sizeof(float), "d_fit"))) return s;
    if ((s = ctx->grow(&d_status.p, &d_status.cap, (size_t)n * sizeof(uint32_t), "d_status"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(d_nodes.p, h_nodes, (size_t)total * sizeof(gp_node), cudaMemcpyHostToDevice, ctx->stream), "H2D nodes"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(d_off.p, h_off, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream), "H2D offsets"))) return s;
    double t1 = now_s();
    host_view_valid = true;
    if (given_fitness) {                 // gp_engine_set_population with known fitness
      s = ctx->cuda(cudaMemcpyAsync(d_fit.p, given_fitness, (size_t)n * sizeof(float),
                                    cudaMemcpyDefault, ctx->stream), "fitness copy");
    } else {
      s = gp_evaluate(ctx, (const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n, total,
                      std::min(max_need, GP_MAX_STACK), X, ldx, y, w, n_rows, n_cols,
                      (gp_metric)cfg.metric, (float*)d_fit.p, (uint32_t*)d_status.p);
    }
    if (s) return s;
    fit.resize(n);
    if ((s = ctx->cuda(cudaMemcpyAsync(fit.data(), d_fit.p, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream), "D2H fitness"))) return s;
    if ((s = ctx->cuda(cudaStreamSynchronize(ctx->stream), "evaluate sync"))) return s;
    double t2 = now_s();
    if (stats) {
      stats->t_h2d_s += t1 - t0;
      stats->t_eval_s += t2 - t1;
    }
    return GP_OK;
  }

  MutConfig mut_config() const {
    MutConfig m{};
    m.k0 = (uint32_t)cfg.seed;
    m.k1 = (uint32_t)(cfg.seed >> 32);
    m.n_features = n_cols;
    m.n_functions = cfg.n_functions;
    for (int i = 0; i < 32; ++i) m.function_set[i] = cfg.function_set[i];
    m.const_lo = cfg.const_lo;
    m.const_hi = cfg.const_hi;
    m.p[0] = cfg.p_crossover;
    m.p[1] = cfg.p_subtree;
    m.p[2] = cfg.p_hoist;
    m.p[3] = cfg.p_point;
    m.p_point_replace = cfg.p_point_replace;
    m.init_depth_min = cfg.init_depth_min;
    m.init_depth_max = cfg.init_depth_max;
    m.stack_capacity = cfg.stack_capacity;
    return m;
  }

  gp_status dev_buffers(int n) {
    gp_status s;
    if ((s = ctx->grow(&d_kinds.p, &d_kinds.cap, (size_t)n * 4, "kinds"))) return s;
    if ((s = ctx->grow(&d_tcnt.p, &d_tcnt.cap, (size_t)n * 4, "tcount"))) return s;
    if ((s = ctx->grow(&d_toff.p, &d_toff.cap, (size_t)(n + 1) * 4, "toff"))) return s;
    if ((s = ctx->grow(&d_win.p, &d_win.cap, (size_t)2 * n * 4, "winners"))) return s;
    if ((s = ctx->grow(&d_recipe.p, &d_recipe.cap, (size_t)n * sizeof(Recipe), "recipes"))) return s;
    if ((s = ctx->grow(&d_len.p, &d_len.cap, (size_t)n * 4, "lens"))) return s;
    if ((s = ctx->grow(&d_off2.p, &d_off2.cap, (size_t)(n + 1) * 8, "off2"))) return s;
    if ((s = ctx->grow(&d_depth.p, &d_depth.cap, (size_t)n * 4, "depth"))) return s;
    if ((s = ctx->grow(&d_stats.p, &d_stats.cap, sizeof(DevGenStats), "stats"))) return s;
    if (!h_stats && cudaMallocHost(&h_stats, sizeof(DevGenStats)) != cudaSuccess)
      return ctx->fail(GP_ERR_OOM, "pinned stats");
    for (cudaEvent_t& x : ev)
      if (!x && cudaEventCreate(&x) != cudaSuccess) return ctx->fail(GP_ERR_CUDA, "event");
    return GP_OK;
  }

  // Statistics of the device population + fitness (pop_stats, fit_stats) -> h_stats [sync].
  gp_status dev_stats(int n) {
    gp_status s;
    DevGenStats* ds = (DevGenStats*)d_stats.p;
    if ((s = ctx->cuda(cudaMemsetAsync(ds, 0, sizeof(DevGenStats), ctx->stream), "stats memset"))) return s;
    if ((s = ctx->launch(launch_pop_stats((const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n,
                                          (int32_t*)d_depth.p, ds, ctx->stream), "pop stats"))) return s;
    if ((s = ctx->launch(launch_fit_stats((const float*)d_fit.p, n, higher ? 1 : 0,
                                          (const int64_t*)d_off.p, (const int32_t*)d_depth.p, ds,
                                          ctx->stream), "fit stats"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(h_stats, ds, sizeof(DevGenStats), cudaMemcpyDeviceToHost, ctx->stream), "D2H stats"))) return s;
    return ctx->cuda(cudaStreamSynchronize(ctx->stream), "stats sync");
  }

  void fill_stats_dev(gp_generation_stats* st) {
    const DevGenStats& d = *h_stats;
    st->generation = generation;
    st->best_index = d.best;
    st->mean_raw = d.mean;
    st->total_nodes = n_nodes;
    max_need = std::max(1, d.max_need);
    st->max_stack_need = max_need;
    std::copy(d.op_count, d.op_count + GP_OP_COUNT, st->op_count);
    std::copy(d.op_count, d.op_count + GP_OP_COUNT, op_count);
    st->const_nodes = const_nodes = d.const_nodes;
    st->const_programs = const_programs = d.const_programs;
    if (d.best >= 0) {
      const float pen = cfg.parsimony * (float)d.best_len;
      st->best_raw = d.best_raw;
      st->best_adjusted = higher ? d.best_raw - pen : d.best_raw + pen;
      st->best_len = d.best_len;
      st->best_depth = d.best_depth;
    } else {
      st->best_raw = st->best_adjusted = NAN;
      st->best_len = st->best_depth = 0;
    }
  }

  // Copies the device population + fitness into the pinned host mirror (host views) [sync].
  gp_status sync_host_view() {
    if (host_view_valid) return GP_OK;
    const int n = cfg.population_size;
    if ((size_t)n_nodes > h_nodes_cap) {
      if (h_nodes) cudaFreeHost(h_nodes);
      h_nodes_cap = (size_t)n_nodes + n_nodes / 2 + 1024;
      if (cudaMallocHost(&h_nodes, h_nodes_cap * sizeof(gp_node)) != cudaSuccess) return ctx->fail(GP_ERR_OOM, "pinned nodes");
    }
    if ((size_t)n + 1 > h_off_cap) {
      if (h_off) cudaFreeHost(h_off);
      h_off_cap = (size_t)n + 1;
      if (cudaMallocHost(&h_off, h_off_cap * sizeof(int64_t)) != cudaSuccess) return ctx->fail(GP_ERR_OOM, "pinned offsets");
    }
    fit.resize(n);
    gp_status s;
    if ((s = ctx->cuda(cudaMemcpyAsync(h_nodes, d_nodes.p, (size_t)n_nodes * sizeof(gp_node), cudaMemcpyDeviceToHost, ctx->stream), "D2H nodes"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(h_off, d_off.p, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream), "D2H offsets"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(fit.data(), d_fit.p, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream), "D2H fitness"))) return s;
    if ((s = ctx->cuda(cudaStreamSynchronize(ctx->stream), "host view sync"))) return s;
    host_view_valid = true;
    return GP_OK;
  }

  // One generation on the GPU: kinds -> tournaments -> plan -> [read the child node
  // total] -> emit -> evaluate -> statistics [read once]. Bit-identical to the host path.
  gp_status device_generation(gp_generation_stats* st_out) {
    const int n = cfg.population_size;
    const uint32_t g = (uint32_t)(generation + 1);
    const double t0 = now_s();
    gp_status s;
    if ((s = dev_buffers(n))) return s;
    const MutConfig mc = mut_config();
    cudaStream_t str = ctx->stream;
    DevGenStats* ds = (DevGenStats*)d_stats.p;
    cudaEventRecord(ev[0], str);
    if ((s = ctx->cuda(cudaMemsetAsync(&ds->err, 0, sizeof(int32_t), str), "err memset"))) return s;
    if ((s = ctx->launch(launch_kinds(n, g, mc, (int32_t*)d_kinds.p, (int32_t*)d_tcnt.p,
                                      (int32_t*)d_toff.p, str), "kinds"))) return s;
    ctx->kernel_launches += 1;                     // kinds + scan
    // tournament t depends only on t: launching the upper bound 2 n gives the same first T
    if ((s = gp_tournament_select(ctx, (const float*)d_fit.p, (const int64_t*)d_off.p, n, 2 * n,
                                  cfg.tournament_size, cfg.parsimony, higher ? 1 : 0, cfg.seed, g,
                                  (int32_t*)d_win.p))) return s;
    if ((s = ctx->launch(launch_plan((const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n, g, mc,
                                     (const int32_t*)d_kinds.p, (const int32_t*)d_toff.p,
                                     (const int32_t*)d_win.p, (Recipe*)d_recipe.p,
                                     (int32_t*)d_len.p, (int64_t*)d_off2.p, &ds->err, str),
                         "plan"))) return s;
    ctx->kernel_launches += 1;                     // plan + scan
    // the child node total sizes the next buffers and the evaluation (one small D2H)
    int64_t hdr[2];
    int32_t T = 0, err = 0;
    if ((s = ctx->cuda(cudaMemcpyAsync(&hdr[0], (int64_t*)d_off2.p + n, 8, cudaMemcpyDeviceToHost, str), "D2H total"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(&T, (int32_t*)d_toff.p + n, 4, cudaMemcpyDeviceToHost, str), "D2H T"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(&err, &ds->err, 4, cudaMemcpyDeviceToHost, str), "D2H err"))) return s;
    cudaEventRecord(ev[1], str);
    if ((s = ctx->cuda(cudaStreamSynchronize(str), "plan sync"))) return s;
    if (err) return ctx->fail(GP_ERR_PROGRAM, "device mutation: program deeper than %d", kMaxDepth);
    const int64_t total = hdr[0];
    if ((s = ctx->grow(&d_nodes2.p, &d_nodes2.cap, (size_t)std::max<int64_t>(total, 1) * sizeof(gp_node), "nodes2"))) return s;
    if ((s = ctx->launch(launch_emit((const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n, g, mc,
                                     (const Recipe*)d_recipe.p, (const int64_t*)d_off2.p,
                                     (gp_node*)d_nodes2.p, str), "emit"))) return s;
    std::swap(d_nodes, d_nodes2);
    std::swap(d_off, d_off2);
    n_nodes = total;
    last_T = T;
    sel_valid = true;
    generation = (int)g;
    host_view_valid = false;
    pop.clear();                                   // the host copy is stale from here on
    cudaEventRecord(ev[2], str);
    // evaluation (Alg. 1 line 7); every program's depth is <= stack_capacity - 1, so its stack
    // need is <= stack_capacity
    if ((s = gp_evaluate(ctx, (const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n, total,
                         std::min(cfg.stack_capacity, GP_MAX_STACK), X, ldx, y, w, n_rows, n_cols,
                         (gp_metric)cfg.metric, (float*)d_fit.p, (uint32_t*)d_status.p))) return s;
    cudaEventRecord(ev[3], str);
    if ((s = dev_stats(n))) return s;
    gp_generation_stats st{};
    float a = 0.f, b = 0.f, c2 = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c2, ev[2], ev[3]);
    st.t_select_s = 1e-3 * a;                      // kinds + tournaments + mutation plans
    st.t_mutate_s = 1e-3 * b;                      // (node total read) + child emission
    st.t_h2d_s = 0.0;                              // nothing crosses PCIe
    st.t_eval_s = 1e-3 * c2;
    st.n_tournaments = T;
    fill_stats_dev(&st);
    st.t_total_s = now_s() - t0;
    if (st_out) *st_out = st;
    return GP_OK;
  }

  // Generation 0 on the GPU (program generation): ramped half-and-half from the same
  // Philox streams as the host path, evaluated, statistics read once. [sync]
  gp_status device_init(gp_generation_stats* st_out) {
    const int n = cfg.population_size;
    const double t0 = now_s();
    gp_status s;
    if ((s = dev_buffers(n))) return s;
    if ((s = ctx->grow(&d_off.p, &d_off.cap, (size_t)(n + 1) * sizeof(int64_t), "d_off"))) return s;
    if ((s = ctx->grow(&d_fit.p, &d_fit.cap, (size_t)n * sizeof(float), "d_fit"))) return s;
    if ((s = ctx->grow(&d_status.p, &d_status.cap, (size_t)n * sizeof(uint32_t), "d_status"))) return s;
    const MutConfig mc = mut_config();
    cudaStream_t str = ctx->stream;
    cudaEventRecord(ev[0], str);
    if ((s = ctx->launch(launch_init_lengths(n, mc, (int32_t*)d_len.p, (int64_t*)d_off.p, str), "init lengths"))) return s;
    ctx->kernel_launches += 1;
    int64_t total = 0;
    if ((s = ctx->cuda(cudaMemcpyAsync(&total, (int64_t*)d_off.p + n, 8, cudaMemcpyDeviceToHost, str), "D2H total"))) return s;
    if ((s = ctx->cuda(cudaStreamSynchronize(str), "init sync"))) return s;
    if ((s = ctx->grow(&d_nodes.p, &d_nodes.cap, (size_t)std::max<int64_t>(total, 1) * sizeof(gp_node), "d_nodes"))) return s;
    if ((s = ctx->launch(launch_init_emit(n, mc, (const int64_t*)d_off.p, (gp_node*)d_nodes.p, str), "init emit"))) return s;
    cudaEventRecord(ev[1], str);
    n_nodes = total;
    generation = 0;
    host_view_valid = false;
    sel_valid = false;
    pop.clear();
    kinds.clear();
    winners.clear();
    last_T = 0;
    if ((s = gp_evaluate(ctx, (const gp_node*)d_nodes.p, (const int64_t*)d_off.p, n, total,
                         std::min(cfg.stack_capacity, GP_MAX_STACK), X, ldx, y, w, n_rows, n_cols,
                         (gp_metric)cfg.metric, (float*)d_fit.p, (uint32_t*)d_status.p))) return s;
    cudaEventRecord(ev[2], str);
    if ((s = dev_stats(n))) return s;
    gp_generation_stats st{};
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    st.t_mutate_s = 1e-3 * a;                     // program generation
    st.t_eval_s = 1e-3 * b;
    fill_stats_dev(&st);
    st.t_total_s = now_s() - t0;
    if (st_out) *st_out = st;
    return GP_OK;
  }

  void fill_stats(gp_generation_stats* st) {
    const int n = (int)pop.size();
    int best = -1;
    double sum = 0.0;
    int nfin = 0;
    for (int i = 0; i < n; ++i) {
      const float f = fit[i];
      if (std::isfinite(f)) { sum += f; ++nfin; }
      if (std::isnan(f)) continue;
      if (best < 0 || (higher ? f > fit[best] : f < fit[best])) best = i;
    }
    st->generation = generation;
    st->best_index = best;
    st->mean_raw = nfin ? sum / nfin : NAN;
    st->total_nodes = n_nodes;
    st->max_stack_need = max_need;
    std::copy(op_count, op_count + GP_OP_COUNT, st->op_count);
    st->const_nodes = const_nodes;
    st->const_programs = const_programs;
    if (best >= 0) {
      const float pen = cfg.parsimony * (float)pop[best].size();
      st->best_raw = fit[best];
      st->best_adjusted = higher ? fit[best] - pen : fit[best] + pen;
      st->best_len = (int)pop[best].size();
      st->best_depth = depth_of(pop[best]);
    } else {
      st->best_raw = st->best_adjusted = NAN;
      st->best_len = st->best_depth = 0;
    }
  }
};

extern "C" {

void gp_config_default(gp_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->population_size = 35;         // Table 6
  c->tournament_size = 4;          // Table 6
  c->parsimony = 0.01f;            // Table 6
  c->metric = GP_RMSE;             // Table 6, regression
  c->p_crossover = 0.7;            // Table 6
  c->p_subtree = 0.1;
  c->p_hoist = 0.05;
  c->p_point = 0.1;                // (P:489); reproduction 0.05 is the residual
  c->p_point_replace = 0.05;
  c->init_depth_min = 2;
  c->init_depth_max = 6;
  c->const_lo = -1.0f;
  c->const_hi = 1.0f;
  const int fs[7] = {GP_OP_ADD, GP_OP_SUB, GP_OP_MUL, GP_OP_DIV, GP_OP_SIN, GP_OP_COS, GP_OP_TAN};
  c->n_functions = 7;              // {+,-,*,/,sin,cos,tan}
  for (int i = 0; i < 7; ++i) c->function_set[i] = fs[i];
  c->stack_capacity = GP_MAX_STACK;
  c->seed = 2110;
  c->n_threads = 0;
  c->device_mutation = 1;          // SURVEY F2 (mutate.cu)
}

gp_status gp_engine_create(gp_engine** out, gp_context* ctx, const gp_config* cfg, const float* X,
                           int64_t ldx, const float* y, const float* w, int64_t n_rows,
                           int32_t n_cols) {
  if (!out || !ctx || !cfg) return GP_ERR_ARG;
  *out = nullptr;
  const gp_config& c = *cfg;
  const double psum = c.p_crossover + c.p_subtree + c.p_hoist + c.p_point;
  bool ok = c.population_size >= 1 && c.tournament_size >= 1 && c.metric >= 0 &&
            c.metric <= GP_SPEARMAN && c.n_functions >= 1 && c.n_functions <= 32 &&
            c.init_depth_min >= 1 && c.init_depth_max >= c.init_depth_min &&
            c.stack_capacity >= 2 && c.stack_capacity <= GP_MAX_STACK &&
            c.init_depth_max <= c.stack_capacity - 1 && psum <= 1.0 + 1e-9 && c.p_crossover >= 0 &&
            c.p_subtree >= 0 && c.p_hoist >= 0 && c.p_point >= 0;
  for (int i = 0; ok && i < c.n_functions; ++i) ok = op_arity(c.function_set[i]) > 0;
  if (!ok) return ctx->fail(GP_ERR_ARG, "invalid gp_config");
  cudaSetDevice(ctx->device);
  gp_engine* e = new gp_engine();
  e->ctx = ctx;
  e->cfg = c;
  e->higher = c.metric == GP_PEARSON || c.metric == GP_SPEARMAN;  // correlations: higher wins
  // default: this rank's share of the host cores (every rank of a node runs the same host steps)
  e->threads = c.n_threads > 0 ? c.n_threads
                               : std::max(1, (int)std::thread::hardware_concurrency() / std::max(1, ctx->world));
  // one generation's host work is O(population); beyond 64 threads wake-ups cost more than they save
  e->pool.reset(new Pool(std::min(e->threads, 64)));
  gp_status s = e->set_dataset(X, ldx, y, w, n_rows, n_cols);
  if (s) { delete e; return s; }
  // device mutation needs the generated donors of subtree mutations to fit kMaxDonorNodes
  e->dev_mut = c.device_mutation != 0 && c.init_depth_max <= kMaxDonorDepth;
  *out = e;
  return GP_OK;
}

gp_status gp_engine_set_dataset(gp_engine* e, const float* X, int64_t ldx, const float* y,
                                const float* w, int64_t n_rows, int32_t n_cols) {
  if (!e) return GP_ERR_ARG;
  cudaSetDevice(e->ctx->device);
  return e->set_dataset(X, ldx, y, w, n_rows, n_cols);
}

gp_status gp_engine_destroy(gp_engine* e) {
  if (!e) return GP_ERR_ARG;
  cudaSetDevice(e->ctx->device);
  cudaStreamSynchronize(e->ctx->stream);
  delete e;
  return GP_OK;
}

gp_status gp_engine_init_population(gp_engine* e, gp_generation_stats* stats_out) {
  if (!e) return GP_ERR_ARG;
  cudaSetDevice(e->ctx->device);
  gp_generation_stats st{};
  const double t0 = now_s();
  const gp_config& c = e->cfg;
  const int n = c.population_size;
  if (e->dev_mut) return e->device_init(stats_out);
  e->pop.assign(n, Prog());
  parallel_for(e->pool.get(), n, [&](int i) {
    Rng r(c.seed, (uint32_t)i, 0u, 3u);
    const int method = i < n / 2 ? FULL : GROW;
    const int md = c.init_depth_min + i % (c.init_depth_max - c.init_depth_min + 1);
    e->pop[i] = random_program(r, method, md, c, e->n_cols);
  });
  st.t_mutate_s = now_s() - t0;
  e->generation = 0;
  gp_status s = e->evaluate(&st);
  if (s) return s;
  e->kinds.clear();
  e->winners.clear();
  e->fill_stats(&st);
  st.t_total_s = now_s() - t0;
  if (stats_out) *stats_out = st;
  return GP_OK;
}

gp_status gp_generation(gp_engine* e, gp_generation_stats* stats_out) {
  if (!e) return GP_ERR_ARG;
  if (e->generation < 0) return e->ctx->fail(GP_ERR_ARG, "gp_generation before gp_engine_init_population");
  cudaSetDevice(e->ctx->device);
  if (e->dev_mut) return e->device_generation(stats_out);
  gp_context* ctx = e->ctx;
  const gp_config& c = e->cfg;
  gp_generation_stats st{};
  const double t0 = now_s();
  const int n = c.population_size;
  const uint32_t g = (uint32_t)(e->generation + 1);
  // (1) mutation kinds first, so the tournament count is known
  e->kinds.resize(n);
  parallel_for(e->pool.get(), n, [&](int i) {
    Rng r(c.seed, (uint32_t)i, g, 1u);
    const double u = r.uniform();
    const double p[4] = {c.p_crossover, c.p_subtree, c.p_hoist, c.p_point};
    double cum = 0.0;
    int kind = K_REPRODUCTION;
    for (int k = 0; k < 4; ++k) {
      cum += p[k];
      if (u < cum) { kind = k; break; }
    }
    e->kinds[i] = kind;
  });
  std::vector<int32_t> toff(n + 1, 0);
  for (int i = 0; i < n; ++i) toff[i + 1] = toff[i] + (e->kinds[i] == K_CROSSOVER ? 2 : 1);
  const int T = toff[n];
  // (2) tournaments on the GPU over the current population's fitness
  gp_status s;
  if ((s = ctx->grow(&e->d_win.p, &e->d_win.cap, (size_t)T * sizeof(int32_t), "winners"))) return s;
  if ((s = gp_tournament_select(ctx, (const float*)e->d_fit.p, (const int64_t*)e->d_off.p, n, T,
                                c.tournament_size, c.parsimony, e->higher ? 1 : 0, c.seed, g,
                                (int32_t*)e->d_win.p))) return s;
  e->winners.resize(T);
  if ((s = ctx->cuda(cudaMemcpyAsync(e->winners.data(), e->d_win.p, (size_t)T * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, ctx->stream), "D2H winners"))) return s;
  if ((s = ctx->cuda(cudaStreamSynchronize(ctx->stream), "select sync"))) return s;
  const double t1 = now_s();
  // (3) host mutations, one Philox stream per child
  std::vector<Prog> next(n);
  const int nf = e->n_cols;
  parallel_for(e->pool.get(), n, [&](int i) {
    Rng r(c.seed, (uint32_t)i, g, 2u);
    const Prog& parent = e->pop[e->winners[toff[i]]];
    switch (e->kinds[i]) {
      case K_CROSSOVER: next[i] = hoisted_crossover(r, parent, e->pop[e->winners[toff[i] + 1]], c); break;
      case K_SUBTREE: next[i] = subtree_mutation(r, parent, c, nf); break;
      case K_HOIST: next[i] = hoist_mutation(r, parent); break;
      case K_POINT: next[i] = point_mutation(r, parent, c, nf); break;
      default: next[i] = parent; break;
    }
  });
  e->pop.swap(next);
  const double t2 = now_s();
  e->generation = (int)g;
  // (4) one H2D copy of the flat population + evaluation (Alg. 1 line 7)
  if ((s = e->evaluate(&st))) return s;
  st.t_select_s = t1 - t0;
  st.t_mutate_s = t2 - t1;
  st.n_tournaments = T;
  e->fill_stats(&st);
  st.t_total_s = now_s() - t0;
  if (stats_out) *stats_out = st;
  return GP_OK;
}

gp_status gp_engine_population(gp_engine* e, const gp_node** nodes, const int64_t** offsets,
                               const float** fitness, int32_t* n_programs, int64_t* n_nodes) {
  if (!e || e->generation < 0) return GP_ERR_ARG;
  cudaSetDevice(e->ctx->device);
  gp_status s = e->sync_host_view();
  if (s) return s;
  if (nodes) *nodes = e->h_nodes;
  if (offsets) *offsets = e->h_off;
  if (fitness) *fitness = e->fit.data();
  if (n_programs) *n_programs = e->cfg.population_size;
  if (n_nodes) *n_nodes = e->n_nodes;
  return GP_OK;
}

gp_status gp_engine_population_device(gp_engine* e, const gp_node** nodes,
                                      const int64_t** offsets, const float** fitness,
                                      int32_t* n_programs, int64_t* n_nodes) {
  if (!e || e->generation < 0) return GP_ERR_ARG;
  if (nodes) *nodes = (const gp_node*)e->d_nodes.p;
  if (offsets) *offsets = (const int64_t*)e->d_off.p;
  if (fitness) *fitness = (const float*)e->d_fit.p;
  if (n_programs) *n_programs = e->cfg.population_size;
  if (n_nodes) *n_nodes = e->n_nodes;
  return GP_OK;
}

gp_status gp_engine_last_selection(gp_engine* e, const int32_t** kinds, const int32_t** winners,
                                   int32_t* n_tournaments) {
  if (!e) return GP_ERR_ARG;
  if (e->dev_mut) {
    if (!e->sel_valid) {                 // no generation since init / set_population
      e->kinds.clear();
      e->winners.clear();
    }
  }
  if (e->dev_mut && e->sel_valid && e->generation > 0 && e->d_kinds.p) {
    cudaSetDevice(e->ctx->device);
    const int n = e->cfg.population_size;
    e->kinds.resize(n);
    e->winners.resize(e->last_T);
    gp_status s;
    if ((s = e->ctx->cuda(cudaMemcpyAsync(e->kinds.data(), e->d_kinds.p, (size_t)n * 4, cudaMemcpyDeviceToHost, e->ctx->stream), "D2H kinds"))) return s;
    if ((s = e->ctx->cuda(cudaMemcpyAsync(e->winners.data(), e->d_win.p, (size_t)e->last_T * 4, cudaMemcpyDeviceToHost, e->ctx->stream), "D2H winners"))) return s;
    if ((s = e->ctx->cuda(cudaStreamSynchronize(e->ctx->stream), "selection sync"))) return s;
  }
  if (kinds) *kinds = e->kinds.data();
  if (winners) *winners = e->winners.data();
  if (n_tournaments) *n_tournaments = (int32_t)e->winners.size();
  return GP_OK;
}

gp_status gp_engine_set_population(gp_engine* e, const gp_node* nodes, const int64_t* offsets,
                                   int32_t n_programs, int64_t n_nodes, const float* fitness,
                                   int32_t generation, gp_generation_stats* stats_out) {
  if (!e || !nodes || !offsets || generation < 0) return GP_ERR_ARG;
  gp_context* ctx = e->ctx;
  cudaSetDevice(ctx->device);
  const gp_config& c = e->cfg;
  if (n_programs != c.population_size || n_nodes < n_programs)
    return ctx->fail(GP_ERR_ARG, "set_population: %d programs (population_size %d), %lld nodes",
                     n_programs, c.population_size, (long long)n_nodes);
  const int n = n_programs;
  gp_status s;
  gp_generation_stats st{};
  const double t0 = now_s();
  if (e->dev_mut && !is_host_pointer(nodes) && !is_host_pointer(offsets) && fitness &&
      !is_host_pointer(fitness)) {
    // device-resident population with known fitness: stream-ordered copies into the engine,
    // statistics on the device (the programs are the caller's responsibility: a program deeper
    // than the device scans makes the next generation fail with GP_ERR_PROGRAM)
    if ((s = e->dev_buffers(n))) return s;
    if ((s = ctx->grow(&e->d_nodes.p, &e->d_nodes.cap, (size_t)n_nodes * sizeof(gp_node), "d_nodes"))) return s;
    if ((s = ctx->grow(&e->d_off.p, &e->d_off.cap, (size_t)(n + 1) * sizeof(int64_t), "d_off"))) return s;
    if ((s = ctx->grow(&e->d_fit.p, &e->d_fit.cap, (size_t)n * sizeof(float), "d_fit"))) return s;
    if ((s = ctx->grow(&e->d_status.p, &e->d_status.cap, (size_t)n * sizeof(uint32_t), "d_status"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(e->d_nodes.p, nodes, (size_t)n_nodes * sizeof(gp_node), cudaMemcpyDeviceToDevice, ctx->stream), "D2D nodes"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(e->d_off.p, offsets, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream), "D2D offsets"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(e->d_fit.p, fitness, (size_t)n * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream), "D2D fitness"))) return s;
    e->n_nodes = n_nodes;
    e->generation = generation;
    e->host_view_valid = false;
    e->sel_valid = false;
    e->pop.clear();
    if (!stats_out) return GP_OK;        // no statistics wanted: stream-ordered, no sync
    if ((s = e->dev_stats(n))) return s;
    e->fill_stats_dev(&st);
  } else {
    // host copy, validated (prefix, depth <= capacity - 1), then the host upload path
    std::vector<int64_t> off(n + 1);
    std::vector<gp_node> nd((size_t)n_nodes);
    if ((s = ctx->cuda(cudaMemcpy(off.data(), offsets, (size_t)(n + 1) * 8, cudaMemcpyDefault), "offsets"))) return s;
    if ((s = ctx->cuda(cudaMemcpy(nd.data(), nodes, (size_t)n_nodes * sizeof(gp_node), cudaMemcpyDefault), "nodes"))) return s;
    if (off[0] != 0 || off[n] != n_nodes) return ctx->fail(GP_ERR_ARG, "set_population: offsets");
    std::vector<Prog> pop(n);
    for (int i = 0; i < n; ++i) {
      if (off[i + 1] <= off[i]) return ctx->fail(GP_ERR_ARG, "set_population: empty program %d", i);
      Prog p(nd.begin() + off[i], nd.begin() + off[i + 1]);
      int64_t needed = 1;
      for (const gp_node& x : p) {
        if (needed == 0 || arity(x.op) < 0) { needed = -1; break; }
        needed += arity(x.op) - 1;
      }
      if (needed != 0) return ctx->fail(GP_ERR_ARG, "set_population: program %d is not a valid prefix list", i);
      if (depth_of(p) > c.stack_capacity - 1) return ctx->fail(GP_ERR_ARG, "set_population: program %d too deep", i);
      pop[i] = std::move(p);
    }
    e->pop.swap(pop);
    e->generation = generation;
    e->sel_valid = false;
    e->kinds.clear();
    e->winners.clear();
    if ((s = e->evaluate(&st, fitness))) return s;
    e->fill_stats(&st);
  }
  st.t_total_s = now_s() - t0;
  if (stats_out) *stats_out = st;
  return GP_OK;
}

}  // extern "C"
