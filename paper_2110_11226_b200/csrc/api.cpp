// api.cpp -- C-ABI implementation: contexts, gp_evaluate / gp_predict / gp_tournament_select
// orchestration, the NCCL all-reduce of per-program partial sums, host-pointer staging.
// Every device step runs in the kernels of aux.cu / eval_s*.cu; this file only validates
// arguments, sizes workspaces and enqueues work on the context stream.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gp_internal.h"

using namespace gpb;

// ---------------------------------------------------------------------------------------------
// NCCL, loaded lazily with dlopen so the library loads (and single-GPU use works) without it.
// ---------------------------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
               api.AllGather && api.Broadcast;
    }
  }
  return api;
}
thread_local std::string g_last_global_error;
}  // namespace

// ---------------------------------------------------------------------------------------------
// Context helpers
// ---------------------------------------------------------------------------------------------
gp_status gp_context::fail(gp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  err = buf;
  return s;
}

gp_status gp_context::cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return GP_OK;
  return fail(e == cudaErrorMemoryAllocation ? GP_ERR_OOM : GP_ERR_CUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

gp_status gp_context::launch(cudaError_t e, const char* what) {
  if (e == cudaSuccess) ++kernel_launches;
  return cuda(e, what);
}

gp_status gp_context::grow(void** p, size_t* cap, size_t bytes, const char* what) {
  if (*cap >= bytes && *p) return GP_OK;
  if (*p) cudaFreeAsync(*p, stream);
  *p = nullptr;
  *cap = 0;
  size_t want = std::max(bytes, (size_t)256);
  want += want / 4;  // amortise growth
  gp_status s = cuda(cudaMallocAsync(p, want, stream), what);
  if (s == GP_OK) *cap = want;
  return s;
}

bool gpb::is_host_pointer(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// Stages a [host|device] input into a context buffer when it is host memory.
gp_status gp_context::stage_in(const void* src, size_t bytes, StageBuf& buf, const void** dst,
                               bool* was_host) {
  *dst = src;
  if (!is_host_pointer(src)) return GP_OK;
  *was_host = true;
  gp_status s = grow(&buf.p, &buf.cap, bytes, "stage_in");
  if (s) return s;
  s = cuda(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, stream), "H2D");
  *dst = buf.p;
  return s;
}

int gpb::sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 148;
}

// Work decomposition shared by every variant launch: items =
// program group x row chunk. Groups are sized for ~8 items per resident CTA slot (large groups
// amortise the per-tile staging of X and y over many programs); row chunks are then cut for ~128
// items per slot. The plan counts every program, but variable-free programs skip the evaluator
// (70 % of an evolved C3 population) and groups differ in total code length, so fine row chunks
// keep the persistent CTAs' queue balanced to the end (C3 SFU frac: 0.72 at 8 items per slot,
// 0.77 at 32, 0.79 at 128). Chunks are whole tiles of the plan tile (kernels.h); the slot count
// assumes 4 resident 128-thread CTAs per SM (the shared-memory shapes run one 512-thread CTA per
// SM, so each CTA takes ~4x the items; measured on C3 with the 512-thread s4, r02).
EvalPlan gpb::plan_eval(int device, int64_t n_rows, int32_t n_programs, int32_t n_cols, int S,
                        bool predict, bool weighted, int force_G, int64_t force_tpc) {
  EvalPlan pl;
  // X is staged in shared memory when the s4 shape's whole layout fits at 128-program groups
  // (8192-row tiles, see kernels.h); otherwise the wide-dataset shapes read X through L1/L2
  pl.xsmem = eval_variant_s4().smem_bytes(128, S, n_cols, weighted, 1, predict) <=
             (size_t)kMaxDynSmem;
  // Largest program group: on the shared-memory path the largest of 512 / 256 / 128 whose
  // accumulators still fit (each staged X / y tile then serves more programs: C3 step 121.7 ->
  // 119.5 -> 118.1 ms at 128 / 256 / 512); 128 on the global-X path, where larger groups keep
  // more distinct code streams' variable loads in flight per row chunk (C4 step 42.0 -> 50.7 ms
  // at 256). Tuning knob GP_G_MAX caps it.
  static const int env_gmax = [] {
    const char* e = getenv("GP_G_MAX");
    return e && atoi(e) > 0 ? std::min(atoi(e), 1024) : 0;
  }();
  int g_max = 128;
  if (pl.xsmem) {
    for (int g : {512, 256}) {
      if (env_gmax > 0 && g > env_gmax) continue;
      if (eval_variant_s4().smem_bytes(g, S, n_cols, weighted, 1, predict) <= (size_t)kMaxDynSmem) {
        g_max = g;
        break;
      }
    }
  }
  if (env_gmax > 0 && env_gmax < g_max) g_max = env_gmax;
  const int tile = pl.xsmem ? kTileSmem : kTileGlobal;
  const int64_t n_tiles = (n_rows + tile - 1) / tile;
  const int occ_guess = 4;
  // row-chunk items per resident CTA slot (tuning knob GP_ITEMS_PER_SLOT)
  static const int per_slot = [] {
    const char* e = getenv("GP_ITEMS_PER_SLOT");
    return e && atoi(e) > 0 ? atoi(e) : 128;
  }();
  const int64_t slots = (int64_t)sm_count(device) * occ_guess;
  const int64_t want_groups = std::max<int64_t>(1, (slots * 8 + n_tiles - 1) / n_tiles);
  int G = (int)std::min<int64_t>(g_max, std::max<int64_t>(1, (n_programs + want_groups - 1) / want_groups));
  static const int env_G = [] {                                 // tuning knob GP_PLAN_G
    const char* e = getenv("GP_PLAN_G");
    return e && atoi(e) > 0 ? atoi(e) : 0;
  }();
  if (env_G > 0) G = std::min(env_G, g_max);
  if (force_G > 0) G = std::min(force_G, g_max);               // gp_context_set_plan
  const int n_groups = (n_programs + G - 1) / G;
  int64_t Q = std::min<int64_t>(n_tiles, std::max<int64_t>(1, (slots * per_slot + n_groups - 1) / n_groups));
  // the fp64 partial buffer (row chunks x evaluated programs x S) is written and tile-reduced
  // every evaluation: at most GP_PARTIAL_MB (default 64) MB of it
  static const int64_t part_mb = [] {
    const char* e = getenv("GP_PARTIAL_MB");
    return (int64_t)(e && atoi(e) > 0 ? atoi(e) : 64);
  }();
  Q = std::min<int64_t>(Q, std::max<int64_t>(1, (part_mb << 20) / ((int64_t)n_programs * S * 8)));
  int64_t tpc = (n_tiles + Q - 1) / Q;
  if (force_tpc > 0) tpc = std::min<int64_t>(force_tpc, n_tiles);
  Q = (n_tiles + tpc - 1) / tpc;
  static const int env_order = [] {                             // tuning knob GP_ITEM_ORDER
    const char* e = getenv("GP_ITEM_ORDER");
    return e ? atoi(e) : 0;
  }();
  pl.item_order = env_order;
  pl.G = G;
  pl.n_groups = n_groups;
  pl.n_chunks = Q;
  pl.rows_per_chunk = tpc * tile;
  return pl;
}

static const EvalVariant& variant(int v, bool global_x = false) {
  if (global_x && v == 0) return eval_variant_w4();
  if (global_x && v == 1) return eval_variant_w8();
  switch (v) {
    case 0: return eval_variant_s4();
    case 1: return eval_variant_s8();
    case 2: return eval_variant_s12();
    default: return eval_variant_s20();
  }
}

// Launches the persistent evaluator of every variant that can hold programs of stack need
// <= max_stack, each over its own bucket (lists / counts written by the bucket kernel).
static gp_status launch_variants(gp_context* ctx, EvalArgs a, const EvalPlan& pl, int32_t max_stack,
                                 bool predict) {
  const int32_t n = a.n_programs;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (ctx->profiling && !predict) {
    if (!ctx->ev_free.empty()) { ev = ctx->ev_free.back(); ctx->ev_free.pop_back(); }
    else { cudaEventCreate(&ev.first); cudaEventCreate(&ev.second); }
    cudaEventRecord(ev.first, ctx->stream);
  }
  for (int v = 0; v < kNumVariants; ++v) {
    if (v > 0 && kVariantStack[v - 1] >= max_stack) break;
    const EvalVariant& var = variant(v, !pl.xsmem);
    if (var.shape.SUB != variant(v).shape.SUB)   // the pack kernel laid out SUB copies per program
      return ctx->fail(GP_ERR_ARG, "evaluator variant %d: wide shape SUB mismatch", v);
    a.stream = (const uint4*)ctx->codestream.p;
    a.item_order = pl.item_order;
    // consecutive variant launches walk the row chunks in opposite directions, so each launch
    // starts on the chunks the previous one left in L2 (C3: X + y = 201 MB vs 126 MB of L2)
    static const bool env_rev = [] {                            // tuning knob GP_CHUNK_REVERSE
      const char* e = getenv("GP_CHUNK_REVERSE");
      return !e || atoi(e) != 0;
    }();
    a.chunk_reverse = env_rev ? (v & 1) : 0;
    a.gstart = (const int64_t*)ctx->gstart.p + (int64_t)v * (n + 1);
    a.prog_ids = (const int32_t*)ctx->lists.p + (int64_t)v * n;
    a.prog_count = (const int32_t*)ctx->counts.p + v;
    a.work_counter = (int32_t*)ctx->counts.p + kNumVariants + v;
    a.part_base = (const int32_t*)ctx->inv.p + n + v;
    a.group_size = (const int32_t*)ctx->inv.p + n + kNumVariants + 1 + v;
    const size_t smem = var.smem_bytes(pl.G, a.metric == GP_PEARSON ? 3 : 1, a.n_cols,
                                       a.w != nullptr, pl.xsmem, predict);
    const int occ = std::max(1, var.occupancy(predict, pl.xsmem, smem));
    gp_status s = ctx->launch(var.launch(a, predict, pl.xsmem, ctx->sms * occ, smem, ctx->stream),
                            predict ? "predict kernel" : "eval kernel");
    if (s) return s;
  }
  if (ctx->profiling && !predict) {
    cudaEventRecord(ev.second, ctx->stream);
    ctx->ev_pending.push_back(ev);
  }
  return GP_OK;
}

// ---------------------------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------------------------
extern "C" {

const char* gp_status_string(gp_status s) {
  switch (s) {
    case GP_OK: return "GP_OK";
    case GP_ERR_ARG: return "GP_ERR_ARG";
    case GP_ERR_PROGRAM: return "GP_ERR_PROGRAM";
    case GP_ERR_UNSUPPORTED: return "GP_ERR_UNSUPPORTED";
    case GP_ERR_CUDA: return "GP_ERR_CUDA";
    case GP_ERR_NCCL: return "GP_ERR_NCCL";
    case GP_ERR_OOM: return "GP_ERR_OOM";
  }
  return "GP_ERR_UNKNOWN";
}

const char* gp_last_error(const gp_context* ctx) {
  return ctx ? ctx->err.c_str() : g_last_global_error.c_str();
}

const char* gp_version(void) { return "gp_b200 0.2 sm_100a"; }

gp_status gp_device_copy(void* dst, const void* src, size_t bytes) {
  if ((!dst || !src) && bytes) return GP_ERR_ARG;
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
  if (e != cudaSuccess) { g_last_global_error = cudaGetErrorString(e); return GP_ERR_CUDA; }
  return GP_OK;
}

gp_status gp_get_unique_id(void* out_id) {
  if (!out_id) return GP_ERR_ARG;
  NcclApi& n = nccl();
  if (!n.ok) { g_last_global_error = "libnccl.so.2 could not be loaded"; return GP_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = n.GetUniqueId(&id);
  if (r != ncclSuccess) { g_last_global_error = n.GetErrorString(r); return GP_ERR_NCCL; }
  memcpy(out_id, &id, sizeof id);
  return GP_OK;
}

gp_status gp_context_create(gp_context** out, int device, void* stream, const void* nccl_unique_id,
                            int rank, int world_size) {
  if (!out || world_size < 1 || rank < 0 || rank >= world_size) return GP_ERR_ARG;
  *out = nullptr;
  if (world_size > 1 && !nccl_unique_id) return GP_ERR_ARG;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { g_last_global_error = cudaGetErrorString(e); return GP_ERR_CUDA; }
  gp_context* c = new gp_context();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->rank = rank;
  c->world = world_size;
  c->sms = sm_count(device);
  if (nccl_unique_id) {
    NcclApi& n = nccl();
    if (!n.ok) { delete c; g_last_global_error = "libnccl.so.2 could not be loaded"; return GP_ERR_NCCL; }
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof id);
    ncclComm_t comm;
    ncclResult_t r = n.CommInitRank(&comm, world_size, id, rank);
    if (r != ncclSuccess) {
      g_last_global_error = n.GetErrorString(r);
      delete c;
      return GP_ERR_NCCL;
    }
    c->comm = comm;
  }
  *out = c;
  return GP_OK;
}

gp_status gp_context_destroy(gp_context* ctx) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (StageBuf* b : ctx->all_buffers())
    if (b->p) cudaFree(b->p);
  for (auto& ev : ctx->ev_pending) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
  for (auto& ev : ctx->ev_free) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
  if (ctx->comm) nccl().CommDestroy((ncclComm_t)ctx->comm);
  delete ctx;
  return GP_OK;
}

gp_status gp_context_set_stream(gp_context* ctx, void* stream) {
  if (!ctx) return GP_ERR_ARG;
  if ((cudaStream_t)stream == ctx->stream) return GP_OK;
  // buffers grown later are freed / allocated stream-ordered on the NEW stream: the old stream's
  // queued work that may still read them must be finished first
  cudaSetDevice(ctx->device);
  gp_status s = ctx->cuda(cudaStreamSynchronize(ctx->stream), "set_stream: old stream");
  if (s) return s;
  ctx->stream = (cudaStream_t)stream;
  return GP_OK;
}

gp_status gp_context_set_plan(gp_context* ctx, int32_t group_size, int64_t tiles_per_chunk) {
  if (!ctx || group_size < 0 || group_size > 512 || tiles_per_chunk < 0) return GP_ERR_ARG;
  ctx->plan_G = group_size;
  ctx->plan_tpc = tiles_per_chunk;
  return GP_OK;
}

gp_status gp_context_set_program_range(gp_context* ctx, int32_t lo, int32_t hi) {
  if (!ctx || lo < 0 || (hi >= 0 && hi < lo)) return GP_ERR_ARG;
  ctx->range_lo = lo;
  ctx->range_hi = hi;
  return GP_OK;
}

gp_status gp_context_set_profiling(gp_context* ctx, int enabled) {
  if (!ctx) return GP_ERR_ARG;
  ctx->profiling = enabled != 0;
  return GP_OK;
}

gp_status gp_context_eval_timing(gp_context* ctx, double* total_ms, int64_t* launches, int reset) {
  if (!ctx) return GP_ERR_ARG;
  for (auto& ev : ctx->ev_pending) {
    cudaEventSynchronize(ev.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.first, ev.second);
    ctx->prof_ms += ms;
    ctx->prof_launches += 1;
    ctx->ev_free.push_back(ev);
  }
  ctx->ev_pending.clear();
  if (total_ms) *total_ms = ctx->prof_ms;
  if (launches) *launches = ctx->prof_launches;
  if (reset) { ctx->prof_ms = 0.0; ctx->prof_launches = 0; }
  return GP_OK;
}

gp_status gp_context_set_shard(gp_context* ctx, gp_shard mode) {
  if (!ctx || (mode != GP_SHARD_ROWS && mode != GP_SHARD_PROGRAMS)) return GP_ERR_ARG;
  ctx->shard = mode;
  return GP_OK;
}

gp_status gp_context_set_const_programs(gp_context* ctx, int closed_form) {
  if (!ctx) return GP_ERR_ARG;
  ctx->const_programs = closed_form != 0;
  return GP_OK;
}

gp_status gp_context_set_eval_order(gp_context* ctx, int sethi_ullman) {
  if (!ctx) return GP_ERR_ARG;
  ctx->sethi_ullman = sethi_ullman != 0;
  return GP_OK;
}

gp_status gp_context_kernel_launches(gp_context* ctx, int64_t* launches, int reset) {
  if (!ctx) return GP_ERR_ARG;
  if (launches) *launches = ctx->kernel_launches;
  if (reset) ctx->kernel_launches = 0;
  return GP_OK;
}

gp_status gp_context_set_reference_row(gp_context* ctx, const float* x_ref, int32_t n_cols,
                                       float y_ref) {
  if (!ctx || !x_ref || n_cols < 1) return GP_ERR_ARG;
  gp_status s = ctx->grow(&ctx->xref.p, &ctx->xref.cap, (size_t)n_cols * sizeof(float) + sizeof(float), "xref");
  if (s) return s;
  ctx->xref_host.assign(x_ref, x_ref + n_cols);
  ctx->xref_host.push_back(y_ref);
  s = ctx->cuda(cudaMemcpyAsync(ctx->xref.p, ctx->xref_host.data(), ctx->xref_host.size() * sizeof(float),
                                cudaMemcpyHostToDevice, ctx->stream), "xref H2D");
  if (s) return s;
  ctx->xref_cols = n_cols;
  return ctx->cuda(cudaStreamSynchronize(ctx->stream), "xref sync");
}

static gp_status bucket_pack(gp_context* ctx, int32_t n_programs, int32_t G, bool skip_const,
                             int32_t p_lo, int32_t p_hi);

// Shared front half of gp_evaluate / gp_predict: argument checks, staging, compile (stage),
// Pearson shift, bucketing by stack need and the per-variant code streams (pack).
static gp_status prepare(gp_context* ctx, const gp_node*& programs, const int64_t*& offsets,
                         int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float*& X,
                         int64_t ldx, int64_t n_rows, int32_t n_cols, int32_t G, bool pearson,
                         const float* y, bool* any_host, bool skip_const = false,
                         int32_t p_lo = 0, int32_t p_hi = -1) {
  if (n_programs < 1 || n_nodes < 1 || max_stack < 1 || max_stack > GP_MAX_STACK || n_rows < 1 ||
      n_cols < 1 || ldx < n_rows || !programs || !offsets || !X)
    return ctx->fail(GP_ERR_ARG, "invalid argument (n_programs=%d n_nodes=%lld max_stack=%d "
                     "n_rows=%lld n_cols=%d ldx=%lld)", n_programs, (long long)n_nodes, max_stack,
                     (long long)n_rows, n_cols, (long long)ldx);
  gp_status s;
  const void* d;
  if ((s = ctx->stage_in(programs, (size_t)n_nodes * sizeof(gp_node), ctx->h_nodes, &d, any_host))) return s;
  programs = (const gp_node*)d;
  if ((s = ctx->stage_in(offsets, (size_t)(n_programs + 1) * sizeof(int64_t), ctx->h_off, &d, any_host))) return s;
  offsets = (const int64_t*)d;
  const size_t xbytes = ((size_t)(n_cols - 1) * ldx + n_rows) * sizeof(float);
  if ((s = ctx->stage_in(X, xbytes, ctx->h_X, &d, any_host))) return s;
  X = (const float*)d;
  const int64_t n = n_programs;
  if ((s = ctx->grow(&ctx->code.p, &ctx->code.cap, (size_t)(n_nodes + 2) * sizeof(uint4), "code"))) return s;
  if ((s = ctx->grow(&ctx->code_off.p, &ctx->code_off.cap, (size_t)n * sizeof(int64_t), "code_off"))) return s;
  if ((s = ctx->grow(&ctx->code_len.p, &ctx->code_len.cap, (size_t)n * sizeof(int32_t), "code_len"))) return s;
  if ((s = ctx->grow(&ctx->need.p, &ctx->need.cap, (size_t)n * sizeof(int32_t), "need"))) return s;
  if ((s = ctx->grow(&ctx->lists.p, &ctx->lists.cap, (size_t)n * kNumVariants * sizeof(int32_t), "lists"))) return s;
  if ((s = ctx->grow(&ctx->pos.p, &ctx->pos.cap, (size_t)n * kNumVariants * sizeof(int64_t), "pos"))) return s;
  if ((s = ctx->grow(&ctx->gstart.p, &ctx->gstart.cap, (size_t)(n + 1) * kNumVariants * sizeof(int64_t), "gstart"))) return s;
  if ((s = ctx->grow(&ctx->counts.p, &ctx->counts.cap, 2 * kNumVariants * sizeof(int32_t) + (kNumVariants + 1) * sizeof(int64_t), "counts"))) return s;
  // stream words <= SUB_max x code words + 2 pad words
  if ((s = ctx->grow(&ctx->codestream.p, &ctx->codestream.cap, ((size_t)4 * (n_nodes + n) + 2) * sizeof(uint4), "stream"))) return s;
  if ((s = ctx->grow(&ctx->status.p, &ctx->status.cap, (size_t)n * sizeof(uint32_t), "status"))) return s;
  if ((s = ctx->grow(&ctx->inv.p, &ctx->inv.cap, (size_t)(n + 2 * kNumVariants + 1) * sizeof(int32_t), "inv"))) return s;
  if ((s = ctx->grow(&ctx->scratch.p, &ctx->scratch.cap, (size_t)4 * n_nodes * sizeof(int32_t), "scratch"))) return s;
  if ((s = ctx->launch(launch_stage(programs, offsets, n_programs, n_nodes, n_cols, max_stack,
                                  (uint4*)ctx->code.p, (int64_t*)ctx->code_off.p,
                                  (int32_t*)ctx->code_len.p, (int32_t*)ctx->need.p,
                                  (uint32_t*)ctx->status.p, (int32_t*)ctx->scratch.p,
                                  ctx->sethi_ullman ? 1 : 0, ctx->stream),
                     "stage kernel"))) return s;
  if (pearson) {  // DESIGN.md C9: K_p = f_p(reference row), K_y = y_ref
    if ((s = ctx->grow(&ctx->shift.p, &ctx->shift.cap, (size_t)n * sizeof(float) + 16, "shift"))) return s;
    float* sh = (float*)ctx->shift.p;
    const float *xref, *yref;
    int64_t stride;
    if (ctx->xref_cols >= n_cols) {
      xref = (const float*)ctx->xref.p;
      stride = 1;
      yref = (const float*)ctx->xref.p + ctx->xref_cols;
    } else if (ctx->comm && ctx->shard == GP_SHARD_ROWS) {
      // no reference row set and rows are sharded: every rank must shift by the SAME row, so
      // rank 0's first row (and y) is broadcast (local rows would mix shifts)
      if ((s = ctx->grow(&ctx->xref_b.p, &ctx->xref_b.cap, (size_t)(n_cols + 1) * sizeof(float), "xref_b"))) return s;
      float* xb = (float*)ctx->xref_b.p;
      if ((s = ctx->launch(launch_gather_row(X, ldx, n_cols, y, xb, ctx->stream), "gather row"))) return s;
      NcclApi& nc = nccl();
      ncclResult_t r = nc.Broadcast(xb, xb, (size_t)n_cols + 1, ncclFloat32, 0,
                                    (ncclComm_t)ctx->comm, ctx->stream);
      if (r != ncclSuccess) return ctx->fail(GP_ERR_NCCL, "ncclBroadcast: %s", nc.GetErrorString(r));
      xref = xb;
      stride = 1;
      yref = xb + n_cols;
    } else {
      xref = X;
      stride = ldx;
      yref = y;
    }
    if ((s = ctx->launch(launch_copy_scalar(yref, sh + n, ctx->stream), "y shift"))) return s;
    if ((s = ctx->launch(launch_shift((const uint4*)ctx->code.p, (const int64_t*)ctx->code_off.p,
                                    (const int32_t*)ctx->code_len.p, n_programs, kCaseStride,
                                    xref, stride, sh, ctx->stream), "shift kernel"))) return s;
  }
  return bucket_pack(ctx, n_programs, G, skip_const, p_lo, p_hi < 0 ? n_programs : p_hi);
}

// Bucketing by stack need of the programs [p_lo, p_hi) (compiled by prepare) and the per-variant
// code streams (pack).
static gp_status bucket_pack(gp_context* ctx, int32_t n_programs, int32_t G, bool skip_const,
                             int32_t p_lo, int32_t p_hi) {
  gp_status s;
  int32_t* counts = (int32_t*)ctx->counts.p;
  int64_t* base = (int64_t*)(counts + 2 * kNumVariants);
  int subs[kNumVariants];  // row passes per program of each variant (its compiled shape)
  for (int v = 0; v < kNumVariants; ++v) subs[v] = variant(v).shape.SUB;
  if ((s = ctx->launch(launch_bucket((const int32_t*)ctx->need.p, (const int32_t*)ctx->code_len.p,
                                   n_programs, G, subs, (int32_t*)ctx->lists.p, (int64_t*)ctx->pos.p,
                                   (int64_t*)ctx->gstart.p, counts, base, skip_const ? 1 : 0,
                                   p_lo, p_hi, (int32_t*)ctx->inv.p, ctx->stream),
                     "bucket kernel"))) return s;
  return ctx->launch(launch_pack((const uint4*)ctx->code.p, (const int64_t*)ctx->code_off.p,
                               (const int32_t*)ctx->code_len.p, (const int32_t*)ctx->lists.p,
                               (const int64_t*)ctx->pos.p, counts, base,
                               (const int64_t*)ctx->gstart.p, n_programs, subs,
                               (const int32_t*)ctx->inv.p, (uint4*)ctx->codestream.p, ctx->stream),
                   "pack kernel");
}

// Population sharding (GP_SHARD_PROGRAMS): in-place all-gather of each rank's [lo, hi) fitness
// and status through a padded buffer (world x chunk entries; ncclAllGather needs equal counts),
// then back into place, so every rank holds all n results.
static gp_status gather_programs(gp_context* ctx, int32_t n_programs, int32_t chunk, int32_t p_lo,
                                 int32_t p_hi, float* fit_dev) {
  gp_status s;
  const size_t cb = (size_t)chunk * 4, own = (size_t)(p_hi - p_lo) * 4;
  if ((s = ctx->grow(&ctx->gather.p, &ctx->gather.cap, 2 * (size_t)ctx->world * cb, "gather"))) return s;
  char* gf = (char*)ctx->gather.p;
  char* gs = gf + (size_t)ctx->world * cb;
  if (own) {
    if ((s = ctx->cuda(cudaMemcpyAsync(gf + ctx->rank * cb, fit_dev + p_lo, own, cudaMemcpyDeviceToDevice, ctx->stream), "gather in"))) return s;
    if ((s = ctx->cuda(cudaMemcpyAsync(gs + ctx->rank * cb, (uint32_t*)ctx->status.p + p_lo, own, cudaMemcpyDeviceToDevice, ctx->stream), "gather in"))) return s;
  }
  NcclApi& n = nccl();
  ncclResult_t r = n.AllGather(gf + ctx->rank * cb, gf, (size_t)chunk, ncclFloat32,
                               (ncclComm_t)ctx->comm, ctx->stream);
  if (r == ncclSuccess)
    r = n.AllGather(gs + ctx->rank * cb, gs, (size_t)chunk, ncclUint32, (ncclComm_t)ctx->comm,
                    ctx->stream);
  if (r != ncclSuccess) return ctx->fail(GP_ERR_NCCL, "ncclAllGather: %s", n.GetErrorString(r));
  if ((s = ctx->cuda(cudaMemcpyAsync(fit_dev, gf, (size_t)n_programs * 4, cudaMemcpyDeviceToDevice, ctx->stream), "gather out"))) return s;
  return ctx->cuda(cudaMemcpyAsync(ctx->status.p, gs, (size_t)n_programs * 4, cudaMemcpyDeviceToDevice, ctx->stream), "gather out");
}

// Spearman fitness: per batch of programs the predict
// kernels write yhat [B][m], spearman.cu ranks each row of it (ties averaged) and correlates the
// ranks with rank(y) (weighted Pearson). Ranks need every row: with row sharding across ranks this
// metric is refused; with GP_SHARD_PROGRAMS each rank ranks its own programs over all rows.
static gp_status evaluate_spearman(gp_context* ctx, const gp_node* programs,
                                   const int64_t* node_offsets, int32_t n_programs, int64_t n_nodes,
                                   int32_t max_stack, const float* X, int64_t ldx, const float* y,
                                   const float* w, int64_t n_rows, int32_t n_cols,
                                   float* fitness_out, uint32_t* status_out, bool fit_host,
                                   bool st_host, bool any_host) {
  gp_status s;
  const bool by_prog = ctx->comm && ctx->shard == GP_SHARD_PROGRAMS;
  if (ctx->comm && !by_prog)
    return ctx->fail(GP_ERR_UNSUPPORTED, "Spearman ranks need every row: use GP_SHARD_PROGRAMS");
  if (n_rows > INT32_MAX / 2)
    return ctx->fail(GP_ERR_ARG, "Spearman: n_rows %lld exceeds the int32 rank range", (long long)n_rows);
  const int32_t m = (int32_t)n_rows;
  const int32_t chunk = by_prog ? (n_programs + ctx->world - 1) / ctx->world : n_programs;
  const int32_t p_lo = by_prog ? std::min(n_programs, ctx->rank * chunk) : 0;
  const int32_t p_hi = by_prog ? std::min(n_programs, p_lo + chunk) : n_programs;
  const EvalPlan pl = plan_eval(ctx->device, n_rows, n_programs, n_cols, 1, true, false,
                                ctx->plan_G, ctx->plan_tpc);
  // compile every program (no bucket work yet: empty range)
  if ((s = prepare(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx, n_rows,
                   n_cols, pl.G, false, nullptr, &any_host, false, 0, 0))) return s;
  // batch size: ~2 GB of per-row buffers (yhat, ranks, sort / scan scratch ~ 32 B per entry)
  const int64_t budget = (int64_t)2 << 30;
  int32_t B = (int32_t)std::max<int64_t>(1, std::min<int64_t>(std::max(1, p_hi - p_lo),
                                                                budget / ((int64_t)m * 32)));
  B = (int32_t)std::min<int64_t>(B, INT32_MAX / m);
  if (const char* e = getenv("GP_SPEARMAN_BATCH")) B = std::max(1, std::min(B, atoi(e)));  // tests
  const size_t scratch = std::max(rank_scratch_bytes(B, m), rank_scratch_bytes(1, m));
  const int32_t Q = spearman_chunks(m);
  const size_t bytes = (size_t)B * m * 4 * 2 + (size_t)m * 4 + (size_t)B * 4 +
                       (size_t)B * Q * 6 * 8 + scratch + 1024;
  if ((s = ctx->grow(&ctx->spear.p, &ctx->spear.cap, bytes, "spearman"))) return s;
  char* p = (char*)ctx->spear.p;
  double* part = (double*)p;                       p += (size_t)B * Q * 6 * 8;
  float* yhat = (float*)p;                         p += (size_t)B * m * 4;
  int32_t* rank2 = (int32_t*)p;                    p += (size_t)B * m * 4;
  int32_t* ry2 = (int32_t*)p;                      p += (size_t)m * 4;
  uint32_t* nonfin = (uint32_t*)p;                 p += (size_t)B * 4;
  void* scr = (void*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
  // rank(y), once
  if ((s = ctx->launch(launch_rank(y, 1, m, scr, scratch, ry2, nullptr, ctx->stream), "rank y"))) return s;
  float* fit_dev = fitness_out;
  if (fit_host) {
    if ((s = ctx->grow(&ctx->h_fit.p, &ctx->h_fit.cap, (size_t)n_programs * sizeof(float), "fit"))) return s;
    fit_dev = (float*)ctx->h_fit.p;
  }
  for (int32_t lo = p_lo; lo < p_hi; lo += B) {
    const int32_t hi = std::min(p_hi, lo + B), nb = hi - lo;
    if ((s = bucket_pack(ctx, n_programs, pl.G, false, lo, hi))) return s;
    EvalArgs a{};
    a.X = X;
    a.ldx = ldx;
    a.n_rows = n_rows;
    a.n_cols = n_cols;
    a.n_programs = n_programs;
    a.metric = GP_MSE;
    a.G = pl.G;
    a.rows_per_chunk = pl.rows_per_chunk;
    a.n_chunks = pl.n_chunks;
    a.out = yhat - (int64_t)lo * m;                // predict writes out[p * m + i], p in [lo, hi)
    a.ld_out = m;
    if ((s = launch_variants(ctx, a, pl, max_stack, true))) return s;
    if ((s = ctx->launch(launch_rank(yhat, nb, m, scr, scratch, rank2, nonfin, ctx->stream), "rank yhat"))) return s;
    if ((s = ctx->launch(launch_spearman(rank2, ry2, w, nb, m, part, nonfin,
                                       (const int32_t*)ctx->code_len.p + lo, fit_dev + lo,
                                       (uint32_t*)ctx->status.p + lo, ctx->stream), "spearman"))) return s;
  }
  if (by_prog && (s = gather_programs(ctx, n_programs, chunk, p_lo, p_hi, fit_dev))) return s;
  if (fit_host) {
    if ((s = ctx->cuda(cudaMemcpyAsync(fitness_out, fit_dev, (size_t)n_programs * sizeof(float),
                                       cudaMemcpyDeviceToHost, ctx->stream), "D2H fitness"))) return s;
  }
  if (status_out) {
    if ((s = ctx->cuda(cudaMemcpyAsync(status_out, ctx->status.p, (size_t)n_programs * sizeof(uint32_t),
                                       st_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                       ctx->stream), "status copy"))) return s;
  }
  if (any_host || fit_host || st_host) return ctx->cuda(cudaStreamSynchronize(ctx->stream), "sync");
  return GP_OK;
}

// The per-rank half of an evaluation: compile, dataset constants, fused evaluator
// launches, fixed-order reduction over row chunks -> ctx->sums (compact layout, kernels.h
// kConstCols). Shared by gp_evaluate and gp_evaluate_partial.
struct EvalRun {
  EvalPlan pl;
  int S = 1;
  bool closed = false, by_prog = false;
  int32_t chunk = 0, p_lo = 0, p_hi = 0;
  int64_t ld_part = 0;
};

static gp_status eval_sums(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                           int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float* X,
                           int64_t ldx, const float* y, const float* w, int64_t n_rows,
                           int32_t n_cols, gp_metric metric, bool* any_host, EvalRun* run) {
  gp_status s;
  const int S = metric == GP_PEARSON ? 3 : 1;
  run->S = S;
  run->pl = plan_eval(ctx->device, n_rows, n_programs, n_cols, S, false, w != nullptr,
                      ctx->plan_G, ctx->plan_tpc);
  const EvalPlan& pl = run->pl;
  // variable-free programs: closed form in finalize for MSE / RMSE / LogLoss / Pearson (not MAE)
  run->closed = ctx->const_programs && metric != GP_MAE;
  // population sharding: every rank holds all rows and evaluates the programs
  // [lo, hi) of equal-count chunks; fitness / status are all-gathered after finalize.
  // Without a communicator gp_context_set_program_range selects the range.
  run->by_prog = ctx->comm && ctx->shard == GP_SHARD_PROGRAMS;
  run->chunk = run->by_prog ? (n_programs + ctx->world - 1) / ctx->world : n_programs;
  if (run->by_prog) {
    run->p_lo = std::min(n_programs, ctx->rank * run->chunk);
    run->p_hi = std::min(n_programs, run->p_lo + run->chunk);
  } else {
    run->p_lo = std::min(n_programs, ctx->range_lo);
    run->p_hi = ctx->range_hi < 0 ? n_programs : std::min(n_programs, ctx->range_hi);
  }
  if ((s = prepare(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx, n_rows,
                   n_cols, pl.G, metric == GP_PEARSON, y, any_host, run->closed, run->p_lo,
                   run->p_hi))) return s;

  // Fused evaluation -> partial sums (compact columns: constants, then evaluated programs)
  const int64_t ld_part = kConstCols + (int64_t)n_programs * S;
  run->ld_part = ld_part;
  if ((s = ctx->grow(&ctx->partial.p, &ctx->partial.cap, (size_t)pl.n_chunks * ld_part * sizeof(double), "partial"))) return s;
  if ((s = ctx->grow(&ctx->sums.p, &ctx->sums.cap, (size_t)ld_part * sizeof(double), "sums"))) return s;
  EvalArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.y = y;
  a.w = w;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.n_programs = n_programs;
  a.metric = metric;
  a.G = pl.G;
  a.rows_per_chunk = pl.rows_per_chunk;
  a.n_chunks = pl.n_chunks;
  a.partial = (double*)ctx->partial.p;
  a.ld_part = ld_part;
  a.shift = metric == GP_PEARSON ? (const float*)ctx->shift.p : nullptr;
  a.y_shift = metric == GP_PEARSON ? (const float*)ctx->shift.p + n_programs : nullptr;
  ctx->last_plan = pl;
  if ((s = ctx->launch(launch_consts(y, w, n_rows, pl.rows_per_chunk, pl.n_chunks, a.y_shift,
                                   a.partial, ld_part, 0, metric == GP_LOGLOSS ? 1 : 0,
                                   ctx->stream),
                     "consts kernel"))) return s;
  if ((s = launch_variants(ctx, a, pl, max_stack, false))) return s;
  return ctx->launch(launch_tile_reduce((const double*)ctx->partial.p, pl.n_chunks, ld_part,
                                        (const int32_t*)ctx->inv.p + n_programs + kNumVariants, S,
                                        (double*)ctx->sums.p, ctx->stream),
                     "tile_reduce");
}

// Fitness / status to the caller's buffers after finalize (+ the program-shard all-gather).
static gp_status deliver(gp_context* ctx, const EvalRun& run, int32_t n_programs, float* fit_dev,
                         float* fitness_out, uint32_t* status_out, bool fit_host, bool st_host,
                         bool any_host) {
  gp_status s;
  if (run.by_prog && (s = gather_programs(ctx, n_programs, run.chunk, run.p_lo, run.p_hi, fit_dev))) return s;
  if (fit_host) {
    if ((s = ctx->cuda(cudaMemcpyAsync(fitness_out, fit_dev, (size_t)n_programs * sizeof(float),
                                       cudaMemcpyDeviceToHost, ctx->stream), "D2H fitness"))) return s;
  }
  if (status_out) {
    if ((s = ctx->cuda(cudaMemcpyAsync(status_out, ctx->status.p, (size_t)n_programs * sizeof(uint32_t),
                                       st_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                       ctx->stream), "status copy"))) return s;
  }
  if (any_host || fit_host || st_host) return ctx->cuda(cudaStreamSynchronize(ctx->stream), "sync");
  return GP_OK;
}

gp_status gp_evaluate(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                      int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float* X,
                      int64_t ldx, const float* y, const float* w, int64_t n_rows, int32_t n_cols,
                      gp_metric metric, float* fitness_out, uint32_t* status_out) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  if ((int)metric < 0 || (int)metric > GP_SPEARMAN || !y || !fitness_out)
    return ctx->fail(GP_ERR_ARG, "invalid metric / y / fitness_out");
  bool any_host = false;
  gp_status s;
  const void* d;
  if ((s = ctx->stage_in(y, (size_t)n_rows * sizeof(float), ctx->h_y, &d, &any_host))) return s;
  y = (const float*)d;
  if (w) {
    if ((s = ctx->stage_in(w, (size_t)n_rows * sizeof(float), ctx->h_w, &d, &any_host))) return s;
    w = (const float*)d;
  }
  const bool fit_host = is_host_pointer(fitness_out);
  const bool st_host = status_out && is_host_pointer(status_out);
  if (metric == GP_SPEARMAN)
    return evaluate_spearman(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx, y,
                             w, n_rows, n_cols, fitness_out, status_out, fit_host, st_host,
                             any_host);
  EvalRun run;
  if ((s = eval_sums(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx, y, w,
                     n_rows, n_cols, metric, &any_host, &run))) return s;
  // A6: one all-reduce of the fp64 sums across ranks (rows are sharded; every rank has the same
  // compact layout because it holds the same population)
  if (ctx->comm && !run.by_prog) {
    NcclApi& n = nccl();
    ncclResult_t r = n.AllReduce(ctx->sums.p, ctx->sums.p, (size_t)run.ld_part, ncclFloat64,
                                 ncclSum, (ncclComm_t)ctx->comm, ctx->stream);
    if (r != ncclSuccess) return ctx->fail(GP_ERR_NCCL, "ncclAllReduce: %s", n.GetErrorString(r));
  }
  // A7: finalize
  float* fit_dev = fitness_out;
  if (fit_host) {
    if ((s = ctx->grow(&ctx->h_fit.p, &ctx->h_fit.cap, (size_t)n_programs * sizeof(float), "fit"))) return s;
    fit_dev = (float*)ctx->h_fit.p;
  }
  const double* sums = (const double*)ctx->sums.p;
  if ((s = ctx->launch(launch_finalize(sums, sums + kConstCols, (const int32_t*)ctx->inv.p,
                                       n_programs, metric,
                                       (const int32_t*)ctx->code_len.p, (const int32_t*)ctx->need.p,
                                       (const uint4*)ctx->code.p, (const int64_t*)ctx->code_off.p,
                                       run.closed ? 1 : 0, fit_dev,
                                       (uint32_t*)ctx->status.p, ctx->stream), "finalize"))) return s;
  return deliver(ctx, run, n_programs, fit_dev, fitness_out, status_out, fit_host, st_host, any_host);
}

gp_status gp_evaluate_partial(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                              int32_t n_programs, int64_t n_nodes, int32_t max_stack,
                              const float* X, int64_t ldx, const float* y, const float* w,
                              int64_t n_rows, int32_t n_cols, gp_metric metric, double* sums_out) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  if ((int)metric < 0 || (int)metric > GP_SPEARMAN || !y || !sums_out)
    return ctx->fail(GP_ERR_ARG, "invalid metric / y / sums_out");
  if (metric == GP_SPEARMAN)
    return ctx->fail(GP_ERR_UNSUPPORTED, "Spearman ranks are not additive over row shards");
  if (ctx->comm && ctx->shard == GP_SHARD_PROGRAMS)
    return ctx->fail(GP_ERR_ARG, "gp_evaluate_partial: program sharding has no row partials");
  bool any_host = false;
  gp_status s;
  const void* d;
  if ((s = ctx->stage_in(y, (size_t)n_rows * sizeof(float), ctx->h_y, &d, &any_host))) return s;
  y = (const float*)d;
  if (w) {
    if ((s = ctx->stage_in(w, (size_t)n_rows * sizeof(float), ctx->h_w, &d, &any_host))) return s;
    w = (const float*)d;
  }
  EvalRun run;
  if ((s = eval_sums(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx, y, w,
                     n_rows, n_cols, metric, &any_host, &run))) return s;
  const bool out_host = is_host_pointer(sums_out);
  double* dst = sums_out;
  const size_t bytes = (size_t)run.ld_part * sizeof(double);
  if (out_host) {
    if ((s = ctx->grow(&ctx->sums_x.p, &ctx->sums_x.cap, bytes, "sums_x"))) return s;
    dst = (double*)ctx->sums_x.p;
  }
  if ((s = ctx->launch(launch_expand_sums((const double*)ctx->sums.p, (const int32_t*)ctx->inv.p,
                                          n_programs, run.S, dst, ctx->stream), "expand sums"))) return s;
  if (out_host) {
    if ((s = ctx->cuda(cudaMemcpyAsync(sums_out, dst, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H sums"))) return s;
  }
  if (any_host || out_host) return ctx->cuda(cudaStreamSynchronize(ctx->stream), "sync");
  return GP_OK;
}

gp_status gp_finalize_sums(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                           int32_t n_programs, int64_t n_nodes, int32_t max_stack, int32_t n_cols,
                           const double* sums, gp_metric metric, float* fitness_out,
                           uint32_t* status_out) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  if ((int)metric < 0 || (int)metric >= GP_SPEARMAN || !sums || !fitness_out)
    return ctx->fail(GP_ERR_ARG, "invalid metric / sums / fitness_out");
  bool any_host = false;
  gp_status s;
  const int S = metric == GP_PEARSON ? 3 : 1;
  const void* d;
  if ((s = ctx->stage_in(sums, ((size_t)n_programs * S + kConstCols) * sizeof(double), ctx->sums_x, &d, &any_host))) return s;
  const double* sd = (const double*)d;
  // compile (status bits, closed-form constants); a dummy 1-row X is never read by the stage
  // kernel, so only the column count matters
  EvalRun run;
  run.S = S;
  run.closed = ctx->const_programs && metric != GP_MAE;
  run.p_lo = 0;
  run.p_hi = n_programs;
  const float* Xdummy = (const float*)sd;
  if ((s = prepare(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, Xdummy, 1, 1,
                   n_cols, 1, false, nullptr, &any_host, run.closed, 0, 0))) return s;
  const bool fit_host = is_host_pointer(fitness_out);
  const bool st_host = status_out && is_host_pointer(status_out);
  float* fit_dev = fitness_out;
  if (fit_host) {
    if ((s = ctx->grow(&ctx->h_fit.p, &ctx->h_fit.cap, (size_t)n_programs * sizeof(float), "fit"))) return s;
    fit_dev = (float*)ctx->h_fit.p;
  }
  if ((s = ctx->launch(launch_finalize(sd + (int64_t)n_programs * S, sd, nullptr, n_programs,
                                       metric, (const int32_t*)ctx->code_len.p,
                                       (const int32_t*)ctx->need.p, (const uint4*)ctx->code.p,
                                       (const int64_t*)ctx->code_off.p, run.closed ? 1 : 0,
                                       fit_dev, (uint32_t*)ctx->status.p, ctx->stream),
                       "finalize"))) return s;
  return deliver(ctx, run, n_programs, fit_dev, fitness_out, status_out, fit_host, st_host, any_host);
}

gp_status gp_predict(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                     int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float* X,
                     int64_t ldx, int64_t n_rows, int32_t n_cols, float* out, int64_t ld_out,
                     uint32_t* status_out) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  if (!out || ld_out < n_rows) return ctx->fail(GP_ERR_ARG, "invalid out / ld_out");
  bool any_host = false;
  const EvalPlan pl = plan_eval(ctx->device, n_rows, n_programs, n_cols, 1, true, false,
                                ctx->plan_G, ctx->plan_tpc);
  gp_status s = prepare(ctx, programs, node_offsets, n_programs, n_nodes, max_stack, X, ldx,
                        n_rows, n_cols, pl.G, false, nullptr, &any_host);
  if (s) return s;
  EvalArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.n_programs = n_programs;
  a.metric = GP_MSE;
  a.G = pl.G;
  a.rows_per_chunk = pl.rows_per_chunk;
  a.n_chunks = pl.n_chunks;
  a.out = out;
  a.ld_out = ld_out;
  if ((s = launch_variants(ctx, a, pl, max_stack, true))) return s;
  if (status_out) {
    const bool st_host = is_host_pointer(status_out);
    if ((s = ctx->cuda(cudaMemcpyAsync(status_out, ctx->status.p, (size_t)n_programs * sizeof(uint32_t),
                                       st_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                       ctx->stream), "status copy"))) return s;
    if (st_host) any_host = true;
  }
  if (any_host) return ctx->cuda(cudaStreamSynchronize(ctx->stream), "sync");
  return GP_OK;
}

gp_status gp_tournament_select(gp_context* ctx, const float* fitness, const int64_t* node_offsets,
                               int32_t n_programs, int32_t n_tournaments, int32_t tournament_size,
                               float parsimony, int32_t higher_is_better, uint64_t seed,
                               uint32_t generation, int32_t* winners_out) {
  if (!ctx) return GP_ERR_ARG;
  cudaSetDevice(ctx->device);
  if (!fitness || !node_offsets || !winners_out || n_programs < 1 || n_tournaments < 1 ||
      tournament_size < 1)
    return ctx->fail(GP_ERR_ARG, "invalid tournament arguments (n=%d T=%d k=%d)", n_programs,
                     n_tournaments, tournament_size);
  return ctx->launch(launch_select(fitness, node_offsets, n_programs, n_tournaments, tournament_size,
                                 parsimony, higher_is_better ? 1 : 0, seed, generation,
                                 winners_out, ctx->stream), "select kernel");
}

}  // extern "C"
