// gp_internal.h -- host-side internals shared by api.cpp and engine.cpp (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/gp.h"
#include "aux.h"

namespace gpb {

struct StageBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct EvalPlan {
  bool xsmem = true;
  int G = 1, n_groups = 1, occupancy = 1;
  int64_t n_chunks = 1, rows_per_chunk = 0;
  int item_order = 0;        // 0: program group fastest, 1: row chunk fastest (EvalArgs)
};

bool is_host_pointer(const void* p);
int sm_count(int device);
EvalPlan plan_eval(int device, int64_t n_rows, int32_t n_programs, int32_t n_cols, int S,
                   bool predict, bool weighted, int force_G = 0, int64_t force_tpc = 0);

}  // namespace gpb

struct gp_context {
  int device = 0, rank = 0, world = 1, sms = 148;
  cudaStream_t stream = nullptr;
  void* comm = nullptr;  // ncclComm_t
  std::string err;
  // device workspaces (grown on demand, stream-ordered)
  gpb::StageBuf gather, spear, code, code_off, code_len, need, lists, pos, gstart, counts, codestream, scratch, status, partial,
      sums, shift, xref, inv, xref_b, sums_x;
  // staging for [host] arguments
  gpb::StageBuf h_nodes, h_off, h_X, h_y, h_w, h_fit;
  std::vector<float> xref_host;
  int xref_cols = 0;
  gpb::EvalPlan last_plan;
  // eval-kernel timing (gp_context_set_profiling)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending, ev_free;
  double prof_ms = 0.0;
  int64_t prof_launches = 0;
  int64_t kernel_launches = 0;   // gp_context_kernel_launches
  bool sethi_ullman = true;      // gp_context_set_eval_order
  bool const_programs = true;    // gp_context_set_const_programs (closed-form constant programs)
  gp_shard shard = GP_SHARD_ROWS;  // gp_context_set_shard
  int plan_G = 0;                // gp_context_set_plan (0 = automatic)
  int64_t plan_tpc = 0;
  int32_t range_lo = 0, range_hi = -1;  // gp_context_set_program_range

  std::vector<gpb::StageBuf*> all_buffers() {
    return {&gather, &spear, &code, &code_off, &code_len, &need, &lists, &pos, &gstart, &counts, &codestream, &scratch, &status,
            &partial, &sums, &shift, &xref, &inv, &xref_b, &sums_x,
            &h_nodes, &h_off, &h_X, &h_y, &h_w, &h_fit};
  }
  gp_status fail(gp_status s, const char* fmt, ...);
  gp_status cuda(cudaError_t e, const char* what);
  gp_status launch(cudaError_t e, const char* what);  // cuda() + counts a successful launch
  gp_status grow(void** p, size_t* cap, size_t bytes, const char* what);
  gp_status stage_in(const void* src, size_t bytes, gpb::StageBuf& buf, const void** dst,
                     bool* was_host);
};
