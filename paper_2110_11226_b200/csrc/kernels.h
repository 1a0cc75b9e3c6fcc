// kernels.h -- internal launch interface between the CUDA translation units and the C-ABI layer.
// Plain C++ (no CUDA-only syntax) so api.cpp / engine.cpp can include it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/gp.h"

namespace gpb {

// Everything the fused evaluator needs for one launch (see eval_impl.cuh).
struct EvalArgs {
  const uint2* code;          // compiled nodes, evaluation order, +2 pad words
  const int64_t* code_off;    // [n_programs] start of each program in code
  const int32_t* code_len;    // [n_programs] length, 0 = invalid (skipped)
  const float* X;             // column-major, X[c * ldx + i]
  int64_t ldx;
  const float* y;             // [n_rows] (FIT mode)
  const float* w;             // [n_rows] or nullptr (all ones)
  int64_t n_rows;
  int32_t n_cols;
  int32_t n_programs;
  int32_t metric;             // gp_metric
  int32_t G;                  // programs per group (grid.y = ceil(n_programs / G))
  int64_t rows_per_chunk;     // rows per work item (grid.x = ceil(n_rows / rows_per_chunk))
  double* partial;            // FIT: [grid.x][ld_part], ld_part = n_programs * S + 3
  int64_t ld_part;
  const float* shift;         // Pearson: K_p per program (nullptr otherwise)
  const float* y_shift;       // Pearson: device scalar K_y
  float* out;                 // PREDICT: out[p * ld_out + i]
  int64_t ld_out;
};

// Static shape of one evaluator variant (chosen by max stack need).
struct EvalShape {
  int stack;                  // register-stack capacity
  int R;                      // rows per thread per pass
  int SUB;                    // passes per program per tile (rows reduced together)
  int NT;                     // threads per CTA
  int tile() const { return NT * R * SUB; }
};

// Per-capacity evaluator translation units (eval_s8.cu, eval_s12.cu, eval_s20.cu).
struct EvalVariant {
  EvalShape shape;
  // Launches the evaluator; xsmem selects X staged in shared memory (small n_cols) versus
  // per-node L1/L2 loads (large n_cols). Returns the CUDA error of the launch.
  cudaError_t (*launch)(const EvalArgs& a, bool predict, bool xsmem, dim3 grid, size_t smem,
                        cudaStream_t s);
  // Resident CTAs per SM for the given dynamic shared memory.
  int (*occupancy)(bool predict, bool xsmem, size_t smem);
};
const EvalVariant& eval_variant_s8();
const EvalVariant& eval_variant_s12();
const EvalVariant& eval_variant_s20();

// aux.cu
cudaError_t launch_stage(const gp_node* nodes, const int64_t* offsets, int32_t n_programs,
                         int64_t n_nodes, int32_t n_cols, int32_t stack_cap, uint2* code,
                         int64_t* code_off, int32_t* code_len, uint32_t* status, cudaStream_t s);
cudaError_t launch_shift(const uint2* code, const int64_t* code_off, const int32_t* code_len,
                         int32_t n_programs, int32_t stack_cap, const float* xref,
                         int64_t xref_stride, float* shift_out, cudaStream_t s);
cudaError_t launch_tile_reduce(const double* partial, int64_t n_chunks, int64_t ld_part,
                               double* sums, cudaStream_t s);
cudaError_t launch_finalize(const double* sums, int32_t n_programs, int32_t metric,
                            const int32_t* code_len, float* fitness, uint32_t* status,
                            cudaStream_t s);
cudaError_t launch_select(const float* fitness, const int64_t* offsets, int32_t n_programs,
                          int32_t n_tournaments, int32_t k, float parsimony, int32_t higher,
                          uint64_t seed, uint32_t generation, int32_t* winners, cudaStream_t s);
cudaError_t launch_copy_scalar(const float* src, float* dst, cudaStream_t s);

}  // namespace gpb
