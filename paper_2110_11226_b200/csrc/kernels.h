// kernels.h -- internal launch interface between the CUDA translation units and the C-ABI layer.
// Plain C++ (no CUDA-only syntax) so api.cpp / engine.cpp can include it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/gp.h"

namespace gpb {

// Case ids of the compiled code use ONE slot stride for every evaluator variant (so the stage
// kernel is variant independent): case id = opv * kCaseStride + slot.
constexpr int kCaseStride = GP_MAX_STACK;
// Row tiles (NT * R * SUB): the shared-memory-X shapes s4..s20 (512 threads) stage 8192-row
// tiles; the wide-dataset shapes w4 / w8 (global-memory X) work on 4096- / 2048-row tiles. Row
// chunks are whole tiles of the plan's tile: kTileSmem when X is staged in shared memory, else
// kTileGlobal (every wide shape's tile divides it).
constexpr int kTile = 2048;
constexpr int kTileGlobal = 4096;
constexpr int kTileSmem = 8192;
// Dynamic shared-memory opt-in of the evaluator kernels (227 KB per CTA minus the kernels' 16 B of
// static shared memory, rounded down).
constexpr int kMaxDynSmem = 227 * 1024 - 256;
// Evaluator variants by register-stack capacity; program p runs in the first variant whose
// capacity >= its stack need (bucketed on the device, no host synchronisation).
constexpr int kNumVariants = 4;
constexpr int kVariantStack[kNumVariants] = {4, 8, 12, 20};

// Pass flags in .w of the LAST code word of each row pass of a program in a code stream:
// bits 0-1 = kEndPass (another pass follows; bits 8.. = its index) or kEndProgram (bits 8.. =
// the program's slot in its group). kEndWin (bit 2) marks the last word of a shared-memory
// stream window (every kStreamWin-th word of a group's stream, and its last word), so the
// evaluator's word loop needs no trip counter.
constexpr uint32_t kEndPass = 1u, kEndProgram = 2u, kEndWin = 4u;
// Code-stream window staged in shared memory per CTA (words of 16 B).
constexpr int kStreamWin = 768;
// Per-warp transposed reduction block of the single-sum metrics (eval_impl.cuh): GP_RED_ROWS
// programs x 32 lanes of fp32 per-lane sums, rows padded to kRedStride floats so the row-part
// LDS.128 reads of a warp hit 32 distinct banks.
constexpr int kRedStride = 36;
// Partial-sum rows (per row chunk): columns 0..2 hold the dataset constants (W, S_y, S_yy; consts
// kernel), then S sums per EVALUATED program in compact bucket order (variable-free programs
// with a closed form and programs outside the evaluated range take no column).
constexpr int kConstCols = 3;

// Everything the fused evaluator needs for one launch (see eval_impl.cuh). Each variant runs a
// packed CODE STREAM per program group: for every program of the group, SUB copies of its code
// words (one per row pass), the last word of each pass flagged in .w -- so the evaluator walks one
// contiguous stream with an uninterrupted prefetch and does the loss / reduction after the flagged
// word, without a separate dispatch.
struct EvalArgs {
  const uint4* stream;        // this variant's packed stream (+2 pad words)
  const int64_t* gstart;      // [n_groups + 1] stream offsets of the program groups
  const int32_t* prog_ids;    // [count] program index of each bucket slot (the bucket list)
  const int32_t* prog_count;  // device: number of programs in the bucket
  int32_t* work_counter;      // device: persistent-CTA work queue (zeroed by the bucket kernel)
  const float* X;             // column-major, X[c * ldx + i]
  int64_t ldx;
  const float* y;             // [n_rows] (FIT mode)
  const float* w;             // [n_rows] or nullptr (all ones)
  int64_t n_rows;
  int32_t n_cols;
  int32_t n_programs;
  int32_t metric;             // gp_metric
  int32_t G;                  // programs per group: the plan's bound (shared-memory layout)
  const int32_t* group_size;  // device: this variant's group size (<= G, bucket_kernel)
  int64_t rows_per_chunk;     // rows per work item (whole plan tiles)
  int64_t n_chunks;           // row chunks; work items = ceil(count / G) * n_chunks
  int32_t item_order;         // work-item order: 0 = program group fastest, 1 = row chunk fastest
  int32_t chunk_reverse;      // 1: row chunks are visited last to first (see launch_variants)
  double* partial;            // FIT: [n_chunks][ld_part], ld_part = kConstCols + n_programs * S
  int64_t ld_part;
  const int32_t* part_base;   // FIT, device: first compact partial slot of this variant's bucket
  const float* shift;         // Pearson: K_p per program
  const float* y_shift;       // Pearson: device scalar K_y
  float* out;                 // PREDICT: out[p * ld_out + i]
  int64_t ld_out;
};

// Static shape of one evaluator variant.
struct EvalShape {
  int stack;                  // register-stack capacity
  int R;                      // rows per thread per pass
  int SUB;                    // passes per program per tile (rows reduced together)
  int NT;                     // threads per CTA
  int tile() const { return NT * R * SUB; }
};

// Per-capacity evaluator translation units (eval_s4.cu, eval_s8.cu, eval_s12.cu, eval_s20.cu).
struct EvalVariant {
  EvalShape shape;
  // Launches the persistent evaluator with n_ctas CTAs; xsmem selects X staged in shared memory
  // (small n_cols) versus per-node L1/L2 loads (large n_cols).
  cudaError_t (*launch)(const EvalArgs& a, bool predict, bool xsmem, int n_ctas, size_t smem,
                        cudaStream_t s);
  // Resident CTAs per SM for the given dynamic shared memory.
  int (*occupancy)(bool predict, bool xsmem, size_t smem);
  // Dynamic shared memory of one launch: accumulators + reduction blocks for G programs x S sums
  // (FIT mode), the y / w tile, the X tile (xsmem) and the code-stream window.
  size_t (*smem_bytes)(int G, int S, int n_cols, int weighted, int xsmem, int predict);
};
const EvalVariant& eval_variant_s4();
const EvalVariant& eval_variant_s8();
const EvalVariant& eval_variant_s12();
const EvalVariant& eval_variant_s20();
// Wide-dataset shapes of the 4- and 8-slot variants (global-memory X only; eval_w4.cu,
// eval_w8.cu): same SUB as s4 / s8, so the packed code streams serve both.
const EvalVariant& eval_variant_w4();
const EvalVariant& eval_variant_w8();

}  // namespace gpb
