// aux.h -- launchers of the small kernels in aux.cu (stage, bucket/layout, pack, shift, consts,
// tile reduce, finalize, select). Included by aux.cu and the host layer only, so the evaluator
// translation units do not depend on it.
#pragma once
#include "kernels.h"

namespace gpb {

// aux.cu
cudaError_t launch_stage(const gp_node* nodes, const int64_t* offsets, int32_t n_programs,
                         int64_t n_nodes, int32_t n_cols, int32_t max_stack, uint4* code,
                         int64_t* code_off, int32_t* code_len, int32_t* need, uint32_t* status,
                         int32_t* scratch /* 4 x n_nodes int32 */, int32_t sethi_ullman,
                         cudaStream_t s);
// Partitions valid programs by stack need into kNumVariants ascending lists, lays out each
// variant's code stream (per-program offsets, group starts for G programs per group), zeroes the
// work counters. lists/pos: [kNumVariants][n_programs]; gstart: [kNumVariants][n_programs + 1];
// counts: [kNumVariants] then counters [kNumVariants]; base: [kNumVariants + 1] stream bases;
// inv: [n] compact partial-sum position of each program (-1: not evaluated), then
// [kNumVariants + 1] bucket start positions and the evaluated total, then [kNumVariants] the
// bucket group sizes (<= G: as many groups per bucket as the plan has for the population).
cudaError_t launch_bucket(const int32_t* need, const int32_t* code_len, int32_t n_programs,
                          int32_t G, const int* subs, int32_t* lists, int64_t* pos,
                          int64_t* gstart, int32_t* counts, int64_t* base, int32_t skip_const,
                          int32_t p_lo, int32_t p_hi, int32_t* inv /* n + 2 kNumVariants + 1 */,
                          cudaStream_t s);
// Copies every bucketed program's code into its variant stream, flagging the end of each pass
// and of each shared-memory stream window (kernels.h kEndWin).
cudaError_t launch_pack(const uint4* code, const int64_t* code_off, const int32_t* code_len,
                        const int32_t* lists, const int64_t* pos, const int32_t* counts,
                        const int64_t* base, const int64_t* gstart, int32_t n_programs,
                        const int* subs, const int32_t* inv /* bucket group sizes at n + 5 */,
                        uint4* stream, cudaStream_t s);
// Dataset constants W, S_y, S_yy per row chunk -> partial[q][col0 .. col0 + 2].
cudaError_t launch_consts(const float* y, const float* w, int64_t n_rows, int64_t rows_per_chunk,
                          int64_t n_chunks, const float* y_shift, double* partial, int64_t ld_part,
                          int64_t col0, int32_t logloss, cudaStream_t s);
cudaError_t launch_shift(const uint4* code, const int64_t* code_off, const int32_t* code_len,
                         int32_t n_programs, int32_t stack_cap, const float* xref,
                         int64_t xref_stride, float* shift_out, cudaStream_t s);
// sums[j] = fixed-order sum over row chunks of partial[q][j], j < kConstCols + S * (*live)
cudaError_t launch_tile_reduce(const double* partial, int64_t n_chunks, int64_t ld_part,
                               const int32_t* live, int32_t S, double* sums, cudaStream_t s);
// compact sums -> program order [n][S] (0 for programs not evaluated) + the kConstCols constants
cudaError_t launch_expand_sums(const double* sums, const int32_t* inv, int32_t n, int32_t S,
                               double* out, cudaStream_t s);
// dst[0 .. n_cols) = row 0 of X, dst[n_cols] = y[0]
cudaError_t launch_gather_row(const float* X, int64_t ldx, int32_t n_cols, const float* y,
                              float* dst, cudaStream_t s);
// closed_const: variable-free programs (need 0) skipped by the evaluator get their loss from the
// dataset moments (MSE / RMSE) or an undefined correlation (Pearson).
// consts: W, S_y, S_yy; psums: S sums per program at position idx[p] (null: p; -1: none)
cudaError_t launch_finalize(const double* consts, const double* psums, const int32_t* idx,
                            int32_t n_programs, int32_t metric,
                            const int32_t* code_len, const int32_t* need, const uint4* code,
                            const int64_t* code_off, int32_t closed_const, float* fitness,
                            uint32_t* status, cudaStream_t s);
cudaError_t launch_select(const float* fitness, const int64_t* offsets, int32_t n_programs,
                          int32_t n_tournaments, int32_t k, float parsimony, int32_t higher,
                          uint64_t seed, uint32_t generation, int32_t* winners, cudaStream_t s);
cudaError_t launch_copy_scalar(const float* src, float* dst, cudaStream_t s);

// ---- Spearman (spearman.cu) ----------------------------------------------------------
// Doubled tie-averaged ranks of B segments of m fp32 keys (B m <= INT32_MAX):
// rank2[b m + i] = 2 rank of keys[b m + i] within segment b; nonfinite[b] (optional) = any
// non-finite key in segment b. scratch >= rank_scratch_bytes(B, m) device bytes.
size_t rank_scratch_bytes(int32_t B, int32_t m);
cudaError_t launch_rank(const float* keys, int32_t B, int32_t m, void* scratch,
                        size_t scratch_bytes, int32_t* rank2, uint32_t* nonfinite, cudaStream_t s);
// Weighted Pearson of rank2 [B][m] against ry2 [m] -> fitness[b], status[b] (|= undefined
// flag); part: [B][spearman_chunks(m)][6] fp64 scratch. code_len[b] == 0 -> -inf.
int32_t spearman_chunks(int32_t m);
cudaError_t launch_spearman(const int32_t* rank2, const int32_t* ry2, const float* w, int32_t B,
                            int32_t m, double* part, const uint32_t* nonfinite,
                            const int32_t* code_len, float* fitness, uint32_t* status,
                            cudaStream_t s);

}  // namespace gpb
