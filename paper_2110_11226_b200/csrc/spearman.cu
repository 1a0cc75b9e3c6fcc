// spearman.cu -- Spearman fitness ("Spearman's Rank Correlation
// Coefficient"; S:201 Pearson of rank_vector(y) and rank_vector(yhat) with the same weights;
// S:209-215 ranks 1..n with ties averaged).
//
// Ranks need every row of a program's predictions at once, so this metric cannot stream through
// the fused evaluator: per batch of B programs the predict kernels write yhat [B][m] (fp32, the
// evaluator's precision), then
//   1. a segmented radix sort (CUB, a library sort step) orders each program's (yhat, row) pairs,
//   2. run starts are max-scanned (CUB) and each run's last element scatters its end to the run's
//      start, so every element knows its tie run [s, e) -> doubled rank s + e + 1 (exact int32),
//      scattered back to the row's position,
//   3. a fixed-order fp64 reduction per (program, row chunk) forms the weighted rank sums about the
//      rank midpoint (m + 1) / 2, and a finalize kernel turns them into r (Pearson).
// rank(y) is computed once per call with the same steps (B = 1). Rows with w = 0 are ranked (S:210
// ranks the whole vector) but skipped in the weighted sums. Non-finite predictions leave the ranks
// undefined -> r = 0 with GP_FLAG_UNDEFINED_CORR, as for an undefined Pearson correlation.
#include <cub/cub.cuh>
#include <cfloat>
#include "aux.h"

namespace gpb {

namespace {
struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

__global__ void rank_prep_kernel(const float* __restrict__ keys, int32_t B, int32_t m,
                                 int32_t* __restrict__ idx, int32_t* __restrict__ seg_off,
                                 uint32_t* __restrict__ nonfinite) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= B) seg_off[i] = (int32_t)(i * m);       // segment b = rows [b m, (b + 1) m)
  if (i >= (int64_t)B * m) return;
  idx[i] = (int32_t)(i % m);
  if (nonfinite && !isfinite(keys[i])) atomicOr(nonfinite + i / m, 1u);
}

// run starts of the sorted keys (a segment start is always a run start)
__global__ void run_start_kernel(const float* __restrict__ k, int32_t total, int32_t m,
                                 int32_t* __restrict__ start) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  start[i] = (i % m == 0 || k[i] != k[i - 1]) ? i : 0;
}

// the last element of each run writes the run's end (exclusive) at the run's start
__global__ void run_end_kernel(const float* __restrict__ k, const int32_t* __restrict__ s,
                               int32_t total, int32_t m, int32_t* __restrict__ end_at_start) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  if (i % m == m - 1 || k[i + 1] != k[i]) end_at_start[s[i]] = i + 1;
}

// doubled average rank (s + 1 + e) in segment-local positions, scattered to the row
__global__ void rank_scatter_kernel(const int32_t* __restrict__ s,
                                    const int32_t* __restrict__ end_at_start,
                                    const int32_t* __restrict__ row, int32_t total, int32_t m,
                                    int32_t* __restrict__ rank2) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int32_t base = (i / m) * m, st = s[i], en = end_at_start[st];
  rank2[base + row[i]] = (st - base) + (en - base) + 1;
}

constexpr int kSumThreads = 256;

// weighted rank sums of program b over row chunk q: W, Sa, Sb, Saa, Sbb, Sab about (m + 1) / 2
__global__ void spearman_sums_kernel(const int32_t* __restrict__ rank2,
                                     const int32_t* __restrict__ ry2, const float* __restrict__ w,
                                     int32_t m, int32_t rows_per_q, double* __restrict__ part) {
  __shared__ double red[6][kSumThreads];
  const int q = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int32_t r0 = q * rows_per_q, r1 = min(m, r0 + rows_per_q);
  const double mid = 0.5 * ((double)m + 1.0);
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int32_t* ra = rank2 + (int64_t)b * m;
  for (int32_t i = r0 + tid; i < r1; i += kSumThreads) {
    const double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    const double x = 0.5 * ra[i] - mid, yv = 0.5 * ry2[i] - mid;
    acc[0] += wi;
    acc[1] += wi * x;
    acc[2] += wi * yv;
    acc[3] += wi * x * x;
    acc[4] += wi * yv * yv;
    acc[5] += wi * x * yv;
  }
  for (int k = 0; k < 6; ++k) red[k][tid] = acc[k];
  __syncthreads();
  for (int o = kSumThreads / 2; o > 0; o >>= 1) {
    if (tid < o)
      for (int k = 0; k < 6; ++k) red[k][tid] += red[k][tid + o];
    __syncthreads();
  }
  if (tid < 6) part[((int64_t)b * gridDim.x + q) * 6 + tid] = red[tid][0];
}

__global__ void spearman_finalize_kernel(const double* __restrict__ part, int32_t B, int32_t Q,
                                         const uint32_t* __restrict__ nonfinite,
                                         const int32_t* __restrict__ code_len,
                                         float* __restrict__ fitness, uint32_t* __restrict__ status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double t[6] = {0, 0, 0, 0, 0, 0};
  for (int q = 0; q < Q; ++q)
    for (int k = 0; k < 6; ++k) t[k] += part[((int64_t)b * Q + q) * 6 + k];
  uint32_t fl = status[b];
  float out;
  if (code_len[b] == 0) {
    out = -INFINITY;
  } else {
    const double W = t[0];
    const double cov = t[5] - t[1] * t[2] / W, va = t[3] - t[1] * t[1] / W,
                 vb = t[4] - t[2] * t[2] / W;
    double r = cov / sqrt(va * vb);
    if (nonfinite[b] || !(va > 0.0) || !(vb > 0.0) || !isfinite(r)) {
      r = 0.0;
      fl |= GP_FLAG_UNDEFINED_CORR;
    }
    r = r > 1.0 ? 1.0 : (r < -1.0 ? -1.0 : r);
    out = (float)r;
  }
  fitness[b] = out;
  status[b] = fl;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

// scratch: idx_in, keys_out, idx_out, run start, run end (B m int32 / fp32 each), segment
// offsets (B + 1), CUB temp storage
size_t rank_scratch_bytes(int32_t B, int32_t m) {
  const int32_t total = B * m;
  size_t sort_tmp = 0, scan_tmp = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sort_tmp, (const float*)nullptr,
                                           (float*)nullptr, (const int32_t*)nullptr,
                                           (int32_t*)nullptr, total, B, (const int32_t*)nullptr,
                                           (const int32_t*)nullptr);
  cub::DeviceScan::InclusiveScan(nullptr, scan_tmp, (const int32_t*)nullptr, (int32_t*)nullptr,
                                 MaxOp(), total);
  const size_t arrays = (size_t)5 * total * 4 + (size_t)(B + 1) * 4;
  return ((arrays + 255) & ~(size_t)255) + std::max(sort_tmp, scan_tmp) + 256;
}

cudaError_t launch_rank(const float* keys, int32_t B, int32_t m, void* scratch,
                        size_t scratch_bytes, int32_t* rank2, uint32_t* nonfinite,
                        cudaStream_t s) {
  const int32_t total = B * m;
  char* p = (char*)scratch;
  int32_t* idx_in = (int32_t*)p;
  float* kout = (float*)(idx_in + total);
  int32_t* iout = (int32_t*)(kout + total);
  int32_t* rs = iout + total;
  int32_t* re = rs + total;
  int32_t* off = re + total;
  const size_t arrays = (size_t)5 * total * 4 + (size_t)(B + 1) * 4;
  void* tmp = p + ((arrays + 255) & ~(size_t)255);
  size_t tmp_bytes = scratch_bytes - ((arrays + 255) & ~(size_t)255);
  const int nt = 256;
  if (nonfinite) {
    cudaError_t e = cudaMemsetAsync(nonfinite, 0, (size_t)B * 4, s);
    if (e != cudaSuccess) return e;
  }
  rank_prep_kernel<<<nblk(std::max<int64_t>(total, B + 1), nt), nt, 0, s>>>(keys, B, m, idx_in,
                                                                             off, nonfinite);
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(tmp, tmp_bytes, keys, kout, idx_in,
                                                           iout, total, B, off, off + 1, 0, 32, s);
  if (e != cudaSuccess) return e;
  run_start_kernel<<<nblk(total, nt), nt, 0, s>>>(kout, total, m, re);
  e = cub::DeviceScan::InclusiveScan(tmp, tmp_bytes, re, rs, MaxOp(), total, s);
  if (e != cudaSuccess) return e;
  run_end_kernel<<<nblk(total, nt), nt, 0, s>>>(kout, rs, total, m, re);
  rank_scatter_kernel<<<nblk(total, nt), nt, 0, s>>>(rs, re, iout, total, m, rank2);
  return cudaGetLastError();
}

int32_t spearman_chunks(int32_t m) { return std::max(1, std::min(64, (m + 65535) / 65536)); }

cudaError_t launch_spearman(const int32_t* rank2, const int32_t* ry2, const float* w, int32_t B,
                            int32_t m, double* part, const uint32_t* nonfinite,
                            const int32_t* code_len, float* fitness, uint32_t* status,
                            cudaStream_t s) {
  const int32_t Q = spearman_chunks(m);
  const int32_t rows_per_q = (m + Q - 1) / Q;
  spearman_sums_kernel<<<dim3(Q, B), kSumThreads, 0, s>>>(rank2, ry2, w, m, rows_per_q, part);
  spearman_finalize_kernel<<<nblk(B, 128), 128, 0, s>>>(part, B, Q, nonfinite, code_len, fitness,
                                                         status);
  return cudaGetLastError();
}

}  // namespace gpb
