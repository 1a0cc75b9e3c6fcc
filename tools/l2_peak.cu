// L2 read bandwidth microbenchmark (the ceiling of the wide-dataset evaluator, whose variable
// operands are L2 loads: DESIGN.md section 8). Every CTA streams a buffer that fits in L2 with
// 16-byte loads, either cached in L2 only (ld.global.cg) or through L1 (ld.global.nc), many times;
// bandwidth = bytes read / CUDA-event time. The buffer is read once before timing (L2 warm).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_peak tools/l2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool CG>
__global__ void l2read(const float4* __restrict__ p, long long n4, int iters, float* out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = CG ? __ldcg(p + i) : __ldg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 123456.0f) out[0] = acc.x;  // keeps the loads live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("%s SMs=%d l2=%d\n", prop.name, sms, prop.l2CacheSize);
  float* out;
  cudaMalloc(&out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (long long mb : {8LL, 16LL, 32LL, 48LL, 64LL, 256LL}) {
    const long long bytes = mb << 20, n4 = bytes / 16;
    float4* p;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0, bytes);
    const int iters = mb >= 256 ? 4 : (int)(4096 / mb);
    for (int cg = 1; cg >= 0; --cg) {
      for (int ctas_per_sm : {4, 8}) {
        const int grid = sms * ctas_per_sm, nt = 256;
        if (cg) l2read<true><<<grid, nt>>>(p, n4, 1, out); else l2read<false><<<grid, nt>>>(p, n4, 1, out);
        cudaEventRecord(a);
        if (cg) l2read<true><<<grid, nt>>>(p, n4, iters, out); else l2read<false><<<grid, nt>>>(p, n4, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        printf("%4lld MB  %s  %d CTAs/SM x 256  %8.3f ms  %8.1f GB/s\n", mb, cg ? "ld.cg (L2)  " : "ld.nc (L1+L2)",
               ctas_per_sm, ms, (double)bytes * iters / (ms * 1e-3) / 1e9);
      }
    }
    cudaFree(p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
