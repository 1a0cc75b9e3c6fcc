// Microbenchmark: per-SM throughput of the pipes the GP interpreter uses
// (MUFU.SIN / MUFU.COS / MUFU.RCP / MUFU.EX2 / MUFU.LG2 on the XU pipe, FFMA on the FMA pipe).
// Used to derive the "alu" roofline denominators in DESIGN.md. Prints ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITERS 4096
template <int OP>
__global__ void k(float* out, float seed, long long* cycles) {
  float a0 = seed + threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N_ITERS; ++i) {
#define STEP(a) \
    if (OP == 0) a = __sinf(a); \
    else if (OP == 1) a = __cosf(a); \
    else if (OP == 2) a = __frcp_rn(a) ; \
    else if (OP == 3) { asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a)); } \
    else if (OP == 4) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); } \
    else if (OP == 5) { asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(a)); } \
    else if (OP == 6) { asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(a)); } \
    else if (OP == 7) a = __fmaf_rn(a, 1.0001f, 0.5f);
    STEP(a0) STEP(a1) STEP(a2) STEP(a3) STEP(a4) STEP(a5) STEP(a6) STEP(a7)
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}
template <int OP> void run(const char* name, int sms) {
  float* out; long long* cyc; cudaMalloc(&out, sizeof(float) * sms * 4 * 1024); cudaMalloc(&cyc, 8);
  int blocks = sms * 4, threads = 512;
  k<OP><<<blocks, threads>>>(out, 0.3f, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, 0.3f, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)blocks * threads * N_ITERS * 8;
  double per_sm_per_clk = ops / sms / (double)c;  // block 0's clock span (all blocks co-resident)
  printf("%-10s %8.3f ms  %.3e ops/s  %.2f ops/clk/SM (block0 cycles %lld)\n", name, ms, ops / (ms * 1e-3), per_sm_per_clk, c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s SMs=%d clockRate=%d kHz regsPerSM=%d smemPerSM=%zu l2=%d\n", p.name, p.multiProcessorCount, clk,
         p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor, p.l2CacheSize);
  int sms = p.multiProcessorCount;
  run<0>("__sinf", sms); run<1>("__cosf", sms); run<2>("frcp_rn", sms); run<3>("rcp.approx", sms);
  run<4>("ex2", sms); run<5>("lg2", sms); run<6>("sin.approx", sms); run<7>("ffma", sms);
  return 0;
}
