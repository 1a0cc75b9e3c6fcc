// common.h -- host/device helpers shared by the CUDA kernels and the host engine (product code;
// the oracle has its own, independent implementations).
#pragma once
#include <cstdint>
#include "../../include/gp.h"

#ifdef __CUDACC__
#define GPB_HD __host__ __device__ __forceinline__
#else
#define GPB_HD inline
#endif

namespace gpb {

// Arity: terminals 0, binary 2 (ADD..POW), unary 1 (SIN..ATAN); -1 = not an opcode.
GPB_HD constexpr int op_arity(int op) {
  return op < 0 ? -1 : op <= GP_OP_CONST ? 0 : (op <= GP_OP_POW ? 2 : (op < GP_OP_COUNT ? 1 : -1));
}

// ---- Philox4x32-10, product implementation ---------------------------------------------
struct u32x4 { uint32_t x, y, z, w; };
GPB_HD u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#ifdef __CUDACC__
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

}  // namespace gpb
