// mutate.h -- launch interface of mutate.cu (GPU-side variation). Plain C++ so the host
// engine (engine.cpp) can include it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/gp.h"

namespace gpb {

// Deepest tree the device scans handle (engine populations have depth <= stack_capacity - 1 <= 19)
constexpr int kMaxDepth = 30;
// Largest generated donor of a subtree mutation (Grow of depth <= 10 has <= 2047 nodes); the GPU
// path is used when init_depth_max <= kMaxDonorDepth
constexpr int kMaxDonorDepth = 10;
constexpr int kMaxDonorNodes = (1 << (kMaxDonorDepth + 1)) - 1;

// The parts of gp_config the device needs (kernel parameter).
struct MutConfig {
  uint32_t k0, k1;              // Philox key = seed
  int32_t n_features, n_functions;
  int32_t function_set[32];
  float const_lo, const_hi;
  double p[4];                  // crossover, subtree, hoist, point
  double p_point_replace;
  int32_t init_depth_min, init_depth_max, stack_capacity;
};

// A child = parent[0, s) + inserted range [a, b) + parent[e, len): the range comes from the parent
// (hoist), the donor program (crossover) or the regenerated donor (subtree mutation);
// reproduction / point mutation copy (and rewrite) the whole parent.
struct Recipe {
  int32_t kind, parent, donor, s, e, a, b, len;
};

// Device-side generation statistics (copied to the host once per phase).
struct DevGenStats {
  int64_t op_count[GP_OP_COUNT];
  int64_t const_nodes, const_programs;
  int32_t max_need, err;
  int32_t best, best_len, best_depth;
  float best_raw;
  double mean;
};

cudaError_t launch_kinds(int32_t n, uint32_t generation, const MutConfig& c, int32_t* kinds,
                         int32_t* tcount, int32_t* toff /* n + 1 */, cudaStream_t s);
cudaError_t launch_plan(const gp_node* nodes, const int64_t* off, int32_t n, uint32_t generation,
                        const MutConfig& c, const int32_t* kinds, const int32_t* toff,
                        const int32_t* winners, Recipe* recipes, int32_t* lens,
                        int64_t* out_off /* n + 1 */, int32_t* err, cudaStream_t s);
cudaError_t launch_emit(const gp_node* nodes, const int64_t* off, int32_t n, uint32_t generation,
                        const MutConfig& c, const Recipe* recipes, const int64_t* out_off,
                        gp_node* out, cudaStream_t s);
// ramped half-and-half initial population: lengths + offsets (n + 1), then the nodes
cudaError_t launch_init_lengths(int32_t n, const MutConfig& c, int32_t* lens, int64_t* off,
                                cudaStream_t s);
cudaError_t launch_init_emit(int32_t n, const MutConfig& c, const int64_t* off, gp_node* out,
                             cudaStream_t s);
cudaError_t launch_pop_stats(const gp_node* nodes, const int64_t* off, int32_t n, int32_t* depth,
                             DevGenStats* st, cudaStream_t s);
cudaError_t launch_fit_stats(const float* fit, int32_t n, int32_t higher, const int64_t* off,
                             const int32_t* depth, DevGenStats* st, cudaStream_t s);

}  // namespace gpb
