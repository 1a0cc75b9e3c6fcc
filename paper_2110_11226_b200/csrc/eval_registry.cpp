// eval_registry.cpp -- assembles the EvalVariant of every evaluator shape (kernels.h) from the
// per-kernel translation units that build.py generates from eval_impl.cuh + shape_<name>.h: one
// translation unit per (shape, PREDICT, XSMEM), so the large dispatch switches compile in
// parallel. Shapes s12 / s20 have all four kernels, s4 / s8 the shared-memory-X pair; the wide-dataset shapes w4 / w8
// only the global-memory-X pair.
#include "kernels.h"

namespace gpb {

#define GP_DECLARE_KERNEL(NS, TAG)                                                             \
  namespace NS {                                                                               \
  cudaError_t launch_k##TAG(const EvalArgs& a, int n_ctas, size_t smem, cudaStream_t s);      \
  int occ_k##TAG(size_t smem);                                                                 \
  }
#define GP_DECLARE_SHAPE(NS)                                                                   \
  namespace NS {                                                                               \
  EvalShape shape_info();                                                                      \
  size_t smem_bytes(int G, int S, int n_cols, int weighted, int xsmem, int predict);           \
  }

// shapes with a shared-memory X tile and a global-X fallback: kernels 00 01 10 11
#define GP_FULL_SHAPE(NS)                                                                      \
  GP_DECLARE_KERNEL(NS, 00) GP_DECLARE_KERNEL(NS, 01) GP_DECLARE_KERNEL(NS, 10)                \
  GP_DECLARE_KERNEL(NS, 11) GP_DECLARE_SHAPE(NS)                                               \
  namespace NS {                                                                               \
  static cudaError_t launch(const EvalArgs& a, bool predict, bool xsmem, int n, size_t smem,   \
                            cudaStream_t s) {                                                  \
    if (predict) return xsmem ? launch_k11(a, n, smem, s) : launch_k10(a, n, smem, s);         \
    return xsmem ? launch_k01(a, n, smem, s) : launch_k00(a, n, smem, s);                      \
  }                                                                                            \
  static int occupancy(bool predict, bool xsmem, size_t smem) {                                \
    if (predict) return xsmem ? occ_k11(smem) : occ_k10(smem);                                 \
    return xsmem ? occ_k01(smem) : occ_k00(smem);                                              \
  }                                                                                            \
  }                                                                                            \
  const EvalVariant& eval_variant_##NS() {                                                     \
    static const EvalVariant v = {NS::shape_info(), &NS::launch, &NS::occupancy,               \
                                  &NS::smem_bytes};                                             \
    return v;                                                                                  \
  }

// shapes with a shared-memory X tile only (kernels 01 11): the global-X path runs their buckets
// in the wide-dataset shapes
#define GP_SMEM_SHAPE(NS)                                                                      \
  GP_DECLARE_KERNEL(NS, 01) GP_DECLARE_KERNEL(NS, 11) GP_DECLARE_SHAPE(NS)                     \
  namespace NS {                                                                               \
  static cudaError_t launch(const EvalArgs& a, bool predict, bool xsmem, int n, size_t smem,   \
                            cudaStream_t s) {                                                  \
    if (!xsmem) return cudaErrorInvalidValue;                                                  \
    return predict ? launch_k11(a, n, smem, s) : launch_k01(a, n, smem, s);                    \
  }                                                                                            \
  static int occupancy(bool predict, bool xsmem, size_t smem) {                                \
    if (!xsmem) return 0;                                                                      \
    return predict ? occ_k11(smem) : occ_k01(smem);                                            \
  }                                                                                            \
  }                                                                                            \
  const EvalVariant& eval_variant_##NS() {                                                     \
    static const EvalVariant v = {NS::shape_info(), &NS::launch, &NS::occupancy,               \
                                  &NS::smem_bytes};                                             \
    return v;                                                                                  \
  }

// wide-dataset shapes: global-memory X only (kernels 00 10)
#define GP_WIDE_SHAPE(NS)                                                                      \
  GP_DECLARE_KERNEL(NS, 00) GP_DECLARE_KERNEL(NS, 10) GP_DECLARE_SHAPE(NS)                     \
  namespace NS {                                                                               \
  static cudaError_t launch(const EvalArgs& a, bool predict, bool xsmem, int n, size_t smem,   \
                            cudaStream_t s) {                                                  \
    if (xsmem) return cudaErrorInvalidValue;                                                   \
    return predict ? launch_k10(a, n, smem, s) : launch_k00(a, n, smem, s);                    \
  }                                                                                            \
  static int occupancy(bool predict, bool xsmem, size_t smem) {                                \
    if (xsmem) return 0;                                                                       \
    return predict ? occ_k10(smem) : occ_k00(smem);                                            \
  }                                                                                            \
  }                                                                                            \
  const EvalVariant& eval_variant_##NS() {                                                     \
    static const EvalVariant v = {NS::shape_info(), &NS::launch, &NS::occupancy,               \
                                  &NS::smem_bytes};                                             \
    return v;                                                                                  \
  }

GP_SMEM_SHAPE(s4)
GP_SMEM_SHAPE(s8)
GP_FULL_SHAPE(s12)
GP_FULL_SHAPE(s20)
GP_WIDE_SHAPE(w4)
GP_WIDE_SHAPE(w8)

}  // namespace gpb
