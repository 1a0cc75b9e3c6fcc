// Evaluator variant for wide datasets (X columns read through L1/L2, no shared-memory X tile):
// register stack of 4 slots, 4 rows per thread, 1024-thread CTAs at a 32-register budget (2 CTAs =
// 64 warps per SM, full occupancy; 4096-row tiles). The variable operands are L2 loads (a tile of
// 28-90 columns does not fit shared memory), so the shape that hides their latency best wins:
// measured on C5 / C4 (r02 A/B, tools/ab_libs.sh): 256 x 8 rows at 80 registers (24 warps) 0.31 /
// 0.39 SFU frac of the step, 512 x 4 at 64 / 40 / 32 registers 0.39 / 0.44, 0.44 / 0.47, 0.46 /
// 0.50; 1024 x 4 (two code streams per SM instead of four) C5 12.2 -> 12.0 ms per step, C4
// gp_evaluate 108.5 -> 105.5 ms (profiles/ab_r02_wide_iso.log).
// (A warp-per-program kernel that staged one warp's rows of every column in shared memory was
// measured slower, C5 12 -> 22 ms per step: the staging costs more than the L2 loads it removes.)
#define GP_STACK 4
#define GP_R 4
#define GP_SUB 1
#define GP_NT 1024
#define GP_MINB 2
#define GP_MINB_GLOBAL 2
#define GP_RED_ROWS 8
#define GP_GLOBAL_X_ONLY 1
// The register-starved wide shapes keep tan = sin * rcp(cos) and the shared case tail: the FMA-pipe
// tan and the per-case continue (eval_impl.cuh) need live registers a 32-register kernel spills
// (r02 A/B, profiles/ab_r02_wide_iso.log: C5 step 15.1 -> 12.8 ms without the polynomial tan,
// 15.1 -> 14.0 ms without the per-case continue).
#define GP_TAN_POLY 0
#define GP_CASE_CONTINUE 0
// one-deep case-id prefetch (as shape_s4.h; C4 step 39.7 -> 39.5 ms, C5 12.12 -> 12.06 ms,
// profiles/ab_r02_s4misc.log)
#define GP_PREFETCH 1
