// Evaluator variant for wide datasets: register stack of 8 slots, 4 rows per thread, 2 passes per
// tile (4096 rows), 512-thread CTAs at a 64-register budget (2 CTAs = 32 warps per SM; r02 A/B:
// 256 threads at 80 registers, 24 warps, C5 gp_evaluate 37.1 ms -> 35.0 ms here,
// profiles/ab_r02_wide_shapes3.log).
#define GP_STACK 8
#define GP_R 4
#define GP_SUB 2
#define GP_NT 512
#define GP_MINB 2
#define GP_MINB_GLOBAL 2
#define GP_RED_ROWS 8
#define GP_GLOBAL_X_ONLY 1

// as shape_w4.h: sin * rcp(cos) tan and the shared case tail
#define GP_TAN_POLY 0
#define GP_CASE_CONTINUE 0
