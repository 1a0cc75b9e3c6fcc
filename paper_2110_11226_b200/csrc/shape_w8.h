// Evaluator variant for wide datasets: register stack of 8 slots, 4 rows per thread, 2 passes per
// tile, 256-thread CTAs at an 80-register budget (see eval_w4.cu).
#define GP_STACK 8
#define GP_R 4
#define GP_SUB 2
#define GP_NT 256
#define GP_MINB 3
#define GP_MINB_GLOBAL 3
#define GP_RED_ROWS 8
#define GP_GLOBAL_X_ONLY 1

// as shape_w4.h: sin * rcp(cos) tan and the shared case tail
#define GP_TAN_POLY 0
#define GP_CASE_CONTINUE 0
