// Evaluator variant: register stack of 12 slots, 4 rows per thread per pass, 4 passes per tile,
// 512-thread CTAs (one per SM, see shape_s4.h).
#define GP_STACK 12
#define GP_R 4
#define GP_SUB 4
#define GP_NT 512
#define GP_MINB 1
