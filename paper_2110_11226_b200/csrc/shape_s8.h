// Evaluator variant: register stack of 8 slots, 8 rows per thread per pass, 2 passes per tile,
// 512-thread CTAs (one per SM, see shape_s4.h).
#define GP_STACK 8
#define GP_R 8
#define GP_SUB 2
#define GP_NT 512
#define GP_MINB 1
