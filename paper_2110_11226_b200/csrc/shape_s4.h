// Evaluator variant: register stack of 4 slots, 16 rows per thread per pass, 1 pass per tile,
// 128-register budget (4 CTAs per SM): measured best on C3 (DESIGN.md performance log).
#define GP_STACK 4
#define GP_R 16
#define GP_SUB 1
#define GP_NT 128
#define GP_MINB 4

