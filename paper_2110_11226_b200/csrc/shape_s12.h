// Evaluator variant: register stack of 12 slots, 4 rows per thread per pass, 4 passes per tile.
#define GP_STACK 12
#define GP_R 4
#define GP_SUB 4
#define GP_NT 128
#define GP_MINB 4

