// Evaluator variant for wide datasets (X columns read through L1/L2, no shared-memory X tile):
// register stack of 4 slots, 8 rows per thread, 256-thread CTAs at an 80-register budget (3 CTAs
// = 24 warps per SM). The L2 latency of the per-word variable loads needs more resident warps
// than the shared-memory-X shape (128 threads x 16 rows, 16 warps) provides; measured on C5
// (Year-shaped 1M x 90): SFU frac 0.35 -> 0.53 (DESIGN.md performance log).
#define GP_STACK 4
#define GP_R 8
#define GP_SUB 1
#define GP_NT 256
#define GP_MINB 3
#define GP_MINB_GLOBAL 3
#define GP_RED_ROWS 8
#define GP_GLOBAL_X_ONLY 1

