// Evaluator variant: register stack of 4 slots, 16 rows per thread per pass, 1 pass per tile,
// 512-thread CTAs at the 128-register budget (1 CTA = 16 warps per SM). One CTA per SM means the
// four warps on each SM sub-partition walk the SAME code stream, so the leading warp's
// instruction-cache misses are the followers' hits (4 CTAs of 128 threads walked 4 different
// streams: gen-0 C3 gp_evaluate 224 -> 197 ms, step 134 -> 128 ms; profiles/ab_r02_nt512.log).
#define GP_STACK 4
#define GP_R 16
#define GP_SUB 1
#define GP_NT 512
#define GP_MINB 1
// one-deep case-id prefetch (r02 A/B on the final build: gen-0 gp_evaluate 181.3 -> 178.6 ms,
// step 118.0 -> 117.8 ms; it was slower before the per-case continue, profiles/ab_r02_s4misc.log)
#define GP_PREFETCH 1
