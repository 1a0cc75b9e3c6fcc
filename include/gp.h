/*
 * gp.h -- C-ABI of the B200-native data-parallel hot path of arXiv 2110.11226
 * ("GPU accelerated stack-based generational GP", the cuML genetic-programming paper).
 *
 * Citation convention: P:L = /root/reference/PAPER.md line L (with its section / equation /
 * algorithm); S:L = /root/reference/SPEC.md line L. DESIGN.md lists every reading of the paper
 * that this interface fixes.
 *
 * Conventions for every entry point
 *  - Memory: pointers are DEVICE pointers unless the argument says [host] or [host|device].
 *    [host|device] arguments are detected with cudaPointerGetAttributes; host data is staged into
 *    library-owned device memory inside the call (this is the end-to-end path).
 *  - Ownership: the caller owns every buffer it passes; the library owns only the context /
 *    engine workspaces it allocates (freed by the matching *_destroy).
 *  - Streams: every call is asynchronous on the context's stream unless marked [sync].
 *  - Errors: nothing throws and nothing aborts. Each call returns a gp_status; argument errors
 *    (GP_ERR_ARG) are detected on the host before any work is enqueued. Per-program problems
 *    (invalid prefix list, stack overflow, variable out of range, non-finite fitness) are NOT
 *    call errors: they are reported per program through status bits (GP_FLAG_*) and the program
 *    receives the worst fitness of the metric. gp_last_error(ctx) returns a message for the
 *    last failing call on that context.
 *  - Thread safety: a context / engine must be used by one host thread at a time.
 */
#ifndef GP_B200_GP_H
#define GP_B200_GP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------------------------------
 * Status codes, metrics, opcodes, nodes
 * -------------------------------------------------------------------------------------------*/
typedef enum {
  GP_OK = 0,
  GP_ERR_ARG = 1,          /* invalid argument (sizes, pointers, metric, config) */
  GP_ERR_PROGRAM = 2,      /* reserved: per-program errors are reported via status bits */
  GP_ERR_UNSUPPORTED = 3,  /* e.g. Spearman with row-sharded ranks, world_size > 1 without NCCL */
  GP_ERR_CUDA = 4,         /* a CUDA runtime call failed; see gp_last_error */
  GP_ERR_NCCL = 5,         /* an NCCL call failed or libnccl could not be loaded */
  GP_ERR_OOM = 6           /* device allocation failed */
} gp_status;

/* Fitness metrics, P:264-275 ("weighted versions of the following 6 standard loss functions").
 * MAE, MSE, RMSE, LogLoss: lower is better. Pearson, Spearman: higher is better.
 * Spearman = weighted Pearson of rank_vector(y) and rank_vector(yhat), ranks
 * 1..n over every row with ties averaged, yhat ranked in fp32. It cannot stream: its
 * gp_evaluate path materialises yhat per batch of programs and sorts it; with a
 * row-sharded multi-rank context it returns GP_ERR_UNSUPPORTED (use GP_SHARD_PROGRAMS). */
typedef enum {
  GP_MAE = 0, GP_MSE = 1, GP_RMSE = 2, GP_LOGLOSS = 3, GP_PEARSON = 4, GP_SPEARMAN = 5
} gp_metric;

/* Opcodes. Terminals: variable (feature column) and constant ("terminals collectively denote
 * both variables and constants"). Functions: maximum arity 2. The catalog is SPEC's
 * -- the paper names only "33 pre-defined functions" and the Table 2 / 6 set
 * {+, -, *, /, sin, cos, tan}. Protected semantics (C2):
 *   div(a,b) = 1 if |b| < 1e-3 else a/b     log(a) = 0 if |a| < 1e-3 else ln|a|
 *   inv(a)   = 1 if |a| < 1e-3 else 1/a     sqrt(a) = sqrt(|a|)     exp(a) = min(e^a, 1e30)
 *   sinh, cosh clamped to +-1e30; asin, acos clamp their argument to [-1, 1];
 *   pow(a,b) = 1 if b == 0, else 0^b = 0 (b > 0) or 1e30 (b < 0), else min(|a|^b, 1e30).
 * Binary operands: the first operand is the first child in prefix order. */
enum {
  GP_OP_VAR = 0, GP_OP_CONST = 1,
  GP_OP_ADD = 2, GP_OP_SUB = 3, GP_OP_MUL = 4, GP_OP_DIV = 5, GP_OP_MIN = 6, GP_OP_MAX = 7,
  GP_OP_POW = 8,
  GP_OP_SIN = 9, GP_OP_COS = 10, GP_OP_TAN = 11, GP_OP_ABS = 12, GP_OP_NEG = 13, GP_OP_SQRT = 14,
  GP_OP_LOG = 15, GP_OP_EXP = 16, GP_OP_INV = 17, GP_OP_SQUARE = 18, GP_OP_CUBE = 19,
  GP_OP_TANH = 20, GP_OP_SINH = 21, GP_OP_COSH = 22, GP_OP_ASIN = 23, GP_OP_ACOS = 24,
  GP_OP_ATAN = 25,
  GP_OP_COUNT = 26
};

/* One node of a program's prefix (Polish) list, P:176 / P:186 (Listing 1 "node *nodes").
 * 8 bytes: op, then the variable index (GP_OP_VAR) or the fp32 constant (GP_OP_CONST); unused
 * for functions. A population is a flat CSR: nodes[] plus int64 node_offsets[n_programs + 1],
 * program i = nodes[node_offsets[i] .. node_offsets[i+1]) -- one contiguous copy per generation
 * instead of the paper's per-program cudaMemcpy loop. */
typedef struct {
  int32_t op;
  union { int32_t var; float value; };
} gp_node;

/* Per-program status bits written to status_out. */
enum {
  GP_FLAG_INVALID_PREFIX = 1,  /* S:44 needed-counter scan failed (or empty program) */
  GP_FLAG_STACK_OVERFLOW = 2,  /* stack need > capacity (capacity m evaluates depth m-1) */
  GP_FLAG_VAR_RANGE = 4,       /* variable index >= n_cols */
  GP_FLAG_NONFINITE = 8,       /* loss fitness non-finite -> +inf (C4) */
  GP_FLAG_UNDEFINED_CORR = 16, /* Pearson with zero variance / non-finite r -> 0 (C4) */
  GP_FLAG_BAD_OPCODE = 32      /* opcode outside [0, GP_OP_COUNT) */
};

/* Largest supported stack capacity (S:165 default 20). */
#define GP_MAX_STACK 20

typedef struct gp_context gp_context;
typedef struct gp_engine gp_engine;

const char* gp_status_string(gp_status s);
const char* gp_last_error(const gp_context* ctx);
/* Library version string, e.g. "gp_b200 0.1 sm_100a". */
const char* gp_version(void);
/* Copies `bytes` between any two [host|device] buffers (cudaMemcpyDefault) [sync]; lets a binding
 * take copies of the borrowed device views below without a second CUDA runtime. */
gp_status gp_device_copy(void* dst, const void* src, size_t bytes);

/* ---------------------------------------------------------------------------------------------
 * Context: device, stream, optional NCCL communicator (data parallelism over dataset rows).
 * -------------------------------------------------------------------------------------------*/

/* Writes a fresh 128-byte NCCL unique id into out_id [host]. Rank 0 calls it and broadcasts the
 * bytes to the other ranks (the Python binding uses torch.distributed for that). */
gp_status gp_get_unique_id(void* out_id);

/* Creates a context on `device`, issuing work on `stream` (a cudaStream_t; NULL = legacy default
 * stream). nccl_unique_id [host]: NULL for a single GPU without a communicator; otherwise the
 * 128-byte id from gp_get_unique_id, and every rank 0 <= rank < world_size must call this
 * collectively (world_size 1 with an id creates a one-rank communicator). With
 * world_size > 1 each rank passes its own contiguous row shard to gp_evaluate, and the
 * per-program partial sums are combined with one fp64 ncclAllReduce per evaluation, so every
 * rank receives bit-identical fitness. */
gp_status gp_context_create(gp_context** out, int device, void* stream, const void* nccl_unique_id,
                            int rank, int world_size);
gp_status gp_context_destroy(gp_context* ctx);
/* Switches the context's stream. Work already queued on the old stream is waited for first
 * (the context's buffers may be reallocated on the new stream). */
gp_status gp_context_set_stream(gp_context* ctx, void* stream);

/* Pearson's single-pass evaluation accumulates about a per-program shift K_p = f_p(x_ref)
 * (C9). All ranks must use the same reference row: pass the GLOBAL first row
 * x_ref [host, n_cols floats] and its label y_ref. If never called, the first row of the X / y
 * passed to gp_evaluate is used; on a row-sharded communicator rank 0's first row is broadcast
 * to every rank inside gp_evaluate (one ncclBroadcast of n_cols + 1 floats), so the shifts
 * always agree. gp_evaluate_partial without a communicator cannot do that: set the row. */
gp_status gp_context_set_reference_row(gp_context* ctx, const float* x_ref, int32_t n_cols,
                                       float y_ref);

/* Kernel timing (for roofline reporting): when enabled, the context records CUDA events on its
 * stream around every fused-evaluator launch. gp_context_eval_timing returns the accumulated
 * device time in milliseconds and the launch count since the last reset [sync: waits for the
 * recorded events]. */
gp_status gp_context_set_profiling(gp_context* ctx, int enabled);
gp_status gp_context_eval_timing(gp_context* ctx, double* total_ms, int64_t* launches, int reset);
/* Evaluation order of the compiled programs. 1 (default): for every binary node whose operands
 * are both computed values, the operand needing more stack slots is evaluated first
 * (Sethi-Ullman), which minimises the register-stack need; 0: the classic reverse-prefix order
 * (second operand first). Results are identical either way (same operations on the same
 * operands); only the stack need, hence the evaluator variant a program runs in, changes. */
gp_status gp_context_set_eval_order(gp_context* ctx, int sethi_ullman);
/* Variable-free programs: a program whose whole tree folds to one constant c at compile time
 * (stage kernel) predicts c on every row. With closed_form = 1 (default) gp_evaluate takes its
 * MSE / RMSE sum from the dataset moments, sum_i w_i (c - y_i)^2 = W c^2 - 2 c S_y + S_yy
 * (fp64, the same per-chunk W, S_y, S_yy the Pearson path uses), its LogLoss sum from the two
 * per-row values it can take, W_1 softplus(-c) + (W - W_1) softplus(c) (W_1 = weight of rows with
 * y > 1/2, clamped as in S:191), and reports its Pearson correlation as undefined (0,
 * GP_FLAG_UNDEFINED_CORR) -- all without a per-row pass. This is the per-row loss of P:256-262
 * with the constant prediction factored out of the sum. MAE still evaluates such programs per
 * row. 0: every program goes through the per-row evaluator. */
gp_status gp_context_set_const_programs(gp_context* ctx, int closed_form);
/* Multi-GPU work split of gp_evaluate on a context with world > 1.
 *  GP_SHARD_ROWS (default): each rank passes its contiguous row shard; the per-program fp64
 *    partial sums are combined by one ncclAllReduce before finalize.
 *  GP_SHARD_PROGRAMS: each rank passes ALL rows and evaluates the programs [r c, min(n, (r+1) c))
 *    with c = ceil(n / world); the fp32 fitness and status words of the chunks are combined by
 *    ncclAllGather (in place, padded to world x c). Suits small datasets with large populations.
 * Results are identical on every rank in both modes. */
typedef enum { GP_SHARD_ROWS = 0, GP_SHARD_PROGRAMS = 1 } gp_shard;
gp_status gp_context_set_shard(gp_context* ctx, gp_shard mode);
/* Work decomposition override (tests and tuning): group_size programs per work item
 * (1..512, 0 = automatic; capped to the largest group whose accumulators fit: 128 on the
 * global-memory-X path) and tiles_per_chunk plan tiles per work item (8192 rows when X is staged
 * in shared memory, 4096 otherwise; 0 = automatic). Only the fp64 summation order of the
 * per-chunk partial sums depends on it. GP_ERR_ARG for values out of range. */
gp_status gp_context_set_plan(gp_context* ctx, int32_t group_size, int64_t tiles_per_chunk);
/* Restricts gp_evaluate / gp_evaluate_partial to the programs [lo, hi) (hi < 0: all) -- the
 * per-rank program chunk of GP_SHARD_PROGRAMS, usable without a communicator (a caller that
 * distributes programs itself, and the single-GPU simulation of that mode). Fitness and status of
 * the programs outside the range are unspecified. */
gp_status gp_context_set_program_range(gp_context* ctx, int32_t lo, int32_t hi);
/* Number of CUDA kernels this context has launched (all entry points) since the last reset. */
gp_status gp_context_kernel_launches(gp_context* ctx, int64_t* launches, int reset);

/* ---------------------------------------------------------------------------------------------
 * gp_evaluate -- Evaluate + fitness of a whole population (Alg. 1 line 7).
 *
 * For every program p and every row i of this rank's shard, evaluates the prefix list with a
 * fixed-capacity register stack, computes the weighted per-row loss
 * and reduces it per program -- fused, with no m x n prediction matrix -- then
 * combines ranks (one all-reduce) and finalizes:
 *   MAE / MSE / LogLoss: sum_i w_i loss_i / sum_i w_i;  RMSE = sqrt(MSE);
 *   Pearson: weighted correlation r (signed).
 * Rows with w_i == 0 are skipped (never multiplied: 0 * inf is not 0). Non-finite loss fitness
 * becomes +inf (GP_FLAG_NONFINITE); undefined Pearson becomes 0 (GP_FLAG_UNDEFINED_CORR).
 * Invalid programs get +inf (lower-better metrics) or -inf (Pearson).
 *
 *  programs      [host|device] gp_node[n_nodes], prefix order
 *  node_offsets  [host|device] int64[n_programs + 1], node_offsets[0] == 0,
 *                node_offsets[n_programs] == n_nodes
 *  n_programs    >= 1
 *  n_nodes       [host] total node count
 *  max_stack     [host] bound on every program's stack need, 1..GP_MAX_STACK. The evaluator keeps
 *                only computed values on its register stack (terminal operands are folded into
 *                their parent), so its need is <= the classic reverse-prefix need (and smaller
 *                still with the Sethi-Ullman order, gp_context_set_eval_order). Programs needing
 *                more than max_stack get GP_FLAG_STACK_OVERFLOW.
 *  X             [host|device] fp32, column-major: feature c of local row i at
 *                X[c * ldx + i]; ldx >= n_rows (ldx > n_rows lets a rank pass a row window of
 *                a global column-major array)
 *  y             [host|device] fp32[n_rows] targets (LogLoss requires y in {0, 1})
 *  w             [host|device] fp32[n_rows] weights >= 0, or NULL for all ones
 *  n_rows        this rank's row count, >= 1;   n_cols >= 1
 *  fitness_out   [host|device] fp32[n_programs] raw fitness ("float raw_fitness_")
 *  status_out    [host|device] uint32[n_programs] GP_FLAG_* bits, or NULL
 * If any pointer is host memory the call synchronizes the stream before returning. */
gp_status gp_evaluate(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                      int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float* X,
                      int64_t ldx, const float* y, const float* w, int64_t n_rows, int32_t n_cols,
                      gp_metric metric, float* fitness_out, uint32_t* status_out);

/* gp_evaluate_partial -- the per-rank half of gp_evaluate, before ranks are combined (SURVEY
 * A2-A5): the fp64 per-program sums of this call's rows,
 *   sums_out[p S + k], S = 3 for Pearson (S_d, S_dd, S_dy about the shifts K_p, K_y of
 *                     DESIGN.md C9), else 1 (sum_i w_i loss_i);
 *   sums_out[n S + 0..2] = W = sum_i w_i, S_y, S_yy (Pearson: about K_y; LogLoss: S_y = weight
 *                     of the rows with y > 1/2; MSE / RMSE: about 0),
 * with zeros for programs the evaluator skipped (invalid; variable-free under a closed-form
 * metric; outside gp_context_set_program_range). Summing the outputs of row shards (any order)
 * and passing the total to gp_finalize_sums gives what gp_evaluate gives with one row-sharded
 * communicator -- this is the data flow of the NCCL path with the all-reduce made explicit.
 * Arguments as gp_evaluate; sums_out [host|device] fp64[n_programs * S + 3]. Spearman is not
 * additive over rows: GP_ERR_UNSUPPORTED. For Pearson every shard must use the same reference
 * row (gp_context_set_reference_row). */
gp_status gp_evaluate_partial(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                              int32_t n_programs, int64_t n_nodes, int32_t max_stack,
                              const float* X, int64_t ldx, const float* y, const float* w,
                              int64_t n_rows, int32_t n_cols, gp_metric metric, double* sums_out);
/* gp_finalize_sums -- the other half: fitness and status from sums laid out as
 * gp_evaluate_partial writes them (summed over shards). The programs are compiled again for
 * their status bits and the closed-form constants. sums [host|device]; fitness_out / status_out
 * as gp_evaluate. */
gp_status gp_finalize_sums(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                           int32_t n_programs, int64_t n_nodes, int32_t max_stack, int32_t n_cols,
                           const double* sums, gp_metric metric, float* fitness_out,
                           uint32_t* status_out);

/* gp_predict -- the execution step alone ("all programs ... evaluated on the given
 * data-set, to produce set of predicted values"): out[p * ld_out + i] = f_p(x_i) in fp32 for
 * p < n_programs, i < n_rows. Same interpreter as gp_evaluate. All pointers device memory;
 * ld_out >= n_rows. Invalid programs' columns are left untouched (status_out says why). */
gp_status gp_predict(gp_context* ctx, const gp_node* programs, const int64_t* node_offsets,
                     int32_t n_programs, int64_t n_nodes, int32_t max_stack, const float* X,
                     int64_t ldx, int64_t n_rows, int32_t n_cols, float* out, int64_t ld_out,
                     uint32_t* status_out);

/* ---------------------------------------------------------------------------------------------
 * gp_tournament_select -- parallel tournament selection (Eqs. 1-2).
 * One thread per tournament t < n_tournaments: draws tournament_size indices with replacement
 * from Philox4x32-10, key = (seed lo, seed hi), counter = (t, generation, i / 4, 0),
 * word i % 4, index = (uint64(word) * n_programs) >> 32; adjusted fitness in fp32 without FMA
 * contraction: raw + parsimony * len (lower-better) or raw - parsimony * len (higher-better,
 * S:257), len = node count; NaN is the worst value; winner = best adjusted fitness, ties
 * to the smallest population index. Bit-exact across launches, devices and ranks.
 *  fitness       device fp32[n_programs]
 *  node_offsets  device int64[n_programs + 1] (program lengths are the differences)
 *  winners_out   device int32[n_tournaments] */
gp_status gp_tournament_select(gp_context* ctx, const float* fitness, const int64_t* node_offsets,
                               int32_t n_programs, int32_t n_tournaments, int32_t tournament_size,
                               float parsimony, int32_t higher_is_better, uint64_t seed,
                               uint32_t generation, int32_t* winners_out);

/* ---------------------------------------------------------------------------------------------
 * Engine: the generational loop of Alg. 1; mutations on the GPU or the
 * host.
 * -------------------------------------------------------------------------------------------*/
typedef struct {
  int32_t population_size;     /* Table 2: 50, Table 6: 35 */
  int32_t tournament_size;     /* Table 6: 4 */
  float parsimony;             /* Table 6: 0.01 (Eq. 1) */
  int32_t metric;              /* gp_metric */
  double p_crossover;          /* Table 6: 0.7 (hoisted crossover) */
  double p_subtree;            /* 0.1 */
  double p_hoist;              /* 0.05 */
  double p_point;              /* 0.1;  residual mass -> reproduction */
  double p_point_replace;      /* per-node replacement probability for point mutation */
  int32_t init_depth_min;      /* ramped half-and-half depth range ([2, 6]) */
  int32_t init_depth_max;
  float const_lo, const_hi;    /* constant range ([-1, 1]) */
  int32_t n_functions;         /* function set size, <= 32 */
  int32_t function_set[32];    /* opcodes; Table 2 / 6: {add, sub, mul, div, sin, cos, tan} */
  int32_t stack_capacity;      /* depth <= stack_capacity - 1, <= GP_MAX_STACK */
  uint64_t seed;               /* Philox key for init, kinds, tournaments and mutations */
  int32_t n_threads;           /* host threads for the host mutation path (0 = cores / ranks) */
  int32_t device_mutation;     /* 1 (default): kinds, mutations and the flat population stay on the
                                  GPU (mutate.cu; needs init_depth_max <= 10, else the
                                  host path runs); 0: host mutation + one H2D copy */
} gp_config;

/* Fills Table 6's parameters with SPEC defaults for the rest. */
void gp_config_default(gp_config* cfg);

typedef struct {
  int32_t generation;          /* 0 = initial population */
  float best_raw;              /* directionally best raw fitness */
  float best_adjusted;         /* its parsimony-adjusted fitness (Eq. 2) */
  int32_t best_index, best_len, best_depth;
  double mean_raw;             /* mean over finite raw fitness */
  int64_t total_nodes;         /* sum of program lengths */
  int32_t max_stack_need;
  int32_t n_tournaments;
  double t_select_s, t_mutate_s, t_h2d_s, t_eval_s, t_total_s; /* phase wall times */
  int64_t op_count[GP_OP_COUNT]; /* opcode histogram of the evaluated population's nodes whose
                                   subtree contains a variable (per-row work) */
  int64_t const_nodes;           /* nodes of variable-free subtrees (per-program constants) */
  int64_t const_programs;        /* programs whose whole tree is variable-free */
} gp_generation_stats;

/* Creates an engine over a dataset. X / y / w are [host|device] (same layouts as gp_evaluate);
 * host data is copied into engine-owned device memory, device data is referenced (the caller
 * keeps it alive). cfg [host] is copied. */
gp_status gp_engine_create(gp_engine** out, gp_context* ctx, const gp_config* cfg, const float* X,
                           int64_t ldx, const float* y, const float* w, int64_t n_rows,
                           int32_t n_cols);
/* Replaces the dataset (same rules as gp_engine_create); used by the end-to-end path to stream
 * a host dataset into HBM every step. */
gp_status gp_engine_set_dataset(gp_engine* e, const float* X, int64_t ldx, const float* y,
                                const float* w, int64_t n_rows, int32_t n_cols);
gp_status gp_engine_destroy(gp_engine* e);
/* Alg. 1 lines 2-3: ramped half-and-half init and evaluation. [sync] */
gp_status gp_engine_init_population(gp_engine* e, gp_generation_stats* stats_out);
/* Alg. 1 lines 5-8 once: kinds, tournaments, mutations, evaluation. With
 * device_mutation the whole step runs on the GPU (two small D2H reads: the child node total,
 * then the statistics); otherwise mutations run on the host followed by one H2D copy of the flat
 * population. Both paths produce bit-identical populations. [sync] */
gp_status gp_generation(gp_engine* e, gp_generation_stats* stats_out);
/* Borrowed [host] views of the current population and its fp32 raw fitness; valid until the
 * next gp_generation / gp_engine_init_population / gp_engine_set_population / gp_engine_destroy.
 * [sync] (with device mutation the population is copied from HBM on this call). */
gp_status gp_engine_population(gp_engine* e, const gp_node** nodes, const int64_t** offsets,
                               const float** fitness, int32_t* n_programs, int64_t* n_nodes);
/* Borrowed DEVICE views of the current population (flat CSR) and its fitness, same validity. */
gp_status gp_engine_population_device(gp_engine* e, const gp_node** nodes,
                                      const int64_t** offsets, const float** fitness,
                                      int32_t* n_programs, int64_t* n_nodes);
/* Replaces the current population (cfg.population_size programs, [host|device] flat CSR with
 * offsets[0] == 0) and declares it generation `generation`. fitness [host|device] fp32[n]: the
 * population's raw fitness, or NULL to evaluate it now. Programs must be valid with depth <=
 * stack_capacity - 1 (GP_ERR_ARG otherwise). Used to resume a run, to seed a population, and by
 * the benchmark to start every step from the same population. [sync], except for a device
 * population with device fitness on a device-mutation engine and stats_out == NULL: then the call
 * only enqueues device-to-device copies on the context stream. */
gp_status gp_engine_set_population(gp_engine* e, const gp_node* nodes, const int64_t* offsets,
                                   int32_t n_programs, int64_t n_nodes, const float* fitness,
                                   int32_t generation, gp_generation_stats* stats_out);
/* [host] views of the last generation's mutation kinds (0 crossover, 1 subtree, 2 hoist,
 * 3 point, 4 reproduction) and tournament winners (for replay tests). */
gp_status gp_engine_last_selection(gp_engine* e, const int32_t** kinds, const int32_t** winners,
                                   int32_t* n_tournaments);

#ifdef __cplusplus
}
#endif
#endif /* GP_B200_GP_H */
