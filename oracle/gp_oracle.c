/*
 * gp_oracle.c -- TEST INFRASTRUCTURE ONLY. The plain, slow, obviously-correct CPU oracle for the
 * data-parallel hot path of arXiv 2110.11226 ("GPU accelerated stack-based generational GP").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this file's shared object. The product (paper_2110_11226_b200/) never links, imports or executes
 * it, and it shares no code, header, table or constant generator with the product: every opcode,
 * threshold and constant below is retyped from the paper / SPEC readings listed in DESIGN.md.
 *
 * Precision: double everywhere (fp32 inputs are widened exactly). Compile with -O2
 * -ffp-contract=off so no FMA contraction changes any rounding (needed for the fp32 tournament
 * arithmetic, which must be replayed bit-exactly).
 *
 * Citation convention: P:L = /root/reference/PAPER.md line L, S:L = /root/reference/SPEC.md line L.
 *
 * What is here, and what pins it (tests/test_oracle_*.py):
 *   - validate / depth / subtree_end / stack_need       S:41-66, P:243      SPEC examples, brute force
 *   - recursive tree-walk evaluation (value + fp32 error bound + branch-ambiguity + overflow flags)
 *                                                        P:176
 *                                                        hand-derived programs, Pagie Eq.3 program,
 *                                                        independent stack walk (tests, brute force)
 *   - weighted metrics MAE/MSE/RMSE/LogLoss/Pearson (two-pass)
 *                                                        SPEC examples, closed forms on Pagie grids,
 *                                                        identities (RMSE^2 = MSE, Pearson(y,y)=1 ...)
 *   - rank_vector (average ties) and Spearman = weighted Pearson of ranks   P:274-277; S:201,
 *     S:209-215, S:219-220                               SPEC examples, scipy rankdata / spearmanr,
 *                                                        monotone-transform invariance
 *   - Philox4x32-10                                      P:202 (Salmon et al. 2011)   Random123 KATs
 *   - tournament selection with parsimony (Eqs. 1-2)
 *                                                        brute force on tiny populations, closed-form
 *                                                        win law (chi-square)
 *   - Pagie polynomial (Eq. 3)                           P:346-352; S:490-507   closed forms
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

/* ------------------------------------------------------------------------------------------------
 * Node encoding (the C-ABI's 8-byte node, retyped here: {int32 op; int32 var | float value}).
 * Opcode numbering is the public interface contract documented in DESIGN.md "Function catalog".
 * ----------------------------------------------------------------------------------------------*/
typedef struct { int32_t op; int32_t payload; } onode;

enum {
  O_VAR = 0, O_CONST = 1,
  O_ADD = 2, O_SUB = 3, O_MUL = 4, O_DIV = 5, O_MIN = 6, O_MAX = 7, O_POW = 8,
  O_SIN = 9, O_COS = 10, O_TAN = 11, O_ABS = 12, O_NEG = 13, O_SQRT = 14, O_LOG = 15, O_EXP = 16,
  O_INV = 17, O_SQUARE = 18, O_CUBE = 19, O_TANH = 20, O_SINH = 21, O_COSH = 22, O_ASIN = 23,
  O_ACOS = 24, O_ATAN = 25,
  O_NUM = 26
};

/* Arity of each opcode: terminals 0, binary functions 2, unary 1 ("maximum arity of 2"). */
int orc_arity(int op) {
  if (op == O_VAR || op == O_CONST) return 0;
  if (op >= O_ADD && op <= O_POW) return 2;
  if (op >= O_SIN && op <= O_ATAN) return 1;
  return -1;
}

static float payload_f(int32_t p) { float f; memcpy(&f, &p, 4); return f; }

/* ------------------------------------------------------------------------------------------------
 * Structure: S:41-66 (validate_prefix, depth, subtree_span), P:243 (stack bound).
 * ----------------------------------------------------------------------------------------------*/

/* validate_prefix: scan left->right with needed := 1, needed := needed - 1 + arity; valid iff
 * needed reaches 0 exactly at the final token and never earlier. Also checks opcodes and var range
 * (S:142 VariableOutOfRange). Returns 0 if valid, else 1 empty, 2 underflow, 3 dangling,
 * 4 unknown opcode, 5 variable out of range. */
int orc_validate(const onode* nodes, int64_t len, int n_cols) {
  if (len <= 0) return 1;
  int64_t needed = 1;
  for (int64_t i = 0; i < len; ++i) {
    if (needed == 0) return 2;                       /* tokens after the tree closed */
    int a = orc_arity(nodes[i].op);
    if (a < 0) return 4;
    if (nodes[i].op == O_VAR && (nodes[i].payload < 0 || nodes[i].payload >= n_cols)) return 5;
    needed = needed - 1 + a;
  }
  return needed == 0 ? 0 : 3;
}

/* subtree_span: end of the subtree rooted at start (same needed-counter scan). */
int64_t orc_subtree_end(const onode* nodes, int64_t len, int64_t start) {
  int64_t needed = 1, i = start;
  while (needed > 0 && i < len) { needed = needed - 1 + orc_arity(nodes[i].op); ++i; }
  return i;
}

/* depth: a lone terminal has depth 0. Recursive definition on the tree. */
static int depth_rec(const onode* nodes, int64_t len, int64_t i, int64_t* next) {
  int a = orc_arity(nodes[i].op);
  int64_t j = i + 1;
  int d = 0;
  for (int c = 0; c < a; ++c) {
    int dc = depth_rec(nodes, len, j, &j);
    if (dc + 1 > d) d = dc + 1;
  }
  *next = j;
  return d;
}
int orc_depth(const onode* nodes, int64_t len) {
  int64_t next;
  return depth_rec(nodes, len, 0, &next);
}

/* Brute-force maximum stack occupancy of the reverse-prefix stack evaluation ("reverse
 * iteration due to the prefix notation"): iterate nodes from last to first, a terminal
 * pushes (+1), a function of arity a pops a and pushes 1 (net 1-a). Only the counter is simulated. */
int orc_stack_need(const onode* nodes, int64_t len) {
  int64_t sp = 0, need = 0;
  for (int64_t i = len - 1; i >= 0; --i) {
    int a = orc_arity(nodes[i].op);
    sp = sp - a + 1;
    if (sp > need) need = sp;
  }
  return (int)need;
}

/* ------------------------------------------------------------------------------------------------
 * Evaluation: recursive tree walk in double (S:155 / S:609 "independent recursive tree-walk
 * evaluator"). Function semantics: SPEC's protected catalog, S:132 and DESIGN.md readings C2:
 *   div(a,b) = 1 if |b| < 1e-3 else a/b        log(a) = 0 if |a| < 1e-3 else ln|a|
 *   inv(a)   = 1 if |a| < 1e-3 else 1/a        sqrt(a) = sqrt(|a|)      exp(a) = min(e^a, 1e30)
 *   sinh, cosh clamped to +-1e30; asin/acos argument clamped to [-1,1];
 *   pow(a,b) = 1 if b == 0; else 0 if a == 0 and b > 0; 1e30 if a == 0 and b < 0;
 *              else min(|a|^b, 1e30)
 *   add sub mul min max sin cos tan abs neg square cube tanh atan: plain.
 * Operand order: the first operand is the first child in prefix order.
 *
 * Alongside the value, each node carries E, a rigorous-to-first-order bound on |fp32 result -
 * exact result| for an fp32 evaluation whose per-op rounding errors are within the budgets of
 * DESIGN.md "Tolerance model" (IEEE ops: 1 ulp; SFU-approximated ops: the budgets below). E uses
 * interval endpoints for monotone functions and Lipschitz constants otherwise. This is the
 * "exact result within the error bound" pin used to set per-row / per-program tolerances.
 * Flags: 1 = fp32 overflow (some |intermediate| > FLT_MAX or non-finite in double),
 *        2 = protected-branch ambiguous (|argument| within E of the 1e-3 threshold).
 * ----------------------------------------------------------------------------------------------*/
#define U32 (5.9604644775390625e-08)      /* 2^-24, fp32 unit roundoff */
#define SFU_ABS (3.5762786865234375e-07)  /* 2^-21.41 ~ 3.6e-7: MUFU sin/cos/lg2 absolute budget */
#define CLAMP_BIG 1e30
#define PROT 1e-3
#define FTZ_IN(v) (fabs(v) < (double)FLT_MIN ? fabs(v) : 0.0)

typedef struct { double v, e; int flags; } oval;

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* Exact (double) semantics of one function application. */
double orc_apply(int op, double a, double b) {
  switch (op) {
    case O_ADD: return a + b;
    case O_SUB: return a - b;
    case O_MUL: return a * b;
    case O_DIV: return fabs(b) < PROT ? 1.0 : a / b;
    case O_MIN: return fmin(a, b);
    case O_MAX: return fmax(a, b);
    case O_POW:
      if (b == 0.0) return 1.0;
      if (a == 0.0) return b > 0.0 ? 0.0 : CLAMP_BIG;
      return fmin(pow(fabs(a), b), CLAMP_BIG);
    case O_SIN: return sin(a);
    case O_COS: return cos(a);
    case O_TAN: return tan(a);
    case O_ABS: return fabs(a);
    case O_NEG: return -a;
    case O_SQRT: return sqrt(fabs(a));
    case O_LOG: return fabs(a) < PROT ? 0.0 : log(fabs(a));
    case O_EXP: return fmin(exp(a), CLAMP_BIG);
    case O_INV: return fabs(a) < PROT ? 1.0 : 1.0 / a;
    case O_SQUARE: return a * a;
    case O_CUBE: return a * a * a;
    case O_TANH: return tanh(a);
    case O_SINH: return clampd(sinh(a), -CLAMP_BIG, CLAMP_BIG);
    case O_COSH: return fmin(cosh(a), CLAMP_BIG);
    case O_ASIN: return asin(clampd(a, -1.0, 1.0));
    case O_ACOS: return acos(clampd(a, -1.0, 1.0));
    case O_ATAN: return atan(a);
  }
  return NAN;
}

/* Spread of a unary function over [a-e, a+e] around f(a) (used for monotone f). */
static double mono_spread(int op, double a, double e) {
  double f = orc_apply(op, a, 0), lo = orc_apply(op, a - e, 0), hi = orc_apply(op, a + e, 0);
  return fmax(fabs(hi - f), fabs(f - lo));
}

/* Is the protected test |x| < 1e-3 undecided for an fp32 value within e of x? */
static int ambiguous(double x, double e) {
  return fabs(fabs(x) - PROT) <= e;
}

static oval eval_rec(const onode* nodes, int64_t* i, const float* X, int64_t ld, int64_t row) {
  onode n = nodes[*i];
  *i += 1;
  oval r = {0.0, 0.0, 0};
  /* a subnormal fp32 input is flushed to zero by an FTZ evaluation: error |v| < FLT_MIN */
  if (n.op == O_VAR) { r.v = (double)X[(int64_t)n.payload * ld + row]; r.e = FTZ_IN(r.v); return r; }
  if (n.op == O_CONST) { r.v = (double)payload_f(n.payload); r.e = FTZ_IN(r.v); return r; }
  int ar = orc_arity(n.op);
  oval A = eval_rec(nodes, i, X, ld, row);
  oval B = {0.0, 0.0, 0};
  if (ar == 2) B = eval_rec(nodes, i, X, ld, row);
  double a = A.v, b = B.v, ea = A.e, eb = B.e;
  r.flags = A.flags | B.flags;
  r.v = orc_apply(n.op, a, b);
  double v = r.v, av = fabs(v);
  switch (n.op) {
    case O_ADD: case O_SUB: r.e = ea + eb + U32 * av; break;
    case O_MUL: r.e = fabs(b) * ea + fabs(a) * eb + ea * eb + U32 * av; break;
    case O_DIV:
      if (ambiguous(b, eb)) { r.flags |= 2; r.e = fabs(a) + ea + 1.0 + av; }
      else if (fabs(b) < PROT) r.e = 0.0;
      else r.e = (fabs(b) > eb ? (ea + av * eb) / (fabs(b) - eb) : INFINITY) + 3 * U32 * av;
      break;
    case O_MIN: case O_MAX: r.e = fmax(ea, eb); break;
    case O_POW:
      if (b == 0.0 && eb == 0.0) r.e = 0.0;
      else if (a == 0.0 || fabs(a) <= ea) r.e = INFINITY;
      else {
        double la = fabs(log(fabs(a)));
        /* |a|^b = 2^(b log2|a|): input sensitivities plus lg2/ex2/mul rounding budgets */
        r.e = av * (fabs(b) * ea / (fabs(a) - ea) + la * eb + (fabs(b) * la + 2.0) * 4 * U32);
      }
      break;
    case O_SIN: case O_COS:
      r.e = fmin(2.0, ea + SFU_ABS + fabs(a) * 2 * U32);
      break;
    case O_TAN: {
      /* interval must not contain a pole; tan increasing on it */
      double lo = a - ea, hi = a + ea;
      double k_lo = floor((lo - M_PI_2) / M_PI), k_hi = floor((hi - M_PI_2) / M_PI);
      if (k_lo != k_hi) { r.e = INFINITY; break; }
      double es = SFU_ABS + fabs(a) * 2 * U32;
      double c = fabs(cos(a));
      double round = (c > es) ? (es + av * es) / (c - es) + 2 * U32 * av : INFINITY;
      r.e = fmax(fabs(tan(hi) - v), fabs(v - tan(lo))) + round;
      break;
    }
    case O_ABS: case O_NEG: r.e = ea; break;
    case O_SQRT: {
      double s = sqrt(ea), d = fabs(a) > 0 ? ea / sqrt(fabs(a)) : INFINITY;
      r.e = fmin(s, d) + 2 * U32 * av;
      break;
    }
    case O_LOG:
      if (ambiguous(a, ea)) { r.flags |= 2; r.e = fabs(log(PROT)) + av + 1.0; }
      else if (fabs(a) < PROT) r.e = 0.0;
      else r.e = (fabs(a) > ea ? ea / (fabs(a) - ea) : INFINITY) + 2 * SFU_ABS + 4 * U32 * av;
      break;
    case O_EXP:
      r.e = mono_spread(O_EXP, a, ea) + av * (4 * U32 + fabs(a) * 2 * U32);
      break;
    case O_INV:
      if (ambiguous(a, ea)) { r.flags |= 2; r.e = 1.0 + av + 1.0 / PROT; }
      else if (fabs(a) < PROT) r.e = 0.0;
      else r.e = (fabs(a) > ea ? ea / (fabs(a) * (fabs(a) - ea)) : INFINITY) + 2 * U32 * av;
      break;
    case O_SQUARE: r.e = 2 * fabs(a) * ea + ea * ea + U32 * av; break;
    case O_CUBE: {
      double m = fabs(a) + ea;
      r.e = 3 * m * m * ea + 2 * U32 * av;
      break;
    }
    case O_TANH: case O_ATAN: case O_ASIN: case O_ACOS:
      r.e = mono_spread(n.op, a, ea) + 2 * SFU_ABS + 4 * U32 * av;
      break;
    case O_SINH:
      r.e = mono_spread(O_SINH, a, ea) + av * (4 * U32 + fabs(a) * 2 * U32) + 2 * SFU_ABS;
      break;
    case O_COSH: {
      double f = v, hi = orc_apply(O_COSH, fabs(a) + ea, 0);
      r.e = fabs(hi - f) + av * (4 * U32 + fabs(a) * 2 * U32);
      break;
    }
  }
  /* underflow: an fp32 result below FLT_MIN is subnormal (IEEE, absolute error <= 2^-150) or
   * flushed to zero (FTZ evaluation, error < FLT_MIN); the relative budgets above do not cover
   * either, so every function result carries an absolute FLT_MIN term */
  r.e += (double)FLT_MIN;
  if (!isfinite(v) || av > (double)FLT_MAX) r.flags |= 1;
  if (isnan(r.e)) r.e = INFINITY;   /* an undefined first-order bound is "unbounded" */
  return r;
}

/* Evaluate one valid program on rows [0, n_rows) of column-major X (ld = leading dimension).
 * out_v/out_e receive value and error bound per row; out_flags (may be NULL) the row flags. */
void orc_eval_program(const onode* nodes, int64_t len, const float* X, int64_t ld, int64_t n_rows,
                      double* out_v, double* out_e, uint8_t* out_flags) {
  (void)len;
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t i = 0;
    oval o = eval_rec(nodes, &i, X, ld, r);
    out_v[r] = o.v;
    out_e[r] = o.e;
    if (out_flags) out_flags[r] = (uint8_t)o.flags;
  }
}

/* Value-only evaluation at a single row (no error bookkeeping). */
double orc_eval_row(const onode* nodes, const float* X, int64_t ld, int64_t row) {
  int64_t i = 0;
  return eval_rec(nodes, &i, X, ld, row).v;
}

/* ------------------------------------------------------------------------------------------------
 * Fitness metrics, P:256-273 (weighted MAE, MSE, RMSE, logistic loss, Pearson).
 * Two-pass, double. Rows with w == 0 contribute nothing and are skipped (reading C5).
 * w == NULL means all ones. Metric ids: 0 MAE, 1 MSE, 2 RMSE, 3 LogLoss, 4 Pearson.
 * Non-finite loss fitness -> +inf (reading C4). Pearson with zero variance or non-finite r -> 0
 * and *undefined = 1 (reading C4; S:202 names the condition).
 * ----------------------------------------------------------------------------------------------*/
static double row_loss(int metric, double y, double yh) {
  switch (metric) {
    case 0: return fabs(y - yh);                       /* S:192 MAE */
    case 1: case 2: return (y - yh) * (y - yh);        /* S:192 MSE / RMSE */
    case 3: {                                          /* S:191-192 logistic loss, literal */
      double p = 1.0 / (1.0 + exp(-yh));
      p = clampd(p, 1e-15, 1.0 - 1e-15);
      return -(y * log(p) + (1.0 - y) * log(1.0 - p));
    }
  }
  return NAN;
}

/* rank_vector: ranks 1..n ascending, ties get the average of the positions they cover
 * ("average-tie rule"). Sorting is a library step (qsort); ties are then averaged per run. */
typedef struct { double v; int64_t i; } vidx;
static int cmp_vidx(const void* a, const void* b) {
  const double x = ((const vidx*)a)->v, y = ((const vidx*)b)->v;
  return x < y ? -1 : (x > y ? 1 : 0);
}
void orc_rank_vector(const double* v, int64_t n, double* ranks) {
  vidx* t = (vidx*)malloc(sizeof(vidx) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) { t[i].v = v[i]; t[i].i = i; }
  qsort(t, (size_t)n, sizeof(vidx), cmp_vidx);
  for (int64_t s = 0; s < n;) {
    int64_t e = s + 1;
    while (e < n && t[e].v == t[s].v) ++e;
    const double r = 0.5 * (double)(s + 1 + e);   /* average of positions s+1 .. e */
    for (int64_t k = s; k < e; ++k) ranks[t[k].i] = r;
    s = e;
  }
  free(t);
}

/* 1 if v takes one value on every live row (w != 0): zero variance exactly. The rounded
 * weighted mean of equal values need not equal them, so this is decided on the values. */
static int live_constant(const double* v, const float* w, int64_t n) {
  int64_t first = -1;
  for (int64_t i = 0; i < n; ++i) {
    if ((w ? (double)w[i] : 1.0) == 0.0) continue;
    if (first < 0) first = i;
    else if (!(v[i] == v[first])) return 0;
  }
  return 1;
}

/* weighted Pearson correlation of a and b: weighted means first, then centred sums
 * (two-pass); w == 0 rows skipped; zero variance or non-finite r -> 0 and *undefined = 1. */
static double pearson_w(const double* a, const double* b, const float* w, int64_t n, double W,
                        int* undefined) {
  if (live_constant(a, w, n) || live_constant(b, w, n)) {
    if (undefined) *undefined = 1;
    return 0.0;
  }
  double ma = 0.0, mb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    ma += wi * a[i];
    mb += wi * b[i];
  }
  ma /= W;
  mb /= W;
  double sab = 0.0, saa = 0.0, sbb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    double da = a[i] - ma, db = b[i] - mb;
    sab += wi * da * db;
    saa += wi * da * da;
    sbb += wi * db * db;
  }
  double r = sab / sqrt(saa * sbb);
  if (!isfinite(r) || !(saa > 0.0) || !(sbb > 0.0)) {
    if (undefined) *undefined = 1;
    return 0.0;
  }
  return r;
}

double orc_fitness(int metric, const double* yh, const float* y, const float* w, int64_t n,
                   int* undefined) {
  if (undefined) *undefined = 0;
  if (metric == 5) {
    /* Spearman: Pearson of rank_vector(y) and rank_vector(yhat) with the same weights.
     * The ranks are taken over every row (rank_vector has no weights). Reading: the predictions
     * are ranked at the evaluator's precision (fp32: where floating point decides an integer,
     * both sides decide in the kernel's precision); non-finite predictions leave the ranks
     * undefined (S:210 pre: finite values) -> 0 and *undefined = 1, as for Pearson. */
    double W = 0.0;
    for (int64_t i = 0; i < n; ++i) W += w ? (double)w[i] : 1.0;
    double* a = (double*)malloc(sizeof(double) * (size_t)n);
    double* b = (double*)malloc(sizeof(double) * (size_t)n);
    double* ra = (double*)malloc(sizeof(double) * (size_t)n);
    double* rb = (double*)malloc(sizeof(double) * (size_t)n);
    int finite = 1;
    for (int64_t i = 0; i < n; ++i) {
      a[i] = (double)(float)yh[i];
      b[i] = (double)y[i];
      if (!isfinite(a[i])) finite = 0;
    }
    double r = 0.0;
    if (!finite) {
      if (undefined) *undefined = 1;
    } else {
      orc_rank_vector(a, n, ra);
      orc_rank_vector(b, n, rb);
      r = pearson_w(ra, rb, w, n, W, undefined);
    }
    free(a); free(b); free(ra); free(rb);
    return r;
  }
  double W = 0.0;
  for (int64_t i = 0; i < n; ++i) W += w ? (double)w[i] : 1.0;
  if (metric <= 3) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double wi = w ? (double)w[i] : 1.0;
      if (wi == 0.0) continue;
      s += wi * row_loss(metric, (double)y[i], yh[i]);
    }
    double f = s / W;
    if (metric == 2) f = sqrt(f);
    if (!isfinite(f)) f = INFINITY;
    return f;
  }
  /* Pearson: weighted means first, then centred sums (two-pass). A prediction that
   * is the same value on every live row has zero variance exactly (S:202 ConstantVector): the
   * rounded mean of equal values need not equal them, so this is decided on the values. */
  if (live_constant(yh, w, n)) {
    if (undefined) *undefined = 1;
    return 0.0;
  }
  double my = 0.0, mh = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    my += wi * (double)y[i];
    mh += wi * yh[i];
  }
  my /= W;
  mh /= W;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    double dy = (double)y[i] - my, dh = yh[i] - mh;
    sxy += wi * dh * dy;
    sxx += wi * dh * dh;
    syy += wi * dy * dy;
  }
  double r = sxy / sqrt(sxx * syy);
  if (!isfinite(r) || !(sxx > 0.0) || !(syy > 0.0)) {
    if (undefined) *undefined = 1;
    return 0.0;
  }
  return r;
}

/* Propagated fitness tolerance: sum_i |d fitness / d yhat_i| * E_i,
 * evaluated at the exact predictions. For RMSE the chain rule through sqrt is applied. */
double orc_fitness_sensitivity(int metric, const double* yh, const double* E, const float* y,
                               const float* w, int64_t n) {
  double W = 0.0;
  for (int64_t i = 0; i < n; ++i) W += w ? (double)w[i] : 1.0;
  double s = 0.0;
  if (metric <= 3) {
    for (int64_t i = 0; i < n; ++i) {
      double wi = w ? (double)w[i] : 1.0;
      if (wi == 0.0) continue;
      double d = yh[i] - (double)y[i], g;
      if (metric == 0) g = 1.0;
      else if (metric <= 2) g = 2.0 * fabs(d) + E[i];
      else g = fabs(1.0 / (1.0 + exp(-yh[i])) - (double)y[i]) + 0.25 * E[i];
      double c = g * E[i];
      /* a clamped log-loss row changes by at most the clamp range -ln(1e-15) */
      if (metric == 3 && !(c <= 34.538776394910684)) c = 34.538776394910684;
      s += wi * c;
    }
    s /= W;
    if (metric == 2) { /* |sqrt(a) - sqrt(b)| <= min(|a-b| / sqrt(a), sqrt(|a-b|)) */
      double rm = sqrt(orc_fitness(1, yh, y, w, n, NULL));
      s = rm > 0 ? fmin(s / rm, sqrt(s)) : sqrt(s);
    }
    return s;
  }
  /* Spearman: ranks change by whole steps, no first-order bound (tests use exactly representable
   * inputs or a rank-swap tolerance) */
  if (metric == 5) return 0.0;
  /* Pearson: |dr/dyh_i| = w_i |(y_i - my)/sqrt(sxx syy) - r (yh_i - mh)/sxx|, bounded by the sum
   * of the two magnitudes */
  double my = 0.0, mh = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    my += wi * (double)y[i];
    mh += wi * yh[i];
  }
  my /= W;
  mh /= W;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    double dy = (double)y[i] - my, dh = yh[i] - mh;
    sxy += wi * dh * dy;
    sxx += wi * dh * dh;
    syy += wi * dy * dy;
  }
  if (!(sxx > 0.0) || !(syy > 0.0)) return INFINITY;
  double r = sxy / sqrt(sxx * syy);
  for (int64_t i = 0; i < n; ++i) {
    double wi = w ? (double)w[i] : 1.0;
    if (wi == 0.0) continue;
    /* triangle inequality instead of the difference: the two terms can cancel to far below
     * their rounding error (outliers near the 1e30 clamps), which would understate the bound */
    double g = fabs((double)y[i] - my) / sqrt(sxx * syy) + fabs(r) * fabs(yh[i] - mh) / sxx;
    s += wi * g * E[i];
  }
  /* r lies in [-1, 1]: a bound of 2 or more says nothing (no usable first-order bound) */
  if (!(s < 2.0)) s = INFINITY;
  return s;
}

/* ------------------------------------------------------------------------------------------------
 * Philox4x32-10 ("Philox counter-based RNG" [Salmon et al. 2011]). Round function and
 * constants from the Random123 definition: multipliers 0xD2511F53, 0xCD9E8D57; Weyl key
 * increments 0x9E3779B9, 0xBB67AE85; 10 rounds. Pinned by the Random123 known-answer vectors.
 * ----------------------------------------------------------------------------------------------*/
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------------------------------
 * Tournament selection, P:218-226 (one tournament = k random indices, keep the best
 * parsimony-adjusted fitness) with Eqs. 1-2: penalty = c * len; adjusted =
 * raw + penalty (lower-better) or raw - penalty (higher-better). Readings (C10):
 *   draws with replacement; draw i of tournament t = word (i mod 4) of
 *   Philox(ctr = (t, generation, i / 4, 0), key = (seed_lo, seed_hi));
 *   index = (uint64(word) * n) >> 32;  adjusted in fp32 with explicit roundings (no FMA);
 *   NaN adjusted fitness is the worst value; ties -> smallest population index.
 * ----------------------------------------------------------------------------------------------*/
int32_t orc_tournament_one(const float* fitness, const int32_t* lens, int32_t n, int32_t t, int32_t k,
                           float c, int higher_better, uint64_t seed, uint32_t generation) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  int32_t best = -1;
  float best_adj = 0.0f;
  for (int32_t i = 0; i < k; ++i) {
    uint32_t ctr[4] = {(uint32_t)t, generation, (uint32_t)(i / 4), 0u}, out[4];
    orc_philox4x32_10(ctr, key, out);
    int32_t idx = (int32_t)(((uint64_t)out[i % 4] * (uint64_t)n) >> 32);
    volatile float pen = c * (float)lens[idx];           /* Eq. 1, fp32 */
    float adj = higher_better ? fitness[idx] - pen : fitness[idx] + pen; /* Eq. 2, fp32 */
    if (isnan(adj)) adj = higher_better ? -INFINITY : INFINITY;
    int better;
    if (best < 0) better = 1;
    else if (higher_better) better = adj > best_adj || (adj == best_adj && idx < best);
    else better = adj < best_adj || (adj == best_adj && idx < best);
    if (better) { best = idx; best_adj = adj; }
  }
  return best;
}

void orc_tournament(const float* fitness, const int32_t* lens, int32_t n, int32_t n_tournaments,
                    int32_t k, float c, int higher_better, uint64_t seed, uint32_t generation,
                    int32_t* winners) {
  for (int32_t t = 0; t < n_tournaments; ++t)
    winners[t] = orc_tournament_one(fitness, lens, n, t, k, c, higher_better, seed, generation);
}

/* ------------------------------------------------------------------------------------------------
 * Pagie polynomial, Eq. 3: f(x, y) = 1/(1 + x^-4) + 1/(1 + y^-4) on [-5, 5]^2.
 * A zero coordinate contributes its limit value 0.
 * ----------------------------------------------------------------------------------------------*/
static double pagie_term(double x) {
  if (x == 0.0) return 0.0;
  return 1.0 / (1.0 + pow(x, -4.0));
}
double orc_pagie(double x, double y) { return pagie_term(x) + pagie_term(y); }

/* ------------------------------------------------------------------------------------------------
 * Whole-population convenience used by tests and by bench.py's cpu_baseline: for every program,
 * evaluate all rows and compute the fitness; also the propagated tolerance and program flags
 * (bit 0 overflow, bit 1 ambiguous branch, bit 2 invalid program, bit 3 undefined correlation).
 * Work buffers are allocated here; single-threaded on purpose (the oracle "as it stands").
 * ----------------------------------------------------------------------------------------------*/
void orc_population_fitness(const onode* nodes, const int64_t* offsets, int32_t n_programs,
                            const float* X, int64_t ld, const float* y, const float* w,
                            int64_t n_rows, int32_t n_cols, int metric, double* out_fitness,
                            double* out_sens, int32_t* out_flags) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n_rows);
  double* e = (double*)malloc(sizeof(double) * (size_t)n_rows);
  uint8_t* f = (uint8_t*)malloc((size_t)n_rows);
  for (int32_t p = 0; p < n_programs; ++p) {
    const onode* prog = nodes + offsets[p];
    int64_t len = offsets[p + 1] - offsets[p];
    int32_t flags = 0;
    if (orc_validate(prog, len, n_cols) != 0) {
      out_fitness[p] = metric >= 4 ? -INFINITY : INFINITY;
      if (out_sens) out_sens[p] = 0.0;
      if (out_flags) out_flags[p] = 4;
      continue;
    }
    orc_eval_program(prog, len, X, ld, n_rows, v, e, f);
    for (int64_t r = 0; r < n_rows; ++r) {
      double wr = w ? (double)w[r] : 1.0;
      if (wr != 0.0) flags |= f[r];
    }
    int undef = 0;
    out_fitness[p] = orc_fitness(metric, v, y, w, n_rows, &undef);
    if (undef) flags |= 8;
    if (out_sens) out_sens[p] = orc_fitness_sensitivity(metric, v, e, y, w, n_rows);
    if (out_flags) out_flags[p] = flags;
  }
  free(v);
  free(e);
  free(f);
}
