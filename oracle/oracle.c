/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential CPU oracle for the reduction of arXiv 1710.07358:
 *   "Given a set X with n values, X = {x_0, x_1, ..., x_{n-1}}, compute
 *    x_0 (x) x_1 (x) ... (x) x_{n-1}"                  (§1.1)
 * evaluated as Algorithm 1 "Summation(A)" -- a single
 * left-to-right fold -- generalised from + to the combiner (x), with a wider
 * accumulator for floating point: double-double (an unevaluated fp64 pair
 * hi + lo, TwoSum / FMA TwoProduct) for fp32 and fp64 data alike (PAPER.md
 * P:50 footnote 3 names double precision and compensated summation as the
 * mitigations). Its own error, <= ~4n 2^-104 sum|x_i|, stays far below the
 * 4 eps sum|x_i| tolerance at every n < 2^40 (a plain fp64 fold of fp32 data
 * would reach 16 eps32 sum|x_i| at n = 2^34 in the worst case). The fold
 * order is exactly Algorithm 1's.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library. It shares no code, header,
 * table or constant with the CUDA path (paper_1710_07358_b200/); the dtype and
 * op codes below are restated numbers, not an include.
 *
 * Readings of the paper taken here (all listed in DESIGN.md "Readings"):
 *  R1  n == 0 returns the initial accumulator of Algorithm 1, i.e. the
 *      combiner's identity (+0.0 for float +, INFINITY for min as Listing 1's
 *      `accumulator = INFINITY`).
 *  R2  n >= 1 folds x_0 (x) x_1 (x) ... literally: the fold starts at
 *      x_0, so the sign of a float zero sum is -0.0 iff every term is -0.0.
 *  R3  Integer + and x wrap modulo 2^w (two's complement); min/max compare
 *      signed for int32/int64 and unsigned for uint32; and/or/xor act on raw
 *      bits (P:23's AND/OR/XOR/intersection/union read as bitwise).
 *  R4  Float min/max are IEEE 754-2019 minimum/maximum: NaN propagates and
 *      -0.0 < +0.0.
 *  R5  Bitwise ops on float dtypes are rejected (status 2).
 *  R6  argmin / argmax (the paper's consumers are
 *      shortest paths and golden-section search): the value of
 *      min / max under R4's order together with the SMALLEST index attaining
 *      it; a NaN anywhere wins (value NaN, index of the first NaN); -0.0 ranks
 *      below +0.0; empty input -> identity value and index -1.
 *  R17 The exact sum ("reproducible": P:50 fn 2 shows
 *      that float + depends on the evaluation order, fn 3 names the
 *      mitigations): the real-number sum of the n float values, computed
 *      exactly, rounded ONCE to the dtype (round to nearest, ties to even).
 *      It is the one float result no evaluation order can change. Specials:
 *      any NaN, or +inf together with -inf -> NaN; else any +-inf -> that inf;
 *      a finite exact sum beyond the dtype's range rounds to +-inf; an exact
 *      zero is -0.0 iff every term is -0.0 (R2), else +0.0; n == 0 -> +0.0.
 *      Integers: identical to the sum (already exact).
 *
 * Parity pins for every function: tests/test_oracle_pins.py (DESIGN.md
 * "Oracle pins"). No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* dtype / op / status numbers (restated, see header comment) */
enum { OR_INT32 = 0, OR_UINT32 = 1, OR_INT64 = 2, OR_FLOAT32 = 3, OR_FLOAT64 = 4 };
enum { OR_SUM = 0, OR_PROD = 1, OR_MIN = 2, OR_MAX = 3, OR_AND = 4, OR_OR = 5, OR_XOR = 6,
       OR_ARGMIN = 7, OR_ARGMAX = 8, OR_SUM_COMPENSATED = 9, OR_SUM_EXACT = 10 };
enum { OR_OK = 0, OR_INVALID = 1, OR_UNSUPPORTED = 2 };

/* R17: the exact sum is a two's-complement fixed-point integer of
 * OR_BIG_LIMBS 32-bit limbs whose unit (bit 0) is the dtype's smallest
 * subnormal, 2^-149 (fp32) / 2^-1074 (fp64): every finite value of the dtype
 * is an integer multiple of it, below 2^(128+149) / 2^(1024+1074), so 2304
 * bits hold any sum of < 2^40 terms with room to spare. */
#define OR_BIG_LIMBS 72

/* Fold state; mirrored by oracle/__init__.py (ctypes). */
typedef struct {
  int32_t dtype, op;
  uint64_t count;       /* elements folded so far                           */
  uint64_t ibits;       /* integer accumulator (unsigned, width of dtype)   */
  double hi, lo;        /* float accumulator; lo used for double-double     */
  double abs_hi, abs_lo;/* sum_i |x_i| as double-double (tolerance input)   */
  int32_t all_negzero;  /* every float term so far is -0.0 (reading R2)     */
  int32_t pad;
  uint64_t best_idx;    /* argmin / argmax: index of the current best (R6)  */
  uint32_t big[OR_BIG_LIMBS]; /* exact sum (R17), little-endian limbs       */
  int32_t nan_seen, pinf_seen, ninf_seen, pad2;   /* exact sum: specials    */
} or_state;

static int is_float(int dt) { return dt == OR_FLOAT32 || dt == OR_FLOAT64; }

/* ---- exact two-term transformations (Knuth TwoSum, Dekker/FMA TwoProduct) -- */
static void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double bp = ss - a;
  *e = (a - (ss - bp)) + (b - bp);
  *s = ss;
}
static void fast_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}

/* double-double += double  (float +, and sum |x|) */
static void dd_add(double* hi, double* lo, double x) {
  if (!isfinite(*hi) || !isfinite(x)) { *hi = *hi + x; *lo = 0.0; return; }
  double s, e;
  two_sum(*hi, x, &s, &e);
  if (!isfinite(s)) { *hi = s; *lo = 0.0; return; }   /* overflow: +-inf (TwoSum's error is NaN) */
  e += *lo;
  fast_two_sum(s, e, hi, lo);
}

/* double-double *= double  (float x) */
static void dd_mul(double* hi, double* lo, double x) {
  double p = *hi * x;
  if (!isfinite(p) || p == 0.0) { *hi = p; *lo = 0.0; return; }
  double e = fma(*hi, x, -p);
  e = fma(*lo, x, e);
  fast_two_sum(p, e, hi, lo);
}

/* IEEE 754-2019 minimum / maximum (reading R4) */
static double ieee_min(double a, double b) {
  if (isnan(a) || isnan(b)) return NAN;
  if (a < b) return a;
  if (b < a) return b;
  if (a == 0.0 && b == 0.0) return (signbit(a) || signbit(b)) ? -0.0 : 0.0;
  return a;
}
static double ieee_max(double a, double b) {
  if (isnan(a) || isnan(b)) return NAN;
  if (a > b) return a;
  if (b > a) return b;
  if (a == 0.0 && b == 0.0) return (signbit(a) && signbit(b)) ? -0.0 : 0.0;
  return a;
}

static int is_arg(int op) { return op == OR_ARGMIN || op == OR_ARGMAX; }

/* ---- exact sum (R17): plain multi-limb integer arithmetic ------------------ */
static int lsb_exp(int dt) { return dt == OR_FLOAT32 ? -149 : -1074; }

/* big += v * 2^(32k) (v < 2^96 given as three limbs), mod 2^(32*OR_BIG_LIMBS) */
static void big_add3(uint32_t* big, int k, const uint32_t v[3]) {
  uint64_t carry = 0;
  for (int i = k; i < OR_BIG_LIMBS; ++i) {
    uint64_t t = (uint64_t)big[i] + carry + (i - k < 3 ? v[i - k] : 0);
    big[i] = (uint32_t)t;
    carry = t >> 32;
    if (i - k >= 2 && carry == 0) break;
  }
}
/* big -= v * 2^(32k) */
static void big_sub3(uint32_t* big, int k, const uint32_t v[3]) {
  uint64_t borrow = 0;
  for (int i = k; i < OR_BIG_LIMBS; ++i) {
    uint64_t sub = (uint64_t)(i - k < 3 ? v[i - k] : 0) + borrow;
    borrow = (uint64_t)big[i] < sub;
    big[i] = (uint32_t)((uint64_t)big[i] - sub);
    if (i - k >= 2 && borrow == 0) break;
  }
}
/* big += x exactly, x finite (x is an integer multiple of 2^lsb) */
static void big_add_float(uint32_t* big, double x, int lsb) {
  if (x == 0.0) return;
  int e;
  double m = frexp(fabs(x), &e);            /* |x| = m * 2^e, 0.5 <= m < 1 */
  uint64_t M = (uint64_t)ldexp(m, 53);      /* |x| = M * 2^(e-53), exact */
  int pos = e - 53 - lsb;                   /* bit position of M's unit */
  while (pos < 0) { M >>= 1; ++pos; }       /* drops only zero bits (x is a multiple of 2^lsb) */
  unsigned __int128 v = (unsigned __int128)M << (pos % 32);
  const uint32_t limbs[3] = {(uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64)};
  if (x > 0) big_add3(big, pos / 32, limbs);
  else big_sub3(big, pos / 32, limbs);
}
static int big_bit(const uint32_t* b, int i) { return i < 0 ? 0 : (int)((b[i / 32] >> (i % 32)) & 1u); }

/* The fixed-point integer `big` times 2^lsb, rounded to p significant bits
 * (round to nearest, ties to even); returned as a double (exact for p <= 53,
 * +-inf past the double range). */
static double big_round(const uint32_t* big_in, int p, int lsb) {
  uint32_t b[OR_BIG_LIMBS];
  memcpy(b, big_in, sizeof(b));
  const int neg = (int)(b[OR_BIG_LIMBS - 1] >> 31);
  if (neg) {                                 /* magnitude: two's complement negation */
    uint64_t carry = 1;
    for (int i = 0; i < OR_BIG_LIMBS; ++i) {
      uint64_t t = (uint64_t)(uint32_t)~b[i] + carry;
      b[i] = (uint32_t)t;
      carry = t >> 32;
    }
  }
  int P = -1;                                /* highest set bit */
  for (int i = 32 * OR_BIG_LIMBS - 1; i >= 0; --i)
    if (big_bit(b, i)) { P = i; break; }
  if (P < 0) return 0.0;
  double mag;
  if (P < p) {                               /* fits: exact */
    uint64_t q = 0;
    for (int i = P; i >= 0; --i) q = 2 * q + (uint64_t)big_bit(b, i);
    mag = ldexp((double)q, lsb);
  } else {
    const int shift = P + 1 - p;             /* bits below the p kept ones */
    uint64_t q = 0;
    for (int i = P; i >= shift; --i) q = 2 * q + (uint64_t)big_bit(b, i);
    const int half = big_bit(b, shift - 1);
    int sticky = 0;
    for (int i = shift - 2; i >= 0 && !sticky; --i) sticky = big_bit(b, i);
    if (half && (sticky || (q & 1u))) q += 1; /* ties to even */
    mag = ldexp((double)q, shift + lsb);     /* q <= 2^p: exact, or inf */
  }
  return neg ? -mag : mag;
}

int or_init(or_state* st, int dtype, int op) {
  if (!st || dtype < 0 || dtype > 4 || op < 0 || op > 10) return OR_INVALID;
  /* integer sums are exact already (R17) */
  if (op == OR_SUM_EXACT && !is_float(dtype)) op = OR_SUM;
  /* the compensated sum of the library has the same definition as
   * the sum; this oracle's sum accumulators are already fp64 / double-double */
  if (op == OR_SUM_COMPENSATED) op = OR_SUM;
  if (is_float(dtype) && op >= OR_AND && op <= OR_XOR) return OR_UNSUPPORTED; /* R5 */
  memset(st, 0, sizeof(*st));
  st->dtype = dtype;
  st->op = op;
  st->all_negzero = 1;
  return OR_OK;
}

/* Integer combine (R3), on the unsigned bit pattern of width 32 or 64. */
static uint64_t int_combine(int dt, int op, uint64_t a, uint64_t b) {
  if (dt == OR_INT64) {
    switch (op) {
      case OR_SUM: return a + b;
      case OR_PROD: return a * b;
      case OR_MIN: return ((int64_t)a < (int64_t)b) ? a : b;
      case OR_MAX: return ((int64_t)a > (int64_t)b) ? a : b;
      case OR_AND: return a & b;
      case OR_OR: return a | b;
      default: return a ^ b;
    }
  } else {
    uint32_t x = (uint32_t)a, y = (uint32_t)b, r;
    switch (op) {
      case OR_SUM: r = x + y; break;
      case OR_PROD: r = x * y; break;
      case OR_MIN: r = (dt == OR_INT32) ? (((int32_t)x < (int32_t)y) ? x : y) : ((x < y) ? x : y); break;
      case OR_MAX: r = (dt == OR_INT32) ? (((int32_t)x > (int32_t)y) ? x : y) : ((x > y) ? x : y); break;
      case OR_AND: r = x & y; break;
      case OR_OR: r = x | y; break;
      default: r = x ^ y; break;
    }
    return r;
  }
}

/* R6: is candidate a strictly better than the current best b? (ties keep b,
 * the earlier index) */
static int int_better(int dt, int op, uint64_t a, uint64_t b) {
  int lt, gt;
  if (dt == OR_INT64) { lt = (int64_t)a < (int64_t)b; gt = (int64_t)a > (int64_t)b; }
  else if (dt == OR_INT32) { lt = (int32_t)(uint32_t)a < (int32_t)(uint32_t)b; gt = (int32_t)(uint32_t)a > (int32_t)(uint32_t)b; }
  else { lt = (uint32_t)a < (uint32_t)b; gt = (uint32_t)a > (uint32_t)b; }
  return op == OR_ARGMIN ? lt : gt;
}
static int float_better(int op, double a, double b) {
  if (isnan(b)) return 0;                 /* a NaN best is never displaced */
  if (isnan(a)) return 1;                 /* the first NaN wins */
  if (op == OR_ARGMIN) {
    if (a < b) return 1;
    return a == 0.0 && b == 0.0 && signbit(a) && !signbit(b);   /* -0 < +0 */
  }
  if (a > b) return 1;
  return a == 0.0 && b == 0.0 && !signbit(a) && signbit(b);
}

/* Algorithm 1, body of the `for i <- 1 to n` loop, one element. */
static void fold_one(or_state* st, const unsigned char* p) {
  const int dt = st->dtype, op = st->op;
  if (is_arg(op)) {
    if (!is_float(dt)) {
      uint64_t v = 0;
      if (dt == OR_INT64) memcpy(&v, p, 8);
      else { uint32_t w; memcpy(&w, p, 4); v = w; }
      if (st->count == 0 || int_better(dt, op, v, st->ibits)) { st->ibits = v; st->best_idx = st->count; }
    } else {
      double x;
      if (dt == OR_FLOAT32) { float f; memcpy(&f, p, 4); x = (double)f; }
      else memcpy(&x, p, 8);
      if (st->count == 0 || float_better(op, x, st->hi)) { st->hi = x; st->best_idx = st->count; }
    }
    st->count++;
    return;
  }
  if (!is_float(dt)) {
    uint64_t v = 0;
    if (dt == OR_INT64) memcpy(&v, p, 8);
    else { uint32_t w; memcpy(&w, p, 4); v = w; }
    st->ibits = (st->count == 0) ? v : int_combine(dt, op, st->ibits, v); /* R2 */
    st->count++;
    return;
  }
  double x;
  if (dt == OR_FLOAT32) { float f; memcpy(&f, p, 4); x = (double)f; } /* exact widening */
  else memcpy(&x, p, 8);
  dd_add(&st->abs_hi, &st->abs_lo, fabs(x));
  if (!(x == 0.0 && signbit(x))) st->all_negzero = 0;
  if (op == OR_SUM_EXACT) {       /* R17: the fold adds x_i to the exact sum */
    if (isnan(x)) st->nan_seen = 1;
    else if (isinf(x)) { if (x > 0) st->pinf_seen = 1; else st->ninf_seen = 1; }
    else big_add_float(st->big, x, lsb_exp(dt));
    st->count++;
    return;
  }
  if (st->count == 0) {           /* R2: the fold starts at x_0 */
    st->hi = x; st->lo = 0.0; st->count = 1;
    return;
  }
  switch (op) {
    case OR_SUM: dd_add(&st->hi, &st->lo, x); break;     /* double-double */
    case OR_PROD: dd_mul(&st->hi, &st->lo, x); break;
    case OR_MIN: st->hi = ieee_min(st->hi, x); break;
    case OR_MAX: st->hi = ieee_max(st->hi, x); break;
    default: break;
  }
  st->count++;
}

/* Fold x[0..n) into the running state (chunked calls == one long fold). */
int or_fold(or_state* st, const void* x, uint64_t n) {
  if (!st || (!x && n)) return OR_INVALID;
  const int s = (st->dtype == OR_INT64 || st->dtype == OR_FLOAT64) ? 8 : 4;
  const unsigned char* p = (const unsigned char*)x;
  for (uint64_t i = 0; i < n; ++i) fold_one(st, p + i * (uint64_t)s);
  return OR_OK;
}

/* Result of an empty fold: Algorithm 1's initial accumulator (R1); argmin /
 * argmax report the min / max identity value (their index is -1). */
int or_identity(int dtype, int op, void* out) {
  if (!out || dtype < 0 || dtype > 4 || op < 0 || op > 10) return OR_INVALID;
  if (op == OR_SUM_COMPENSATED || op == OR_SUM_EXACT) op = OR_SUM;
  if (op == OR_ARGMIN) op = OR_MIN;
  if (op == OR_ARGMAX) op = OR_MAX;
  if (is_float(dtype) && op >= OR_AND) return OR_UNSUPPORTED;
  if (dtype == OR_FLOAT32 || dtype == OR_FLOAT64) {
    double v = (op == OR_SUM) ? 0.0 : (op == OR_PROD) ? 1.0 : (op == OR_MIN) ? INFINITY : -INFINITY;
    if (dtype == OR_FLOAT32) { float f = (float)v; memcpy(out, &f, 4); }
    else memcpy(out, &v, 8);
    return OR_OK;
  }
  uint64_t v = 0;
  switch (op) {
    case OR_SUM: case OR_OR: case OR_XOR: v = 0; break;
    case OR_PROD: v = 1; break;
    case OR_AND: v = ~0ULL; break;
    case OR_MIN: v = (dtype == OR_INT32) ? 0x7FFFFFFFULL : (dtype == OR_UINT32) ? 0xFFFFFFFFULL : 0x7FFFFFFFFFFFFFFFULL; break;
    case OR_MAX: v = (dtype == OR_INT32) ? 0x80000000ULL : (dtype == OR_UINT32) ? 0ULL : 0x8000000000000000ULL; break;
  }
  if (dtype == OR_INT64) memcpy(out, &v, 8);
  else { uint32_t w = (uint32_t)v; memcpy(out, &w, 4); }
  return OR_OK;
}

/*
 * Final value, narrowed to the dtype with ONE rounding (value_out, s bytes),
 * plus the unrounded accumulator (hi + lo) and sum |x_i| for the tolerance.
 */
int or_result(const or_state* st, void* value_out, double* hi, double* lo, double* sum_abs) {
  if (!st || !value_out) return OR_INVALID;
  if (st->count == 0) {
    or_identity(st->dtype, st->op, value_out);
    if (hi) { double v = 0.0; if (is_float(st->dtype)) { if (st->dtype == OR_FLOAT32) { float f; memcpy(&f, value_out, 4); v = f; } else memcpy(&v, value_out, 8); } *hi = v; }
    if (lo) *lo = 0.0;
    if (sum_abs) *sum_abs = 0.0;
    return OR_OK;
  }
  if (is_arg(st->op) && is_float(st->dtype)) {
    double v = st->hi;
    if (st->dtype == OR_FLOAT32) { float f = (float)v; memcpy(value_out, &f, 4); }
    else memcpy(value_out, &v, 8);
    if (hi) *hi = v;
    if (lo) *lo = 0.0;
    if (sum_abs) *sum_abs = 0.0;
    return OR_OK;
  }
  if (!is_float(st->dtype)) {
    if (st->dtype == OR_INT64) memcpy(value_out, &st->ibits, 8);
    else { uint32_t w = (uint32_t)st->ibits; memcpy(value_out, &w, 4); }
    if (hi) *hi = 0.0;
    if (lo) *lo = 0.0;
    if (sum_abs) *sum_abs = 0.0;
    return OR_OK;
  }
  if (st->op == OR_SUM_EXACT) {   /* R17: one rounding of the exact sum */
    double v;
    if (st->nan_seen || (st->pinf_seen && st->ninf_seen)) v = NAN;
    else if (st->pinf_seen) v = INFINITY;
    else if (st->ninf_seen) v = -INFINITY;
    else {
      v = big_round(st->big, st->dtype == OR_FLOAT32 ? 24 : 53, lsb_exp(st->dtype));
      if (v == 0.0) v = st->all_negzero ? -0.0 : 0.0;
    }
    if (st->dtype == OR_FLOAT32) { float f = (float)v; memcpy(value_out, &f, 4); } /* exact or inf */
    else memcpy(value_out, &v, 8);
    if (hi) *hi = v;
    if (lo) *lo = 0.0;
    if (sum_abs) *sum_abs = st->abs_hi + st->abs_lo;
    return OR_OK;
  }
  double v = (st->lo == 0.0) ? st->hi : st->hi + st->lo; /* double-double -> double; keeps -0.0 */
  if (!isfinite(st->hi)) v = st->hi;
  if (v == 0.0 && (st->op == OR_SUM)) v = st->all_negzero ? -0.0 : 0.0; /* R2 */
  if (v == 0.0 && (st->op == OR_PROD)) v = st->hi;  /* sign of an exact zero product */
  if (st->dtype == OR_FLOAT32) { float f = (float)v; memcpy(value_out, &f, 4); }
  else memcpy(value_out, &v, 8);
  if (hi) *hi = isfinite(st->hi) ? st->hi : v;
  if (lo) *lo = isfinite(st->hi) ? st->lo : 0.0;
  if (sum_abs) *sum_abs = st->abs_hi + st->abs_lo;
  return OR_OK;
}

/* One-shot: Algorithm 1 over x[0..n). */
int or_reduce(const void* x, uint64_t n, int dtype, int op, void* value_out,
              double* hi, double* lo, double* sum_abs) {
  or_state st;
  int rc = or_init(&st, dtype, op);
  if (rc) return rc;
  rc = or_fold(&st, x, n);
  if (rc) return rc;
  return or_result(&st, value_out, hi, lo, sum_abs);
}

/* Combine two fold states whose inputs are consecutive blocks A then B of one
 * array, in that order: result = fold(A) (x) fold(B). Used only by the
 * multi-rank host-logic tests (rank-order combine); for floats
 * the two accumulators are combined in the oracle's own wide precision. */
int or_merge(or_state* a, const or_state* b) {
  if (!a || !b || a->dtype != b->dtype || a->op != b->op) return OR_INVALID;
  if (b->count == 0) return OR_OK;
  if (a->count == 0) { *a = *b; return OR_OK; }
  const int dt = a->dtype, op = a->op;
  if (is_arg(op)) {
    /* b covers the block after a: its indices shift by a->count; ties keep a */
    if (!is_float(dt)) {
      if (int_better(dt, op, b->ibits, a->ibits)) { a->ibits = b->ibits; a->best_idx = a->count + b->best_idx; }
    } else if (float_better(op, b->hi, a->hi)) {
      a->hi = b->hi;
      a->best_idx = a->count + b->best_idx;
    }
    a->count += b->count;
    return OR_OK;
  }
  if (!is_float(dt)) {
    a->ibits = int_combine(dt, op, a->ibits, b->ibits);
  } else if (op == OR_SUM_EXACT) {  /* exact sums add exactly */
    uint64_t carry = 0;
    for (int i = 0; i < OR_BIG_LIMBS; ++i) {
      uint64_t t = (uint64_t)a->big[i] + b->big[i] + carry;
      a->big[i] = (uint32_t)t;
      carry = t >> 32;
    }
    a->nan_seen |= b->nan_seen;
    a->pinf_seen |= b->pinf_seen;
    a->ninf_seen |= b->ninf_seen;
    dd_add(&a->abs_hi, &a->abs_lo, b->abs_hi);
    dd_add(&a->abs_hi, &a->abs_lo, b->abs_lo);
    a->all_negzero = a->all_negzero && b->all_negzero;
  } else {
    switch (op) {
      case OR_SUM: dd_add(&a->hi, &a->lo, b->hi); dd_add(&a->hi, &a->lo, b->lo); break;
      case OR_PROD: {
        double h = a->hi, l = a->lo;
        dd_mul(&h, &l, b->hi);          /* a * b.hi */
        double h2 = a->hi, l2 = a->lo;
        dd_mul(&h2, &l2, b->lo);        /* a * b.lo (tiny) */
        dd_add(&h, &l, h2);
        a->hi = h; a->lo = l;
        break;
      }
      case OR_MIN: a->hi = ieee_min(a->hi, b->hi); break;
      case OR_MAX: a->hi = ieee_max(a->hi, b->hi); break;
      default: break;
    }
    dd_add(&a->abs_hi, &a->abs_lo, b->abs_hi);
    dd_add(&a->abs_hi, &a->abs_lo, b->abs_lo);
    a->all_negzero = a->all_negzero && b->all_negzero;
  }
  a->count += b->count;
  return OR_OK;
}

/* argmin / argmax: index of the best element (R6), -1 for an empty fold. */
int64_t or_result_index(const or_state* st) {
  if (!st || st->count == 0) return -1;
  return (int64_t)st->best_idx;
}

uint64_t or_state_size(void) { return (uint64_t)sizeof(or_state); }
