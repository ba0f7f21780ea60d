// rd_exact.cuh -- the exact float sum (RD_SUM_EXACT; SURVEY §8(f) row f2,
// reading R17): the real sum of the n float values, rounded ONCE to nearest-
// even. PAPER.md P:50 fn 2 shows that a float sum depends on the order of the
// additions ("the floating point computed value can result in 0 or 1.5");
// the exact sum is the one result no order, grid, variant, base alignment or
// GPU count can change -- so it is bitwise reproducible by construction.
//
// Design (one single-pass launch; a vector-load form, its one-cluster form
// for small inputs, and a bulk-copy form):
//  a1  each thread streams vectors (32-byte loads, or LDS.128 from the bulk
//      ring) and adds every element (fp32 widened to fp64, exactly) into one
//      of E three-term expansions (a0, a1, a2), a0 + a1 + a2 exact. Per
//      vector it SPECULATES branch-free -- fp32 data: every add into a0 is
//      exact, tested by compares only (fl(s - a0) == x && fl(s - x) == a0;
//      3 DADD + 2 compares per element); fp64 data: a0's TwoSum error goes into
//      a1 exactly -- with ONE branch per vector; the streaming loops do the
//      same per GROUP of 8 terms with one tested add (fold_group_exact32/64).
//      A group they cannot take goes out of line to the BINS (binned
//      extraction into 8 fixed-exponent fp64 bins per lane, exact by its
//      invariants, bins_group); inf/NaN terms and fp64 spreads past the bins
//      go element by element (replay_vec: a0 -> a1 -> a2 TwoSums; only a
//      nonzero third error, an fp64 overflow or inf/NaN reaches the
//      superaccumulator). Loops end with __syncwarp so replays reconverge.
//  superaccumulator: a fixed-point integer whose unit is the dtype's smallest
//      subnormal (2^-149 / 2^-1074), held as kWords carry-save int64 words of
//      32-bit digits in shared memory (one per warp). A finite double is
//      deposited exactly as three signed digits (shared 64-bit atomics); a word
//      nearing 2^60 moves its high part to the next word (value-preserving).
//  a3-a5  at the end the warp deposits its lanes' expansions cooperatively
//      (no atomics), carries its words to digits in [0, 2^32), and the CTA
//      adds its warps' digits.
//  a6  every CTA adds its words into one workspace accumulator with native
//      64-bit global reductions (integers: any order is exact); the last CTA
//      (atomic ticket) reads it, zeroes it for the next launch, carries
//      (one-cluster form: rank 0 adds the CTAs' words over DSMEM), and
//  a7  rounds once: the 64 bits below the leading one give the p kept bits,
//      the guard bit and (with every lower digit) the sticky bit; ties to even;
//      the float is assembled as (shift << (p-1)) + q, which carries a rounded-
//      up mantissa into the exponent and reaches inf exactly at the IEEE
//      overflow threshold. Specials: flags for NaN, +inf, -inf and "some term
//      is not -0.0" (reading R2's sign of a zero sum). Or (mode 1) the carried
//      words leave as an rd_exact_record, or (mode 2) go through the fused
//      multi-GPU mailboxes (exact_fused_exchange).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rd_bulk.cuh"

namespace rd {

template <typename T> struct ExactTraits;
template <> struct ExactTraits<float> {
  static constexpr int kLsb = -149;    // 2^-149: the fp32 subnormal unit
  static constexpr int kWords = 12;    // 384 bits >= 128 + 149 + 40 (n < 2^40) + sign
  static constexpr int kPrec = 24;
  static constexpr uint64_t kInfBits = 0x7f800000ull;
  static constexpr uint64_t kSignBit = 0x80000000ull;
  static constexpr uint64_t kQNaN = 0x7fc00000ull;
};
template <> struct ExactTraits<double> {
  static constexpr int kLsb = -1074;   // 2^-1074: the fp64 subnormal unit
  static constexpr int kWords = 68;    // 2176 bits >= 1024 + 1074 + 40 + sign
  static constexpr int kPrec = 53;
  static constexpr uint64_t kInfBits = 0x7ff0000000000000ull;
  static constexpr uint64_t kSignBit = 0x8000000000000000ull;
  static constexpr uint64_t kQNaN = 0x7ff8000000000000ull;
};
static_assert(ExactTraits<double>::kWords <= RD_EXACT_MAX_WORDS, "rd_exact_record too small");

constexpr uint32_t kXNaN = 1u, kXPosInf = 2u, kXNegInf = 4u, kXNotNegZero = 8u;
constexpr uint64_t kNegZeroBits = 0x8000000000000000ull;

struct XArgs {
  const unsigned char* x;
  uint64_t n, head, nvec, tail_start, tail;
  void* out;                 // mode 0: one element
  rd_exact_record* rec;      // mode 1: one exact record
  long long* partials;       // the grid accumulator: kWords + 1 words, zero between launches
  unsigned* ticket;
  uint32_t tag;
  int mode;
  // bulk variant only: the chunk schedule (as KArgs; the exact sum does not
  // depend on which CTA takes which chunk, so no per-chunk partials)
  uint64_t chunk_bytes, tail_chunk_bytes, head_region_bytes;
  uint32_t nchunks, nhead_chunks;
  unsigned* work;
  // mode 2 (fused multi-GPU exchange, rd_kernels.cuh Mailbox) only
  Mailbox* const* peers;
  Mailbox* self;
  int* err;
  int nranks, rank;
};

// ------------------------------------------------------------ superaccumulator
// w[k] += v (carry-save). A word whose magnitude passes 2^60 hands its high
// part to w[k+1]: both are atomic adds of opposite value, so the represented
// number never changes, whatever other lanes do meanwhile.
template <int NW>
__device__ __forceinline__ void sacc_word_add(long long* w, int k, long long v) {
  for (;;) {
    const long long now = (long long)atomicAdd((unsigned long long*)&w[k], (unsigned long long)v) + v;
    if (k == NW - 1 || (now < (1ll << 60) && now > -(1ll << 60))) return;
    const long long c = now >> 32;   // arithmetic shift
    atomicAdd((unsigned long long*)&w[k], (unsigned long long)(-(c << 32)));
    ++k;
    v = c;
  }
}

// deposit a finite double d exactly: d = +-m * 2^(e-1075), m < 2^53
template <typename T>
__device__ __forceinline__ void sacc_add(long long* w, double d) {
  using TR = ExactTraits<T>;
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  int e = (int)((b >> 52) & 0x7ff);
  uint64_t m = b & ((1ull << 52) - 1);
  if (e) m |= 1ull << 52;
  else e = 1;
  if (m == 0) return;
  int p = e - 1075 - TR::kLsb;       // bit position of m's unit
  if (p < 0) { m >>= -p; p = 0; }    // only zero bits (d is a multiple of 2^kLsb)
  const int k = p >> 5, r = p & 31;
  const uint64_t lo = m << r;
  const long long d0 = (long long)(lo & 0xffffffffull), d1 = (long long)(lo >> 32);
  const long long d2 = r ? (long long)(m >> (64 - r)) : 0;
  const bool neg = (int64_t)b < 0;
  if (d0) sacc_word_add<TR::kWords>(w, k, neg ? -d0 : d0);
  if (d1) sacc_word_add<TR::kWords>(w, k + 1, neg ? -d1 : d1);
  if (d2) sacc_word_add<TR::kWords>(w, k + 2, neg ? -d2 : d2);
}

// deposit the signed integer v (|v| < 2^62) times 2^e exactly, e an exponent
// at or above the dtype's smallest unit whenever v has bits below it (the
// bins' contents are sums of terms, so multiples of 2^kLsb)
template <typename T>
__device__ __forceinline__ void sacc_add_units(long long* w, long long v, int e) {
  using TR = ExactTraits<T>;
  const bool neg = v < 0;
  uint64_t m = neg ? (uint64_t)(-v) : (uint64_t)v;
  int p = e - TR::kLsb;              // bit position of v's unit
  if (p < 0) { m >>= -p; p = 0; }    // only zero bits
  const int k = p >> 5, r = p & 31;
  const uint64_t lo = m << r;
  const long long d0 = (long long)(lo & 0xffffffffull), d1 = (long long)(lo >> 32);
  const long long d2 = r ? (long long)(m >> (64 - r)) : 0;
  if (d0) sacc_word_add<TR::kWords>(w, k, neg ? -d0 : d0);
  if (d1) sacc_word_add<TR::kWords>(w, k + 1, neg ? -d1 : d1);
  if (d2) sacc_word_add<TR::kWords>(w, k + 2, neg ? -d2 : d2);
}

// carry the words into digits [0, 2^32) (the top word keeps the sign); one thread
template <int NW>
__device__ __forceinline__ void sacc_normalise(long long* w) {
  long long c = 0;
  for (int k = 0; k < NW - 1; ++k) {
    const long long t = w[k] + c;
    w[k] = t & 0xffffffffll;
    c = t >> 32;
  }
  w[NW - 1] += c;
}

// The same result as sacc_normalise, by one whole (converged) warp: lane l
// owns words [l*R, l*R + R). Each lane carries its own words, then the lanes'
// carries move one lane per shift step until they are all in {-1, 0, +1} and
// of one sign, when a carry-lookahead over ballots (generate = the lane's
// carry, propagate = its digits all ones for +1 / all zero for -1) settles
// every ripple chain in one step -- the chain of 0xffffffff digits a negative
// total leaves above its top digit included. The value is kept at every step,
// and the digits of a value are unique, so the words equal the sequential's.
template <int NW>
__device__ __forceinline__ void sacc_normalise_warp(long long* w) {
  constexpr int R = (NW + 31) / 32;
  constexpr int L = (NW + R - 1) / R;                 // lanes that own words; L-1 owns the top word
  constexpr long long M = 0xffffffffll;
  const int ln = threadIdx.x & 31, k0 = ln * R;
  const bool top = ln == L - 1;
  long long d[R];
#pragma unroll
  for (int i = 0; i < R; ++i) d[i] = (ln < L && k0 + i < NW) ? w[k0 + i] : 0;
  long long c = 0, hi = 0;                            // hi: the top lane's carry out (kept, not shipped)
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (k0 + i < NW) { const long long t = d[i] + c; d[i] = t & M; c = t >> 32; }
  if (top) { hi = c; c = 0; }
  const unsigned below_top = (1u << (L - 1)) - 1u;    // lanes whose carry goes to the next lane
  while (__any_sync(0xffffffffu, c != 0)) {
    const unsigned gp = __ballot_sync(0xffffffffu, c == 1), gm = __ballot_sync(0xffffffffu, c == -1);
    const bool lookahead = __all_sync(0xffffffffu, c >= -1 && c <= 1) && (gp == 0u || gm == 0u);
    long long cin;
    const bool gen = c != 0;
    if (lookahead) {
      const bool plus = gp != 0u;
      bool prop = ln < L - 1;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (k0 + i < NW) prop = prop && d[i] == (plus ? M : 0);
      const unsigned G = plus ? gp : gm;
      const unsigned P = __ballot_sync(0xffffffffu, prop) & below_top & ~G;
      const unsigned into = ((G | P) + G) ^ P;        // bit l: a unit enters lane l
      cin = ((into >> ln) & 1u) ? (plus ? 1 : -1) : 0;
    } else {
      cin = __shfl_up_sync(0xffffffffu, c, 1);
      if (ln == 0) cin = 0;
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (k0 + i < NW) { const long long t = d[i] + cin; d[i] = t & M; cin = t >> 32; }
    // cin is now the lane's carry out: the top lane keeps it; after a shift
    // step it is the lane's next carry; after a lookahead step the chains
    // already account for a propagating lane's, and only a generating lane
    // that also wrapped has one left
    if (top) { hi += cin; c = 0; }
    else c = (!lookahead || gen) ? cin : 0;
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (ln < L && k0 + i < NW) w[k0 + i] = d[i] + ((k0 + i == NW - 1) ? (long long)((unsigned long long)hi << 32) : 0);
}

// what a whole warp calls: the lookahead form for the fp64 68 words (measured
// ~0.45 us less per small launch), lane 0's sequential carry for fp32's 12
// (there the warp form costs ~0.1 us more; profiles/r01_exact_small_norm.txt)
template <int NW>
__device__ __forceinline__ void sacc_normalise_by_warp(long long* w) {
  if constexpr (NW > 32) sacc_normalise_warp<NW>(w);
  else if ((threadIdx.x & 31) == 0) sacc_normalise<NW>(w);
}

// ------------------------------------------------------------------ expansions
struct Ex { double a0, a1, a2; };   // a0 + a1 + a2 exactly; |a0| >> |a1| >> |a2| in practice

// TwoSum (Knuth): s + e == a + b exactly (when s is finite)
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bp = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bp)), __dsub_rn(b, bp));
}

// the rare cases, out of line (keeps the hot loop small): an inf/NaN term,
// an fp64 overflow of a0 + x, or a nonzero error of the second TwoSum, which
// goes into a2 by a third TwoSum; only a third nonzero error reaches the
// superaccumulator. Recomputes from the state before the element.
struct ExSlow { Ex ex; uint32_t flags; };
template <typename T>
__device__ __noinline__ ExSlow ex_slow(Ex ex, double x, long long* w, uint32_t flags) {
  if (!(fabs(x) <= 1.7976931348623157e308)) {   // inf or NaN term: flags only
    flags |= (x != x) ? kXNaN : (x > 0 ? kXPosInf : kXNegInf);
    return ExSlow{ex, flags};
  }
  flags |= kXNotNegZero;
  double s, e;
  two_sum(ex.a0, x, s, e);
  if (!(fabs(s) <= 1.7976931348623157e308)) {   // a0 + x overflows (fp64 data): deposit x
    sacc_add<T>(w, x);
    return ExSlow{ex, flags};
  }
  ex.a0 = s;
  if (e == 0.0) return ExSlow{ex, flags};
  double s1, e1;
  two_sum(ex.a1, e, s1, e1);
  if (!(fabs(s1) <= 1.7976931348623157e308)) {
    sacc_add<T>(w, e);
    return ExSlow{ex, flags};
  }
  ex.a1 = s1;
  if (e1 == 0.0) return ExSlow{ex, flags};
  double s2, e2;
  two_sum(ex.a2, e1, s2, e2);
  if (!(fabs(s2) <= 1.7976931348623157e308)) {
    sacc_add<T>(w, e1);
    return ExSlow{ex, flags};
  }
  ex.a2 = s2;
  if (e2 != 0.0) sacc_add<T>(w, e2);
  return ExSlow{ex, flags};
}

// a0 + x = s + e exactly (TwoSum). e == 0: done (fp32 data with a narrow
// exponent spread: nearly every term). Else e -- finite and nonzero unless x
// is inf/NaN or s overflowed -- goes into a1 by a second TwoSum, inline (fp64
// data: most terms); only a nonzero second error or a non-finite value leaves
// the inline path.
template <typename T>
__device__ __forceinline__ void ex_add(Ex& ex, double x, long long* w, uint32_t& flags) {
  double s, e;
  two_sum(ex.a0, x, s, e);
  if (__builtin_expect(e == 0.0, 1)) {
    ex.a0 = s;
    return;
  }
  double s1, e1;
  two_sum(ex.a1, e, s1, e1);                     // NaN throughout for the non-finite cases
  if (__builtin_expect(e1 == 0.0 && fabs(s1) <= 1.7976931348623157e308, 1)) {
    ex.a0 = s;
    ex.a1 = s1;
    flags |= kXNotNegZero;                       // e != 0: x is not a zero
    return;
  }
  const ExSlow r = ex_slow<T>(ex, x, w, flags);
  ex = r.ex;
  flags = r.flags;
}

template <typename T>
__device__ __forceinline__ double widen(T v) { return (double)v; }   // exact for fp32

// One loaded vector, speculatively and branch-free: every element's TwoSum(s)
// are computed on the lane's expansion (the E expansions are independent
// dependency chains) and their "inexact / non-finite" tests OR-ed; ONE branch
// per vector. fp32 data: one TwoSum per element, speculating e == 0 (every
// term of a narrow-exponent workload). fp64 data: both TwoSums, speculating
// that the second error is 0 (a 53-bit term almost always leaves an error in
// a0, almost never in a1). If the speculation fails the vector is replayed
// element by element from the saved state through ex_add.
template <int L>
struct ExVals { double v[L]; };

// two-level speculation over one vector: both TwoSums per element, branch-free
template <int E, int L>
__device__ __forceinline__ bool spec2(Ex (&ex)[E], const double (&xs)[L]) {
  bool bad = false;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    Ex& q = ex[l % E];
    double s, e;
    two_sum(q.a0, xs[l], s, e);
    // a1 + e exact? the symmetric difference test (see fold_vec_exact): 3 DADD
    // + 2 compares instead of a second TwoSum; NaN (inf/NaN term, overflow)
    // fails a compare
    const double s1 = __dadd_rn(q.a1, e);
    bad |= (__dsub_rn(s1, q.a1) != e) | (__dsub_rn(s1, e) != q.a1);
    q.a0 = s;
    q.a1 = s1;
  }
  return bad;
}

// the replay of a vector whose speculation failed, out of line: one copy of
// this code for the whole kernel (inlined into every unrolled vector slot it
// thrashed the instruction cache whenever it ran)
template <int E, int L>
struct ExState { Ex ex[E]; uint32_t flags; };
template <typename T, int E, int L>
__device__ __noinline__ ExState<E, L> replay_vec(ExState<E, L> st, const ExVals<L> xs, long long* w) {
  // The full cascade a0 -> a1 -> a2 for every element, computed the same way in
  // every lane (no data-dependent branch but the rare superaccumulator
  // deposits): replaying lanes stay converged. (Per-element early exits made
  // the lanes diverge per element and run this ~1-2 lanes at a time: ncu avg
  // threads per DADD 1.5 on the adversarial `wide` workload.)
  constexpr double kMax = 1.7976931348623157e308;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    Ex& q = st.ex[l % E];
    const double x = xs.v[l];
    const bool fin = fabs(x) <= kMax;                        // false for inf / NaN
    st.flags |= fin ? (x != 0.0 ? kXNotNegZero : 0u) : ((x != x) ? kXNaN : (x > 0 ? kXPosInf : kXNegInf));
    const double xf = fin ? x : 0.0;
    double s, e;
    two_sum(q.a0, xf, s, e);
    if (__builtin_expect(!(fabs(s) <= kMax), 0)) {          // a0 + x overflows (fp64 data): deposit x
      sacc_add<T>(w, xf);
      s = q.a0;
      e = 0.0;
    }
    q.a0 = s;
    double s1, e1;
    two_sum(q.a1, e, s1, e1);
    if (__builtin_expect(!(fabs(s1) <= kMax), 0)) {
      sacc_add<T>(w, e);
      s1 = q.a1;
      e1 = 0.0;
    }
    q.a1 = s1;
    double s2, e2;
    two_sum(q.a2, e1, s2, e2);
    if (__builtin_expect(!(fabs(s2) <= kMax), 0)) {
      sacc_add<T>(w, e1);
      s2 = q.a2;
      e2 = 0.0;
    }
    q.a2 = s2;
    if (__builtin_expect(e2 != 0.0, 0)) sacc_add<T>(w, e2);
  }
  return st;
}

template <typename T, int E, int L>
__device__ __forceinline__ void fold_vec_exact(Ex (&ex)[E], const double (&xs)[L], long long* w,
                                               uint32_t& flags) {
  const unsigned mask = __activemask();
  Ex save[E];
#pragma unroll
  for (int j = 0; j < E; ++j) save[j] = ex[j];
  bool bad = false;
  if constexpr (sizeof(T) == 4) {
    // fp32 terms: speculate that every add into a0 is exact, tested without
    // TwoSum's error term: s == a0 + x exactly iff fl(s - a0) == x and
    // fl(s - x) == a0. (If s is inexact, the difference taken from the
    // operand of larger magnitude is exact -- Dekker's Fast2Sum lemma -- and
    // differs from the other operand by the nonzero rounding error; if s is
    // exact both differences are.) 3 DADD + 2 compares per element instead of
    // 6 + 1: the FP64 pipe is the limiter. inf/NaN terms and overflow fail a
    // compare (inf - inf, NaN).
#pragma unroll
    for (int l = 0; l < L; ++l) {
      Ex& q = ex[l % E];
      const double s = __dadd_rn(q.a0, xs[l]);
      bad |= (__dsub_rn(s, q.a0) != xs[l]) | (__dsub_rn(s, xs[l]) != q.a0);
      q.a0 = s;
    }
    // warp-uniform decisions: a lane whose speculation failed takes the whole
    // (converged) warp to the next level -- every level is exact for any data
    if (__builtin_expect(!__any_sync(mask, bad), 1)) return;
#pragma unroll
    for (int j = 0; j < E; ++j) ex[j] = save[j];
  }
  bad = spec2<E, L>(ex, xs);
  if (__builtin_expect(__any_sync(mask, bad), 0)) {   // replay element by element
    ExState<E, L> st;
#pragma unroll
    for (int j = 0; j < E; ++j) st.ex[j] = save[j];
    st.flags = flags;
    ExVals<L> v;
#pragma unroll
    for (int l = 0; l < L; ++l) v.v[l] = xs[l];
    st = replay_vec<T, E, L>(st, v, w);
#pragma unroll
    for (int j = 0; j < E; ++j) ex[j] = st.ex[j];
    flags = st.flags;
  }
}

// The end-of-thread deposit, warp-cooperative, in registers and without
// atomics: every lane of the (converged) warp passes its NV doubles (0 =
// nothing). The warp walks the superaccumulator words its lanes' digits land
// in (the next occupied word comes from one redux.min); per word each lane
// sums its own digits there (|c| < 2^35), the warp adds the 32 lane sums with
// three 13-bit-chunk redux.sync adds (offset to be nonnegative: no chunk sum
// overflows), and lane 0 adds the total to the word. (Per-lane shared 64-bit
// atomics are CAS loops on sm_100a, ATOMS.CAST.SPIN.64, and a smem-staged
// transposed sum costs ~2000 instructions per warp: both dominated small n.)
// Only this warp writes its superaccumulator, and its slow-path atomics are
// complete (__syncwarp). `mask`: the lanes taking part (all of them converged
// here; the lowest adds the word sums).
template <typename T, int NV>
__device__ __forceinline__ void sacc_flush_warp(long long* w, const double (&d)[NV], unsigned mask = 0xffffffffu) {
  using TR = ExactTraits<T>;
  constexpr int kNone = 0x7fffffff;
  int k[NV];
  long long s0[NV], s1[NV], s2[NV];
  int first = kNone;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    k[v] = kNone;
    s0[v] = s1[v] = s2[v] = 0;
    if (d[v] != 0.0) {
      const uint64_t b = (uint64_t)__double_as_longlong(d[v]);
      int e = (int)((b >> 52) & 0x7ff);
      uint64_t m = b & ((1ull << 52) - 1);
      if (e) m |= 1ull << 52;
      else e = 1;
      int p = e - 1075 - TR::kLsb;
      if (p < 0) { m >>= -p; p = 0; }
      const int r = p & 31;
      const uint64_t lo = m << r;
      s0[v] = (long long)(lo & 0xffffffffull);
      s1[v] = (long long)(lo >> 32);
      s2[v] = r ? (long long)(m >> (64 - r)) : 0;
      if ((int64_t)b < 0) { s0[v] = -s0[v]; s1[v] = -s1[v]; s2[v] = -s2[v]; }
      k[v] = p >> 5;
      first = min(first, k[v]);
    }
  }
  const bool writer = (int)(threadIdx.x & 31) == __ffs(mask) - 1;
  const long long offset = (long long)__popc(mask) << 38;
  // value slots no lane of the warp fills (e.g. a1, a2 of fp32 data, which the
  // group path never touches) are skipped by a warp-uniform branch
  bool used[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) used[v] = __any_sync(mask, k[v] != kNone);
  int word = __reduce_min_sync(mask, first);
  while (word != kNone) {                            // warp-uniform
    long long c = 0;
    int next = kNone;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!used[v]) continue;
      const int r = word - k[v];                     // digit r of value v lands here (r in 0..2)
      c += r == 0 ? s0[v] : r == 1 ? s1[v] : r == 2 ? s2[v] : 0;
      // this lane's next occupied word above `word` (k, k+1, k+2 of each value)
      const int x = word + 1 - k[v];
      next = min(next, x <= 0 ? k[v] : (x <= 2 ? word + 1 : kNone));
    }
    const unsigned long long u = (unsigned long long)(c + (1ll << 38));   // in [0, 2^39)
    const unsigned c0 = __reduce_add_sync(mask, (unsigned)(u & 0x1fff));
    const unsigned c1 = __reduce_add_sync(mask, (unsigned)((u >> 13) & 0x1fff));
    const unsigned c2 = __reduce_add_sync(mask, (unsigned)(u >> 26));
    if (writer) {
      const long long v = (long long)c0 + ((long long)c1 << 13) + ((long long)c2 << 26) - offset;
      // a partial warp (a tail loop): the lanes outside it may be depositing
      // stragglers into the same words by atomics meanwhile
      if (mask == 0xffffffffu) w[word] += v;
      else atomicAdd((unsigned long long*)&w[word], (unsigned long long)v);
    }
    word = __reduce_min_sync(mask, next);
  }
  __syncwarp(mask);
}

// ------------------------------------------------------------------- bins
// The fallback for groups the group paths cannot sum exactly (exponents
// spread wider than one fp64 significand can hold: the `wide` workload, where
// nearly every group fails): BINNED EXTRACTION after Demmel & Nguyen's
// indexed summation (the technique of ReproBLAS), with enough bins and a
// bounded number of additions that it is EXACT, not only reproducible.
// Each lane keeps K = 8 fp64 bins with fixed exponents a_j = a_0 - j*W
// (W = 38; the anchor a_0 is the same in every lane of a warp): bin j holds
// S_j = 1.5*2^(a_j) + (sum of the pieces it took), and every piece is a
// multiple of its unit u_j = ulp(S_j) = 2^(a_j - 52). A term x passes down
// the bins: t = fl(S_j + r); q = t - S_j (exact: Sterbenz); r = r - q
// (exact: the error of rounding r to a multiple of u_j); S_j = t. Bounds that
// keep every step exact: |x| <= 2^(a_0 + W - 53) (floor(log2|x|) <= a_0 - 16,
// else the warp re-anchors higher) and at most 4096 < 2^(51 - W) additions
// between re-anchorings, so |S_j - 1.5*2^(a_j)| < 2^(a_j - 2) and S_j never
// leaves its binade. A group runs the fewest bins whose last unit is <= every
// term's lowest bit (from the exponent fields; per warp: 2, 3, 4 or 8), so
// nothing falls below the last bin and it is one plain add: 3 DADD per bin
// but the last (1) -- 7 per term for `wide` fp32 (3 bins), 10 for `wide`
// fp64 (4), 22 at most -- branch-free and independent of the order of the
// terms (round 1's per-element TwoSum cascade: ~20 dependent FP64 ops per
// term). 8 bins span 52 + 7 * 38 = 318 bits: every fp32 exponent; fp64
// groups that reach past them take the per-element levels. Re-anchoring
// moves each bin's content (the difference of the bit patterns of S_j and
// 1.5*2^(a_j), in units of u_j) into the warp's superaccumulator, summed over
// the warp first.
constexpr int kBinW = 38;                  // bits per bin
constexpr int kBinHead = 54 - kBinW;       // bins take floor(log2|x|) <= a_0 - kBinHead
constexpr int kBinSlack = 4;               // a new anchor leaves this many binades of room above the max
constexpr int kBinMaxAdds = 4096;          // additions per bin between re-anchorings (< 2^(51 - kBinW))
template <typename T> struct BinK;
template <> struct BinK<float> { static constexpr int K = 8; };    // 52 + 7 * 38 bits: every fp32 exponent
template <> struct BinK<double> { static constexpr int K = 8; };

template <int K>
struct Bins {
  double s[K];   // S_j
  int top;       // the largest floor(log2|x|) the bins take: a_0 - kBinHead
  int count;     // terms added since the last (re)anchoring
};
// Each lane's bins live in shared memory (the warp's block, lane-strided: no
// bank conflicts), not in registers: only the out-of-line fallback touches
// them, and the hot loop keeps its registers (8-10 per thread otherwise).
template <int K>
struct WarpBins {
  double s[K][32];
  int top[32];
  int count[32];
};
// the lowest anchor whose K bins are all normal doubles
template <int K> __host__ __device__ constexpr int bins_min_a0() { return -1022 + (K - 1) * kBinW; }
// the largest floor(log2|x|) any anchor takes (a_0 <= 1023)
constexpr int kBinMaxTop = 1023 - kBinHead;

__device__ __forceinline__ double bin_anchor(int a) {   // 1.5 * 2^a, a in [-1022, 1023]
  return __hiloint2double(((a + 1023) << 20) | 0x80000, 0);
}
template <int K>
__device__ __forceinline__ void bins_init(WarpBins<K>* wb) {
  constexpr int a0 = bins_min_a0<K>();
  const int ln = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < K; ++j) wb->s[j][ln] = bin_anchor(a0 - j * kBinW);
  wb->top[ln] = a0 - kBinHead;
  wb->count[ln] = 0;
}
template <int K>
__device__ __forceinline__ Bins<K> bins_load(const WarpBins<K>* wb) {
  const int ln = threadIdx.x & 31;
  Bins<K> bn;
#pragma unroll
  for (int j = 0; j < K; ++j) bn.s[j] = wb->s[j][ln];
  bn.top = wb->top[ln];
  bn.count = wb->count[ln];
  return bn;
}
template <int K>
__device__ __forceinline__ void bins_store(WarpBins<K>* wb, const Bins<K>& bn) {
  const int ln = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < K; ++j) wb->s[j][ln] = bn.s[j];
  wb->top[ln] = bn.top;
  wb->count[ln] = bn.count;
}
// bin j's content, exact (S_j and 1.5 * 2^(a_j) are within a factor 2)
template <int K>
__device__ __forceinline__ double bin_value(const Bins<K>& bn, int j) {
  return __dsub_rn(bn.s[j], bin_anchor(bn.top + kBinHead - j * kBinW));
}

// One group of GL finite terms (gmax >= every floor(log2|x|), gmax <=
// kBinMaxTop; glow <= the exponent of every nonzero term's lowest bit) into
// this lane's bins; called from the out-of-line group fallbacks. Returns the
// flags.
// KE of this lane's K bins, straight from / to shared memory, every term a
// multiple of bin KE-1's unit, so nothing falls below it and the last bin is
// one plain add: 3 (KE - 1) + 1 DADD per term
constexpr int kBinPre = 4;                 // bins loaded at entry, before the checks
template <int K, int KE, int GL>
__device__ __forceinline__ void bins_run(WarpBins<K>* wb, const ExVals<GL>& xs, const double (&pre)[kBinPre]) {
  const int ln = threadIdx.x & 31;
  double s[KE];
#pragma unroll
  for (int j = 0; j < KE; ++j) s[j] = j < kBinPre ? pre[j < kBinPre ? j : 0] : wb->s[j][ln];
#pragma unroll
  for (int l = 0; l < GL; ++l) {
    double r = xs.v[l];
#pragma unroll
    for (int j = 0; j < KE - 1; ++j) {
      const double t = __dadd_rn(s[j], r);
      r = __dsub_rn(r, __dsub_rn(t, s[j]));
      s[j] = t;
    }
    s[KE - 1] = __dadd_rn(s[KE - 1], r);
  }
#pragma unroll
  for (int j = 0; j < KE; ++j) wb->s[j][ln] = s[j];
}
// this lane needs k bins -> the warp runs 2, 3, 4 or K (more than needed is
// exact too: the extra bins take zeros; four forms, not K, keep the
// fallback's code small), decided by votes (cheaper than a redux.max on the
// path to the first DADD). k > K: not taken (returns false).
template <int K, int GL>
__device__ __forceinline__ bool bins_run_dispatch(WarpBins<K>* wb, const ExVals<GL>& xs, int k, unsigned mask,
                                                  const double (&pre)[kBinPre]) {
  static_assert(K >= 4, "K >= 4 bins");
  if (!__any_sync(mask, k > 3)) {
    if (__any_sync(mask, k > 2)) bins_run<K, 3, GL>(wb, xs, pre);
    else bins_run<K, 2, GL>(wb, xs, pre);
  } else if (!__any_sync(mask, k > 4)) {
    bins_run<K, 4, GL>(wb, xs, pre);
  } else {
    if (__any_sync(mask, k > K)) return false;
    bins_run<K, K, GL>(wb, xs, pre);
  }
  return true;
}

// One group of GL finite terms (gmax >= every floor(log2|x|), gmax <=
// kBinMaxTop; glow <= the exponent of every nonzero term's lowest bit) into
// this lane's bins; called from the out-of-line group fallbacks. fp64 terms
// that reach below the K-th bin (exponents spread over more than ~300
// binades in one warp's groups) are not taken (returns false: the caller's
// per-element levels); fp32 terms always fit (K = 8 bins span the format).
template <typename T, int K, int GL>
__device__ __forceinline__ bool bins_group(WarpBins<K>* wb, uint32_t& flags, const ExVals<GL>& xs, int gmax,
                                           int glow, bool nonzero, long long* w) {
  const unsigned mask = __activemask();
  const int ln = threadIdx.x & 31;
  int top = wb->top[ln];
  int count = wb->count[ln];
  double pre[kBinPre];
#pragma unroll
  for (int j = 0; j < kBinPre; ++j) pre[j] = wb->s[j][ln];
  if (__any_sync(mask, gmax > top || count > kBinMaxAdds - GL)) {
    // re-anchor, the whole warp at once (rare). The anchor is the same in
    // every lane of a warp, so the warp re-anchors when ITS maximum grows (a
    // few times per launch, not once per lane), and bin j holds a multiple of
    // the same unit u_j in every lane: its content in units, m = bits(S_j) -
    // bits(1.5 * 2^a_j) (same binade: the difference of the bit patterns;
    // |m| < 2^50), is summed over the warp exactly by three 17-bit-chunk
    // redux adds, and ONE lane deposits the total (< 2^55 units) -- per-lane
    // atomic deposits were CAS loops contended by 32 lanes on the same words
    // (~40 us per launch at 2^24). The bins then start empty, re-anchored
    // higher if the warp's maximum grew.
    const int a0 = top + kBinHead;
    const bool writer = (int)ln == __ffs(mask) - 1;
    const long long off = (long long)__popc(mask) << 50;
    // (the anchors agree across the lanes by construction -- every re-anchoring
    // is the warp's -- but a lane left out of a partial-warp call would not
    // follow one; then each lane deposits its own bins, atomically)
    const bool uniform = __all_sync(mask, top == __shfl_sync(mask, top, __ffs(mask) - 1));
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const long long m = __double_as_longlong(wb->s[j][ln]) - __double_as_longlong(bin_anchor(a0 - j * kBinW));
      if (!uniform) {
        if (m != 0) sacc_add_units<T>(w, m, a0 - j * kBinW - 52);
        continue;
      }
      const unsigned long long u = (unsigned long long)(m + (1ll << 50));          // [0, 2^51)
      const long long tot = (long long)__reduce_add_sync(mask, (unsigned)(u & 0x1ffffu)) +
                            ((long long)__reduce_add_sync(mask, (unsigned)((u >> 17) & 0x1ffffu)) << 17) +
                            ((long long)__reduce_add_sync(mask, (unsigned)(u >> 34)) << 34) - off;
      if (writer && tot != 0) sacc_add_units<T>(w, tot, a0 - j * kBinW - 52);
    }
    const int wmax = __reduce_max_sync(mask, gmax);
    const int na0 = wmax > top ? min(max(wmax + kBinHead + kBinSlack, bins_min_a0<K>()), 1023) : a0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double sj = bin_anchor(na0 - j * kBinW);
      wb->s[j][ln] = sj;
      if (j < kBinPre) pre[j < kBinPre ? j : 0] = sj;
    }
    top = na0 - kBinHead;
    wb->top[ln] = top;
    count = 0;
  }
  __syncwarp(mask);
  // the bins this lane needs: the fewest k whose last unit 2^(a_0 - (k-1)W -
  // 52) is <= every term's lowest bit, k = 1 + ceil(span / W); the quotient
  // by multiply-shift ((x * 1725) >> 16 == x / 38 for 0 <= x <= 2400; span <=
  // 2046 for any double)
  static_assert(kBinW == 38, "the multiply-shift divides by 38");
  const int span = max(top + kBinHead - 52 - glow, 0);
  const int k = 1 + (((span + kBinW - 1) * 1725) >> 16);
  if (!bins_run_dispatch<K, GL>(wb, xs, k, mask, pre)) return false;   // (the re-anchoring kept the value)
  wb->count[ln] = count + GL;
  // "some term is not -0.0": a nonzero term (the caller's max |bits| != 0), or a +0.0
  bool nz = nonzero;
  if (!nz) {
#pragma unroll
    for (int l = 0; l < GL; ++l) nz |= (uint64_t)__double_as_longlong(xs.v[l]) != kNegZeroBits;
  }
  if (nz) flags |= kXNotNegZero;
  return true;
}

// The per-element levels for a group whose group speculation failed, in
// pieces of P elements: each piece speculates (fold_vec_exact) and replays on
// its own, so one inexact element replays P elements, not the whole group --
// on data whose adds are mostly inexact (the `wide` workload) the replay
// probability grows with the piece size (round 1 speculated per LDS.128
// vector: 4 floats / 2 doubles; whole groups of 8 had cost `wide` 25% / 11%).
template <typename T, int E, int GL, int P>
__device__ __forceinline__ void elementwise_pieces(ExState<E, GL>& st, const ExVals<GL>& xs, long long* w) {
#pragma unroll
  for (int p = 0; p < GL; p += P) {
    double piece[P];
#pragma unroll
    for (int l = 0; l < P; ++l) piece[l] = xs.v[p + l];
    fold_vec_exact<T, E, P>(st.ex, piece, w, st.flags);
  }
}

// fp32 data, one group the group path could not take, out of line (one
// copy per kernel): inf/NaN terms in the warp -> fold_vec_exact's
// per-element levels (tested adds into a0, two TwoSum levels, the element
// replay) per 4 elements, which keep the flags (exact32_special); else the
// bins (exact32_bins: no expansion state crosses the call). mx / mn: the
// group's max |bits| and min |bits| - 1 (zeros skipped).
template <int E, int GL>
__device__ __noinline__ ExState<E, GL> exact32_special(ExState<E, GL> st, const ExVals<GL> xs, long long* w) {
  elementwise_pieces<float, E, GL, (GL < 4 ? GL : 4)>(st, xs, w);
  return st;
}
template <int GL, int K>
__device__ __noinline__ uint32_t exact32_bins(uint32_t flags, const ExVals<GL> xs, WarpBins<K>* wb, uint32_t mx,
                                              uint32_t mn, long long* w) {
  // floor(log2|x|) <= (mx >> 23) - 127; every nonzero term's lowest bit is at
  // least 2^((mn >> 23) - 150) (mn's field may be one below the term's)
  static_assert(K >= 8, "fp32: the bins must span every exponent");   // 52 + 7 * 38 >= 277 + slack
  bins_group<float, K, GL>(wb, flags, xs, (int)(mx >> 23) - 127, (int)(mn >> 23) - 150, mx != 0, w);
  return flags;
}

// fp32 data, a GROUP of GL elements (one LDG.256, or two LDS.128 of the bulk
// ring): each element is m * 2^(e-150) with m < 2^24, so when the group's
// exponent fields span at most 29 - log2(GL) (zeros excluded), every partial
// sum of the group is an integer multiple of 2^(e_min-150) below
// 2^(53+e_min-150): the group's fp64 tree sum is EXACT whatever the order.
// Then ONE tested add puts it into a0 (fl(t - a0) == s && fl(t - s) == a0,
// as in fold_vec_exact). Per element: the F2F widening, 7/8 DADD and 4
// integer ops (|b|, max |b|, |b| - 1, min) -- 1.5 FP64 ops per element
// instead of the per-element test's 5: the FP64 work and its power were
// what held the sustained exact sum at 85% of the read probe.
// Decisions are per warp, with ONE vote on the common path: inf/NaN terms
// send the group to the per-element path (which keeps the flags); an
// exponent spread past the bound (e_min from |b| - 1, so zeros drop out and
// subnormals count as exponent 0) or an inexact add into a0 to the bins.
template <int E, int GL, int K>
__device__ __forceinline__ void fold_group_exact32(Ex (&ex)[E], WarpBins<K>* wb, int g, const uint32_t (&b)[GL],
                                                   long long* w, uint32_t& flags) {
  static_assert(GL == 4 || GL == 8 || GL == 16, "group of 4, 8 or 16 floats");
  constexpr int kMaxSpread = 29 - (GL == 4 ? 2 : GL == 8 ? 3 : 4);
  const unsigned mask = __activemask();
  uint32_t mx = 0, mn = 0xffffffffu;
  double x[GL];
#pragma unroll
  for (int l = 0; l < GL; ++l) {
    const uint32_t a = b[l] & 0x7fffffffu;
    mx = max(mx, a);
    mn = min(mn, a - 1u);                            // zero -> 0xffffffff: no effect
    x[l] = (double)__uint_as_float(b[l]);            // exact widening
  }
  const bool special = mx >= 0x7f800000u;
  const bool wide = (int)(mx >> 23) - (int)(mn >> 23) > kMaxSpread;
  if (__builtin_expect(!__any_sync(mask, special | wide), 1)) {   // (no group work thrown away on wide data)
    const double s = tree_sum<GL>(x);                // exact: the spread test holds
    Ex& q = ex[g % E];
    const double t = __dadd_rn(q.a0, s);
    const bool bad = (__dsub_rn(t, q.a0) != s) | (__dsub_rn(t, s) != q.a0);
    if (__builtin_expect(!__any_sync(mask, bad), 1)) {
      q.a0 = t;
      return;
    }
  }
  ExVals<GL> v;
#pragma unroll
  for (int l = 0; l < GL; ++l) v.v[l] = x[l];
  if (__any_sync(mask, special)) {
    ExState<E, GL> st;
#pragma unroll
    for (int j = 0; j < E; ++j) st.ex[j] = ex[j];
    st.flags = flags;
    st = exact32_special<E, GL>(st, v, w);
#pragma unroll
    for (int j = 0; j < E; ++j) ex[j] = st.ex[j];
    flags = st.flags;
  } else {
    flags = exact32_bins<GL, K>(flags, v, wb, mx, mn, w);
  }
}

// fp64 data, one group the group path could not take, out of line (one
// copy per kernel): the exponent fields are recomputed with the low words
// (a subnormal below 2^-1042 has a zero high word but counts as exponent 0);
// inf/NaN terms or a term past the bins' range (> 2^1007) in the warp, or
// terms that reach below the K-th bin -> the per-element levels per 2
// elements; else the bins.
template <int E, int GL, int K>
__device__ __noinline__ ExState<E, GL> exact64_fallback(ExState<E, GL> st, const ExVals<GL> xs, WarpBins<K>* wb,
                                                        long long* w) {
  uint32_t xmax = 0, xmin = 0xffffffffu;
#pragma unroll
  for (int l = 0; l < GL; ++l) {
    const uint32_t xh = ((uint32_t)__double2hiint(xs.v[l]) & 0x7fffffffu) | min((uint32_t)__double2loint(xs.v[l]), 1u);
    xmax = max(xmax, xh);
    xmin = min(xmin, xh - 1u);                       // zero -> 0xffffffff: no effect
  }
  // floor(log2|x|) <= (xmax >> 20) - 1023; every nonzero term's lowest bit is
  // at least 2^((xmin >> 20) - 1075)
  if (__any_sync(__activemask(), (xmax >> 20) > (uint32_t)(1023 + kBinMaxTop)) ||
      !bins_group<double, K, GL>(wb, st.flags, xs, (int)(xmax >> 20) - 1023, (int)(xmin >> 20) - 1075, xmax != 0,
                                 w))
    elementwise_pieces<double, E, GL, 2>(st, xs, w);
  return st;
}

template <int E, int GL, int K>
__device__ __forceinline__ void exact64_fallback_call(Ex (&ex)[E], uint32_t& flags, const double (&x)[GL],
                                                      WarpBins<K>* wb, long long* w) {
  ExState<E, GL> st;
#pragma unroll
  for (int j = 0; j < E; ++j) st.ex[j] = ex[j];
  st.flags = flags;
  ExVals<GL> v;
#pragma unroll
  for (int l = 0; l < GL; ++l) v.v[l] = x[l];
  st = exact64_fallback<E, GL, K>(st, v, wb, w);
#pragma unroll
  for (int j = 0; j < E; ++j) ex[j] = st.ex[j];
  flags = st.flags;
}

// fp64 data, a GROUP of GL elements into one expansion (a0, a1): the GL
// errors of the adds into a0 are summed in a tree and ONE tested add puts that
// sum into a1 (as spec2's test). The error tree is exact when every error is
// a multiple of 2^m (m: the smallest ulp among the terms and the starting a0
// -- every running sum, rounded or not, is a multiple of the finest of their
// grids) and below half an ulp of the largest running sum: the exponent
// spread <= 54 - log2(GL) -- or trivially when every error is 0 (e.g. terms
// on a common grid, such as the normalish workload's multiples of 2^-24).
// Two forms, chosen per warp BEFORE the group work from facts the terms and
// the current a0 give:
//  * Fast2Sum (3 DADD per element instead of TwoSum's 6) when every lane's
//    |a0| >= GL * max |x| (exponent of a0 >= that of max |x| + 1 + log2 GL):
//    then every running sum outweighs every term, so a0 + x = s + e with
//    e = x - (s - a0) exactly. 3 + 7/8 + 5/8 FP64 ops per element (spec2:
//    11). Same-sign data (u01) lives here after its first groups.
//  * TwoSum otherwise (zero-mean data whose running sums cross zero, every
//    thread's first groups): 6 + 7/8 + 5/8 -- still below spec2's 11, with no
//    wasted speculation. (Speculating Fast2Sum and replaying on failure had
//    cost zero-mean fp64 data 15-29%: with 32 lanes per warp some lane's sum
//    is nearly always near zero.)
// Per warp: inf/NaN terms or a term above the bins' range (> 2^1007): the
// per-element levels (out of line); a spread of the terms alone past the
// bound: the bins (no group work to throw away); an overflow, a spread past
// the bound (with the running sums) with a nonzero error, or an inexact a1
// add: the bins after the group work, told floor(log2|x|) <= (xmax >> 20) -
// 1023 and that every nonzero term's lowest bit is >= 2^((xmin >> 20) - 1075).
template <int E, int GL, int K>
__device__ __forceinline__ void fold_group_exact64(Ex (&ex)[E], WarpBins<K>* wb, int g, const double (&x)[GL],
                                                   long long* w, uint32_t& flags) {
  static_assert(GL == 4 || GL == 8, "group of 4 or 8 doubles");
  constexpr int kLog2GL = (GL == 4 ? 2 : 3);
  constexpr int kMaxSpread = 54 - kLog2GL;
  const unsigned mask = __activemask();
  Ex& q = ex[g % E];
  // exponent fields from the high words: xmax = max |hi|, xmin = SIGNED min
  // of |hi| - 1, which is -1 exactly when some high word is 0 -- a zero, or a
  // subnormal below 2^-1042 whose bits are all in the low word and which must
  // count as exponent 0 (else an error tree that mixes it with errors 2^53
  // larger passes the spread test). Only such groups read the low words, in
  // the rare branch, which recomputes the fields with zeros dropped out.
  uint32_t xmax = 0;
  int xmin_s = 0x7fffffff;
#pragma unroll
  for (int l = 0; l < GL; ++l) {
    const uint32_t xh = (uint32_t)__double2hiint(x[l]) & 0x7fffffffu;
    xmax = max(xmax, xh);
    xmin_s = min(xmin_s, (int)xh - 1);
  }
  uint32_t xmin = (uint32_t)xmin_s;
  const bool special = (xmax >> 20) > (uint32_t)(1023 + kBinMaxTop);   // inf/NaN, or past the bins
  const bool wide = (int)(xmax >> 20) - (xmin_s >> 20) > kMaxSpread;
  if (__builtin_expect(__any_sync(mask, special | wide | (xmin_s < 0)), 0)) {
    bool out = __any_sync(mask, special | wide);
    if (!out) {                                      // zeros (or subnormals below 2^-1042) only
      xmin = 0xffffffffu;
#pragma unroll
      for (int l = 0; l < GL; ++l) {
        const uint32_t xh = ((uint32_t)__double2hiint(x[l]) & 0x7fffffffu) | min((uint32_t)__double2loint(x[l]), 1u);
        xmin = min(xmin, xh - 1u);                   // zero -> 0xffffffff: no effect
      }
      out = __any_sync(mask, (int)(xmax >> 20) - (int)(xmin >> 20) > kMaxSpread);
    }
    if (out) {                                       // the fallback: per element or the bins, no group work
      exact64_fallback_call<E, GL, K>(ex, flags, x, wb, w);
      return;
    }
    // zeros only: the group work with the zeros dropped out of xmin
  }
  const uint32_t a0h = (uint32_t)__double2hiint(q.a0) & 0x7fffffffu;
  const bool fast = __all_sync(mask, (a0h >> 20) >= (xmax >> 20) + 1 + kLog2GL);
  double a = q.a0, e[GL];
  uint32_t smax = 0, amin = 0xffffffffu;   // amin: the starting a0 (the running sums' grids follow from it and the terms)
  if (fast) {
#pragma unroll
    for (int l = 0; l < GL; ++l) {
      const double sl = __dadd_rn(a, x[l]);
      e[l] = __dsub_rn(x[l], __dsub_rn(sl, a));      // Fast2Sum: |a| >= |x| here
      a = sl;
      smax = max(smax, (uint32_t)__double2hiint(a) & 0x7fffffffu);
    }
  } else {
    amin = (a0h | min((uint32_t)__double2loint(q.a0), 1u)) - 1u;   // a zero a0 drops out
#pragma unroll
    for (int l = 0; l < GL; ++l) {
      double sl;
      two_sum(a, x[l], sl, e[l]);
      a = sl;
      smax = max(smax, (uint32_t)__double2hiint(a) & 0x7fffffffu);
    }
  }
  bool nz = false;
#pragma unroll
  for (int l = 0; l < GL; ++l) nz |= (e[l] != 0.0);
  const uint32_t mn = min(xmin, amin);
  const double se = tree_sum<GL>(e);
  const double t = __dadd_rn(q.a1, se);
  const bool bad = (smax >= 0x7ff00000u) |
                   (nz & ((int)(smax >> 20) - (int)(mn >> 20) > kMaxSpread)) |
                   (__dsub_rn(t, q.a1) != se) | (__dsub_rn(t, se) != q.a1);
  if (__builtin_expect(!__any_sync(mask, bad), 1)) {
    q.a0 = a;
    q.a1 = t;
    return;
  }
  exact64_fallback_call<E, GL, K>(ex, flags, x, wb, w);
}

// round the normalised words (value = sum w[k] 2^(32k) * 2^kLsb) once; returns the float's bits
template <typename T>
__device__ uint64_t exact_round(const long long* w, uint32_t flags, uint64_t n) {
  using TR = ExactTraits<T>;
  constexpr int NW = TR::kWords, p = TR::kPrec;
  if ((flags & kXNaN) || ((flags & kXPosInf) && (flags & kXNegInf))) return TR::kQNaN;
  if (flags & kXPosInf) return TR::kInfBits;
  if (flags & kXNegInf) return TR::kInfBits | TR::kSignBit;
  const bool neg = w[NW - 1] < 0;
  uint32_t D[NW];
  uint64_t c = neg ? 1 : 0;
  for (int k = 0; k < NW; ++k) {                // magnitude digits (two's complement negation)
    const uint32_t dk = (uint32_t)w[k];
    const uint64_t t = (uint64_t)(neg ? ~dk : dk) + c;
    D[k] = (uint32_t)t;
    c = neg ? (t >> 32) : 0;
  }
  int kt = NW - 1;
  while (kt >= 0 && D[kt] == 0) --kt;
  if (kt < 0) return (n == 0 || (flags & kXNotNegZero)) ? 0ull : TR::kSignBit;   // exact zero (R2)
  const int lz = __clz(D[kt]);
  const int P = 32 * kt + 31 - lz;              // leading one
  uint64_t bits;
  if (P < p) {
    // the integer itself is the bit pattern: subnormal (exponent field 0) or
    // the smallest normal binade (field 1 = the 2^(p-1) bit)
    bits = ((uint64_t)(kt >= 1 ? D[1] : 0) << 32) | D[0];
  } else {
    const uint32_t Dm1 = kt >= 1 ? D[kt - 1] : 0, Dm2 = kt >= 2 ? D[kt - 2] : 0;
    const unsigned __int128 win = ((unsigned __int128)D[kt] << 64) | ((unsigned __int128)Dm1 << 32) | Dm2;
    const int sh = 32 - lz;                     // 96-bit window -> leading one at bit 63
    const uint64_t W64 = (uint64_t)(win >> sh);
    bool sticky = ((uint64_t)win & ((1ull << sh) - 1)) != 0;
    for (int k = 0; k < kt - 2 && !sticky; ++k) sticky = D[k] != 0;
    uint64_t q = W64 >> (64 - p);
    const bool guard = (W64 >> (63 - p)) & 1;
    const bool rest = (W64 & ((1ull << (63 - p)) - 1)) != 0 || sticky;
    if (guard && (rest || (q & 1))) ++q;        // ties to even
    bits = ((uint64_t)(P + 1 - p) << (p - 1)) + q;   // a carry out of q bumps the exponent
    if (bits >= TR::kInfBits) bits = TR::kInfBits;   // beyond the range: inf (IEEE overflow)
  }
  return neg ? (bits | TR::kSignBit) : bits;
}

template <typename T>
__device__ __forceinline__ void exact_store(const long long* w, uint32_t flags, uint64_t n, void* out) {
  const uint64_t b = exact_round<T>(w, flags, n);
  if constexpr (sizeof(T) == 4) *(uint32_t*)out = (uint32_t)b;
  else *(uint64_t*)out = b;
}

// The fused multi-GPU exchange of exact records (reduce_fused with
// RD_SUM_EXACT; the LL protocol of rd_kernels.cuh fused_exchange, 4 + 2*NW
// self-validating words per rank): warp 0 of the last CTA pushes this rank's
// carried words into slot [epoch&1][rank] of every mailbox, polls its own
// until the W records of this epoch are complete, adds them word by word
// (integers: the same bits on every rank, whatever the arrival order), and
// rounds once.
template <typename T>
__device__ __noinline__ void exact_fused_exchange(long long* words, unsigned flags, const XArgs& args) {
  constexpr int NW = ExactTraits<T>::kWords;
  constexpr int NP = 4 + 2 * NW;                     // payload words
  static_assert(NP <= kExactLLWords, "mailbox too small");
  const int ln = threadIdx.x & 31;
  const unsigned long long epoch = *(volatile unsigned long long*)&args.self->epoch + 1;
  const int par = (int)(epoch & 1);
  const unsigned long long eflag = (unsigned long long)(uint32_t)epoch << 32;
  const int W = args.nranks;
  auto payload = [&](int k) -> uint32_t {
    if (k == 0) return args.tag;
    if (k == 1) return (uint32_t)args.n;
    if (k == 2) return (uint32_t)(args.n >> 32);
    if (k == 3) return flags;
    const unsigned long long v = (unsigned long long)words[(k - 4) >> 1];
    return (k & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
  };
  // the common 32-byte LL header {tag, 0, n lo, n hi, 0...} goes through the
  // same ll slots as every plain record, so a peer that runs another op or
  // dtype (plain or exact) sees this tag and reports RD_ERR_MISMATCH instead
  // of waiting for words it would never receive
  for (int p = 0; p < W; ++p) {
    volatile unsigned long long* dst = args.peers[p]->xll[par][args.rank];
    for (int k = ln; k < NP; k += 32) dst[k] = eflag | payload(k);   // peer stores over NVLink
    if (ln < 8) {
      const uint32_t h = ln == 0 ? args.tag : ln == 2 ? (uint32_t)args.n : ln == 3 ? (uint32_t)(args.n >> 32) : 0u;
      args.peers[p]->ll[par][args.rank][ln] = eflag | h;
    }
  }
  bool timeout = false, bad = false;
  for (int q = ln; q < W; q += 32) {                 // the peers' headers first
    const volatile unsigned long long* src = args.self->ll[par][q];
    uint32_t spins = 0;
    unsigned long long v;
    while (((v = src[0]) & 0xffffffff00000000ull) != eflag) {
      if (++spins > 4096) __nanosleep(128);
      if (spins > (1u << 25)) { timeout = true; break; }
    }
    bad |= !timeout && (uint32_t)v != args.tag;
  }
  timeout = __any_sync(0xffffffffu, timeout);
  bad = __any_sync(0xffffffffu, bad);
  for (int q = 0; q < W && !timeout && !bad; ++q) {
    const volatile unsigned long long* src = args.self->xll[par][q];
    for (int k = ln; k < NP; k += 32) {
      uint32_t spins = 0;
      while ((src[k] & 0xffffffff00000000ull) != eflag) {
        if (++spins > 4096) __nanosleep(128);
        if (spins > (1u << 25)) { timeout = true; break; }
      }
      if (timeout) break;
    }
    timeout = __any_sync(0xffffffffu, timeout);
  }
  __syncwarp();
  // every word of every record is in: sum them (lane j: words j, j+32, ...)
  unsigned long long n = 0;
  unsigned fl = 0;
  if (!timeout && !bad) {
    for (int q = 0; q < W; ++q) {
      const volatile unsigned long long* src = args.self->xll[par][q];
      bad |= (uint32_t)src[0] != args.tag;
      n += ((unsigned long long)(uint32_t)src[2] << 32) | (uint32_t)src[1];
      fl |= (uint32_t)src[3];
    }
    for (int j = ln; j < NW; j += 32) {
      long long s = 0;
      for (int q = 0; q < W; ++q) {
        const volatile unsigned long long* src = args.self->xll[par][q];
        s += (long long)((((unsigned long long)(uint32_t)src[5 + 2 * j]) << 32) | (uint32_t)src[4 + 2 * j]);
      }
      words[j] = s;                                  // < W * 2^32 per word
    }
  }
  __syncwarp();
  // timeout, bad and n are warp-uniform (every lane read the same headers)
  if (!timeout && !bad && n != 0) {
    sacc_normalise_by_warp<NW>(words);
    __syncwarp();
  }
  if (ln == 0) {
    if (timeout) atomicExch(args.err, (int)RD_ERR_TIMEOUT);
    else if (bad) atomicExch(args.err, (int)RD_ERR_MISMATCH);
    if (timeout || bad || n == 0) {
      if constexpr (sizeof(T) == 4) *(uint32_t*)args.out = 0u;
      else *(uint64_t*)args.out = 0ull;
    } else {
      exact_store<T>(words, fl, n, args.out);
    }
    *(volatile unsigned long long*)&args.self->epoch = epoch;
  }
}

// a3-a5, shared by the exact kernels: the expansions -> warp
// superaccumulators -> the CTA's carried-digit sums in cta[0..NW) (< 2^35 per
// word) and its flags in cta[NW]. Ends with __syncthreads.
template <typename T, int B, int E, int K>
__device__ __forceinline__ void exact_cta_words(Ex (&ex)[E], const WarpBins<K>* wbins, uint32_t flags,
                                                long long (*sacc)[ExactTraits<T>::kWords], unsigned& s_flags,
                                                long long* cta) {
  constexpr int NW = ExactTraits<T>::kWords;
  constexpr int NWARP = B / 32;
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  long long* w = sacc[warp];
  // a3: the expansions into the warp's superaccumulator. Every term passes
  // through some a0 (or the slow path, which flags itself), and an a0 that
  // has seen a term other than -0.0 is never -0.0 again (x + -x = +0), so a0
  // alone decides reading R2's "every term is -0.0".
  __syncwarp();
  double dv[3 * E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    if ((uint64_t)__double_as_longlong(ex[j].a0) != kNegZeroBits) flags |= kXNotNegZero;
    dv[3 * j] = ex[j].a0;
    dv[3 * j + 1] = ex[j].a1;
    dv[3 * j + 2] = ex[j].a2;
  }
  sacc_flush_warp<T, 3 * E>(w, dv);
  // the bins' contents (flags set by bins_group), only if some lane of the warp
  // added to its bins since the last re-anchoring (count > 0): most data never
  // reaches them, and small launches are epilogue-bound
  if (__any_sync(0xffffffffu, wbins[warp].count[ln] > 0)) {
    const Bins<K> bn = bins_load(&wbins[warp]);
    double bv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) bv[j] = bin_value(bn, j);
    sacc_flush_warp<T, K>(w, bv);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (ln == 0 && flags) atomicOr(&s_flags, flags);
  __syncwarp();
  // a4: each warp carries its words into digits
  sacc_normalise_by_warp<NW>(w);
  __syncthreads();
  // a5: the CTA's words (sum of NWARP digit vectors)
  if (threadIdx.x < NW) {
    long long s = 0;
#pragma unroll
    for (int q = 0; q < NWARP; ++q) s += sacc[q][threadIdx.x];
    cta[threadIdx.x] = s;
  }
  if (threadIdx.x == NW) cta[NW] = (long long)s_flags;
  __syncthreads();
}

// a7: the carried total (words, normalised) -> the result (mode 0, thread 0),
// an exact record (mode 1, thread 0) or the fused exchange (mode 2, warp 0)
template <typename T>
__device__ __forceinline__ void exact_emit(long long* words, unsigned flags, const XArgs& args) {
  constexpr int NW = ExactTraits<T>::kWords;
  if (threadIdx.x == 0) {
    if (args.mode == 0) {
      exact_store<T>(words, flags, args.n, args.out);
    } else if (args.mode == 1) {
      rd_exact_record* r = args.rec;
      r->tag = args.tag;
      r->status = 0;
      r->n = args.n;
      r->flags = flags;
      r->nwords = NW;
      r->reserved = 0;
      for (int k = 0; k < NW; ++k) r->word[k] = words[k];
      for (int k = NW; k < RD_EXACT_MAX_WORDS; ++k) r->word[k] = 0;
    }
  }
  if (args.mode == 2 && threadIdx.x < 32) {
    __syncwarp();
    exact_fused_exchange<T>(words, flags, args);
  }
}

// a3-a7 for the persistent grids: the CTA's words go to workspace slot
// blockIdx; the last CTA (atomic ticket) adds the G slots and emits.
template <typename T, int B, int E, int K>
__device__ __forceinline__ void exact_finish(Ex (&ex)[E], const WarpBins<K>* wbins, uint32_t flags,
                                             long long (*sacc)[ExactTraits<T>::kWords],
                                             long long* tot, unsigned& s_flags, unsigned& s_last,
                                             const XArgs& args) {
  constexpr int NW = ExactTraits<T>::kWords;
  static_assert(B > NW, "one thread per word");
  // a6: the launch's accumulator -- NW + 1 words at the head of the exact
  // workspace, zero between launches. Every CTA adds its carried words
  // (< 2^35 each: < 2^47 over any grid) with native 64-bit global reductions
  // and ORs its flags; integer adds are exact in any order, so the last CTA
  // (atomic ticket) reads NW + 1 words instead of folding G slots of NW + 1
  // words (fp64: 296 CTAs x 69 words were ~80 dependent-ish L2 loads per
  // thread of the last CTA) and zeroes them for the next launch.
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(args.partials);
  exact_cta_words<T, B, E, K>(ex, wbins, flags, sacc, s_flags, tot);
  if (threadIdx.x < NW) {
    if (tot[threadIdx.x] != 0) atomicAdd(acc + threadIdx.x, (unsigned long long)tot[threadIdx.x]);
  } else if (threadIdx.x == NW) {
    if (tot[NW] != 0) atomicOr(acc + NW, (unsigned long long)tot[NW]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = ticket_acq_rel(args.ticket);   // release the CTA's additions, acquire the others'
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x <= NW) {
    const long long v = (long long)__ldcg(acc + threadIdx.x);
    acc[threadIdx.x] = 0ull;                         // zero for the next launch (kernel boundary orders it)
    if (threadIdx.x < NW) sacc[0][threadIdx.x] = v;
    else s_flags = (unsigned)v;
  }
  __syncthreads();
  if (threadIdx.x < 32) sacc_normalise_by_warp<NW>(sacc[0]);
  if (threadIdx.x == 0) {
    *args.ticket = 0u;
    if (args.work) *args.work = 0u;
  }
  __syncthreads();
  exact_emit<T>(sacc[0], s_flags, args);
}

// a6-a7 when the grid is one thread-block cluster (small inputs): rank 0 adds
// the G CTAs' words over distributed shared memory -- no slot, fence or ticket.
__device__ __forceinline__ long long dsmem_load_i64(const long long* local, unsigned rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(a), "r"(rank));
  long long v;
  asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(remote) : "memory");
  return v;
}

template <typename T, int B, int E, int K>
__device__ __forceinline__ void exact_finish_cluster(Ex (&ex)[E], const WarpBins<K>* wbins, uint32_t flags,
                                                     long long (*sacc)[ExactTraits<T>::kWords], long long* cta,
                                                     unsigned& s_flags, const XArgs& args) {
  constexpr int NW = ExactTraits<T>::kWords;
  exact_cta_words<T, B, E, K>(ex, wbins, flags, sacc, s_flags, cta);
  cluster_sync();
  if (cluster_ctarank() == 0) {
    const unsigned G = cluster_nctarank();
    if (threadIdx.x <= NW) {
      const int j = threadIdx.x;
      long long v[16];                               // all G remote loads in flight at once
#pragma unroll
      for (unsigned r = 0; r < 16; ++r) v[r] = r < G ? dsmem_load_i64(cta + j, r) : 0;
      long long s = 0;
#pragma unroll
      for (unsigned r = 0; r < 16; ++r) s = (j == NW) ? (s | v[r]) : (s + v[r]);
      if (j < NW) sacc[0][j] = s;
      else s_flags = (unsigned)s;
    }
    __syncthreads();
    if (threadIdx.x < 32) sacc_normalise_by_warp<NW>(sacc[0]);
    __syncthreads();
    exact_emit<T>(sacc[0], s_flags, args);
  }
  cluster_sync();   // the other CTAs' words stay alive until rank 0 has read them
}

// --------------------------------------------------------------------- kernel
// The exact vector kernels' streaming part (a1, a2): every thread's E
// expansions over its grid-stride share of 32-byte vectors, and the head/tail
// stragglers. The main loop's trip count is warp-uniform (tested on the warp's
// last lane, whose index is the largest), so every iteration can end with a
// __syncwarp: a lane that replayed a vector (divergent) rejoins its warp
// there. Without it the warp stayed split after the first divergent replay
// and ran the loop ~2 lanes at a time (ncu: 2.0 avg threads per F2F).
template <typename T, int B, int U, int E>
__device__ __forceinline__ void exact_vector_body(const XArgs& args, Ex (&ex)[E], WarpBins<BinK<T>::K>* wb,
                                                  long long* w, uint32_t& flags) {
  constexpr int VB = 32;
  constexpr int L = VB / (int)sizeof(T);
  const int ln = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < E; ++j) ex[j] = Ex{-0.0, -0.0, -0.0};
  bins_init(wb);
  const uint64_t tid = (uint64_t)blockIdx.x * B + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * B;
  const unsigned char* body = args.x + args.head * sizeof(T);
  pdl_wait();
  const uint64_t nvec = args.nvec;
  uint64_t i = tid;
  const uint64_t lag = 31 - (uint64_t)ln;        // lane 31's index = i + lag
  for (; i + lag + (uint64_t)(U - 1) * stride < nvec; i += (uint64_t)U * stride) {
    Vec<VB> v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream<VB>(body + (i + (uint64_t)u * stride) * VB);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int u = 0; u < U; ++u) fold_group_exact32<E, L>(ex, wb, u, v[u].w, w, flags);
    } else if constexpr (U % 2 == 0) {
      // fp64: groups of 8 (two 32-byte vectors)
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        double xs[2 * L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
          xs[l] = lane<T, VB>(v[u], l);
          xs[L + l] = lane<T, VB>(v[u + 1], l);
        }
        fold_group_exact64<E, 2 * L>(ex, wb, u / 2, xs, w, flags);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double xs[L];
#pragma unroll
        for (int l = 0; l < L; ++l) xs[l] = lane<T, VB>(v[u], l);
        fold_group_exact64<E, L>(ex, wb, u, xs, w, flags);
      }
    }
    __syncwarp();
  }
  for (; i < nvec; i += stride) {
    Vec<VB> v = ldg_stream<VB>(body + i * VB);
    if constexpr (sizeof(T) == 4) {
      fold_group_exact32<E, L>(ex, wb, 0, v.w, w, flags);
    } else {
      double xs[L];
#pragma unroll
      for (int l = 0; l < L; ++l) xs[l] = widen(lane<T, VB>(v, l));
      fold_vec_exact<T, E, L>(ex, xs, w, flags);
    }
  }
  pdl_trigger();
  // a2: head and tail stragglers
  if (tid < args.head) ex_add<T>(ex[0], widen(ldg_scalar<T>(args.x + tid * sizeof(T))), w, flags);
  if (tid < args.tail) ex_add<T>(ex[E - 1], widen(ldg_scalar<T>(args.x + (args.tail_start + tid) * sizeof(T))), w, flags);
}

// The persistent vector form: grid-stride, then slots + the atomic ticket.
template <typename T, int B, int U, int E, int MINB>
__global__ void __launch_bounds__(B, MINB) rd_exact_kernel(const __grid_constant__ XArgs args) {
  constexpr int NW = ExactTraits<T>::kWords;
  constexpr int NWARP = B / 32;
  __shared__ long long sacc[NWARP][NW];
  __shared__ long long tot[B];
  __shared__ unsigned s_flags, s_last;
  for (int i = threadIdx.x; i < NWARP * NW; i += B) (&sacc[0][0])[i] = 0;
  if (threadIdx.x == 0) s_flags = 0;
  __syncthreads();
  __shared__ WarpBins<BinK<T>::K> wbins[NWARP];
  Ex ex[E];
  uint32_t flags = 0;
  exact_vector_body<T, B, U, E>(args, ex, &wbins[threadIdx.x >> 5], sacc[threadIdx.x >> 5], flags);
  exact_finish<T, B, E>(ex, wbins, flags, sacc, tot, s_flags, s_last, args);
}

// The same on a grid that is ONE thread-block cluster (<= 16 CTAs): AUTO's
// choice for small inputs (n*s <= 1 MiB), like rd_cluster_kernel -- the CTA
// words are added over distributed shared memory (no slots, fence or ticket).
template <typename T, int B, int U, int E, int MINB>
__global__ void __launch_bounds__(B, MINB) rd_exact_cluster_kernel(const __grid_constant__ XArgs args) {
  constexpr int NW = ExactTraits<T>::kWords;
  constexpr int NWARP = B / 32;
  __shared__ long long sacc[NWARP][NW];
  __shared__ long long cta[NW + 1];
  __shared__ unsigned s_flags;
  for (int i = threadIdx.x; i < NWARP * NW; i += B) (&sacc[0][0])[i] = 0;
  if (threadIdx.x == 0) s_flags = 0;
  __syncthreads();
  __shared__ WarpBins<BinK<T>::K> wbins[NWARP];
  Ex ex[E];
  uint32_t flags = 0;
  exact_vector_body<T, B, U, E>(args, ex, &wbins[threadIdx.x >> 5], sacc[threadIdx.x >> 5], flags);
  exact_finish_cluster<T, B, E>(ex, wbins, flags, sacc, cta, s_flags, args);
}

// The bulk-copy form (like rd_bulk_kernel): one producer lane streams
// chunks (static first chunk, then a global counter) into a STAGES-deep
// shared-memory ring with cp.async.bulk; CW consumer warps LDS.128 their
// slice of each stage into fold_vec_exact. Memory parallelism comes from the
// ring (STAGES * STAGE_BYTES in flight per SM), not from registers -- the
// vector kernel's 118 registers/thread cap it at 16 warps/SM.
// the exact bulk kernel's dynamic shared memory: the ring, its barriers and
// stage metadata (BulkSmem), then one WarpBins block per warp
template <typename T, int STAGES, int STAGE_BYTES, int CW>
struct ExactBulkSmem {
  static constexpr int kBins = BulkSmem<STAGES, STAGE_BYTES, CW>::kBytes;
  static constexpr int kBytes = kBins + (CW + 1) * (int)sizeof(WarpBins<BinK<T>::K>);
};

template <typename T, int STAGES, int STAGE_BYTES, int CW, int E>
__global__ void __launch_bounds__(32 * (CW + 1), 1) rd_exact_bulk_kernel(const __grid_constant__ XArgs args) {
  using TR = ExactTraits<T>;
  constexpr int NW = TR::kWords;
  constexpr int B = 32 * (CW + 1);
  constexpr int CT = 32 * CW;
  constexpr int L = 16 / (int)sizeof(T);
  constexpr int PER_THREAD = STAGE_BYTES / (16 * CT);
  static_assert(STAGE_BYTES % (16 * CT) == 0, "stage must split evenly over consumer threads");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint32_t* st_bytes = reinterpret_cast<uint32_t*>(empty + STAGES);   // 0 = no more chunks
  __shared__ long long sacc[B / 32][NW];
  WarpBins<BinK<T>::K>* wbins =                      // dynamic: past the 48 KB static limit
      reinterpret_cast<WarpBins<BinK<T>::K>*>(smem_raw + ExactBulkSmem<T, STAGES, STAGE_BYTES, CW>::kBins);
  __shared__ long long tot[B];
  __shared__ unsigned s_flags, s_last;

  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (B / 32) * NW; i += B) (&sacc[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    s_flags = 0;
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], RD_EMPTY_COUNT(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Ex ex[E];
#pragma unroll
  for (int j = 0; j < E; ++j) ex[j] = Ex{-0.0, -0.0, -0.0};
  bins_init(&wbins[warp]);
  uint32_t flags = 0;
  const unsigned char* body = args.x + args.head * sizeof(T);
  const uint64_t body_bytes = args.nvec * 16;
  pdl_wait();
  if (warp == CW) {
    if (ln == 0) {                                   // producer
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      uint32_t c = blockIdx.x;
      uint32_t next = atomicAdd(args.work, 1u) + gridDim.x;
      for (;; c = next, next = atomicAdd(args.work, 1u) + gridDim.x) {
        if (c >= args.nchunks) {
          mbar_wait(&empty[stage], phase ^ 1);
          st_bytes[stage] = 0;
          mbar_arrive(&full[stage]);
          break;
        }
        uint64_t cbeg, clen;
        chunk_range(args, c, body_bytes, &cbeg, &clen);
        const uint64_t cend = cbeg + clen;
        for (uint64_t off = cbeg; off < cend; off += STAGE_BYTES) {
          const uint32_t bytes = (uint32_t)min((uint64_t)STAGE_BYTES, cend - off);
          mbar_wait(&empty[stage], phase ^ 1);
          st_bytes[stage] = bytes;
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(ring + (size_t)stage * STAGE_BYTES, body + off, bytes, &full[stage], pol);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {                                           // consumers
    long long* w = sacc[warp];
    const int t = threadIdx.x;
    const uint32_t ring_addr = smem_addr(ring);
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      mbar_wait(&full[stage], phase);
      const uint32_t bytes = st_bytes[stage];
      if (bytes == 0) break;
      const uint32_t base = ring_addr + stage * STAGE_BYTES;
      if (bytes == STAGE_BYTES) {
        uint4 v[PER_THREAD];
#pragma unroll
        for (int k = 0; k < PER_THREAD; ++k) v[k] = lds128(base + (k * CT + t) * 16);
        if constexpr (sizeof(T) == 4 && PER_THREAD % 2 == 0) {
          // fp32: groups of 8 (two LDS.128), one tested add per group
#pragma unroll
          for (int k = 0; k < PER_THREAD; k += 2) {
            const uint32_t b8[8] = {v[k].x, v[k].y, v[k].z, v[k].w, v[k + 1].x, v[k + 1].y, v[k + 1].z, v[k + 1].w};
            fold_group_exact32<E, 8>(ex, &wbins[warp], k / 2, b8, w, flags);
          }
        } else if constexpr (sizeof(T) == 8 && PER_THREAD % 4 == 0) {
          // fp64: groups of 8 (four LDS.128)
#pragma unroll
          for (int k = 0; k < PER_THREAD; k += 4) {
            double d8[8];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              Vec<16> q{{v[k + j].x, v[k + j].y, v[k + j].z, v[k + j].w}};
              d8[2 * j] = lane<T, 16>(q, 0);
              d8[2 * j + 1] = lane<T, 16>(q, 1);
            }
            fold_group_exact64<E, 8>(ex, &wbins[warp], k / 4, d8, w, flags);
          }
        } else {
#pragma unroll
          for (int k = 0; k < PER_THREAD; ++k) {
            Vec<16> q{{v[k].x, v[k].y, v[k].z, v[k].w}};
            double xs[L];
#pragma unroll
            for (int l = 0; l < L; ++l) xs[l] = widen(lane<T, 16>(q, l));
            fold_vec_exact<T, E, L>(ex, xs, w, flags);
          }
        }
      } else {
        for (int k = 0; k < PER_THREAD; ++k) {
          const uint32_t off = (k * CT + t) * 16;
          if (off < bytes) {
            const uint4 r = lds128(base + off);
            Vec<16> q{{r.x, r.y, r.z, r.w}};
            double xs[L];
#pragma unroll
            for (int l = 0; l < L; ++l) xs[l] = widen(lane<T, 16>(q, l));
            fold_vec_exact<T, E, L>(ex, xs, w, flags);
          }
        }
      }
      // reconverge (a replayed vector diverges), then release the stage
      RD_RELEASE_STAGE(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    // a2: head and tail stragglers (< 16 bytes each), CTA 0's first threads
    if (blockIdx.x == 0) {
      if ((uint64_t)t < args.head) ex_add<T>(ex[0], widen(ldg_scalar<T>(args.x + t * sizeof(T))), w, flags);
      if ((uint64_t)t < args.tail)
        ex_add<T>(ex[E - 1], widen(ldg_scalar<T>(args.x + (args.tail_start + t) * sizeof(T))), w, flags);
    }
  }
  pdl_trigger();
  exact_finish<T, B, E>(ex, wbins, flags, sacc, tot, s_flags, s_last, args);
}

// Fold `count` exact records (any order gives the same integer): one CTA.
template <typename T>
__global__ void rd_exact_combine_kernel(const rd_exact_record* recs, int count, uint32_t tag, void* out,
                                        rd_exact_record* rec_out, int* d_status) {
  using TR = ExactTraits<T>;
  constexpr int NW = TR::kWords;
  __shared__ long long s[NW];
  __shared__ unsigned s_flags, s_bad;
  __shared__ unsigned long long s_n;
  if (threadIdx.x == 0) { s_flags = 0; s_bad = 0; s_n = 0; }
  __syncthreads();
  for (int r = threadIdx.x; r < count; r += blockDim.x) {
    const rd_exact_record* q = recs + r;
    if (q->tag != tag || q->nwords != (uint32_t)NW) atomicOr(&s_bad, 1u);
    else {
      atomicOr(&s_flags, q->flags);
      atomicAdd(&s_n, (unsigned long long)q->n);
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < NW) {
    long long a = 0;
    for (int r = 0; r < count; ++r)
      if (recs[r].tag == tag && recs[r].nwords == (uint32_t)NW) a += recs[r].word[threadIdx.x];
    s[threadIdx.x] = a;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  sacc_normalise_by_warp<NW>(s);                    // launched with 128 threads: warp 0 is whole
  __syncwarp();
  if (threadIdx.x != 0) return;
  if (s_bad && d_status) *d_status = (int)RD_ERR_MISMATCH;
  if (out) {
    if (s_bad || s_n == 0) {
      if constexpr (sizeof(T) == 4) *(uint32_t*)out = 0u;
      else *(uint64_t*)out = 0ull;
    } else {
      exact_store<T>(s, s_flags, s_n, out);
    }
  }
  if (rec_out) {
    rec_out->tag = tag;
    rec_out->status = s_bad ? (uint32_t)RD_ERR_MISMATCH : 0u;
    rec_out->n = s_n;
    rec_out->flags = s_flags;
    rec_out->nwords = NW;
    rec_out->reserved = 0;
    for (int k = 0; k < NW; ++k) rec_out->word[k] = s[k];
    for (int k = NW; k < RD_EXACT_MAX_WORDS; ++k) rec_out->word[k] = 0;
  }
}

}  // namespace rd
