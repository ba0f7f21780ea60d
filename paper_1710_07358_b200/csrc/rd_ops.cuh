// rd_ops.cuh -- the combiner (x) of PAPER.md P:23 for every (dtype, op) pair,
// as device-side traits used by every kernel of the library.
//
// Each trait defines
//   T         storage type of one element (raw bit pattern for integers)
//   Acc       accumulator type (wider for fp32 x and fp64 x; see b200reduce.h)
//   identity  the padding element: combine(identity, a) == a for every a
//             (Algorithm 1's initial accumulator; -0.0 for float +,
//             because +0.0 is not an identity for -0.0)
//   fold      acc (x) x_i for one element (the body of Algorithm 1's loop)
//   combine   acc (x) acc
//   warp_reduce  butterfly over the 32 lanes (Luitjens' SHFL tree),
//             or redux.sync for 32-bit integer add/min/max/and/or/xor
//   store     narrow to T with one rounding and write one element
//   store_empty  the empty-input result (b200reduce.h table)
//   pack/unpack  16-byte slot for partials and rd_record.acc
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "b200reduce.h"

namespace rd {

struct Slot { uint64_t a, b; };

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_idx_u64(uint64_t v, int src) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ double shfl_xor_f64(double v, int m) {
  return __longlong_as_double((long long)shfl_xor_u64((uint64_t)__double_as_longlong(v), m));
}

// ------------------------------------------------------------------ integers
template <typename U, rd_op OP, bool SIGNED>
struct IntOp {
  using T = U;
  using Acc = U;
  static constexpr bool kFloat = false;
  static constexpr bool kIndexed = false;
  static constexpr bool kOrderFree = true;   // mod-2^w ring / lattice ops: any order, same bits
  using S = typename std::conditional<sizeof(U) == 4, int32_t, int64_t>::type;

  __device__ __forceinline__ static Acc identity() {
    if (OP == RD_SUM || OP == RD_OR || OP == RD_XOR) return (U)0;
    if (OP == RD_PROD) return (U)1;
    if (OP == RD_AND) return (U)~(U)0;
    constexpr U smax = (U)(~(U)0) >> 1;         // 0x7fff..
    if (OP == RD_MIN) return SIGNED ? smax : (U)~(U)0;
    /* RD_MAX */ return SIGNED ? (U)(smax + (U)1) : (U)0;
  }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) {
    if (OP == RD_SUM) return a + b;                       // wraps mod 2^w
    if (OP == RD_PROD) return a * b;                      // wraps mod 2^w
    if (OP == RD_AND) return a & b;
    if (OP == RD_OR) return a | b;
    if (OP == RD_XOR) return a ^ b;
    if (OP == RD_MIN) {
      if (SIGNED) return ((S)a < (S)b) ? a : b;
      return a < b ? a : b;
    }
    if (SIGNED) return ((S)a > (S)b) ? a : b;
    return a > b ? a : b;
  }
  __device__ __forceinline__ static Acc fold(Acc a, T x) { return combine(a, x); }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
    if constexpr (sizeof(U) == 4 && OP != RD_PROD) {
      // redux.sync (sm_80+): one instruction for the whole warp
      if (OP == RD_SUM) return __reduce_add_sync(0xffffffffu, (unsigned)a);
      if (OP == RD_AND) return __reduce_and_sync(0xffffffffu, (unsigned)a);
      if (OP == RD_OR) return __reduce_or_sync(0xffffffffu, (unsigned)a);
      if (OP == RD_XOR) return __reduce_xor_sync(0xffffffffu, (unsigned)a);
      if (OP == RD_MIN)
        return SIGNED ? (U)__reduce_min_sync(0xffffffffu, (int)a) : (U)__reduce_min_sync(0xffffffffu, (unsigned)a);
      return SIGNED ? (U)__reduce_max_sync(0xffffffffu, (int)a) : (U)__reduce_max_sync(0xffffffffu, (unsigned)a);
    } else {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        U o = (sizeof(U) == 4) ? (U)__shfl_xor_sync(0xffffffffu, (uint32_t)a, m) : (U)shfl_xor_u64((uint64_t)a, m);
        a = combine(a, o);
      }
      return a;
    }
  }
  __device__ __forceinline__ static void store(Acc a, void* out) { *(T*)out = a; }
  __device__ __forceinline__ static void store_empty(void* out) { *(T*)out = identity(); }
  __device__ __forceinline__ static Slot pack(Acc a) { return Slot{(uint64_t)a, 0}; }
  __device__ __forceinline__ static Acc unpack(Slot s) { return (Acc)s.a; }
};

// ------------------------------------------------- float32 x (fp64 accumulator)
struct Float32Prod {
  using T = float;
  using Acc = double;
  static constexpr bool kFloat = true;
  static constexpr bool kIndexed = false;
  __device__ __forceinline__ static Acc identity() { return 1.0; }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static Acc fold(Acc a, T x) { return __dmul_rn(a, (double)x); }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) a = __dmul_rn(a, shfl_xor_f64(a, m));
    return a;
  }
  __device__ __forceinline__ static void store(Acc a, void* out) { *(float*)out = __double2float_rn(a); }
  __device__ __forceinline__ static void store_empty(void* out) { *(float*)out = 1.0f; }
  __device__ __forceinline__ static Slot pack(Acc a) { return Slot{(uint64_t)__double_as_longlong(a), 0}; }
  __device__ __forceinline__ static Acc unpack(Slot s) { return __longlong_as_double((long long)s.a); }
};

// ---------------------------------------- float64 x (double-double accumulator)
// (hi, lo) represents hi + lo. hi is always the plainly rounded running product
// and lo carries the exact rounding errors (TwoProduct by FMA), scaled along:
//   fold:    hi' = fl(hi*x),  lo' = lo*x + (hi*x - hi')        (3 DP ops)
// lo is not renormalised into hi: |lo| grows at most ~n ulp(hi), and its own
// rounding (2^-53 |lo|) stays ~n 2^-106 |hi| -- far below the fp64 result's
// half ulp for any n < 2^40. Zero / inf / NaN products: hi is exact in class
// and sign, and the result is hi alone.
struct DD { double hi, lo; };

struct Float64Prod {
  using T = double;
  using Acc = DD;
  static constexpr bool kFloat = true;
  static constexpr bool kIndexed = false;
  __device__ __forceinline__ static Acc identity() { return DD{1.0, 0.0}; }
  __device__ __forceinline__ static Acc fold(Acc a, T x) {
    const double p = __dmul_rn(a.hi, x);
    const double e = __fma_rn(a.hi, x, -p);   // exact error of a.hi * x
    return DD{p, __fma_rn(a.lo, x, e)};
  }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) {
    const double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __fma_rn(a.hi, b.lo, e);
    e = __fma_rn(a.lo, b.hi, e);
    return DD{p, e};
  }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      DD o{shfl_xor_f64(a.hi, m), shfl_xor_f64(a.lo, m)};
      a = combine(a, o);
    }
    return a;
  }
  __device__ __forceinline__ static double value(Acc a) {
    const bool ok = (a.hi != 0.0) && (fabs(a.hi) < __longlong_as_double(0x7ff0000000000000LL));
    return ok ? __dadd_rn(a.hi, a.lo) : a.hi;
  }
  __device__ __forceinline__ static void store(Acc a, void* out) { *(double*)out = value(a); }
  __device__ __forceinline__ static void store_empty(void* out) { *(double*)out = 1.0; }
  __device__ __forceinline__ static Slot pack(Acc a) {
    return Slot{(uint64_t)__double_as_longlong(a.hi), (uint64_t)__double_as_longlong(a.lo)};
  }
  __device__ __forceinline__ static Acc unpack(Slot s) {
    return DD{__longlong_as_double((long long)s.a), __longlong_as_double((long long)s.b)};
  }
};

// ------------------------------------------------------------- float min / max
// IEEE 754-2019 minimum/maximum, bit-exact and order-independent:
//   key(x)  = the float's bits with the magnitude bits flipped when negative,
//             compared as a signed integer: a total order with -0 < +0;
//   amax    = max over |x| bit patterns: > inf's pattern iff some x is NaN.
// The integer min/max are exactly associative, so every order gives the same
// key; the paper's (a<b)*a + (a>=b)*b select is replaced by a
// native integer min (IMNMX / redux.sync), which is branch-free and IEEE-safe.
template <typename F, rd_op OP>
struct FloatMinMax {
  using T = F;
  // LaneOps folds a loaded vector key-only and marks NaN once per vector
  // (a paired unordered compare) instead of tracking max |x| per element
  static constexpr bool kLazyNan = true;
  using U = typename std::conditional<sizeof(F) == 4, uint32_t, uint64_t>::type;
  using S = typename std::conditional<sizeof(F) == 4, int32_t, int64_t>::type;
  struct Acc { S key; U amax; };
  static constexpr bool kFloat = true;
  static constexpr bool kIndexed = false;
  static constexpr bool kOrderFree = true;   // IEEE minimum/maximum on total-order keys
  static constexpr U kAbsMask = (U)(~(U)0) >> 1;
  static constexpr U kInfBits = sizeof(F) == 4 ? (U)0x7f800000u : (U)0x7ff0000000000000ull;

  __device__ __forceinline__ static U bits(F x) {
    if constexpr (sizeof(F) == 4) return __float_as_uint(x);
    else return (U)__double_as_longlong(x);
  }
  __device__ __forceinline__ static S key_of(U b) { return (S)(b ^ ((U)((S)b >> (8 * sizeof(F) - 1)) & kAbsMask)); }
  __device__ __forceinline__ static Acc identity() {
    // min: key(+inf); max: key(-inf)
    return OP == RD_MIN ? Acc{key_of(kInfBits), 0} : Acc{key_of(kInfBits | ~kAbsMask), 0};
  }
  __device__ __forceinline__ static S kmin(S a, S b) { return OP == RD_MIN ? (a < b ? a : b) : (a > b ? a : b); }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) {
    return Acc{kmin(a.key, b.key), a.amax > b.amax ? a.amax : b.amax};
  }
  __device__ __forceinline__ static Acc fold(Acc a, T x) {
    U b = bits(x);
    U m = b & kAbsMask;
    return Acc{kmin(a.key, key_of(b)), a.amax > m ? a.amax : m};
  }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
    if constexpr (sizeof(F) == 4) {
      a.key = OP == RD_MIN ? __reduce_min_sync(0xffffffffu, (int)a.key) : __reduce_max_sync(0xffffffffu, (int)a.key);
      a.amax = __reduce_max_sync(0xffffffffu, (unsigned)a.amax);
      return a;
    } else {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        Acc o{(S)shfl_xor_u64((uint64_t)a.key, m), (U)shfl_xor_u64((uint64_t)a.amax, m)};
        a = combine(a, o);
      }
      return a;
    }
  }
  __device__ __forceinline__ static void store(Acc a, void* out) {
    U b = (a.amax > kInfBits) ? (kInfBits | ((U)1 << (sizeof(F) == 4 ? 22 : 51)))  // quiet NaN
                              : (U)key_of((U)a.key);                              // key is an involution
    *(U*)out = b;
  }
  __device__ __forceinline__ static void store_empty(void* out) {
    *(U*)out = OP == RD_MIN ? kInfBits : (kInfBits | ~kAbsMask);
  }
  __device__ __forceinline__ static Slot pack(Acc a) { return Slot{(uint64_t)(U)a.key, (uint64_t)a.amax}; }
  __device__ __forceinline__ static Acc unpack(Slot s) { return Acc{(S)(U)s.a, (U)s.b}; }
};

// ------------------------------------------- compensated float + 
// fp32: fp64 accumulator (every fp32 term exact in fp64); fp64: double-double
// with an error-free TwoSum per term (6 DP ops), lo not renormalised (its own
// error stays ~n u^2 sum|x|). The result is the exact sum rounded once in all
// but near-tie cases, hence (in practice) independent of the evaluation order,
// the grid and the number of GPUs (P:50 fn 3: "strategies to reduce truncation
// errors, like the one proposed by Kahan").
struct Float32SumComp {
  using T = float;
  using Acc = double;
  static constexpr bool kFloat = true;
  static constexpr bool kIndexed = false;
  __device__ __forceinline__ static Acc identity() { return -0.0; }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static Acc fold(Acc a, T x) { return __dadd_rn(a, (double)x); }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) a = __dadd_rn(a, shfl_xor_f64(a, m));
    return a;
  }
  __device__ __forceinline__ static void store(Acc a, void* out) { *(float*)out = __double2float_rn(a); }
  __device__ __forceinline__ static void store_empty(void* out) { *(float*)out = 0.0f; }
  __device__ __forceinline__ static Slot pack(Acc a) { return Slot{(uint64_t)__double_as_longlong(a), 0}; }
  __device__ __forceinline__ static Acc unpack(Slot s) { return __longlong_as_double((long long)s.a); }
};

struct Float64SumComp {
  using T = double;
  using Acc = DD;
  static constexpr bool kFloat = true;
  static constexpr bool kIndexed = false;
  __device__ __forceinline__ static Acc identity() { return DD{-0.0, -0.0}; }
  // TwoSum (Knuth): s + e == a + b exactly
  __device__ __forceinline__ static Acc two_sum_into(double hi, double lo, double x) {
    const double s = __dadd_rn(hi, x);
    const double bp = __dsub_rn(s, hi);
    const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bp)), __dsub_rn(x, bp));
    return DD{s, __dadd_rn(lo, e)};
  }
  __device__ __forceinline__ static Acc fold(Acc a, T x) { return two_sum_into(a.hi, a.lo, x); }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) {
    Acc r = two_sum_into(a.hi, a.lo, b.hi);
    r.lo = __dadd_rn(r.lo, b.lo);
    return r;
  }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      DD o{shfl_xor_f64(a.hi, m), shfl_xor_f64(a.lo, m)};
      a = combine(a, o);
    }
    return a;
  }
  __device__ __forceinline__ static double value(Acc a) {
    // non-finite: the plain sum decides (TwoSum's error term is NaN there);
    // lo == 0 keeps the sign of a zero sum (-0.0 iff every term is -0.0)
    if (!(fabs(a.hi) < __longlong_as_double(0x7ff0000000000000LL))) return a.hi;
    return a.lo == 0.0 ? a.hi : __dadd_rn(a.hi, a.lo);
  }
  __device__ __forceinline__ static void store(Acc a, void* out) { *(double*)out = value(a); }
  __device__ __forceinline__ static void store_empty(void* out) { *(double*)out = 0.0; }
  __device__ __forceinline__ static Slot pack(Acc a) {
    return Slot{(uint64_t)__double_as_longlong(a.hi), (uint64_t)__double_as_longlong(a.lo)};
  }
  __device__ __forceinline__ static Acc unpack(Slot s) {
    return DD{__longlong_as_double((long long)s.a), __longlong_as_double((long long)s.b)};
  }
};

// ------------------------------------------------ float32 / float64 + (RD_SUM)
// The north-star bound |result - exact| <= 4 eps sum|x_i| for EVERY input
// (whose partial sums stay finite: e.g. sum|x_i| <= the dtype's max) by
// blocked pairwise summation, at the plain sum's cost per element:
//   * the K <= 32 elements a thread has loaded in one iteration (U vectors in
//     the vector kernel, one ring stage's slice in the bulk kernel) are summed
//     as a balanced binary tree in the INPUT precision (depth t <= 5):
//     |tree - sum| <= t u sum|x| (u = eps/2 = 2^-24 / 2^-53);
//   * the block sum enters a WIDE accumulator exactly or nearly so: fp32 data
//     -> fp64 (exact widening + one DADD), fp64 data -> double-double (TwoSum);
//     every later combine (lanes, warp, CTA, chunk slots, records) stays wide,
//     so chains of any length d add only d u_w sum|x| (u_w = 2^-53 / ~2^-106);
//   * one rounding to the dtype at the end: <= u |S|.
// Total <= (t + 1) u sum|x| + d u_w sum|x| < 3.01 eps sum|x|: t <= 5, and the
// wide chains of these kernels are d < 2^21 deep for any n < 2^40 (DESIGN.md
// R6) -- whatever the values, so no input can push a long input-precision
// chain past the bound (per-lane fp32 chains missed it by 7x at 2^28 on an
// input that places 1.0 at the head of every chain).
// P:50 fn 3: "double precision floating points" as the mitigation, applied
// to the block sums instead of to every element.
template <typename F>
struct FloatSum;

template <>
struct FloatSum<float> : Float32SumComp {
  static constexpr bool kBlocked = true;
  __device__ __forceinline__ static Acc add_block(Acc a, float s) { return __dadd_rn(a, (double)s); }
};

template <>
struct FloatSum<double> : Float64SumComp {
  static constexpr bool kBlocked = true;
  __device__ __forceinline__ static Acc add_block(Acc a, double s) { return two_sum_into(a.hi, a.lo, s); }
};

// Ops whose result is the same for EVERY evaluation order (not only the same
// bits for a fixed order): integers, float min/max, argmin/argmax. The bulk
// kernel folds their chunks into one running partial per CTA instead of one
// fixed-tree partial per chunk (rd_bulk.cuh).
template <class O, class = void> struct OrderFree : std::false_type {};
template <class O> struct OrderFree<O, std::void_t<decltype(O::kOrderFree)>> : std::bool_constant<O::kOrderFree> {};

// 32-bit integer + (int32 / uint32 sum and their compensated / exact aliases):
// the grid combine adds every CTA's partial and counts the CTA in ONE 64-bit
// atomic add on {partial << 32 | 1} (rd_kernels.cuh packed_arrive) -- the sum
// wraps mod 2^32 in the high word (carries leave the 64 bits), the count in
// the low word never carries -- so the last CTA has the total from its
// atomic's return value: no slots to fold.
template <class O> struct PackedSum32 : std::false_type {};
template <bool S> struct PackedSum32<IntOp<uint32_t, RD_SUM, S>> : std::true_type {};

template <class O, class = void> struct Blocked : std::false_type {};
template <class O> struct Blocked<O, std::void_t<decltype(O::kBlocked)>> : std::bool_constant<O::kBlocked> {};

// the largest block summed as one tree (depth <= 5)
constexpr int kMaxTreeBlock = 32;

// balanced binary tree over v[0..N) in the element precision: depth ceil(log2 N)
template <int N, typename T>
__device__ __forceinline__ T tree_sum(const T* v) {
  if constexpr (N == 1) return v[0];
  else {
    constexpr int H = N / 2;
    return tree_sum<N - H>(v) + tree_sum<H>(v + (N - H));
  }
}

// acc <- acc (+) tree(v[C..C+32)) (+) tree(v[C+32..)) ... for a blocked sum
template <class OpT, int N, int C = 0, typename T>
__device__ __forceinline__ void add_blocks(typename OpT::Acc& acc, const T* v) {
  if constexpr (C < N) {
    constexpr int M = (N - C < kMaxTreeBlock) ? N - C : kMaxTreeBlock;
    acc = OpT::add_block(acc, tree_sum<M>(v + C));
    add_blocks<OpT, N, C + M>(acc, v);
  }
}

// ------------------------------------------------- argmin / argmax
// Value and the SMALLEST index attaining it (reading R6). Every element maps
// to an unsigned order key K (ints: sign-flipped bits; floats: the total-order
// key of FloatMinMax, with any NaN mapped to the winning end), and (K, index)
// is compared lexicographically -- exactly associative and commutative, so
// any evaluation order gives the same (value, index).
template <typename U, rd_dtype DT, rd_op OP>
struct ArgOp {
  using T = U;
  static constexpr bool kMin = (OP == RD_ARGMIN);
  struct Acc { U key; uint64_t idx; };
  static constexpr bool kFloat = (DT == RD_FLOAT32 || DT == RD_FLOAT64);
  static constexpr bool kIndexed = true;
  static constexpr bool kOrderFree = true;   // lexicographic (key, index): any order, same result
  static constexpr int kBits = 8 * sizeof(U);
  static constexpr U kSign = (U)1 << (kBits - 1);
  static constexpr U kAbs = kSign - 1;
  static constexpr U kInf = sizeof(U) == 4 ? (U)0x7f800000u : (U)0x7ff0000000000000ull;

  __device__ __forceinline__ static U key_of(U b) {
    if constexpr (DT == RD_UINT32) return b;
    else if constexpr (!kFloat) return b ^ kSign;
    else {
      // unsigned total-order key in two ops: negative -> ~b, positive -> b ^ sign
      const U sgn = (U)((typename std::make_signed<U>::type)b >> (kBits - 1));
      const U k = b ^ (sgn | kSign);
      // any NaN wins (maps to the winning end); one unordered float compare
      bool nan;
      if constexpr (sizeof(U) == 4) { const float f = __uint_as_float((uint32_t)b); nan = (f != f); }
      else { const double f = __longlong_as_double((long long)b); nan = (f != f); }
      return nan ? (OP == RD_ARGMIN ? (U)0 : (U)~(U)0) : k;
    }
  }
  // the order key without the NaN mapping (exact for every non-NaN element)
  __device__ __forceinline__ static U raw_key(U b) {
    if constexpr (DT == RD_UINT32) return b;
    else if constexpr (!kFloat) return b ^ kSign;
    else {
      const U sgn = (U)((typename std::make_signed<U>::type)b >> (kBits - 1));
      return b ^ (sgn | kSign);
    }
  }
  __device__ __forceinline__ static U bits_of(U k) {   // inverse of key_of (non-NaN)
    if constexpr (DT == RD_UINT32) return k;
    else if constexpr (!kFloat) return k ^ kSign;
    else {
      if (k == (OP == RD_ARGMIN ? (U)0 : (U)~(U)0)) return kInf | ((U)1 << (sizeof(U) == 4 ? 22 : 51));
      const U skey = k ^ kSign;
      return skey ^ ((U)((typename std::make_signed<U>::type)skey >> (kBits - 1)) & kAbs);
    }
  }
  __device__ __forceinline__ static Acc identity() {
    return OP == RD_ARGMIN ? Acc{(U)~(U)0, ~0ull} : Acc{(U)0, ~0ull};
  }
  __device__ __forceinline__ static bool better(const Acc& a, const Acc& b) {   // a strictly before b
    if (a.key != b.key) return OP == RD_ARGMIN ? a.key < b.key : a.key > b.key;
    return a.idx < b.idx;
  }
  __device__ __forceinline__ static Acc combine(Acc a, Acc b) { return better(b, a) ? b : a; }
  __device__ __forceinline__ static Acc fold_idx(Acc a, T x, uint64_t i) { return combine(a, Acc{key_of(x), i}); }
  __device__ __forceinline__ static Acc fold(Acc a, T x) { return fold_idx(a, x, 0); }
  __device__ __forceinline__ static Acc warp_reduce(Acc a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      Acc o;
      if constexpr (sizeof(U) == 4) o.key = __shfl_xor_sync(0xffffffffu, a.key, m);
      else o.key = (U)shfl_xor_u64((uint64_t)a.key, m);
      o.idx = shfl_xor_u64(a.idx, m);
      a = combine(a, o);
    }
    return a;
  }
  // out -> rd_arg_result {value bits (low sizeof(T) bytes), int64 index}
  __device__ __forceinline__ static void store(Acc a, void* out) {
    uint64_t* r = (uint64_t*)out;
    r[0] = (uint64_t)bits_of(a.key);
    r[1] = a.idx;
  }
  __device__ __forceinline__ static void store_empty(void* out) {
    uint64_t* r = (uint64_t*)out;
    U v;
    if constexpr (kFloat) v = OP == RD_ARGMIN ? kInf : (kInf | kSign);
    else if constexpr (DT == RD_UINT32) v = OP == RD_ARGMIN ? (U)~(U)0 : (U)0;
    else v = OP == RD_ARGMIN ? kAbs : kSign;
    r[0] = (uint64_t)v;
    r[1] = ~0ull;   // index -1
  }
  __device__ __forceinline__ static Slot pack(Acc a) { return Slot{(uint64_t)a.key, a.idx}; }
  __device__ __forceinline__ static Acc unpack(Slot s) { return Acc{(U)s.a, s.b}; }
};

// fold with the element's global index (indexed ops), else plain fold
template <class OpT>
__device__ __forceinline__ typename OpT::Acc fold_at(typename OpT::Acc a, typename OpT::T x, uint64_t i) {
  if constexpr (OpT::kIndexed) return OpT::fold_idx(a, x, i);
  else return OpT::fold(a, x);
}
// partial of a later block: indices shift by the elements before it
template <class OpT>
__device__ __forceinline__ typename OpT::Acc shifted(typename OpT::Acc a, uint64_t off) {
  if constexpr (OpT::kIndexed) {
    if (a.idx != ~0ull) a.idx += off;
  }
  return a;
}

#define OP_IS_MIN(OpT) (OpT::kMin)

// any NaN among L lanes, two lanes per unordered compare (setp.nan[.or])
template <int L, typename T>
__device__ __forceinline__ bool any_nan(const T (&x)[L]) {
  uint32_t r = 0;
  if constexpr (sizeof(T) == 4 && L == 4) {
    asm("{ .reg .pred p; setp.nan.f32 p, %1, %2; setp.nan.or.f32 p, %3, %4, p; selp.u32 %0, 1, 0, p; }"
        : "=r"(r) : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]));
  } else if constexpr (sizeof(T) == 4 && L == 8) {
    asm("{ .reg .pred p; setp.nan.f32 p, %1, %2; setp.nan.or.f32 p, %3, %4, p; "
        "setp.nan.or.f32 p, %5, %6, p; setp.nan.or.f32 p, %7, %8, p; selp.u32 %0, 1, 0, p; }"
        : "=r"(r) : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]));
  } else if constexpr (sizeof(T) == 8 && L == 2) {
    asm("{ .reg .pred p; setp.nan.f64 p, %1, %2; selp.u32 %0, 1, 0, p; }" : "=r"(r) : "l"(x[0]), "l"(x[1]));
  } else if constexpr (sizeof(T) == 8 && L == 4) {
    asm("{ .reg .pred p; setp.nan.f64 p, %1, %2; setp.nan.or.f64 p, %3, %4, p; selp.u32 %0, 1, 0, p; }"
        : "=r"(r) : "l"(x[0]), "l"(x[1]), "l"(x[2]), "l"(x[3]));
  } else {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      typename std::conditional<sizeof(T) == 4, float, double>::type f;
      memcpy(&f, &x[l], sizeof(T));
      r |= (f != f);
    }
  }
  return r != 0;
}


// ---------------------------------------------------------- lane accumulators
// What the hot loops keep per thread. fold_vec folds one loaded vector (L
// lanes, consecutive elements); finish combines the lanes into one Acc.
// Plain ops keep one accumulator per lane (L independent dependency chains).
// Indexed ops (argmin / argmax) keep per lane the best order key and the STEP
// at which it was seen: along one lane the element index grows with the step,
// so a strict comparison keeps the earliest of equal keys, and the 64-bit
// index is formed once, in finish().
template <class O, class = void> struct LazyNan : std::false_type {};
template <class O> struct LazyNan<O, std::void_t<decltype(O::kLazyNan)>> : std::bool_constant<O::kLazyNan> {};

template <class OpT, bool IDX = OpT::kIndexed>
struct LaneOps {
  using T = typename OpT::T;
  using Lane = typename OpT::Acc;
  __device__ __forceinline__ static Lane identity() { return OpT::identity(); }
  template <int L>
  __device__ __forceinline__ static void fold_vec(Lane (&acc)[L], const T (&x)[L], uint32_t) {
    if constexpr (LazyNan<OpT>::value) {
      // float min / max: the order key per element; NaN is detected per
      // vector (setp.nan on pairs) and recorded as amax = all ones (> the
      // inf pattern), the same state OpT::fold leaves -- 2/3 of the integer
      // work per element, which matters when the ALU and the power cap, not
      // HBM, bound a sustained run (float64 max: 85.7% of the read probe)
      using U = typename OpT::U;
      U b[L];
#pragma unroll
      for (int l = 0; l < L; ++l) b[l] = OpT::bits(x[l]);
#pragma unroll
      for (int l = 0; l < L; ++l) acc[l].key = OpT::kmin(acc[l].key, OpT::key_of(b[l]));
      if (__builtin_expect(any_nan<L>(b), 0)) {
#pragma unroll
        for (int l = 0; l < L; ++l) acc[l].amax = (U)~(U)0;
      }
    } else {
#pragma unroll
      for (int l = 0; l < L; ++l) acc[l] = OpT::fold(acc[l], x[l]);
    }
  }
  // the K vectors one thread loaded in one iteration (vector k's elements
  // come at step step0 + k). Blocked sums (FloatSum): one input-precision
  // tree per <= 32 elements into the wide lane accumulator 0.
  template <int K, int L>
  __device__ __forceinline__ static void fold_vecs(Lane (&acc)[L], const T (&x)[K][L], uint32_t step0) {
    if constexpr (Blocked<OpT>::value) {
      add_blocks<OpT, K * L>(acc[0], &x[0][0]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) fold_vec(acc, x[k], step0 + k);
    }
  }
  template <int L, class F>
  __device__ __forceinline__ static typename OpT::Acc finish(const Lane (&acc)[L], F) {
    typename OpT::Acc a = acc[0];
#pragma unroll
    for (int l = 1; l < L; ++l) a = OpT::combine(a, acc[l]);
    return a;
  }
};

template <class OpT>
struct LaneOps<OpT, true> {
  using T = typename OpT::T;
  struct Lane { T key; uint32_t step; };
  static constexpr uint32_t kEmpty = 0xffffffffu;
  __device__ __forceinline__ static Lane identity() { return Lane{OpT::identity().key, kEmpty}; }
#ifdef RD_ARG_PER_LANE
  // (A/B builds only) one (key, step) per lane: L independent select chains
  template <int L>
  __device__ __forceinline__ static void fold_vec(Lane (&acc)[L], const T (&x)[L], uint32_t step) {
    const bool nan = OpT::kFloat && any_nan<L>(x);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const T k = nan ? OpT::key_of(x[l]) : OpT::raw_key(x[l]);
      bool better = OP_IS_MIN(OpT) ? (k < acc[l].key) : (k > acc[l].key);
      if constexpr (!OpT::kFloat) better = better || (acc[l].step == kEmpty);
      acc[l] = better ? Lane{k, step} : acc[l];
    }
  }
  template <int K, int L>
  __device__ __forceinline__ static void fold_vecs(Lane (&acc)[L], const T (&x)[K][L], uint32_t step0) {
#pragma unroll
    for (int k = 0; k < K; ++k) fold_vec(acc, x[k], step0 + k);
  }
  template <int L, class Fn>
  __device__ __forceinline__ static typename OpT::Acc finish(const Lane (&acc)[L], Fn index_of) {
    typename OpT::Acc a = OpT::identity();
#pragma unroll
    for (int l = 0; l < L; ++l)
      if (acc[l].step != kEmpty) a = OpT::combine(a, typename OpT::Acc{acc[l].key, index_of(acc[l].step, (uint32_t)l)});
    return a;
  }
#else
  // Group-best: ONE (key, position) per thread, in acc[0]. A group of G
  // vectors (G*L <= 8 keys) is reduced to its best key by a min/max tree
  // (IMNMX / VIMNMX3: no select chains), then compared once with the
  // thread's best; only an improvement -- rare after the first groups, about
  // ln(groups) times per thread -- takes the (divergent) branch that finds the
  // group's FIRST position holding that key and records step * L + lane. A
  // strict comparison keeps the earliest of equal keys across groups, the
  // first position within one: the lowest index, as the per-lane form did, at
  // ~3 integer ops per element instead of ~5 (sustained float32 argmax was
  // 88.8% of the read probe, the lowest of all (dtype, op)).
  template <int N>
  __device__ __forceinline__ static T best_of(const T* k) {
    if constexpr (N == 1) return k[0];
    else {
      const T a = best_of<N - N / 2>(k), b = best_of<N / 2>(k + (N - N / 2));
      return OP_IS_MIN(OpT) ? (a < b ? a : b) : (a > b ? a : b);
    }
  }
  using F = typename std::conditional<sizeof(T) == 4, float, double>::type;
  __device__ __forceinline__ static F as_float(T b) {
    if constexpr (sizeof(T) == 4) return __uint_as_float((uint32_t)b);
    else return __longlong_as_double((long long)b);
  }
  template <int N>
  __device__ __forceinline__ static F fbest_of(const T* x) {    // FMNMX / FMNMX3, DSETP.MAX
    if constexpr (N == 1) return as_float(x[0]);
    else {
      const F a = fbest_of<N - N / 2>(x), b = fbest_of<N / 2>(x + (N - N / 2));
      return OP_IS_MIN(OpT) ? fmin(a, b) : fmax(a, b);
    }
  }
  template <int G, int L>
  __device__ __forceinline__ static void fold_group(Lane& best, const T* x, uint32_t step0) {
    constexpr int N = G * L;
    bool nan = false;
    if constexpr (OpT::kFloat) {
#pragma unroll
      for (int g = 0; g < G; ++g) nan |= any_nan<L>(*reinterpret_cast<const T(*)[L]>(x + g * L));
      // floats: the group's best by the float min/max instructions (1 op per
      // element, no key transform); fmin/fmax return one of the operands, so
      // its bits are an element's -- unless the best is a zero (-0 vs +0 are
      // not ordered by fmin/fmax) or a NaN is present: then the key path below
      const F m = fbest_of<N>(x);
      if (__builtin_expect(!nan && m != (F)0, 1)) {
        T mb;
        if constexpr (sizeof(T) == 4) mb = (T)__float_as_uint(m);
        else mb = (T)__double_as_longlong(m);
        const T vb = OpT::raw_key(mb);
        if (__builtin_expect(OP_IS_MIN(OpT) ? (vb < best.key) : (vb > best.key), 0)) {
          uint32_t j0 = N - 1;
#pragma unroll
          for (int j = N - 1; j >= 0; --j) j0 = (x[j] == mb) ? (uint32_t)j : j0;
          best.key = vb;
          best.step = step0 * L + j0;
        }
        return;
      }
    }
    T k[N];
    if (__builtin_expect(!nan, 1)) {
#pragma unroll
      for (int j = 0; j < N; ++j) k[j] = OpT::raw_key(x[j]);
    } else {                                            // NaN maps to the winning end
#pragma unroll
      for (int j = 0; j < N; ++j) k[j] = OpT::key_of(x[j]);
    }
    const T vb = best_of<N>(k);
    bool upd = OP_IS_MIN(OpT) ? (vb < best.key) : (vb > best.key);
    // integer keys can equal the identity key: an empty thread takes its first group
    if constexpr (!OpT::kFloat) upd = upd || (best.step == kEmpty);
    if (__builtin_expect(upd, 0)) {
      uint32_t j0 = N - 1;
#pragma unroll
      for (int j = N - 1; j >= 0; --j) j0 = (k[j] == vb) ? (uint32_t)j : j0;
      best.key = vb;
      best.step = step0 * L + j0;                       // = (step0 + j0 / L) * L + j0 % L
    }
  }
  template <int L>
  __device__ __forceinline__ static void fold_vec(Lane (&acc)[L], const T (&x)[L], uint32_t step) {
    fold_group<1, L>(acc[0], x, step);
  }
  template <int K, int L>
  __device__ __forceinline__ static void fold_vecs(Lane (&acc)[L], const T (&x)[K][L], uint32_t step0) {
    constexpr int G0 = (L >= 8) ? 1 : 8 / L;
    constexpr int G = (K % G0 == 0) ? G0 : 1;
#pragma unroll
    for (int k = 0; k < K; k += G) fold_group<G, L>(acc[0], &x[k][0], step0 + k);
  }
  template <int L, class Fn>
  __device__ __forceinline__ static typename OpT::Acc finish(const Lane (&acc)[L], Fn index_of) {
    typename OpT::Acc a = OpT::identity();
    if (acc[0].step != kEmpty)
      a = typename OpT::Acc{acc[0].key, index_of(acc[0].step / L, acc[0].step % L)};
    return a;
  }
#endif
};

// ---------------------------------------------------------------- type map
template <rd_dtype DT, rd_op OP> struct OpFor;
#define RD_INT_OPS(DT, U, SIGNED)                                                  \
  template <> struct OpFor<DT, RD_SUM> { using type = IntOp<U, RD_SUM, SIGNED>; }; \
  template <> struct OpFor<DT, RD_PROD> { using type = IntOp<U, RD_PROD, SIGNED>; }; \
  template <> struct OpFor<DT, RD_MIN> { using type = IntOp<U, RD_MIN, SIGNED>; }; \
  template <> struct OpFor<DT, RD_MAX> { using type = IntOp<U, RD_MAX, SIGNED>; }; \
  template <> struct OpFor<DT, RD_AND> { using type = IntOp<U, RD_AND, SIGNED>; }; \
  template <> struct OpFor<DT, RD_OR> { using type = IntOp<U, RD_OR, SIGNED>; };   \
  template <> struct OpFor<DT, RD_XOR> { using type = IntOp<U, RD_XOR, SIGNED>; };
RD_INT_OPS(RD_INT32, uint32_t, true)
RD_INT_OPS(RD_UINT32, uint32_t, false)
RD_INT_OPS(RD_INT64, uint64_t, true)
#undef RD_INT_OPS
#define RD_ARG_OPS(DT, U)                                                              \
  template <> struct OpFor<DT, RD_ARGMIN> { using type = ArgOp<U, DT, RD_ARGMIN>; }; \
  template <> struct OpFor<DT, RD_ARGMAX> { using type = ArgOp<U, DT, RD_ARGMAX>; };
RD_ARG_OPS(RD_INT32, uint32_t)
RD_ARG_OPS(RD_UINT32, uint32_t)
RD_ARG_OPS(RD_INT64, uint64_t)
RD_ARG_OPS(RD_FLOAT32, uint32_t)
RD_ARG_OPS(RD_FLOAT64, uint64_t)
#undef RD_ARG_OPS
// compensated sum: exact already for integers
template <> struct OpFor<RD_INT32, RD_SUM_COMPENSATED> { using type = IntOp<uint32_t, RD_SUM, true>; };
template <> struct OpFor<RD_UINT32, RD_SUM_COMPENSATED> { using type = IntOp<uint32_t, RD_SUM, false>; };
template <> struct OpFor<RD_INT64, RD_SUM_COMPENSATED> { using type = IntOp<uint64_t, RD_SUM, true>; };
// exact sum (rd_exact.cuh for floats): integer sums are exact already
template <> struct OpFor<RD_INT32, RD_SUM_EXACT> { using type = IntOp<uint32_t, RD_SUM, true>; };
template <> struct OpFor<RD_UINT32, RD_SUM_EXACT> { using type = IntOp<uint32_t, RD_SUM, false>; };
template <> struct OpFor<RD_INT64, RD_SUM_EXACT> { using type = IntOp<uint64_t, RD_SUM, true>; };
template <> struct OpFor<RD_FLOAT32, RD_SUM_COMPENSATED> { using type = Float32SumComp; };
template <> struct OpFor<RD_FLOAT64, RD_SUM_COMPENSATED> { using type = Float64SumComp; };
template <> struct OpFor<RD_FLOAT32, RD_SUM> { using type = FloatSum<float>; };
template <> struct OpFor<RD_FLOAT64, RD_SUM> { using type = FloatSum<double>; };
template <> struct OpFor<RD_FLOAT32, RD_PROD> { using type = Float32Prod; };
template <> struct OpFor<RD_FLOAT64, RD_PROD> { using type = Float64Prod; };
template <> struct OpFor<RD_FLOAT32, RD_MIN> { using type = FloatMinMax<float, RD_MIN>; };
template <> struct OpFor<RD_FLOAT32, RD_MAX> { using type = FloatMinMax<float, RD_MAX>; };
template <> struct OpFor<RD_FLOAT64, RD_MIN> { using type = FloatMinMax<double, RD_MIN>; };
template <> struct OpFor<RD_FLOAT64, RD_MAX> { using type = FloatMinMax<double, RD_MAX>; };

__host__ __device__ __forceinline__ constexpr uint32_t record_tag(int dtype, int op) {
  return 0x52440000u | ((uint32_t)dtype << 8) | (uint32_t)op;
}

}  // namespace rd
