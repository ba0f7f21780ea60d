/*
 * inputs/gen.h -- seeded, counter-based synthetic input generator.
 *
 * This module is shared by BOTH sides of the parity check (the CUDA path's
 * tests/bench and the CPU oracle's tests).  It holds NONE of the reduction's
 * arithmetic: it only maps (seed, workload, global index i) to the value x_i
 * of a synthetic input vector X = {x_0 .. x_{n-1}} (§1.1).
 * The same header is compiled by gcc (host twin, gen_host.c) and by nvcc
 * (device twin, gen_device.cu), so host and device outputs are bit-identical
 * by construction: only integer ops and exact int->float conversions are used
 * (the one rounding conversion, `normalish`, is a single IEEE round-to-nearest
 * int->float conversion on both sides).
 *
 * Workload recipe: DESIGN.md "Input recipe"; SURVEY.md §8(d) table.
 */
#ifndef B200_INPUTS_GEN_H
#define B200_INPUTS_GEN_H

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

/* dtype codes (same numbering as the public ABI, restated here so this
 * module depends on neither the oracle nor the CUDA library). */
enum { GEN_INT32 = 0, GEN_UINT32 = 1, GEN_INT64 = 2, GEN_FLOAT32 = 3, GEN_FLOAT64 = 4 };

/* workload codes */
enum {
  GEN_IOTA = 0,            /* x_i = i                                         */
  GEN_UNIFORM_BITS = 1,    /* ints: raw hash bits; floats: same as u01         */
  GEN_ODD = 2,             /* ints: hash | 1 (products stay odd mod 2^w)       */
  GEN_SPARSE_CLEAR = 3,    /* ints: all ones, one bit cleared w.p. 2^-12       */
  GEN_SPARSE_SET = 4,      /* ints: zero, one bit set w.p. 2^-12               */
  GEN_U01 = 5,             /* floats: uniform [0,1) on a 2^-24 / 2^-53 grid    */
  GEN_NORMALISH = 6,       /* floats: Irwin-Hall(4) centred, sd ~ 0.577        */
  GEN_NEAR_ONE = 7,        /* floats: 1 + k*eps, k in [-64, 64]                */
  GEN_POW2_SPARSE = 8,     /* floats: 1.0, ~100 hashed positions hold 2 or 0.5 */
  GEN_PLANTED = 9,         /* one planted max and one planted min              */
  GEN_INT_SMALL = 10,      /* integers in [-65536, 65536] (exact in fp64 sums) */
  GEN_SPARSE_PM1 = 11,     /* 0, or +-1 at <= ~2^20 hashed positions           */
  GEN_WIDE = 12,           /* floats: random sign, mantissa, exponent in [-40, 40] */
  GEN_WIDE_FULL = 13,      /* floats: random sign, mantissa, ANY finite exponent
                              field (subnormals through the largest binade)    */
  GEN_NUM_WORKLOADS = 14
};

#define GEN_GOLDEN 0x9E3779B97F4A7C15ULL

/* splitmix64 finaliser (Steele, Lea, Flood 2014). */
GEN_HD uint64_t gen_mix(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

/* per-(seed, workload, draw) stream key */
GEN_HD uint64_t gen_key(uint64_t seed, int workload, int draw) {
  return gen_mix(seed * GEN_GOLDEN + (uint64_t)workload * 0xD1B54A32D192ED03ULL +
                 (uint64_t)draw * 0x632BE59BD9B4E019ULL + 1ULL);
}

/* counter-based hash of global index i */
GEN_HD uint64_t gen_h(uint64_t key, uint64_t i) { return gen_mix(key + (i + 1ULL) * GEN_GOLDEN); }

/* threshold on (h >> 32) so that about `expect` of n_total positions are hit */
GEN_HD uint64_t gen_threshold(uint64_t expect, uint64_t n_total) {
  if (n_total <= expect) return 1ULL << 32;
  return (expect << 32) / n_total;
}

/* The two planted positions of GEN_PLANTED: p_max (holds the maximum) and
 * p_min (holds the minimum); distinct whenever n_total >= 2. */
GEN_HD void gen_planted_positions(uint64_t seed, uint64_t n_total, uint64_t* p_max, uint64_t* p_min) {
  uint64_t k = gen_key(seed, GEN_PLANTED, 7);
  if (n_total == 0) { *p_max = *p_min = 0; return; }
  *p_max = gen_h(k, 0) % n_total;
  if (n_total == 1) { *p_min = *p_max; return; }
  *p_min = (*p_max + 1ULL + gen_h(k, 1) % (n_total - 1ULL)) % n_total;
}

GEN_HD float gen_bits_to_f32(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
GEN_HD double gen_bits_to_f64(uint64_t b) { double f; memcpy(&f, &b, 8); return f; }

/* 2^e for small |e| as exact constants built from bits (no libm). */
GEN_HD float gen_pow2f(int e) { return gen_bits_to_f32((uint32_t)(127 + e) << 23); }
GEN_HD double gen_pow2d(int e) { return gen_bits_to_f64((uint64_t)(1023 + e) << 52); }

/*
 * Element i (global index) of workload `wl` for dtype `dt`, written as the
 * raw little-endian bits in *out (4 or 8 bytes). Returns 0, or -1 when the
 * workload is not defined for the dtype.
 */
GEN_HD int gen_element(int dt, int wl, uint64_t seed, uint64_t i, uint64_t n_total, void* out) {
  const int is_float = (dt == GEN_FLOAT32 || dt == GEN_FLOAT64);
  const int w = (dt == GEN_INT64 || dt == GEN_FLOAT64) ? 64 : 32;
  const uint64_t h = gen_h(gen_key(seed, wl, 0), i);
  uint64_t ib = 0;     /* integer result bits */
  double fd = 0.0;     /* float result (fp64 path) */
  float ff = 0.0f;     /* float result (fp32 path) */
  switch (wl) {
    case GEN_IOTA:
      if (is_float) { fd = (double)i; ff = (float)i; } else ib = i;
      break;
    case GEN_UNIFORM_BITS:
      if (is_float) { ff = (float)(h >> 40) * gen_pow2f(-24); fd = (double)(h >> 11) * gen_pow2d(-53); }
      else ib = h;
      break;
    case GEN_ODD:
      if (is_float) return -1;
      ib = h | 1ULL;
      break;
    case GEN_SPARSE_CLEAR:
      if (is_float) return -1;
      ib = ~0ULL;
      if ((h >> 52) == 0) ib &= ~(1ULL << (h & (uint64_t)(w - 1)));
      break;
    case GEN_SPARSE_SET:
      if (is_float) return -1;
      ib = 0;
      if ((h >> 52) == 0) ib |= (1ULL << (h & (uint64_t)(w - 1)));
      break;
    case GEN_U01:
      if (!is_float) return -1;
      ff = (float)(h >> 40) * gen_pow2f(-24);
      fd = (double)(h >> 11) * gen_pow2d(-53);
      break;
    case GEN_NORMALISH: {
      if (!is_float) return -1;
      uint64_t s24 = 0, s53 = 0;
      for (int j = 0; j < 4; ++j) {
        uint64_t hj = gen_h(gen_key(seed, wl, j), i);
        s24 += hj >> 40;
        s53 += hj >> 11;
      }
      ff = (float)((int64_t)s24 - (int64_t)(1ULL << 25)) * gen_pow2f(-24);
      fd = (double)((int64_t)s53 - (int64_t)(1ULL << 54)) * gen_pow2d(-53);
      break;
    }
    case GEN_NEAR_ONE: {
      if (!is_float) return -1;
      int k = (int)((h >> 32) % 129ULL) - 64;
      ff = 1.0f + (float)k * gen_pow2f(-23);
      fd = 1.0 + (double)k * gen_pow2d(-52);
      break;
    }
    case GEN_POW2_SPARSE:
      if (!is_float) return -1;
      ff = 1.0f; fd = 1.0;
      if ((h >> 32) < gen_threshold(100, n_total)) {
        ff = (h & 1ULL) ? 2.0f : 0.5f;
        fd = (h & 1ULL) ? 2.0 : 0.5;
      }
      break;
    case GEN_PLANTED: {
      uint64_t pmax, pmin;
      gen_planted_positions(seed, n_total, &pmax, &pmin);
      if (is_float) {
        ff = 1.0f + (float)(h >> 40) * gen_pow2f(-24);
        fd = 1.0 + (double)(h >> 11) * gen_pow2d(-53);
        if (i == pmax) { ff = gen_pow2f(20); fd = gen_pow2d(20); }
        if (i == pmin) { ff = -gen_pow2f(20); fd = -gen_pow2d(20); }
      } else {
        ib = (h % (1ULL << 21)) + 16ULL;
        if (i == pmax) ib = 1ULL << 30;
        if (i == pmin) ib = 3ULL;
      }
      break;
    }
    case GEN_INT_SMALL: {
      int64_t v = (int64_t)(h % 131073ULL) - 65536;
      ff = (float)v; fd = (double)v; ib = (uint64_t)v;
      break;
    }
    case GEN_SPARSE_PM1: {
      int64_t v = 0;
      if ((h >> 32) < gen_threshold(1ULL << 20, n_total)) v = (h & 1ULL) ? 1 : -1;
      ff = (float)v; fd = (double)v; ib = (uint64_t)v;
      break;
    }
    case GEN_WIDE:
    case GEN_WIDE_FULL: {
      /* built from bits: sign = bit 63, mantissa = low bits, exponent field
       * from bits 32.. (wide: 2^-40 .. 2^40; full: 0 .. max finite field) */
      if (!is_float) return -1;
      const uint64_t sg = h >> 63;
      const uint64_t e32 = (wl == GEN_WIDE) ? 127 - 40 + ((h >> 32) % 81ULL) : (h >> 32) % 255ULL;
      const uint64_t e64 = (wl == GEN_WIDE) ? 1023 - 40 + ((h >> 32) % 81ULL) : (h >> 32) % 2047ULL;
      ff = gen_bits_to_f32((uint32_t)((sg << 31) | (e32 << 23) | (h & 0x7FFFFFULL)));
      fd = gen_bits_to_f64((sg << 63) | (e64 << 52) | ((h * GEN_GOLDEN) & 0xFFFFFFFFFFFFFULL));
      break;
    }
    default:
      return -1;
  }
  switch (dt) {
    case GEN_INT32: case GEN_UINT32: { uint32_t v = (uint32_t)ib; memcpy(out, &v, 4); break; }
    case GEN_INT64: memcpy(out, &ib, 8); break;
    case GEN_FLOAT32: memcpy(out, &ff, 4); break;
    case GEN_FLOAT64: memcpy(out, &fd, 8); break;
    default: return -1;
  }
  return 0;
}

GEN_HD int gen_dtype_size(int dt) {
  return (dt == GEN_INT64 || dt == GEN_FLOAT64) ? 8 : ((dt >= 0 && dt <= 4) ? 4 : 0);
}

#endif /* B200_INPUTS_GEN_H */
