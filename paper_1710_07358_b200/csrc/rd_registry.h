// rd_registry.h -- compiled kernel configurations, looked up by the planner.
#pragma once
#include "rd_kernels.cuh"

namespace rd {

using ReduceFn = void (*)(const KArgs);
using CombineFn = void (*)(const rd_record*, int, uint32_t, void*, rd_record*, int*);

struct KernelRef {
  ReduceFn fn;
  int block, unroll, vec_bytes, variant;
};

constexpr int kBlock = 256;          // threads per CTA for every reduce kernel
constexpr int kMaxGrid = 4096;       // workspace slots
// Default configuration per element size (chosen by the U x V sweep).
constexpr int kDefaultUnroll4 = 4;   // 4-byte elements
constexpr int kDefaultUnroll8 = 4;   // 8-byte elements
constexpr int kDefaultVec = 32;      // LDG.256

// Translation units rd_inst_*.cu each define one of these.
bool lookup_int(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
bool lookup_float(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
bool lookup_ablation(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
CombineFn lookup_combine(int dtype, int op);

// Helpers used by the instantiation units.
template <class OpT>
inline bool lookup_default(int variant, int unroll, int vec_bytes, KernelRef* r) {
  using T = typename OpT::T;
  constexpr int du = sizeof(T) == 4 ? kDefaultUnroll4 : kDefaultUnroll8;
  if (variant != RD_VARIANT_AUTO && variant != RD_VARIANT_VECTOR) return false;
  const int u = unroll ? unroll : du;
  const int vb = vec_bytes ? vec_bytes : kDefaultVec;
  if (u == du && vb == kDefaultVec) {
    *r = KernelRef{rd_vector_kernel<OpT, kBlock, du, kDefaultVec>, kBlock, du, kDefaultVec, RD_VARIANT_VECTOR};
    return true;
  }
  return false;
}

}  // namespace rd
