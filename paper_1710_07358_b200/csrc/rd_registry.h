// rd_registry.h -- compiled kernel configurations, looked up by the planner.
#pragma once
#include "rd_bulk.cuh"
#include "rd_kernels.cuh"

namespace rd {

using ReduceFn = void (*)(const KArgs);
using CombineFn = void (*)(const rd_record*, int, uint32_t, void*, rd_record*, int*);

struct KernelRef {
  ReduceFn fn;
  int block, unroll, vec_bytes, variant;
  int smem_bytes = 0;   // dynamic shared memory (bulk variant: the ring)
};

constexpr int kBlock = 256;          // threads per CTA for every reduce kernel
constexpr int kMaxGrid = 4096;       // CTAs at most (vector / paper variants)
constexpr int kMaxSlots = 8192;      // workspace partial slots (per CTA, or per chunk for bulk)
// Default configuration per element size (chosen by the U x V sweep).
constexpr int kDefaultUnroll4 = 4;   // 4-byte elements
constexpr int kDefaultUnroll8 = 4;   // 8-byte elements
constexpr int kDefaultVec = 32;      // LDG.256

// Translation units rd_inst_*.cu each define one of these.
bool lookup_int(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
bool lookup_float(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
bool lookup_ablation(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r);
CombineFn lookup_combine(int dtype, int op);

// exact float sum (RD_SUM_EXACT, rd_exact.cuh): one vector-load kernel per
// float dtype, launched by launch_exact (rd_api.cu)
struct XArgs;
using ExactFn = void (*)(const XArgs);
using ExactCombineFn = void (*)(const rd_exact_record*, int, uint32_t, void*, rd_exact_record*, int*);
struct ExactRef {
  ExactFn fn;
  int block, unroll, vec_bytes;
  int variant = RD_VARIANT_VECTOR;   // or RD_VARIANT_BULK (unroll = stages, vec_bytes = stage bytes)
  int smem_bytes = 0;
};
constexpr int kExactUnroll = 6;       // 32-byte loads in flight per thread per iteration (tools/tune_exact.py)
constexpr int kExactExpansions = 2;   // independent (a0, a1) expansions per thread
constexpr int kExactMinBlocks = 2;    // __launch_bounds__ min CTAs/SM (register cap: <= 128)
constexpr int kExactBulkConsumerWarps = 16;   // bulk variant: the fold is FP64-latency bound
constexpr int kExactBulkExpansions = 1;       // bulk variant (tools/gpu/tune_exact_bulk.sh)
bool lookup_exact(int dtype, int variant, ExactRef* r);
ExactCombineFn lookup_exact_combine(int dtype);

// bulk variant: CW consumer warps + 1 producer warp per CTA. 8 consumer warps
// keep up with HBM for the cheap combiners; the ALU-heavier float argmin /
// argmax folds get 16 (more warps to hide the dependent integer chains).
constexpr int kBulkConsumerWarps = 8;
template <class OpT>
struct BulkWarps { static constexpr int value = (OpT::kIndexed && OpT::kFloat) ? 16 : kBulkConsumerWarps; };

template <class OpT, int STAGES, int STAGE_BYTES>
inline bool bulk_entry(int stages, int stage_bytes, KernelRef* r) {
  if (stages != STAGES || stage_bytes != STAGE_BYTES) return false;
  constexpr int CW = BulkWarps<OpT>::value;
  *r = KernelRef{rd_bulk_kernel<OpT, STAGES, STAGE_BYTES, CW>, 32 * (CW + 1), STAGES, STAGE_BYTES,
                 RD_VARIANT_BULK, BulkSmem<STAGES, STAGE_BYTES, CW>::kBytes};
  return true;
}

// Default bulk ring (chosen by the stage sweep): 4 x 32 KB.
constexpr int kBulkStages = 4;
constexpr int kBulkStageBytes = 32768;
// AUTO picks the bulk pipeline at or above this many input bytes (below it the
// vector kernel's shorter latency chain wins).
constexpr uint64_t kBulkMinBytes = 128ull << 20;
constexpr uint64_t kBulkMinBytesF64Blocked = 1ull << 30;   // fp64 float + / x / compensated + (rd_api.cu)
// AUTO picks the one-cluster kernel (at most kClusterMax = 16 CTAs, a
// non-portable cluster size allowed on sm_100) for 32 KB < n*s <= 1 MiB: up to
// 512 KB the vector plan needs 2..16 CTAs anyway; at 512 KB - 1 MiB 16 CTAs
// doing two passes still beat 32 ticketed CTAs (graph-captured float32 Σ
// 2^18: 2.85 vs 3.11 us; at 2 MiB they lose: 3.42 vs 3.21; tools/gpu/cl_probe.py).
constexpr int kClusterMax = 16;
constexpr uint64_t kClusterMaxBytes = 1ull << 20;

// Helpers used by the instantiation units: the default kernels of one (dtype, op).
template <class OpT>
inline bool lookup_default(int variant, int unroll, int vec_bytes, KernelRef* r) {
  using T = typename OpT::T;
  constexpr int du = sizeof(T) == 4 ? kDefaultUnroll4 : kDefaultUnroll8;
  if (variant == RD_VARIANT_BULK) {
    return bulk_entry<OpT, kBulkStages, kBulkStageBytes>(unroll ? unroll : kBulkStages,
                                                         vec_bytes ? vec_bytes : kBulkStageBytes, r);
  }
  if (variant == RD_VARIANT_CLUSTER) {
    if ((unroll && unroll != du) || (vec_bytes && vec_bytes != kDefaultVec)) return false;
    *r = KernelRef{rd_cluster_kernel<OpT, kBlock, du, kDefaultVec>, kBlock, du, kDefaultVec, RD_VARIANT_CLUSTER};
    return true;
  }
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
