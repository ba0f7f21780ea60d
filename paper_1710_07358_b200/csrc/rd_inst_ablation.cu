// rd_inst_ablation.cu -- the configurations of the loads-in-flight ablation,
// the B200 form of PAPER.md Table 2: float32 and int32 sums
//   VECTOR variant: U in {1..8, 16} x VB in {4, 8, 16, 32} bytes per load
//   PAPER  variant: F in {1..8, 16} consecutive elements per work-item
//                   (Listing "Unrolling the step 1")
#include "rd_registry.h"

namespace rd {

namespace {

template <class OpT, int U, int VB>
bool vec_entry(int u, int vb, KernelRef* r) {
  if (u != U || vb != VB) return false;
  *r = KernelRef{rd_vector_kernel<OpT, kBlock, U, VB>, kBlock, U, VB, RD_VARIANT_VECTOR};
  return true;
}

template <class OpT, int VB>
bool vec_row(int u, int vb, KernelRef* r) {
  return vec_entry<OpT, 1, VB>(u, vb, r) || vec_entry<OpT, 2, VB>(u, vb, r) ||
         vec_entry<OpT, 3, VB>(u, vb, r) || vec_entry<OpT, 4, VB>(u, vb, r) ||
         vec_entry<OpT, 5, VB>(u, vb, r) || vec_entry<OpT, 6, VB>(u, vb, r) ||
         vec_entry<OpT, 7, VB>(u, vb, r) || vec_entry<OpT, 8, VB>(u, vb, r) ||
         vec_entry<OpT, 16, VB>(u, vb, r);
}

template <class OpT, int F>
bool paper_entry(int f, KernelRef* r) {
  if (f != F) return false;
  *r = KernelRef{rd_paper_kernel<OpT, kBlock, F>, kBlock, F, (int)sizeof(typename OpT::T), RD_VARIANT_PAPER};
  return true;
}

template <class OpT>
bool lookup_sweep(int variant, int unroll, int vec_bytes, KernelRef* r) {
  if (variant == RD_VARIANT_BULK) {
    const int st = unroll ? unroll : kBulkStages;
    const int sb = vec_bytes ? vec_bytes : kBulkStageBytes;
    return bulk_entry<OpT, 4, 32768>(st, sb, r) || bulk_entry<OpT, 6, 32768>(st, sb, r) ||
           bulk_entry<OpT, 3, 32768>(st, sb, r) || bulk_entry<OpT, 5, 32768>(st, sb, r) ||
           bulk_entry<OpT, 2, 65536>(st, sb, r) || bulk_entry<OpT, 4, 49152>(st, sb, r) ||
           bulk_entry<OpT, 3, 65536>(st, sb, r) || bulk_entry<OpT, 12, 16384>(st, sb, r) ||
           bulk_entry<OpT, 8, 16384>(st, sb, r) || bulk_entry<OpT, 6, 16384>(st, sb, r) ||
           bulk_entry<OpT, 24, 8192>(st, sb, r);
  }
  if (variant == RD_VARIANT_PAPER) {
    const int f = unroll ? unroll : 8;
    return paper_entry<OpT, 1>(f, r) || paper_entry<OpT, 2>(f, r) || paper_entry<OpT, 3>(f, r) ||
           paper_entry<OpT, 4>(f, r) || paper_entry<OpT, 5>(f, r) || paper_entry<OpT, 6>(f, r) ||
           paper_entry<OpT, 7>(f, r) || paper_entry<OpT, 8>(f, r) || paper_entry<OpT, 16>(f, r);
  }
  if (variant != RD_VARIANT_VECTOR) return false;   // AUTO resolves to the default kernels
  const int u = unroll ? unroll : kDefaultUnroll4;
  const int vb = vec_bytes ? vec_bytes : kDefaultVec;
  return vec_row<OpT, 4>(u, vb, r) || vec_row<OpT, 8>(u, vb, r) || vec_row<OpT, 16>(u, vb, r) ||
         vec_row<OpT, 32>(u, vb, r);
}

}  // namespace

bool lookup_ablation(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r) {
  if (op != RD_SUM) return false;
  if (dtype == RD_FLOAT32) return lookup_sweep<OpFor<RD_FLOAT32, RD_SUM>::type>(variant, unroll, vec_bytes, r);
  if (dtype == RD_INT32) return lookup_sweep<OpFor<RD_INT32, RD_SUM>::type>(variant, unroll, vec_bytes, r);
  return false;
}

}  // namespace rd
