// rd_inst_exact.cu -- the exact-sum kernels (RD_SUM_EXACT on float dtypes,
// rd_exact.cuh) and their record-combine kernels.
#include <cstdio>
#include <cstdlib>

#include "rd_exact.cuh"
#include "rd_internal.h"
#include "rd_registry.h"

namespace rd {

// RD_TUNING builds only: RD_TUNE_EXACT="U,E,M" picks another compiled
// configuration (loads in flight, expansions, min CTAs/SM for the register
// cap); the default is the measured best and the only one shipped.
template <typename T>
static bool pick(int u, int e, int m, ExactRef* r) {
#define RD_X(U, E, M)                                                                              \
  if (u == U && e == E && m == M) {                                                                \
    *r = ExactRef{rd_exact_kernel<T, kBlock, U, E, M>, kBlock, U, 32};                            \
    return true;                                                                                   \
  }
  RD_X(6, 2, 2)
#ifdef RD_TUNING
  RD_X(6, 2, 1) RD_X(4, 2, 2) RD_X(8, 1, 2) RD_X(2, 2, 3)
#endif
#undef RD_X
  return false;
}

template <typename T, int CW, int E, int STAGES = kBulkStages, int SB = kBulkStageBytes>
static bool bulk_ref(ExactRef* r) {
  *r = ExactRef{rd_exact_bulk_kernel<T, STAGES, SB, CW, E>, 32 * (CW + 1), STAGES, SB, RD_VARIANT_BULK,
                ExactBulkSmem<T, STAGES, SB, CW>::kBytes};
  return true;
}

// RD_TUNING builds only: RD_TUNE_EXACT_BULK="CW,E" (consumer warps, expansions)
template <typename T>
static bool pick_bulk(ExactRef* r) {
  static int tcw = 0, te = 0;
  static bool once = [] {
    const char* v = tune_env("RD_TUNE_EXACT_BULK");
    if (v && std::sscanf(v, "%d,%d", &tcw, &te) != 2) tcw = te = 0;
    return true;
  }();
  (void)once;
  const int cw = tcw ? tcw : kExactBulkConsumerWarps, e = te ? te : kExactBulkExpansions;
  if (cw == 16 && e == 1) return bulk_ref<T, 16, 1>(r);
#ifdef RD_TUNING
  if (cw == 16 && e == 2) return bulk_ref<T, 16, 2>(r);
  if (cw == 24 && e == 1) return bulk_ref<T, 24, 1, 5, 24576>(r);
  if (cw == 24 && e == 2) return bulk_ref<T, 24, 2, 5, 24576>(r);
  if (cw == 8 && e == 2) return bulk_ref<T, 8, 2>(r);
#endif
  return false;
}

bool lookup_exact(int dtype, int variant, ExactRef* r) {
  if (variant == RD_VARIANT_CLUSTER) {
    if (dtype == RD_FLOAT32) {
      *r = ExactRef{rd_exact_cluster_kernel<float, kBlock, kExactUnroll, kExactExpansions, kExactMinBlocks>, kBlock,
                    kExactUnroll, 32, RD_VARIANT_CLUSTER};
      return true;
    }
    if (dtype == RD_FLOAT64) {
      *r = ExactRef{rd_exact_cluster_kernel<double, kBlock, kExactUnroll, kExactExpansions, kExactMinBlocks>, kBlock,
                    kExactUnroll, 32, RD_VARIANT_CLUSTER};
      return true;
    }
    return false;
  }
  if (variant == RD_VARIANT_BULK) {
    if (dtype == RD_FLOAT32) return pick_bulk<float>(r);
    if (dtype == RD_FLOAT64) return pick_bulk<double>(r);
    return false;
  }
  static int tu = 0, te = 0, tm = 0;
  static bool once = [] {
    const char* v = tune_env("RD_TUNE_EXACT");
    if (v && std::sscanf(v, "%d,%d,%d", &tu, &te, &tm) != 3) tu = te = tm = 0;
    return true;
  }();
  (void)once;
  const int u = tu ? tu : kExactUnroll, e = te ? te : kExactExpansions, m = tm ? tm : kExactMinBlocks;
  if (dtype == RD_FLOAT32) return pick<float>(u, e, m, r);
  if (dtype == RD_FLOAT64) return pick<double>(u, e, m, r);
  return false;
}

ExactCombineFn lookup_exact_combine(int dtype) {
  if (dtype == RD_FLOAT32) return rd_exact_combine_kernel<float>;
  if (dtype == RD_FLOAT64) return rd_exact_combine_kernel<double>;
  return nullptr;
}

}  // namespace rd
