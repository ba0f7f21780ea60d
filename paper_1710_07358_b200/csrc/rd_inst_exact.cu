// rd_inst_exact.cu -- the exact-sum kernels (RD_SUM_EXACT on float dtypes,
// rd_exact.cuh) and their record-combine kernels.
#include <cstdio>
#include <cstdlib>

#include "rd_exact.cuh"
#include "rd_registry.h"

namespace rd {

// Tuning only (measurement): RD_TUNE_EXACT="U,E,M" picks another compiled
// (loads in flight, expansions, min CTAs/SM for the register cap); the
// default is the measured best.
template <typename T>
static bool pick(int u, int e, int m, ExactRef* r) {
#define RD_X(U, E, M)                                                                              \
  if (u == U && e == E && m == M) {                                                                \
    *r = ExactRef{rd_exact_kernel<T, kBlock, U, E, M>, kBlock, U, 32};                            \
    return true;                                                                                   \
  }
  RD_X(6, 2, 2) RD_X(6, 2, 1) RD_X(4, 2, 2) RD_X(8, 1, 2) RD_X(2, 2, 3)
#undef RD_X
  return false;
}

template <typename T>
static bool pick_bulk(ExactRef* r) {
  constexpr int CW = kExactBulkConsumerWarps;
  *r = ExactRef{rd_exact_bulk_kernel<T, kBulkStages, kBulkStageBytes, CW, kExactExpansions>, 32 * (CW + 1),
                kBulkStages, kBulkStageBytes, RD_VARIANT_BULK, BulkSmem<kBulkStages, kBulkStageBytes, CW>::kBytes};
  return true;
}

bool lookup_exact(int dtype, int variant, ExactRef* r) {
  if (variant == RD_VARIANT_BULK) {
    if (dtype == RD_FLOAT32) return pick_bulk<float>(r);
    if (dtype == RD_FLOAT64) return pick_bulk<double>(r);
    return false;
  }
  static int tu = 0, te = 0, tm = 0;
  static bool once = [] {
    const char* v = std::getenv("RD_TUNE_EXACT");
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
