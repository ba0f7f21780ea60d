// rd_inst_default.cu -- default-configuration kernels for all 29 (dtype, op)
// pairs, and the record-combine kernels.
#include "rd_registry.h"

namespace rd {

#define RD_CASE_DEFAULT(DT, OP) \
  case OP: return lookup_default<typename OpFor<DT, OP>::type>(variant, unroll, vec_bytes, r);

bool lookup_int(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r) {
#define RD_INT_DTYPE(DT)                                                        \
  case DT:                                                                      \
    switch (op) {                                                               \
      RD_CASE_DEFAULT(DT, RD_SUM) RD_CASE_DEFAULT(DT, RD_PROD)                  \
      RD_CASE_DEFAULT(DT, RD_MIN) RD_CASE_DEFAULT(DT, RD_MAX)                   \
      RD_CASE_DEFAULT(DT, RD_AND) RD_CASE_DEFAULT(DT, RD_OR)                    \
      RD_CASE_DEFAULT(DT, RD_XOR)                                               \
      RD_CASE_DEFAULT(DT, RD_ARGMIN) RD_CASE_DEFAULT(DT, RD_ARGMAX)             \
      RD_CASE_DEFAULT(DT, RD_SUM_COMPENSATED)                                   \
      RD_CASE_DEFAULT(DT, RD_SUM_EXACT)                                         \
      default: return false;                                                    \
    }
  switch (dtype) {
    RD_INT_DTYPE(RD_INT32)
    RD_INT_DTYPE(RD_UINT32)
    RD_INT_DTYPE(RD_INT64)
    default: return false;
  }
#undef RD_INT_DTYPE
}

bool lookup_float(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r) {
#define RD_FLOAT_DTYPE(DT)                                                      \
  case DT:                                                                      \
    switch (op) {                                                               \
      RD_CASE_DEFAULT(DT, RD_SUM) RD_CASE_DEFAULT(DT, RD_PROD)                  \
      RD_CASE_DEFAULT(DT, RD_MIN) RD_CASE_DEFAULT(DT, RD_MAX)                   \
      RD_CASE_DEFAULT(DT, RD_ARGMIN) RD_CASE_DEFAULT(DT, RD_ARGMAX)             \
      RD_CASE_DEFAULT(DT, RD_SUM_COMPENSATED)                                   \
      default: return false;                                                    \
    }
  switch (dtype) {
    RD_FLOAT_DTYPE(RD_FLOAT32)
    RD_FLOAT_DTYPE(RD_FLOAT64)
    default: return false;
  }
#undef RD_FLOAT_DTYPE
}

CombineFn lookup_combine(int dtype, int op) {
#define RD_C(DT, OP) \
  if (dtype == DT && op == OP) return rd_combine_kernel<typename OpFor<DT, OP>::type>;
#define RD_C_INT(DT) RD_C(DT, RD_SUM) RD_C(DT, RD_PROD) RD_C(DT, RD_MIN) RD_C(DT, RD_MAX) \
  RD_C(DT, RD_AND) RD_C(DT, RD_OR) RD_C(DT, RD_XOR) RD_C(DT, RD_ARGMIN) RD_C(DT, RD_ARGMAX)   \
  RD_C(DT, RD_SUM_COMPENSATED) RD_C(DT, RD_SUM_EXACT)
#define RD_C_FLT(DT) RD_C(DT, RD_SUM) RD_C(DT, RD_PROD) RD_C(DT, RD_MIN) RD_C(DT, RD_MAX) \
  RD_C(DT, RD_ARGMIN) RD_C(DT, RD_ARGMAX) RD_C(DT, RD_SUM_COMPENSATED)
  RD_C_INT(RD_INT32) RD_C_INT(RD_UINT32) RD_C_INT(RD_INT64)
  RD_C_FLT(RD_FLOAT32) RD_C_FLT(RD_FLOAT64)
#undef RD_C_FLT
#undef RD_C_INT
#undef RD_C
  return nullptr;
}

}  // namespace rd

