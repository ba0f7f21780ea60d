// tools/cub_ref.cu -- CUB DeviceReduce::Reduce as a context row for bench.py
// (measurement tooling, not the product; SURVEY §8(d) "context rows on the
// same box: torch.sum / torch.amax and CUB DeviceReduce::Reduce").
// PAPER.md Table 3 puts the paper's kernel beside the best
// library-grade reduction of its day (Harris K7); CUB's device-wide reduce is
// that kernel's descendant. Library code: it is timed, never used on the
// product path.
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

namespace {
struct MaxOp {
  template <typename T>
  __device__ __forceinline__ T operator()(const T& a, const T& b) const { return a < b ? b : a; }
};
struct SumOp {
  template <typename T>
  __device__ __forceinline__ T operator()(const T& a, const T& b) const { return a + b; }
};

template <typename T, class Op>
int run(const void* x, int64_t n, void* out, void* tmp, size_t* tmp_bytes, T init, cudaStream_t s) {
  cudaError_t e = cub::DeviceReduce::Reduce(tmp, *tmp_bytes, static_cast<const T*>(x), static_cast<T*>(out), n,
                                            Op{}, init, s);
  return (int)e;
}
}  // namespace

extern "C" {
// dtype: 0 = int32, 3 = float32 (the metric's dtypes); op: 0 = sum, 3 = max.
// tmp == NULL: writes the temp storage size to *tmp_bytes and launches nothing.
int cub_ref_reduce(const void* x, int64_t n, int dtype, int op, void* out, void* tmp, size_t* tmp_bytes,
                   cudaStream_t s) {
  if (dtype == 3 && op == 0) return run<float, SumOp>(x, n, out, tmp, tmp_bytes, 0.0f, s);
  if (dtype == 3 && op == 3) return run<float, MaxOp>(x, n, out, tmp, tmp_bytes, -INFINITY, s);
  if (dtype == 0 && op == 0) return run<int32_t, SumOp>(x, n, out, tmp, tmp_bytes, 0, s);
  if (dtype == 0 && op == 3) return run<int32_t, MaxOp>(x, n, out, tmp, tmp_bytes, INT32_MIN, s);
  return -1;
}
}
