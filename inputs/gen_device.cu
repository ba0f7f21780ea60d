/*
 * inputs/gen_device.cu -- device twin of the seeded input generator (gen.h).
 * Holds no reduction arithmetic; see gen.h. Bit-identical to gen_host.c
 * because both compile the same gen_element().
 */
#include "gen.h"
#include <cuda_runtime.h>

template <int S>
__global__ void in_fill_kernel(unsigned char* out, uint64_t count, int dtype, int workload,
                               uint64_t seed, uint64_t offset, uint64_t n_total, int* err) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    if (gen_element(dtype, workload, seed, offset + j, n_total, out + j * S) != 0 && err) *err = 1;
  }
}

extern "C" int in_fill_device(void* out, uint64_t count, int dtype, int workload, uint64_t seed,
                              uint64_t offset, uint64_t n_total, void* stream) {
  const int s = gen_dtype_size(dtype);
  if (s == 0) return -1;
  {
    /* validate (dtype, workload) on the host with element 0 */
    unsigned char tmp[8];
    if (gen_element(dtype, workload, seed, offset, n_total ? n_total : 1, tmp) != 0) return -1;
  }
  if (count == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  cudaStream_t st = (cudaStream_t)stream;
  if (s == 4)
    in_fill_kernel<4><<<(unsigned)blocks, 256, 0, st>>>((unsigned char*)out, count, dtype, workload, seed, offset, n_total, nullptr);
  else
    in_fill_kernel<8><<<(unsigned)blocks, 256, 0, st>>>((unsigned char*)out, count, dtype, workload, seed, offset, n_total, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
