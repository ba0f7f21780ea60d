// tools/probe.cu -- HBM read-bandwidth probe (measurement tooling, not the product).
// Streams a buffer with 256-bit non-allocating loads and xor-folds into a
// per-thread sink that is written only on an impossible value, so the loads
// cannot be elided. Its best configuration is the "measured HBM read bandwidth"
// that the reduction kernels are compared with (SURVEY §8(d) peak 3).
//   mode 0: grid-stride over the whole buffer (like rd_vector_kernel)
//   mode 1: CTA-contiguous spans (CTA b reads [b*span, (b+1)*span), threads stride by B)
#include <cstdint>
#include <cuda_runtime.h>

template <int U, int B>
__global__ void __launch_bounds__(B, 1) probe_kernel(const unsigned char* __restrict__ base, uint64_t nvec32,
                                                     uint32_t* sink, int mode) {
  uint32_t acc = 0;
  uint64_t i, stride, end;
  if (mode == 0) {
    stride = (uint64_t)gridDim.x * B;
    i = (uint64_t)blockIdx.x * B + threadIdx.x;
    end = nvec32;
  } else {
    const uint64_t span = (nvec32 + gridDim.x - 1) / gridDim.x;
    stride = B;
    i = (uint64_t)blockIdx.x * span + threadIdx.x;
    end = min(nvec32, (uint64_t)(blockIdx.x + 1) * span);
  }
  for (; i + (U - 1) * stride < end; i += U * stride) {
    uint32_t w[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(w[u][0]), "=r"(w[u][1]), "=r"(w[u][2]), "=r"(w[u][3]), "=r"(w[u][4]), "=r"(w[u][5]),
            "=r"(w[u][6]), "=r"(w[u][7])
          : "l"(base + (i + u * stride) * 32));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= w[u][k];
  }
  for (; i < end; i += stride) {
    uint32_t w[8];
    asm("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
        : "l"(base + i * 32));
    for (int k = 0; k < 8; ++k) acc ^= w[k];
  }
  if (acc == 0x9E3779B9u) sink[threadIdx.x] = acc;
}

template <int B>
static int launch_b(const void* x, uint64_t nvec, int unroll, int blocks, void* sink, cudaStream_t s, int mode) {
  const unsigned char* p = (const unsigned char*)x;
  switch (unroll) {
    case 1: probe_kernel<1, B><<<blocks, B, 0, s>>>(p, nvec, (uint32_t*)sink, mode); break;
    case 2: probe_kernel<2, B><<<blocks, B, 0, s>>>(p, nvec, (uint32_t*)sink, mode); break;
    case 4: probe_kernel<4, B><<<blocks, B, 0, s>>>(p, nvec, (uint32_t*)sink, mode); break;
    case 8: probe_kernel<8, B><<<blocks, B, 0, s>>>(p, nvec, (uint32_t*)sink, mode); break;
    default: return -1;
  }
  return 0;
}

extern "C" int probe_read(const void* x, uint64_t nbytes, int unroll, int blocks, int threads, void* sink,
                          void* stream, int mode) {
  uint64_t nvec = nbytes / 32;
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  switch (threads) {
    case 256: rc = launch_b<256>(x, nvec, unroll, blocks, sink, s, mode); break;
    case 512: rc = launch_b<512>(x, nvec, unroll, blocks, sink, s, mode); break;
    case 1024: rc = launch_b<1024>(x, nvec, unroll, blocks, sink, s, mode); break;
    default: return -1;
  }
  if (rc) return rc;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int probe_occupancy(int unroll, int threads) {
  int c = 0;
  const void* f = nullptr;
#define PO(B)                                                       \
  if (threads == B) {                                               \
    if (unroll == 1) f = (const void*)probe_kernel<1, B>;           \
    if (unroll == 2) f = (const void*)probe_kernel<2, B>;           \
    if (unroll == 4) f = (const void*)probe_kernel<4, B>;           \
    if (unroll == 8) f = (const void*)probe_kernel<8, B>;           \
  }
  PO(256) PO(512) PO(1024)
#undef PO
  if (!f) return -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, f, threads, 0);
  return c;
}

// Launch-gap instrumentation (tools/timeline.py): one thread writes
// %globaltimer to buf[idx]; and a kernel that only allocates `smem` bytes of
// dynamic shared memory (switches the SM's L1/shared carveout).
__global__ void stamp_kernel(unsigned long long* buf, int idx) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  buf[idx] = t;
}
__global__ void smem_hog_kernel(int* sink) {
  extern __shared__ int sm[];
  if (threadIdx.x == 1023) sm[0] = 1;
  if (threadIdx.x == 1024) sink[0] = sm[0];
}

extern "C" int probe_stamp(void* buf, int idx, void* stream) {
  stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)buf, idx);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int probe_smem_hog(int smem_bytes, int blocks, void* sink, void* stream) {
  cudaFuncSetAttribute(smem_hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  smem_hog_kernel<<<blocks, 32, smem_bytes, (cudaStream_t)stream>>>((int*)sink);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
