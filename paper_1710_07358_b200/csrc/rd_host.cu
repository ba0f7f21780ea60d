// rd_host.cu -- reduce_host: end-to-end reduction of a host array.
//
// Chunks of the host array are copied to a double-buffered device staging
// area on a copy stream while the previous chunk is reduced to an rd_record
// on a compute stream (copy/compute overlap); the chunk records are folded in
// chunk order (rd_combine_kernel) and the one result is copied back.
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>

#include "b200reduce.h"
#include "rd_internal.h"

namespace rd {
namespace {

constexpr size_t kChunkBytes = 32ull << 20;   // 32 MiB per staging buffer

struct HostPipe {
  cudaStream_t copy = nullptr, comp = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  void* stage[2] = {nullptr, nullptr};
  rd_record* recs = nullptr;
  int rec_cap = 0;
  rd_exact_record* xrecs = nullptr;   // RD_SUM_EXACT on floats
  int xrec_cap = 0;
  void* d_out = nullptr;
  std::mutex mu;
};

std::mutex g_pipes_mu;
std::map<int, HostPipe*> g_pipes;

rd_status make_pipe(HostPipe* p) {
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&p->copy, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
  if ((e = cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
  for (int b = 0; b < 2; ++b) {
    if ((e = cudaEventCreateWithFlags(&p->copied[b], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaEventCreateWithFlags(&p->consumed[b], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaMalloc(&p->stage[b], kChunkBytes)) != cudaSuccess) return cuda_fail(e, "staging cudaMalloc");
  }
  if ((e = cudaMalloc(&p->d_out, 16)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return RD_OK;
}

rd_status get_pipe(int dev, HostPipe** out) {
  std::lock_guard<std::mutex> lk(g_pipes_mu);
  auto it = g_pipes.find(dev);
  if (it != g_pipes.end()) { *out = it->second; return RD_OK; }
  HostPipe* p = new HostPipe();
  rd_status st = make_pipe(p);
  if (st != RD_OK) { delete p; return st; }
  g_pipes[dev] = p;
  *out = p;
  return RD_OK;
}

}  // namespace

void release_host_pipelines() {
  std::lock_guard<std::mutex> lk(g_pipes_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_pipes) {
    HostPipe* p = kv.second;
    cudaSetDevice(kv.first);
    cudaStreamSynchronize(p->comp);
    cudaStreamSynchronize(p->copy);
    for (int b = 0; b < 2; ++b) {
      cudaFree(p->stage[b]);
      cudaEventDestroy(p->copied[b]);
      cudaEventDestroy(p->consumed[b]);
    }
    cudaFree(p->recs);
    cudaFree(p->xrecs);
    cudaFree(p->d_out);
    cudaStreamDestroy(p->copy);
    cudaStreamDestroy(p->comp);
    delete p;
  }
  g_pipes.clear();
  cudaSetDevice(cur);
}

}  // namespace rd

extern "C" rd_status reduce_host(const void* x_host, size_t n, rd_dtype dtype, rd_op op, void* out_host) {
  using namespace rd;
  rd_status st = check_dtype_op(dtype, op);
  if (st != RD_OK) return st;
  const int s = dtype_size(dtype);
  if (!x_host && n > 0) { set_error("x_host is NULL"); return RD_ERR_INVALID_ARG; }
  if (!out_host) { set_error("out_host is NULL"); return RD_ERR_INVALID_ARG; }
  if ((uintptr_t)x_host % s) { set_error("x_host misaligned"); return RD_ERR_MISALIGNED; }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  HostPipe* p = nullptr;
  if ((st = get_pipe(dev, &p)) != RD_OK) return st;
  std::lock_guard<std::mutex> lk(p->mu);

  const uint64_t bytes = (uint64_t)n * s;
  const uint64_t nchunks = (bytes + kChunkBytes - 1) / kChunkBytes;
  if (nchunks > (uint64_t)p->rec_cap) {
    if (p->recs) cudaFree(p->recs);
    p->recs = nullptr;
    p->rec_cap = 0;
    int cap = (int)(nchunks < 64 ? 64 : nchunks);
    if ((e = cudaMalloc(&p->recs, sizeof(rd_record) * cap)) != cudaSuccess) return cuda_fail(e, "records cudaMalloc");
    p->rec_cap = cap;
  }
  const bool exact = is_exact_float(dtype, op);
  if (exact && nchunks > (uint64_t)p->xrec_cap) {
    if (p->xrecs) cudaFree(p->xrecs);
    p->xrecs = nullptr;
    p->xrec_cap = 0;
    int cap = (int)(nchunks < 64 ? 64 : nchunks);
    if ((e = cudaMalloc(&p->xrecs, sizeof(rd_exact_record) * cap)) != cudaSuccess) return cuda_fail(e, "records cudaMalloc");
    p->xrec_cap = cap;
  }
  const unsigned char* src = (const unsigned char*)x_host;
  for (uint64_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    const uint64_t off = k * kChunkBytes;
    const uint64_t len = (bytes - off < kChunkBytes) ? bytes - off : kChunkBytes;
    if (k >= 2 && (e = cudaStreamWaitEvent(p->copy, p->consumed[b], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = cudaMemcpyAsync(p->stage[b], src + off, len, cudaMemcpyHostToDevice, p->copy)) != cudaSuccess)
      return cuda_fail(e, "H2D copy");
    if ((e = cudaEventRecord(p->copied[b], p->copy)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(p->comp, p->copied[b], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    st = exact ? launch_exact(p->stage[b], len / s, dtype, 1, nullptr, p->xrecs + k, p->comp, nullptr, nullptr)
               : launch_reduce(p->stage[b], len / s, dtype, op, 1, nullptr, p->recs + k, p->comp, nullptr, nullptr);
    if (st != RD_OK) return st;
    if ((e = cudaEventRecord(p->consumed[b], p->comp)) != cudaSuccess) return cuda_fail(e, "event record");
  }
  st = exact ? launch_exact_combine(p->xrecs, (int)nchunks, dtype, p->d_out, nullptr, nullptr, p->comp)
             : launch_combine(p->recs, (int)nchunks, dtype, op, p->d_out, nullptr, nullptr, p->comp);
  if (st != RD_OK) return st;
  if ((e = cudaMemcpyAsync(out_host, p->d_out, out_size(dtype, op), cudaMemcpyDeviceToHost, p->comp)) != cudaSuccess)
    return cuda_fail(e, "D2H copy");
  if ((e = cudaStreamSynchronize(p->comp)) != cudaSuccess) return cuda_fail(e, "synchronize");
  return RD_OK;
}
