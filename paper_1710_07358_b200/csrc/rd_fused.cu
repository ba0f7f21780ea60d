// rd_fused.cu -- SURVEY f1: the multi-GPU exchange fused into the reduce
// kernel (rd_kernels.cuh fused_exchange). Host side: mailbox allocation, CUDA
// IPC handle export / import, epoch counting, error readback.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "b200reduce.h"
#include "rd_internal.h"
#include "rd_kernels.cuh"

static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "IPC handle fits the 64-byte slot");

struct rd_fused {
  int nranks = 0, rank = 0, device = 0;
  rd::Mailbox* self = nullptr;          // this rank's mailbox (+ err word after it)
  int* d_err = nullptr;
  rd::Mailbox** d_peers = nullptr;      // device array of nranks pointers
  std::vector<void*> opened;            // IPC-opened peer mappings to close
  bool connected = false;
};

namespace {
// restores the caller's current device on scope exit
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { if (cudaGetDevice(&prev) != cudaSuccess) prev = -1; }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// zero / fill device memory without synchronising the device or the legacy
// stream (other streams, e.g. the ranks of a running exchange, may be busy):
// a private non-blocking stream, waited for alone
cudaError_t private_copy(void* dst, const void* src, size_t bytes) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  e = src ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) : cudaMemsetAsync(dst, 0, bytes, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return e != cudaSuccess ? e : e2;
}
cudaError_t zero_sync(void* p, size_t bytes) { return private_copy(p, nullptr, bytes); }

rd_status upload_peers(rd_fused* f, const std::vector<rd::Mailbox*>& ptrs) {
  cudaError_t e = private_copy(f->d_peers, ptrs.data(), sizeof(rd::Mailbox*) * f->nranks);
  if (e != cudaSuccess) return rd::cuda_fail(e, "copy of the peer table");
  // no lazy kernel loading once ranks may be spinning (rd_api.cu)
  rd_status st = rd::preload_default_kernels(f->device);
  if (st != RD_OK) return st;
  f->connected = true;
  return RD_OK;
}
}  // namespace

extern "C" {

rd_status rd_fused_create(rd_fused_t* out, int nranks, int rank, int device, void* ipc_handle_out) {
  if (!out || nranks < 1 || nranks > rd::kMaxRanks || rank < 0 || rank >= nranks || device < 0) {
    rd::set_error("bad rd_fused_create arguments (nranks <= 32)");
    return RD_ERR_INVALID_ARG;
  }
  DeviceGuard guard;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaSetDevice");
  rd_fused* f = new rd_fused();
  f->nranks = nranks;
  f->rank = rank;
  f->device = device;
  void* p = nullptr;
  const size_t bytes = sizeof(rd::Mailbox) + 256;
  e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = zero_sync(p, bytes);
  if (e == cudaSuccess) e = cudaMalloc((void**)&f->d_peers, sizeof(rd::Mailbox*) * rd::kMaxRanks);
  if (e != cudaSuccess) { cudaFree(p); delete f; return rd::cuda_fail(e, "mailbox allocation"); }
  f->self = (rd::Mailbox*)p;
  f->d_err = (int*)((char*)p + sizeof(rd::Mailbox));
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) { cudaFree(p); cudaFree(f->d_peers); delete f; return rd::cuda_fail(e, "cudaIpcGetMemHandle"); }
    std::memset(ipc_handle_out, 0, 64);
    std::memcpy(ipc_handle_out, &h, sizeof(h));
  }
  *out = f;
  return RD_OK;
}

rd_status rd_fused_connect(rd_fused_t f, const void* ipc_handles) {
  if (!f || !ipc_handles) { rd::set_error("bad rd_fused_connect arguments"); return RD_ERR_INVALID_ARG; }
  DeviceGuard guard;
  cudaError_t e = cudaSetDevice(f->device);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaSetDevice");
  std::vector<rd::Mailbox*> ptrs(f->nranks);
  for (int p = 0; p < f->nranks; ++p) {
    if (p == f->rank) { ptrs[p] = f->self; continue; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const char*)ipc_handles + 64 * p, sizeof(h));
    void* q = nullptr;
    e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return rd::cuda_fail(e, "cudaIpcOpenMemHandle");
    f->opened.push_back(q);
    ptrs[p] = (rd::Mailbox*)q;
  }
  return upload_peers(f, ptrs);
}

rd_status rd_fused_mailbox(rd_fused_t f, void** mailbox) {
  if (!f || !mailbox) { rd::set_error("bad rd_fused_mailbox arguments"); return RD_ERR_INVALID_ARG; }
  *mailbox = f->self;
  return RD_OK;
}

rd_status rd_fused_connect_local(rd_fused_t f, void* const* mailboxes) {
  if (!f || !mailboxes) { rd::set_error("bad rd_fused_connect_local arguments"); return RD_ERR_INVALID_ARG; }
  std::vector<rd::Mailbox*> ptrs(f->nranks);
  for (int p = 0; p < f->nranks; ++p) {
    if (!mailboxes[p]) { rd::set_error("NULL mailbox"); return RD_ERR_INVALID_ARG; }
    ptrs[p] = (rd::Mailbox*)mailboxes[p];
  }
  if (ptrs[f->rank] != f->self) { rd::set_error("mailboxes[rank] is not this rank's mailbox"); return RD_ERR_INVALID_ARG; }
  DeviceGuard guard;
  cudaError_t e = cudaSetDevice(f->device);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaSetDevice");
  // mailboxes on other devices are written by this rank's kernel (peer stores):
  // peer access from this device to each of them must be enabled
  for (int p = 0; p < f->nranks; ++p) {
    cudaPointerAttributes pa;
    e = cudaPointerGetAttributes(&pa, ptrs[p]);
    if (e != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      rd::set_error("mailbox is not device memory");
      return RD_ERR_INVALID_ARG;
    }
    if (pa.device == f->device) continue;
    int can = 0;
    e = cudaDeviceCanAccessPeer(&can, f->device, pa.device);
    if (e != cudaSuccess) return rd::cuda_fail(e, "cudaDeviceCanAccessPeer");
    if (!can) {
      rd::set_error("no peer access between the devices of two mailboxes");
      return RD_ERR_UNSUPPORTED;
    }
    e = cudaDeviceEnablePeerAccess(pa.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();   // already on: fine
    else if (e != cudaSuccess) return rd::cuda_fail(e, "cudaDeviceEnablePeerAccess");
  }
  return upload_peers(f, ptrs);
}

rd_status reduce_fused(const void* x_local, size_t n_local, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, rd_fused_t f) {
  if (!f) { rd::set_error("fused communicator is NULL"); return RD_ERR_INVALID_ARG; }
  if (!f->connected) { rd::set_error("fused communicator not connected"); return RD_ERR_INVALID_ARG; }
  rd::FusedArgs fa;
  fa.peers = f->d_peers;
  fa.self = f->self;
  fa.err = f->d_err;
  fa.nranks = f->nranks;
  fa.rank = f->rank;
  return rd::launch_reduce(x_local, n_local, dtype, op, 2, out, nullptr, (cudaStream_t)stream,
                           nullptr, nullptr, &fa);
}

rd_status rd_fused_check(rd_fused_t f, rd_stream_t stream) {
  if (!f) { rd::set_error("fused communicator is NULL"); return RD_ERR_INVALID_ARG; }
  // stream-ordered read-back and clear (no legacy-stream or device-wide sync)
  int h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, f->d_err, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaMemcpyAsync");
  e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaStreamSynchronize");
  if (h) {
    e = cudaMemsetAsync(f->d_err, 0, sizeof(int), (cudaStream_t)stream);
    if (e != cudaSuccess) return rd::cuda_fail(e, "cudaMemsetAsync");
    rd::set_error(h == RD_ERR_TIMEOUT ? "a peer's record never arrived" : "ranks disagree on dtype/op");
    return (rd_status)h;
  }
  return RD_OK;
}

rd_status rd_fused_destroy(rd_fused_t f) {
  if (!f) { rd::set_error("fused communicator is NULL"); return RD_ERR_INVALID_ARG; }
  DeviceGuard guard;
  cudaSetDevice(f->device);
  cudaDeviceSynchronize();   // no call of this communicator may still be in flight
  for (void* q : f->opened) cudaIpcCloseMemHandle(q);
  cudaFree(f->d_peers);
  cudaFree(f->self);
  delete f;
  return RD_OK;
}

}  // extern "C"
