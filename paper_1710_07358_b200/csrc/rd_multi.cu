// rd_multi.cu -- the sharded form: one process per
// GPU; each rank reduces its contiguous block in local HBM to an rd_record,
// the W records are all-gathered over NCCL (NVLink 5 / NVSwitch), and every
// rank folds them in RANK ORDER (rd_combine_kernel), so all ranks hold the
// bitwise-identical result and float results do not depend on NCCL's
// reduction order. NCCL lacks bitwise reductions and may reorder float ones;
// the gather is 32 B per rank (latency-bound).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "b200reduce.h"
#include "rd_internal.h"

static_assert(sizeof(rd_unique_id) == sizeof(ncclUniqueId), "unique id size");
static_assert(sizeof(rd_record) == 32, "rd_record is 32 bytes");

struct rd_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 0, rank = 0, device = 0;
  rd_record* d_send = nullptr;   // this rank's record
  rd_record* d_recv = nullptr;   // nranks records, rank order
  int* d_err = nullptr;          // sticky mismatch flag (rd_comm_check clears it)
  rd_exact_record* d_xsend = nullptr;   // RD_SUM_EXACT on floats: this rank's exact record
  rd_exact_record* d_xrecv = nullptr;   // nranks exact records
};

namespace {
rd_status nccl_fail(ncclResult_t r, const char* what) {
  rd::set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return RD_ERR_NCCL;
}

// restores the caller's current device on scope exit
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { if (cudaGetDevice(&prev) != cudaSuccess) prev = -1; }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// zero device memory on a private stream and wait for that stream only (no
// device-wide synchronisation: other streams may hold running work)
cudaError_t zero_sync(void* p, size_t bytes) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p, 0, bytes, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return e != cudaSuccess ? e : e2;
}
}  // namespace

extern "C" {

rd_status rd_get_unique_id(rd_unique_id* id) {
  if (!id) { rd::set_error("id is NULL"); return RD_ERR_INVALID_ARG; }
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return RD_OK;
}

rd_status rd_comm_init(rd_comm_t* comm, int nranks, int rank, const rd_unique_id* id, int device) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks || device < 0) {
    rd::set_error("bad rd_comm_init arguments");
    return RD_ERR_INVALID_ARG;
  }
  DeviceGuard guard;                    // the caller's current device is restored
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaSetDevice");
  rd_comm* c = new rd_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank"); }
  void* p = nullptr;
  e = cudaMalloc(&p, sizeof(rd_record) * (nranks + 1) + 64);
  if (e != cudaSuccess) { ncclCommDestroy(c->nccl); delete c; return rd::cuda_fail(e, "cudaMalloc"); }
  e = zero_sync(p, sizeof(rd_record) * (nranks + 1) + 64);
  if (e != cudaSuccess) { cudaFree(p); ncclCommDestroy(c->nccl); delete c; return rd::cuda_fail(e, "comm buffers"); }
  c->d_send = (rd_record*)p;
  c->d_recv = c->d_send + 1;
  c->d_err = (int*)(c->d_recv + nranks);
  void* q = nullptr;
  e = cudaMalloc(&q, sizeof(rd_exact_record) * (nranks + 1));
  if (e == cudaSuccess) e = zero_sync(q, sizeof(rd_exact_record) * (nranks + 1));
  if (e != cudaSuccess) {
    if (q) cudaFree(q);
    cudaFree(p);
    ncclCommDestroy(c->nccl);
    delete c;
    return rd::cuda_fail(e, "exact comm buffers");
  }
  c->d_xsend = (rd_exact_record*)q;
  c->d_xrecv = c->d_xsend + 1;
  *comm = c;
  return RD_OK;
}

rd_status rd_comm_destroy(rd_comm_t comm) {
  if (!comm) { rd::set_error("comm is NULL"); return RD_ERR_INVALID_ARG; }
  DeviceGuard guard;
  cudaSetDevice(comm->device);
  cudaDeviceSynchronize();   // no call of this communicator may still be in flight
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  cudaFree(comm->d_send);
  cudaFree(comm->d_xsend);
  delete comm;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return RD_OK;
}

rd_status reduce_multi(const void* x_local, size_t n_local, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, rd_comm_t comm) {
  if (!comm) { rd::set_error("comm is NULL"); return RD_ERR_INVALID_ARG; }
  if (!out) { rd::set_error("out is NULL"); return RD_ERR_INVALID_ARG; }
  rd_status st = rd::check_dtype_op(dtype, op);
  if (st != RD_OK) return st;
  if ((uintptr_t)out % (rd::is_arg_op(op) ? 8 : rd::dtype_size(dtype))) { rd::set_error("out misaligned"); return RD_ERR_MISALIGNED; }
  cudaStream_t s = (cudaStream_t)stream;
  if (rd::is_exact_float(dtype, op)) {
    // exact sum: the local shard's exact record (608 B), all-gathered; the W
    // fixed-point integers add exactly, so every rank and every W gives the
    // same bits (reading R17)
    st = rd::launch_exact(x_local, n_local, dtype, 1, nullptr, comm->d_xsend, s, nullptr, nullptr);
    if (st != RD_OK) return st;
    const rd_exact_record* recs = comm->d_xsend;
    if (comm->nranks > 1) {
      ncclResult_t r = ncclAllGather(comm->d_xsend, comm->d_xrecv, sizeof(rd_exact_record), ncclUint8, comm->nccl, s);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
      recs = comm->d_xrecv;
    }
    return rd::launch_exact_combine(recs, comm->nranks, dtype, out, nullptr, comm->d_err, s);
  }
  // a0-a7 on the local shard -> this rank's record
  st = rd::launch_reduce(x_local, n_local, dtype, op, 1, nullptr, comm->d_send, s, nullptr, nullptr);
  if (st != RD_OK) return st;
  // a8: exchange the W records (rank order), then fold them identically on every rank
  if (comm->nranks > 1) {
    ncclResult_t r = ncclAllGather(comm->d_send, comm->d_recv, sizeof(rd_record), ncclUint8, comm->nccl, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    return rd::launch_combine(comm->d_recv, comm->nranks, dtype, op, out, nullptr, comm->d_err, s);
  }
  return rd::launch_combine(comm->d_send, 1, dtype, op, out, nullptr, comm->d_err, s);
}

rd_status rd_comm_check(rd_comm_t comm, rd_stream_t stream) {
  if (!comm) { rd::set_error("comm is NULL"); return RD_ERR_INVALID_ARG; }
  // stream-ordered read-back and clear (no legacy-stream or device-wide sync)
  int h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, comm->d_err, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaMemcpyAsync");
  e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return rd::cuda_fail(e, "cudaStreamSynchronize");
  if (h) {
    e = cudaMemsetAsync(comm->d_err, 0, sizeof(int), (cudaStream_t)stream);
    if (e != cudaSuccess) return rd::cuda_fail(e, "cudaMemsetAsync");
    rd::set_error("ranks disagree on dtype/op");
    return RD_ERR_MISMATCH;
  }
  return RD_OK;
}

}  // extern "C"
