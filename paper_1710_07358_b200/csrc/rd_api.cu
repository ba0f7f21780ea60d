// rd_api.cu -- the C ABI (include/b200reduce.h): validation, the launch
// planner and the per-(device, stream) workspace.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "b200reduce.h"
#include "rd_exact.cuh"
#include "rd_internal.h"
#include "rd_registry.h"

namespace rd {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

rd_status cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return RD_ERR_CUDA;
}

int dtype_size(int dtype) {
  return (dtype == RD_INT64 || dtype == RD_FLOAT64) ? 8 : 4;
}

bool is_arg_op(int op) { return op == RD_ARGMIN || op == RD_ARGMAX; }

bool is_exact_float(int dtype, int op) {
  return op == RD_SUM_EXACT && (dtype == RD_FLOAT32 || dtype == RD_FLOAT64);
}

int out_size(int dtype, int op) { return is_arg_op(op) ? (int)sizeof(rd_arg_result) : dtype_size(dtype); }

rd_status check_dtype_op(int dtype, int op) {
  if (dtype < RD_INT32 || dtype > RD_FLOAT64) { set_error("unknown dtype"); return RD_ERR_INVALID_ARG; }
  if (op < RD_SUM || op > RD_SUM_EXACT) { set_error("unknown op"); return RD_ERR_INVALID_ARG; }
  if ((dtype == RD_FLOAT32 || dtype == RD_FLOAT64) && op >= RD_AND && op <= RD_XOR) {
    set_error("bitwise op on a float dtype");
    return RD_ERR_UNSUPPORTED;
  }
  return RD_OK;
}

// ------------------------------------------------------------------ workspace
namespace {

// exact-sum CTA slots: kMaxGrid x (kWords + 1) int64 (the largest, fp64)
// the exact sum's grid accumulator (kWords + 1 words, zero between launches;
// rd_exact.cuh exact_finish), one 128-byte-aligned block
constexpr size_t kExactSlotBytes = (sizeof(long long) * (ExactTraits<double>::kWords + 1) + 127) / 128 * 128;

struct Workspace {
  Slot* partials = nullptr;   // kMaxGrid slots (per CTA, or per chunk for the bulk variant)
  long long* xpart = nullptr; // exact-sum grid accumulator (RD_SUM_EXACT), zero between launches
  unsigned* ticket = nullptr; // CTAs finished, zero between launches
  unsigned* work = nullptr;   // bulk variant: next chunk, zero between launches
};

struct DeviceInfo {
  int sms = 0;
};

std::mutex g_mu;
std::map<std::pair<int, uintptr_t>, Workspace> g_ws;
std::map<int, DeviceInfo> g_dev;
std::map<std::pair<int, const void*>, int> g_occ;   // (device, kernel) -> CTAs/SM
std::map<std::pair<int, const void*>, int> g_regs;  // (device, kernel) -> regs/thread

rd_status get_workspace(int dev, cudaStream_t stream, Workspace* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, (uintptr_t)stream);
  auto it = g_ws.find(key);
  if (it != g_ws.end()) { *out = it->second; return RD_OK; }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
    set_error("first call on a stream must happen outside CUDA graph capture (workspace allocation)");
    return RD_ERR_CUDA;
  }
  Workspace w;
  void* p = nullptr;
  const size_t bytes = sizeof(Slot) * kMaxSlots + 256 + kExactSlotBytes;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "workspace cudaMalloc");
  // zeroed in stream order (no device-wide synchronisation: kernels on other
  // streams, e.g. the ranks of a fused exchange, may be running and waiting)
  e = cudaMemsetAsync(p, 0, bytes, stream);
  if (e != cudaSuccess) { cudaFree(p); return cuda_fail(e, "workspace init"); }
  w.partials = (Slot*)p;
  w.ticket = (unsigned*)((char*)p + sizeof(Slot) * kMaxSlots);
  w.work = w.ticket + 32;     // separate 128-byte line
  w.xpart = (long long*)((char*)p + sizeof(Slot) * kMaxSlots + 256);
  g_ws[key] = w;
  *out = w;
  return RD_OK;
}

rd_status device_info(int dev, DeviceInfo* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) { *out = it->second; return RD_OK; }
  DeviceInfo d;
  cudaError_t e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  g_dev[dev] = d;
  *out = d;
  return RD_OK;
}

rd_status occupancy(int dev, const KernelRef& k, int* ctas, int* regs) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, (const void*)k.fn);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) { *ctas = it->second; *regs = g_regs[key]; return RD_OK; }
  int c = 0;
  cudaError_t e = cudaSuccess;
  if (k.smem_bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
  }
  if (k.variant == RD_VARIANT_CLUSTER) {   // clusters of up to 16 CTAs (non-portable size)
    e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(NonPortableClusterSizeAllowed)");
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k.fn, k.block, k.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, k.fn);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
  if (c < 1) c = 1;
  g_occ[key] = c;
  g_regs[key] = fa.numRegs;
  *ctas = c;
  *regs = fa.numRegs;
  return RD_OK;
}

bool lookup(int dtype, int op, int variant, int unroll, int vec_bytes, KernelRef* r) {
  if (lookup_ablation(dtype, op, variant, unroll, vec_bytes, r)) return true;
  if (dtype == RD_FLOAT32 || dtype == RD_FLOAT64) return lookup_float(dtype, op, variant, unroll, vec_bytes, r);
  return lookup_int(dtype, op, variant, unroll, vec_bytes, r);
}

// Tuning knobs for the bulk chunk schedule and the mid-size grid cap: read
// only by RD_TUNING builds (rd_internal.h tune_env); the shipped library
// always takes the defaults, the documented schedule.
uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = tune_env(name);
  if (!v || !*v) return dflt;
  const unsigned long long x = std::strtoull(v, nullptr, 10);
  return x ? (uint64_t)x : dflt;
}

// Bulk chunk schedule, fixed by the body size, the stage size and the op
// class only (determinism): a head region in chunks of C0 (about 16 per SM,
// at most 5000), then a tail region of 148*P chunks of C1 = Q stages, so the
// dynamic schedule ends with short chunks and the per-SM tail imbalance is
// < one C1 chunk. Plain ops: P = 16, Q = 1 (measured best of a sweep,
// tools/tune_bulk.sh: +0.9% over 12/4/2). Indexed ops (argmin / argmax) pay
// more per chunk end (global indices for the lane bests), so they take fewer,
// longer tail chunks: P = 4, Q = 4 -- still so after chunk ends became
// per-thread folds into a running best (rd_bulk.cuh, order-free ops): 4 / 4
// beat 16 / 1 by 0.9-1.9% on float32 / int32 / uint32 arg ops, float64 even,
// int64 -0.7% (profiles/ab/r02_ab_cta_partials.jsonl; RD_ARG_TAIL_NARROW
// builds take 16 / 1).
struct BulkPlan {
  uint64_t c0, c1, head_region;
  uint32_t nhead, nchunks;
};
bool plan_bulk(uint64_t body_bytes, uint64_t stage_bytes, BulkPlan* p, bool indexed = false) {
  static const uint64_t kHeadPerSm = env_u64("RD_TUNE_HEAD_PER_SM", 16);
  static const uint64_t kTailPerSmEnv = env_u64("RD_TUNE_TAIL_PER_SM", 0);
  static const uint64_t kTailStagesEnv = env_u64("RD_TUNE_TAIL_STAGES", 0);
#ifdef RD_ARG_TAIL_NARROW
  indexed = false;
#endif
  const uint64_t kTailPerSm = kTailPerSmEnv ? kTailPerSmEnv : (indexed ? 4 : 16);
  const uint64_t kTailStages = kTailStagesEnv ? kTailStagesEnv : (indexed ? 4 : 1);
  const uint64_t T = body_bytes;
  const uint64_t S = stage_bytes;
  const uint64_t C1 = kTailStages * S;
  const uint64_t R = T < 148ull * kTailPerSm * C1 ? T : 148ull * kTailPerSm * C1;
  uint64_t c0 = T / (148ull * kHeadPerSm);
  if (c0 < T / 5000) c0 = T / 5000;   // head <= 5000 chunks: head + tail <= kMaxSlots
  c0 = (c0 + S - 1) / S * S;
  if (c0 < 4 * S) c0 = 4 * S;
  const uint64_t nhead = (T - R + c0 - 1) / c0;       // the head region is T - R bytes exactly
  const uint64_t ntail = (R + C1 - 1) / C1;           // <= 148 * kTailPerSm
  p->c0 = c0;
  p->c1 = C1;
  p->head_region = T - R;
  p->nhead = (uint32_t)nhead;
  p->nchunks = (uint32_t)(nhead + ntail);
  return p->nchunks <= (uint32_t)kMaxSlots;
}

}  // namespace

// Load (and configure) every default kernel now. With CUDA lazy loading, the
// first launch of a kernel loads it, and loading can wait for running kernels
// to finish -- which deadlocks spinning producer/consumer kernels such as
// the ranks of a fused exchange driven from one process. Called when a fused
// communicator is connected.
rd_status preload_default_kernels(int dev) {
  for (int dt = RD_INT32; dt <= RD_FLOAT64; ++dt) {
    if (dt == RD_FLOAT32 || dt == RD_FLOAT64) {     // the exact-sum kernels (fused mode 2 too)
      for (int variant : {RD_VARIANT_VECTOR, RD_VARIANT_BULK, RD_VARIANT_CLUSTER}) {
        ExactRef x;
        if (!lookup_exact(dt, variant, &x)) continue;
        int occ = 0, regs = 0;
        rd_status st = occupancy(dev, KernelRef{(ReduceFn)x.fn, x.block, x.unroll, x.vec_bytes, x.variant, x.smem_bytes},
                                 &occ, &regs);
        if (st != RD_OK) return st;
      }
    }
    for (int op = RD_SUM; op <= RD_SUM_EXACT; ++op) {
      if (check_dtype_op(dt, op) != RD_OK) continue;
      for (int variant : {RD_VARIANT_VECTOR, RD_VARIANT_BULK, RD_VARIANT_CLUSTER}) {
        KernelRef k;
        if (!lookup(dt, op, variant, 0, 0, &k)) continue;
        int occ = 0, regs = 0;
        rd_status st = occupancy(dev, k, &occ, &regs);
        if (st != RD_OK) return st;
      }
      CombineFn c = lookup_combine(dt, op);
      cudaFuncAttributes fa;
      if (c) {
        cudaError_t e = cudaFuncGetAttributes(&fa, c);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes(combine)");
      }
    }
  }
  set_error("");
  return RD_OK;
}

#ifdef RD_TIMELINE
// measurement builds only (tools/timeline.py): the bulk kernel's per-CTA
// %globaltimer stamps, one device buffer for the process (current device)
unsigned long long* timeline_buffer() {
  static unsigned long long* buf = nullptr;
  if (!buf && cudaMalloc(&buf, (size_t)kMaxGrid * 8 * sizeof(unsigned long long)) == cudaSuccess)
    cudaMemset(buf, 0, (size_t)kMaxGrid * 8 * sizeof(unsigned long long));
  return buf;
}
#endif

// a0: validate, plan, launch.
rd_status launch_reduce(const void* x, size_t n, int dtype, int op, int mode, void* out,
                        rd_record* rec, cudaStream_t stream, const rd_config* cfg,
                        rd_launch_info* info, const FusedArgs* fused) {
  rd_status st = check_dtype_op(dtype, op);
  if (st != RD_OK) return st;
  const int s = dtype_size(dtype);
  if (x == nullptr && n > 0) { set_error("x is NULL"); return RD_ERR_INVALID_ARG; }
  if ((mode == 0 || mode == 2) && out == nullptr) { set_error("out is NULL"); return RD_ERR_INVALID_ARG; }
  if (mode == 2 && fused == nullptr) { set_error("fused args missing"); return RD_ERR_INVALID_ARG; }
  if (mode == 1 && rec == nullptr) { set_error("rec is NULL"); return RD_ERR_INVALID_ARG; }
  if ((uintptr_t)x % s != 0) { set_error("x is not aligned to sizeof(dtype)"); return RD_ERR_MISALIGNED; }
  if (mode != 1 && (uintptr_t)out % (is_arg_op(op) ? 8 : s) != 0) { set_error("out is not aligned"); return RD_ERR_MISALIGNED; }
  if (mode == 1 && (uintptr_t)rec % 8 != 0) { set_error("rec is not 8-byte aligned"); return RD_ERR_MISALIGNED; }
  if (n >= (1ull << 40)) { set_error("n >= 2^40"); return RD_ERR_INVALID_ARG; }
  if (is_exact_float(dtype, op)) {
    if (mode == 1) {
      set_error("RD_SUM_EXACT on floats: the 32-byte rd_record cannot carry an exact partial "
                "(use reduce_exact_partial / reduce_multi)");
      return RD_ERR_UNSUPPORTED;
    }
    return launch_exact(x, n, dtype, mode, out, nullptr, stream, cfg, info, fused);
  }

  int variant = cfg ? cfg->variant : RD_VARIANT_AUTO;
  const int unroll = cfg ? cfg->unroll : 0;
  const int vec_bytes = cfg ? cfg->vec_bytes : 0;
  if (cfg && cfg->block != 0 && !(cfg->block == kBlock && variant != RD_VARIANT_BULK)) {
    set_error("block size not compiled for this variant (only the vector/paper variants' 256)");
    return RD_ERR_UNSUPPORTED;
  }
  if (variant < RD_VARIANT_AUTO || variant > RD_VARIANT_CLUSTER || unroll < 0 || vec_bytes < 0 ||
      (cfg && cfg->grid < 0) || (variant == RD_VARIANT_CLUSTER && cfg && cfg->grid > kClusterMax)) {
    set_error("bad rd_config");
    return RD_ERR_INVALID_ARG;
  }
  if (vec_bytes && vec_bytes < s && variant != RD_VARIANT_BULK) { set_error("vec_bytes < sizeof(dtype)"); return RD_ERR_INVALID_ARG; }
  if (variant == RD_VARIANT_AUTO && unroll == 0 && vec_bytes == 0) {
    const uint64_t bytes = (uint64_t)n * s;
    // fp64 float + / x / compensated + (fixed-tree partials per bulk chunk): the
    // vector grid stays ahead up to 1 GiB (2^24-2^26: 3-15% cold, 1-10%
    // graph-captured; even at 2^27; the ring from 2^28, profiles/
    // r02_variants_big.json); every other (dtype, op) from 128 MiB
    const bool f64_blocked = dtype == RD_FLOAT64 && (op == RD_SUM || op == RD_PROD || op == RD_SUM_COMPENSATED);
    if (bytes >= (f64_blocked ? kBulkMinBytesF64Blocked : kBulkMinBytes)) {
      variant = RD_VARIANT_BULK;      // planner: large inputs take the bulk-copy pipeline
    } else if (bytes > (uint64_t)kBlock * kDefaultUnroll4 * kDefaultVec && bytes <= kClusterMaxBytes &&
               !(cfg && cfg->grid > kClusterMax)) {
      variant = RD_VARIANT_CLUSTER;   // 2..16 CTAs: one cluster, combine over DSMEM
    }
  }
  KernelRef k;
  if (!lookup(dtype, op, variant, unroll, vec_bytes, &k)) {
    set_error("no compiled kernel for this (dtype, op, variant, unroll, vec_bytes)");
    return RD_ERR_UNSUPPORTED;
  }

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  DeviceInfo di;
  if ((st = device_info(dev, &di)) != RD_OK) return st;
  int occ = 1, regs = 0;
  if ((st = occupancy(dev, k, &occ, &regs)) != RD_OK) return st;
  Workspace ws;
  if ((st = get_workspace(dev, stream, &ws)) != RD_OK) return st;

  KArgs a;
  std::memset(&a, 0, sizeof(a));
  a.x = (const unsigned char*)x;
  a.n = n;
  uint64_t g = (uint64_t)di.sms * occ;   // persistent grid
  if (k.variant == RD_VARIANT_VECTOR || k.variant == RD_VARIANT_BULK || k.variant == RD_VARIANT_CLUSTER) {
    const int vb = k.variant == RD_VARIANT_BULK ? 16 : k.vec_bytes;   // body alignment
    const uint64_t L = (uint64_t)(vb / s);
    const uint64_t mis = (uint64_t)((uintptr_t)x % (uintptr_t)vb);
    uint64_t head = ((vb - mis) % vb) / s;
    if (head > n) head = n;
    a.head = head;
    a.nvec = (n - head) / L;
    a.tail_start = head + a.nvec * L;
    a.tail = n - a.tail_start;
  } else {  // PAPER: F consecutive elements per work-item
    a.head = 0;
    a.nvec = 0;
    a.tail_start = n;
    a.tail = 0;
  }
  if (k.variant == RD_VARIANT_BULK) {
    BulkPlan bp;
    if (!plan_bulk(a.nvec * 16, (uint64_t)k.vec_bytes, &bp, is_arg_op(op))) {
      set_error("chunk schedule exceeds the workspace");
      return RD_ERR_INVALID_ARG;
    }
    a.chunk_bytes = bp.c0;
    a.tail_chunk_bytes = bp.c1;
    a.head_region_bytes = bp.head_region;
    a.nhead_chunks = bp.nhead;
    a.nchunks = bp.nchunks;
    a.work = ws.work;
    uint64_t need = a.nchunks ? a.nchunks : 1;
    if (g > need) g = need;
  } else {
    // work units handed out by the grid-stride loop; fewer CTAs than one
    // resident wave when there is less work than one unrolled pass
    const bool vec = k.variant == RD_VARIANT_VECTOR || k.variant == RD_VARIANT_CLUSTER;
    const uint64_t units = vec ? a.nvec : (n + k.unroll - 1) / k.unroll;
    const uint64_t per_cta = (uint64_t)k.block * (vec ? k.unroll : 1);
    uint64_t need = (units + per_cta - 1) / per_cta;
    if (need < 1) need = 1;
    if (g > need) g = need;
    // Mid sizes (the vector kernel runs below kBulkMinBytes): at 12-48 MiB the
    // grid is capped at 2 CTAs/SM; from 48 MiB it is the occupancy grid.
    // Measured per (dtype, op) and grid, cold (L2 read-flushed) and L2-warm
    // (graph-captured), tools/timeline.py --exp grids, profiles/
    // r02_midsizes_grids.jsonl: float32 sum 2^23 6.2 -> 5.05 us warm, 14.1 ->
    // 12.3 us cold against round 1's 1 CTA/SM (12-48 MiB) / 2 (48-128 MiB)
    // cap, argmin 2^24 10.4 -> 8.9 us warm (round 1's graph-captured sweep
    // had favoured the tighter cap; this build and box do not reproduce it).
    // Below 12 MiB the work (units / per-CTA) limits the grid anyway.
    // RD_TUNE_VEC_CTAS_PER_SM (RD_TUNING builds only): 0 / unset = this rule,
    // k = k CTAs per SM from 12 MiB, kNoCap = the uncapped occupancy grid.
    constexpr uint64_t kNoCap = 1000;
    static const uint64_t kMidCap = env_u64("RD_TUNE_VEC_CTAS_PER_SM", 0);
    const uint64_t bytes_in = (uint64_t)n * s;
    if (k.variant == RD_VARIANT_VECTOR && kMidCap != kNoCap && bytes_in >= (12ull << 20) &&
        (kMidCap || bytes_in < (48ull << 20))) {
      const uint64_t per_sm = kMidCap ? kMidCap : 2;
      const uint64_t cap = (uint64_t)di.sms * per_sm;
      if (g > cap) g = cap;
    }
  }
  if (cfg && cfg->grid > 0) g = (uint64_t)cfg->grid;
  if (g > (uint64_t)kMaxGrid) g = kMaxGrid;
  if (k.variant == RD_VARIANT_CLUSTER && g > (uint64_t)kClusterMax) g = kClusterMax;
  if (g < 1) g = 1;

  a.out = out;
  a.rec = rec;
  a.partials = ws.partials;
  a.ticket = ws.ticket;
  a.tag = record_tag(dtype, op);
  a.mode = mode;
  if (fused) {
    a.peers = fused->peers;
    a.self = fused->self;
    a.err = fused->err;
    a.nranks = fused->nranks;
    a.rank = fused->rank;
  }
#ifdef RD_TIMELINE
  a.tl = timeline_buffer();
#endif

  // programmatic dependent launch: the grid may be scheduled while the previous
  // kernel on the stream drains; the kernels call griddepcontrol.wait before
  // touching global memory (rd_kernels.cuh pdl_wait).
  cudaLaunchConfig_t lc;
  std::memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3((unsigned)g);
  lc.blockDim = dim3((unsigned)k.block);
  lc.dynamicSmemBytes = (size_t)k.smem_bytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  if (k.variant == RD_VARIANT_CLUSTER) {   // the whole grid is one cluster
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)g;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    lc.numAttrs = 2;
  }
  e = cudaLaunchKernelEx(&lc, k.fn, a);
  if (e != cudaSuccess) return cuda_fail(e, "reduce kernel launch");
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->variant = k.variant;
    info->vec_bytes = k.vec_bytes;
    info->unroll = k.unroll;
    info->block = k.block;
    info->grid = (int32_t)g;
    info->regs_per_thread = regs;
    info->ctas_per_sm = occ;
    info->head = a.head;
    info->nvec = a.nvec;
    info->tail = a.tail;
  }
  return RD_OK;
}

// RD_SUM_EXACT on a float dtype (rd_exact.cuh): validate, plan, launch.
// mode 0 writes one element to `out`, mode 1 one rd_exact_record to `xrec`.
rd_status launch_exact(const void* x, size_t n, int dtype, int mode, void* out, rd_exact_record* xrec,
                       cudaStream_t stream, const rd_config* cfg, rd_launch_info* info, const FusedArgs* fused) {
  if (dtype != RD_FLOAT32 && dtype != RD_FLOAT64) {
    set_error("exact partials are for float dtypes (integer sums are exact: use reduce_partial)");
    return RD_ERR_UNSUPPORTED;
  }
  const int s = dtype_size(dtype);
  if (x == nullptr && n > 0) { set_error("x is NULL"); return RD_ERR_INVALID_ARG; }
  if ((mode == 0 || mode == 2) && out == nullptr) { set_error("out is NULL"); return RD_ERR_INVALID_ARG; }
  if (mode == 1 && xrec == nullptr) { set_error("rec is NULL"); return RD_ERR_INVALID_ARG; }
  if (mode == 2 && fused == nullptr) { set_error("fused args missing"); return RD_ERR_INVALID_ARG; }
  if ((uintptr_t)x % s != 0) { set_error("x is not aligned to sizeof(dtype)"); return RD_ERR_MISALIGNED; }
  if (mode != 1 && (uintptr_t)out % s != 0) { set_error("out is not aligned"); return RD_ERR_MISALIGNED; }
  if (mode == 1 && (uintptr_t)xrec % 8 != 0) { set_error("rec is not 8-byte aligned"); return RD_ERR_MISALIGNED; }
  if (n >= (1ull << 40)) { set_error("n >= 2^40"); return RD_ERR_INVALID_ARG; }
  int variant = cfg ? cfg->variant : RD_VARIANT_AUTO;
  if (variant != RD_VARIANT_AUTO && variant != RD_VARIANT_VECTOR && variant != RD_VARIANT_BULK &&
      variant != RD_VARIANT_CLUSTER) {
    set_error("RD_SUM_EXACT: variant must be auto, vector, bulk or cluster");
    return RD_ERR_UNSUPPORTED;
  }
  if (variant == RD_VARIANT_CLUSTER && cfg && cfg->grid > kClusterMax) {
    set_error("cluster variant: grid <= 16");
    return RD_ERR_INVALID_ARG;
  }
  if (variant == RD_VARIANT_AUTO) {
    // fp64 terms: the bulk ring above the one-cluster range (the vector form's
    // 128-register threads trail it at every size from 2 MiB, cold and
    // graph-captured: 2^22 20.5 vs 27.7 us; profiles/r02_exact_variants.json);
    // fp32 terms: the vector form below 128 MiB (ahead graph-captured at 4-64 MiB)
    const uint64_t bytes = (uint64_t)n * s;
    const uint64_t bulk_from = dtype == RD_FLOAT64 ? kClusterMaxBytes + 1 : kBulkMinBytes;
    variant = bytes >= bulk_from ? RD_VARIANT_BULK
              : (bytes > (uint64_t)kBlock * kExactUnroll * 32 && bytes <= kClusterMaxBytes &&
                 !(cfg && cfg->grid > kClusterMax)) ? RD_VARIANT_CLUSTER : RD_VARIANT_VECTOR;
  }
  ExactRef k;
  if (!lookup_exact(dtype, variant, &k)) { set_error("no compiled exact-sum kernel"); return RD_ERR_UNSUPPORTED; }
  if (cfg && ((cfg->unroll && cfg->unroll != k.unroll) || (cfg->vec_bytes && cfg->vec_bytes != k.vec_bytes) ||
              (cfg->block && cfg->block != k.block))) {
    set_error("RD_SUM_EXACT: one compiled configuration per variant (vector: 32 B loads, U=6, 256 threads; "
              "bulk: the default ring)");
    return RD_ERR_UNSUPPORTED;
  }
  if (cfg && cfg->grid < 0) { set_error("bad rd_config"); return RD_ERR_INVALID_ARG; }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  rd_status st;
  DeviceInfo di;
  if ((st = device_info(dev, &di)) != RD_OK) return st;
  int occ = 1, regs = 0;
  KernelRef kr{(ReduceFn)k.fn, k.block, k.unroll, k.vec_bytes, k.variant, k.smem_bytes};
  if ((st = occupancy(dev, kr, &occ, &regs)) != RD_OK) return st;
  Workspace ws;
  if ((st = get_workspace(dev, stream, &ws)) != RD_OK) return st;

  XArgs a;
  std::memset(&a, 0, sizeof(a));
  a.x = (const unsigned char*)x;
  a.n = n;
  const int vb = k.variant == RD_VARIANT_BULK ? 16 : k.vec_bytes;   // body alignment
  const uint64_t L = (uint64_t)(vb / s);
  const uint64_t mis = (uint64_t)((uintptr_t)x % (uintptr_t)vb);
  uint64_t head = ((vb - mis) % vb) / s;
  if (head > n) head = n;
  a.head = head;
  a.nvec = (n - head) / L;
  a.tail_start = head + a.nvec * L;
  a.tail = n - a.tail_start;
  uint64_t g = (uint64_t)di.sms * occ;
  if (k.variant == RD_VARIANT_BULK) {
    BulkPlan bp;
    if (!plan_bulk(a.nvec * 16, (uint64_t)k.vec_bytes, &bp)) { set_error("chunk schedule exceeds the workspace"); return RD_ERR_INVALID_ARG; }
    a.chunk_bytes = bp.c0;
    a.tail_chunk_bytes = bp.c1;
    a.head_region_bytes = bp.head_region;
    a.nhead_chunks = bp.nhead;
    a.nchunks = bp.nchunks;
    a.work = ws.work;
    const uint64_t need = a.nchunks ? a.nchunks : 1;
    if (g > need) g = need;
  } else {
    uint64_t need = (a.nvec + (uint64_t)k.block * k.unroll - 1) / ((uint64_t)k.block * k.unroll);
    if (need < 1) need = 1;
    if (g > need) g = need;
  }
  if (cfg && cfg->grid > 0) g = (uint64_t)cfg->grid;
  if (g > (uint64_t)kMaxGrid) g = kMaxGrid;
  if (k.variant == RD_VARIANT_CLUSTER && g > (uint64_t)kClusterMax) g = kClusterMax;
  a.out = out;
  a.rec = xrec;
  a.partials = ws.xpart;
  a.ticket = ws.ticket;
  a.tag = record_tag(dtype, RD_SUM_EXACT);
  a.mode = mode;
  if (fused) {
    a.peers = fused->peers;
    a.self = fused->self;
    a.err = fused->err;
    a.nranks = fused->nranks;
    a.rank = fused->rank;
  }

  cudaLaunchConfig_t lc;
  std::memset(&lc, 0, sizeof(lc));
  lc.gridDim = dim3((unsigned)g);
  lc.blockDim = dim3((unsigned)k.block);
  lc.dynamicSmemBytes = (size_t)k.smem_bytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  if (k.variant == RD_VARIANT_CLUSTER) {   // the whole grid is one cluster
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)g;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    lc.numAttrs = 2;
  }
  e = cudaLaunchKernelEx(&lc, k.fn, a);
  if (e != cudaSuccess) return cuda_fail(e, "exact-sum kernel launch");
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->variant = k.variant;
    info->vec_bytes = k.vec_bytes;
    info->unroll = k.unroll;
    info->block = k.block;
    info->grid = (int32_t)g;
    info->regs_per_thread = regs;
    info->ctas_per_sm = occ;
    info->head = a.head;
    info->nvec = a.nvec;
    info->tail = a.tail;
  }
  return RD_OK;
}

rd_status launch_exact_combine(const rd_exact_record* recs, int count, int dtype, void* out,
                               rd_exact_record* rec_out, int* d_status, cudaStream_t stream) {
  if (dtype < RD_INT32 || dtype > RD_FLOAT64) { set_error("unknown dtype"); return RD_ERR_INVALID_ARG; }
  ExactCombineFn fn = lookup_exact_combine(dtype);
  if (!fn) { set_error("exact records are for float dtypes"); return RD_ERR_UNSUPPORTED; }
  if (count < 0 || (count > 0 && recs == nullptr)) { set_error("bad recs/count"); return RD_ERR_INVALID_ARG; }
  if ((uintptr_t)recs % 16) { set_error("recs must be 16-byte aligned"); return RD_ERR_MISALIGNED; }
  if (out == nullptr && rec_out == nullptr) { set_error("no output"); return RD_ERR_INVALID_ARG; }
  if (out && (uintptr_t)out % dtype_size(dtype)) { set_error("out misaligned"); return RD_ERR_MISALIGNED; }
  if (rec_out && (uintptr_t)rec_out % 8) { set_error("rec_out misaligned"); return RD_ERR_MISALIGNED; }
  fn<<<1, 128, 0, stream>>>(recs, count, record_tag(dtype, RD_SUM_EXACT), out, rec_out, d_status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "exact combine kernel launch");
  return RD_OK;
}

rd_status launch_combine(const rd_record* recs, int count, int dtype, int op, void* out,
                         rd_record* rec_out, int* d_status, cudaStream_t stream) {
  rd_status st = check_dtype_op(dtype, op);
  if (st != RD_OK) return st;
  if (is_exact_float(dtype, op)) {
    set_error("RD_SUM_EXACT on floats: use rd_combine_exact_records (the 32-byte rd_record cannot carry it)");
    return RD_ERR_UNSUPPORTED;
  }
  if (count < 0 || (count > 0 && recs == nullptr)) { set_error("bad recs/count"); return RD_ERR_INVALID_ARG; }
  if ((uintptr_t)recs % 16) { set_error("recs must be 16-byte aligned"); return RD_ERR_MISALIGNED; }
  if (out == nullptr && rec_out == nullptr) { set_error("no output"); return RD_ERR_INVALID_ARG; }
  if (out && (uintptr_t)out % (is_arg_op(op) ? 8 : dtype_size(dtype))) { set_error("out misaligned"); return RD_ERR_MISALIGNED; }
  if (rec_out && (uintptr_t)rec_out % 16) { set_error("rec_out must be 16-byte aligned"); return RD_ERR_MISALIGNED; }
  CombineFn fn = lookup_combine(dtype, op);
  if (!fn) { set_error("no combine kernel"); return RD_ERR_UNSUPPORTED; }
  fn<<<1, 32, 0, stream>>>(recs, count, record_tag(dtype, op), out, rec_out, d_status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "combine kernel launch");
  return RD_OK;
}

static void release_all_workspaces() {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : g_ws) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(kv.first.first);
    cudaFree(kv.second.partials);
    cudaSetDevice(cur);
  }
  g_ws.clear();
}

}  // namespace rd

// ====================================================================== C ABI
#ifdef RD_TIMELINE
extern "C" int rd_timeline_read(void* host, int nctas) {
  if (nctas > rd::kMaxGrid) nctas = rd::kMaxGrid;
  return (int)cudaMemcpy(host, rd::timeline_buffer(), (size_t)nctas * 8 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost);
}
extern "C" int rd_timeline_clear(void) {
  return (int)cudaMemset(rd::timeline_buffer(), 0, (size_t)rd::kMaxGrid * 8 * sizeof(unsigned long long));
}
#endif

extern "C" {

rd_status reduce(const void* x, size_t n, rd_dtype dtype, rd_op op, void* out, rd_stream_t stream) {
  return rd::launch_reduce(x, n, dtype, op, 0, out, nullptr, (cudaStream_t)stream, nullptr, nullptr);
}

rd_status reduce_partial(const void* x, size_t n, rd_dtype dtype, rd_op op, rd_record* rec,
                         rd_stream_t stream) {
  return rd::launch_reduce(x, n, dtype, op, 1, nullptr, rec, (cudaStream_t)stream, nullptr, nullptr);
}

rd_status rd_reduce_ex(const void* x, size_t n, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, const rd_config* cfg, rd_launch_info* info) {
  return rd::launch_reduce(x, n, dtype, op, 0, out, nullptr, (cudaStream_t)stream, cfg, info);
}

rd_status reduce_exact_partial(const void* x, size_t n, rd_dtype dtype, rd_exact_record* rec,
                               rd_stream_t stream) {
  return rd::launch_exact(x, n, dtype, 1, nullptr, rec, (cudaStream_t)stream, nullptr, nullptr);
}

rd_status rd_combine_exact_records(const rd_exact_record* recs, int count, rd_dtype dtype, void* out,
                                   rd_exact_record* rec_out, int* d_status, rd_stream_t stream) {
  return rd::launch_exact_combine(recs, count, dtype, out, rec_out, d_status, (cudaStream_t)stream);
}

rd_status rd_combine_records(const rd_record* recs, int count, rd_dtype dtype, rd_op op, void* out,
                             rd_record* rec_out, int* d_status, rd_stream_t stream) {
  return rd::launch_combine(recs, count, dtype, op, out, rec_out, d_status, (cudaStream_t)stream);
}

rd_status rd_identity(rd_dtype dtype, rd_op op, void* host_out) {
  rd_status st = rd::check_dtype_op(dtype, op);
  if (st != RD_OK) return st;
  if (!host_out) { rd::set_error("host_out is NULL"); return RD_ERR_INVALID_ARG; }
  if (rd::is_arg_op(op)) {
    rd_arg_result r;
    r.value = 0;
    r.index = -1;
    rd_identity(dtype, op == RD_ARGMIN ? RD_MIN : RD_MAX, &r.value);
    std::memcpy(host_out, &r, sizeof(r));
    return RD_OK;
  }
  if (op == RD_SUM_COMPENSATED || op == RD_SUM_EXACT) op = RD_SUM;
  if (dtype == RD_FLOAT32 || dtype == RD_FLOAT64) {
    const double inf = __builtin_huge_val();
    double v = op == RD_SUM ? 0.0 : op == RD_PROD ? 1.0 : op == RD_MIN ? inf : -inf;
    if (dtype == RD_FLOAT32) { float f = (float)v; std::memcpy(host_out, &f, 4); }
    else std::memcpy(host_out, &v, 8);
    return RD_OK;
  }
  const bool w64 = dtype == RD_INT64;
  uint64_t v = 0;
  switch (op) {
    case RD_PROD: v = 1; break;
    case RD_AND: v = ~0ull; break;
    case RD_MIN: v = dtype == RD_UINT32 ? 0xFFFFFFFFull : (w64 ? 0x7FFFFFFFFFFFFFFFull : 0x7FFFFFFFull); break;
    case RD_MAX: v = dtype == RD_UINT32 ? 0ull : (w64 ? 0x8000000000000000ull : 0x80000000ull); break;
    default: v = 0; break;
  }
  if (w64) std::memcpy(host_out, &v, 8);
  else { uint32_t u = (uint32_t)v; std::memcpy(host_out, &u, 4); }
  return RD_OK;
}

rd_status rd_shard_range(uint64_t n, int nranks, int rank, uint64_t* begin, uint64_t* count) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !begin || !count) {
    rd::set_error("bad shard arguments");
    return RD_ERR_INVALID_ARG;
  }
  const uint64_t W = (uint64_t)nranks, r = (uint64_t)rank;
  const uint64_t q = n / W, rem = n % W;
  *begin = r * q + (r < rem ? r : rem);
  *count = q + (r < rem ? 1 : 0);
  return RD_OK;
}

rd_status rd_release_workspaces(void) {
  rd::release_all_workspaces();
  rd::release_host_pipelines();
  return RD_OK;
}

const char* rd_status_string(rd_status s) {
  switch (s) {
    case RD_OK: return "RD_OK";
    case RD_ERR_INVALID_ARG: return "RD_ERR_INVALID_ARG";
    case RD_ERR_UNSUPPORTED: return "RD_ERR_UNSUPPORTED";
    case RD_ERR_MISALIGNED: return "RD_ERR_MISALIGNED";
    case RD_ERR_CUDA: return "RD_ERR_CUDA";
    case RD_ERR_NCCL: return "RD_ERR_NCCL";
    case RD_ERR_MISMATCH: return "RD_ERR_MISMATCH";
    case RD_ERR_TIMEOUT: return "RD_ERR_TIMEOUT";
    default: return "RD_ERR_UNKNOWN";
  }
}

const char* rd_last_error(void) { return rd::g_last_error.c_str(); }

}  // extern "C"
