// rd_kernels.cuh -- the sm_100a reduction kernels.
//
// rd_vector_kernel: single-pass persistent reduction.
//   a1  Step 1 of the two-stage reduction (Listing 1 ln042-045,
//       and the paper's unrolled Step 1): each thread walks the
//       32-byte-aligned body grid-stride ("skipping GS positions at every
//       step"), issuing U independent 256-bit non-allocating loads
//       (LDG.E.ENL2.256) before folding them into L = VB/sizeof(T) independent
//       accumulators -- the paper's unrolling factor F realised as loads in
//       flight rather than as scalar index arithmetic.
//   a2  head/tail (< VB/sizeof(T) elements each) by predicated scalar loads:
//       never out of bounds (the listing's (i<len)*x read is not reproduced).
//   a3  in-thread fold of the L lane accumulators.
//   a4  warp combine: redux.sync or a shfl_xor butterfly.
//   a5  block combine ("Step 3"): warp leaders -> smem[warp],
//       ONE __syncthreads, warp 0 folds (the barrier-free tree of P:317-326 is
//       a cross-warp race on sm_100 and is not reproduced).
//   a6  grid combine (replaces the second launch): CTA b stores its
//       partial, fences, takes an atomic ticket; the CTA that draws the last
//       ticket folds partials[0..G) in index order and resets the ticket.
//   a7  narrow Acc -> T once and store (or emit an rd_record).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rd_ops.cuh"

namespace rd {

// Fused-exchange mailbox: one per rank, in device memory that every
// rank can address (CUDA IPC over NVLink, or the same device in tests).
// Slots are double-buffered by epoch parity: a rank can be at most one
// reduction ahead of a peer (it cannot finish epoch e+1 before that peer has
// sent its e+1 record, which the peer does only after folding epoch e).
constexpr int kMaxRanks = 32;
// Records travel in "LL" form (NCCL's low-latency idea): each 8-byte word holds
// 4 bytes of the 32-byte record and the 32-bit epoch, and is written with one
// single-copy-atomic 8-byte store. A reader polls the 8 words until all carry
// the expected epoch -- no fences, no release/acquire round trips.
// Exact-sum records (rd_exact.cuh) travel the same way: 4 + 2 * 68 payload
// words {tag, n lo, n hi, flags, word[0] lo, word[0] hi, ...} per sender.
constexpr int kExactLLWords = 4 + 2 * 68;
struct Mailbox {
  unsigned long long ll[2][kMaxRanks][8];  // [epoch parity][sender][word]
  unsigned long long epoch;                // calls completed by this rank (device-side:
                                           // the exchange is CUDA-graph capturable)
  unsigned long long xll[2][kMaxRanks][kExactLLWords];   // exact records, same protocol
};

struct KArgs {
  const unsigned char* x;   // element 0
  uint64_t n;               // elements
  uint64_t head;            // elements before the VB-aligned body
  uint64_t nvec;            // VB-byte vectors in the body
  uint64_t tail_start;      // first element after the body
  uint64_t tail;            // elements after the body
  void* out;                // mode 0: one element of T (rd_arg_result for arg ops)
  rd_record* rec;           // mode 1: one record
  Slot* partials;           // gridDim.x slots (workspace)
  unsigned* ticket;         // zero between launches (workspace)
  uint32_t tag;             // record tag
  int mode;                 // 0 = value, 1 = record, 2 = fused multi-GPU exchange
  // bulk variant only: the chunk schedule (fixed by n and the base alignment)
  uint64_t chunk_bytes;     // head-region chunk size C0 (a multiple of the stage size)
  uint64_t tail_chunk_bytes;// tail-region chunk size C1 (smaller: short tail imbalance)
  uint64_t head_region_bytes;// bytes covered by the head chunks
  uint32_t nchunks;         // chunks in the body
  uint32_t nhead_chunks;    // chunks of size C0; the rest have size C1
  unsigned* work;           // dynamic chunk counter, zero between launches
  // mode 2 (fused multi-GPU exchange) only
  Mailbox* const* peers;    // device array: peers[p] = rank p's mailbox
  Mailbox* self;            // this rank's mailbox
  int* err;                 // sticky status (RD_ERR_MISMATCH / RD_ERR_TIMEOUT)
  int nranks, rank;
#ifdef RD_TIMELINE
  unsigned long long* tl;   // measurement builds: [kMaxGrid][8] %globaltimer stamps (rd_bulk.cuh)
#endif
};

// Programmatic dependent launch: a kernel launched right behind another may be
// scheduled while the previous grid drains; it must not touch global memory
// before griddepcontrol.wait (which returns once the previous grid completed
// and its writes are visible). launch_dependents lets the NEXT grid be
// scheduled early. Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// RD_TIMELINE (measurement builds only, tools/timeline.py): %globaltimer
// stamps per CTA -- 0 entry, 1 first full stage (bulk), 2 stream end, 3 the
// producer out of chunks (bulk), 4 ticket, and the last CTA's 5 fold / 6 block
// reduce / 7 output -- read back with rd_timeline_read (rd_api.cu).
#ifdef RD_TIMELINE
__device__ __forceinline__ unsigned long long rd_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RD_TL(slot) (args.tl[blockIdx.x * 8 + (slot)] = rd_gtimer())
#else
#define RD_TL(slot) ((void)0)
#endif

// Thread-block cluster primitives (sm_90+): a full cluster barrier with
// release/acquire semantics (orders shared-memory writes before the DSMEM
// reads of other CTAs), the CTA's rank and the cluster size, and a 16-byte
// load from the same shared variable in another CTA of the cluster.
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ Slot dsmem_load_slot(const Slot* local, unsigned rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(a), "r"(rank));
  unsigned long long x, y;
  asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(remote) : "memory");
  return Slot{x, y};
}

// chunk c of the bulk schedule -> [off, off + len) of the body (A: KArgs or XArgs)
template <class A>
__device__ __forceinline__ void chunk_range(const A& a, uint32_t c, uint64_t body_bytes,
                                            uint64_t* off, uint64_t* len) {
  if (c < a.nhead_chunks) {
    *off = (uint64_t)c * a.chunk_bytes;
    *len = min(a.chunk_bytes, a.head_region_bytes - *off);   // the last head chunk may be short
  } else {
    *off = a.head_region_bytes + (uint64_t)(c - a.nhead_chunks) * a.tail_chunk_bytes;
    *len = min(a.tail_chunk_bytes, body_bytes - *off);
  }
}

// ---------------------------------------------------------------- loads
template <int VB> struct Vec { uint32_t w[VB / 4]; };

// Streaming, read-only, no L1 allocation; L2 fetches a 256-byte sector group.
template <int VB>
__device__ __forceinline__ Vec<VB> ldg_stream(const unsigned char* p) {
  Vec<VB> v;
  if constexpr (VB == 32) {
    asm("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]),
          "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]), "=r"(v.w[7])
        : "l"(p));
  } else if constexpr (VB == 16) {
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3])
        : "l"(p));
  } else if constexpr (VB == 8) {
    asm("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0,%1}, [%2];"
        : "=r"(v.w[0]), "=r"(v.w[1])
        : "l"(p));
  } else {
    static_assert(VB == 4, "VB");
    asm("ld.global.nc.L1::no_allocate.L2::256B.u32 %0, [%1];" : "=r"(v.w[0]) : "l"(p));
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T ldg_scalar(const unsigned char* p) {
  return __ldg(reinterpret_cast<const T*>(p));
}

template <typename T, int VB>
__device__ __forceinline__ T lane(const Vec<VB>& v, int l) {
  if constexpr (sizeof(T) == 4) {
    uint32_t u = v.w[l];
    T t;
    memcpy(&t, &u, 4);
    return t;
  } else {
    uint64_t u = ((uint64_t)v.w[2 * l + 1] << 32) | v.w[2 * l];
    T t;
    memcpy(&t, &u, 8);
    return t;
  }
}

// ---------------------------------------------------------- block combine
template <class OpT, int B>
__device__ __forceinline__ typename OpT::Acc block_reduce(typename OpT::Acc a, typename OpT::Acc* smem) {
  static_assert(B % 32 == 0 && B <= 1024, "B");
  a = OpT::warp_reduce(a);
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if constexpr (B > 32) {
    if (ln == 0) smem[warp] = a;
    __syncthreads();
    if (warp == 0) {
      a = (ln < B / 32) ? smem[ln] : OpT::identity();
      a = OpT::warp_reduce(a);
    }
  }
  return a;  // valid in thread 0
}

template <class OpT>
__device__ __forceinline__ void finish(const typename OpT::Acc& a, const KArgs& args) {
  if (args.mode == 0) {
    if (args.n == 0) OpT::store_empty(args.out);
    else OpT::store(a, args.out);
  } else {
    Slot s = OpT::pack(a);
    args.rec->tag = args.tag;
    args.rec->status = 0;
    args.rec->n = args.n;
    args.rec->acc[0] = s.a;
    args.rec->acc[1] = s.b;
  }
}

// Fold `count` records in INDEX order with one warp: lanes load 32 records at
// a time in parallel (one memory round trip per 32), then every lane folds
// them sequentially from shuffles (same order, same result in every lane).
// Indexed ops shift each record's indices by the n of the records before it.
template <class OpT, class Load>
__device__ __forceinline__ void fold_records_warp(int count, uint32_t tag, Load load, typename OpT::Acc* acc_out,
                                                  uint64_t* n_out, bool* bad_out) {
  using Acc = typename OpT::Acc;
  const int ln = threadIdx.x & 31;
  Acc a = OpT::identity();
  uint64_t n = 0;
  bool bad = false;
  for (int base = 0; base < count; base += 32) {
    uint32_t t = 0;
    uint64_t rn = 0, a0 = 0, a1 = 0;
    if (base + ln < count) load(base + ln, &t, &rn, &a0, &a1);
    const int m = min(32, count - base);
    for (int j = 0; j < m; ++j) {
      const uint32_t tj = __shfl_sync(0xffffffffu, t, j);
      const uint64_t nj = shfl_idx_u64(rn, j), x0 = shfl_idx_u64(a0, j), x1 = shfl_idx_u64(a1, j);
      if (tj != tag) { bad = true; continue; }
      a = OpT::combine(a, shifted<OpT>(OpT::unpack(Slot{x0, x1}), n));
      n += nj;
    }
  }
  *acc_out = a;
  *n_out = n;
  *bad_out = bad;
}

// a8 fused into the kernel: warp 0 of the last CTA pushes this
// rank's record into slot [epoch&1][rank] of every peer's mailbox (peer
// stores over NVLink) as 8 self-validating 8-byte words {payload, epoch},
// polls its own mailbox until the W records of this epoch are complete, and
// folds them in RANK ORDER -- every rank computes the identical result, with
// no host call, no second kernel and no memory fence. A bounded wait reports
// RD_ERR_TIMEOUT.
template <class OpT>
__device__ __forceinline__ void fused_exchange(typename OpT::Acc a, const KArgs& args) {
  const int ln = threadIdx.x & 31;
  Slot s = OpT::pack(a);                               // valid in lane 0
  s.a = __shfl_sync(0xffffffffu, s.a, 0);
  s.b = __shfl_sync(0xffffffffu, s.b, 0);
  // this call's epoch: calls on one rank are stream-ordered, so the counter in
  // its own mailbox is read and bumped without races
  const unsigned long long epoch = *(volatile unsigned long long*)&args.self->epoch + 1;
  const int par = (int)(epoch & 1);
  const unsigned long long eflag = (unsigned long long)(uint32_t)epoch << 32;
  const int W = args.nranks;
  // the record as 8 x 32-bit payload words: {tag, status=0, n lo, n hi, a lo, a hi, b lo, b hi}
  uint32_t w[8] = {args.tag, 0u, (uint32_t)args.n, (uint32_t)(args.n >> 32),
                   (uint32_t)s.a, (uint32_t)(s.a >> 32), (uint32_t)s.b, (uint32_t)(s.b >> 32)};
  for (int p = ln; p < W; p += 32) {
    volatile unsigned long long* dst = args.peers[p]->ll[par][args.rank];
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[k] = eflag | w[k];   // peer store over NVLink (or local)
  }
  bool timeout = false;
  uint32_t got[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int q = ln; q < W; q += 32) {
    const volatile unsigned long long* src = args.self->ll[par][q];
    uint32_t spins = 0;
    for (;;) {
      bool all = true;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const unsigned long long v = src[k];
        got[k] = (uint32_t)v;
        all = all && ((v & 0xffffffff00000000ull) == eflag);
      }
      if (all) break;
      if (++spins > 4096) __nanosleep(128);           // tight spin first, then back off
      if (spins > (1u << 25)) { timeout = true; break; }
    }
  }  timeout = __any_sync(0xffffffffu, timeout);
  using Acc = typename OpT::Acc;
  Acc acc = OpT::identity();
  uint64_t nn = 0;
  bool bad = false;
  if (!timeout) {
    // lane q already holds record q (its 8 payload words)
    fold_records_warp<OpT>(W, args.tag, [&](int, uint32_t* t, uint64_t* n, uint64_t* a0, uint64_t* a1) {
      *t = got[0];
      *n = ((uint64_t)got[3] << 32) | got[2];
      *a0 = ((uint64_t)got[5] << 32) | got[4];
      *a1 = ((uint64_t)got[7] << 32) | got[6];
    }, &acc, &nn, &bad);
  }
  if (ln == 0) {
    if (timeout) atomicExch(args.err, (int)RD_ERR_TIMEOUT);
    else if (bad) atomicExch(args.err, (int)RD_ERR_MISMATCH);
    if (timeout || bad || nn == 0) OpT::store_empty(args.out);
    else OpT::store(acc, args.out);
    *(volatile unsigned long long*)&args.self->epoch = epoch;
  }
}

// the end of every reduce kernel: warp 0 of the finishing CTA, result in lane 0
template <class OpT>
__device__ __forceinline__ void finish_warp0(const typename OpT::Acc& a, const KArgs& args) {
  if (args.mode == 2) fused_exchange<OpT>(a, args);
  else if ((threadIdx.x & 31) == 0) finish<OpT>(a, args);
}

// Thread t folds slots t, t+B, t+2B, ... in increasing order (a fixed tree);
// NF independent loads in flight per thread (the bulk kernel's last CTA: 16,
// one L2 round trip for up to 16 * B chunk slots).
template <class OpT, int B, int NF = 8>
__device__ __forceinline__ typename OpT::Acc fold_slots(const Slot* slots, uint32_t count) {
  using Acc = typename OpT::Acc;
  Acc b = OpT::identity();
  for (uint32_t j0 = threadIdx.x; j0 < count; j0 += NF * B) {
    ulonglong2 v[NF];
#pragma unroll
    for (int k = 0; k < NF; ++k) {
      const uint32_t j = j0 + k * B;
      v[k] = (j < count) ? __ldcg(reinterpret_cast<const ulonglong2*>(slots + j)) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int k = 0; k < NF; ++k)
      if (j0 + k * B < count) b = OpT::combine(b, OpT::unpack(Slot{v[k].x, v[k].y}));
  }
  return b;
}

// a6 ticket, drawn by thread 0 after a CTA barrier: ONE gpu-scope acq_rel
// atomic. Its release covers every write the CTA made before the barrier
// (release is cumulative through bar.sync); its acquire, followed by the next
// barrier, orders the other CTAs' released writes before every thread's
// later loads -- the fence + atomic + fence of the classic last-block
// pattern in one operation (RD_TICKET_FENCES restores that form for A/B).
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* p) {
#ifdef RD_TICKET_FENCES
  __threadfence();
  const unsigned r = atomicAdd(p, 1u);
  __threadfence();
  return r;
#else
  unsigned r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(r) : "l"(p) : "memory");
  return r;
#endif
}

// a6 for 32-bit integer + (PackedSum32): thread 0 adds {a << 32 | 1} to the
// 64-bit word at the ticket. The vector kernels read no other CTA's memory --
// the total arrives in the atomic's return value -- so relaxed suffices (the
// reset is ordered after every add by the word's own coherence order); the
// bulk kernel (ACQ_REL) also orders every producer's chunk-counter atomics
// before the last CTA resets that counter. Returns true in the last CTA's
// thread 0 with *total = the grid's sum; that thread has reset the word.
#ifndef RD_NO_PACKED_SUM
#define RD_PACKED_SUM 1
#else
#define RD_PACKED_SUM 0
#endif
template <bool ACQ_REL = false>
__device__ __forceinline__ bool packed_arrive(unsigned* ticket, uint32_t a, uint32_t* total) {
  unsigned long long old;
  const unsigned long long add = ((unsigned long long)a << 32) | 1ull;
  if constexpr (ACQ_REL)
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(ticket), "l"(add) : "memory");
  else
    asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(ticket), "l"(add) : "memory");
  if ((uint32_t)old != gridDim.x - 1) return false;
  *total = (uint32_t)(old >> 32) + a;
  *reinterpret_cast<unsigned long long*>(ticket) = 0ull;   // reusable by the next launch
  return true;
}

// a6: one partial per CTA, the last CTA to arrive folds them in index order.
template <class OpT, int B>
__device__ __forceinline__ void grid_combine(typename OpT::Acc a, const KArgs& args,
                                             typename OpT::Acc* smem) {
  using Acc = typename OpT::Acc;
  if (gridDim.x == 1) {
    if (threadIdx.x < 32) finish_warp0<OpT>(a, args);
    return;
  }
  if constexpr (RD_PACKED_SUM && PackedSum32<OpT>::value) {
    __shared__ unsigned s_done;
    __shared__ uint32_t s_total;
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      s_done = packed_arrive(args.ticket, a, &tot);
      s_total = tot;
      RD_TL(4);
    }
    __syncthreads();
    if (!s_done) return;
    if (threadIdx.x < 32) finish_warp0<OpT>(s_total, args);
    if (threadIdx.x == 0) RD_TL(7);
    return;
  }
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    Slot s = OpT::pack(a);
    __stcg(reinterpret_cast<ulonglong2*>(args.partials + blockIdx.x), make_ulonglong2(s.a, s.b));
    const unsigned t = ticket_acq_rel(args.ticket);    // release the partial, acquire the others
    s_last = (t == gridDim.x - 1);
    RD_TL(4);
  }
  __syncthreads();
  if (!s_last) return;
  Acc b = fold_slots<OpT, B>(args.partials, gridDim.x);
  if (threadIdx.x == 0) RD_TL(5);
  b = block_reduce<OpT, B>(b, smem);
  if (threadIdx.x == 0) {
    RD_TL(6);
    *args.ticket = 0u;                                 // reusable by the next launch
  }
  if (threadIdx.x < 32) finish_warp0<OpT>(b, args);
  if (threadIdx.x == 0) RD_TL(7);
}

// ---------------------------------------------------------------- a1-a5
// The vector kernels' body: a1-a3 per thread, a2 stragglers, a4-a5 block
// combine. Returns the CTA's partial (valid in thread 0).
template <class OpT, int B, int U, int VB>
__device__ __forceinline__ typename OpT::Acc vector_body(const KArgs& args, typename OpT::Acc* smem) {
  using T = typename OpT::T;
  using Acc = typename OpT::Acc;
  constexpr int L = VB / (int)sizeof(T);
  static_assert(L >= 1, "vector narrower than the element");

  using LO = LaneOps<OpT>;
  typename LO::Lane acc[L];
#pragma unroll
  for (int l = 0; l < L; ++l) acc[l] = LO::identity();

  const uint64_t tid = (uint64_t)blockIdx.x * B + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * B;
  const unsigned char* body = args.x + args.head * sizeof(T);
  pdl_wait();
  if (threadIdx.x == 0) RD_TL(0);
  const uint64_t nvec = args.nvec;
  uint64_t i = tid;
  uint32_t step = 0;   // vector slot tid + step*stride (indexed ops only)
  if constexpr (U > 1) {
    for (; i + (uint64_t)(U - 1) * stride < nvec; i += (uint64_t)U * stride, step += U) {
      Vec<VB> v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldg_stream<VB>(body + (i + (uint64_t)u * stride) * VB);
      T xs[U][L];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int l = 0; l < L; ++l) xs[u][l] = lane<T, VB>(v[u], l);
      LO::fold_vecs(acc, xs, step);
    }
  }
  for (; i < nvec; i += stride, ++step) {
    Vec<VB> v = ldg_stream<VB>(body + i * VB);
    T xs[1][L];
#pragma unroll
    for (int l = 0; l < L; ++l) xs[0][l] = lane<T, VB>(v, l);
    LO::fold_vecs(acc, xs, step);
  }
  pdl_trigger();
  // a3: lanes -> one accumulator (indexed ops: element index = head + (tid + step*stride)*L + lane)
  Acc a = LO::finish(acc, [&](uint32_t st, uint32_t ln) { return args.head + (tid + (uint64_t)st * stride) * L + ln; });
  // a2: head and tail stragglers
  if (tid < args.head) a = fold_at<OpT>(a, ldg_scalar<T>(args.x + tid * sizeof(T)), tid);
  if (tid < args.tail)
    a = fold_at<OpT>(a, ldg_scalar<T>(args.x + (args.tail_start + tid) * sizeof(T)), args.tail_start + tid);
  // a4, a5
  return block_reduce<OpT, B>(a, smem);
}

// a1-a7: the single-pass persistent grid (a6 by the last CTA's atomic ticket)
template <class OpT, int B, int U, int VB>
__global__ void __launch_bounds__(B, 1) rd_vector_kernel(const KArgs args) {
  __shared__ typename OpT::Acc smem[32];
  typename OpT::Acc a = vector_body<OpT, B, U, VB>(args, smem);
  if (threadIdx.x == 0) RD_TL(2);
  __syncthreads();  // smem is reused by the grid combine
  grid_combine<OpT, B>(a, args, smem);
}

// a1-a7 for small inputs (2..16 CTAs): the grid is ONE thread-block cluster,
// and a6 happens in distributed shared memory -- each CTA leaves its partial
// in its own shared memory, one cluster barrier, and warp 0 of rank 0 reads
// the G partials over DSMEM (in rank order: deterministic) and folds them. No
// workspace slot, no global fence or atomic ticket: those cost ~1.6 us per
// launch at 64 KB - 512 KB (tools/sweep.py sizes: a 2-CTA ticketed grid at
// 2^14 float32 took 3.0 us in a CUDA graph against 1.4 us for one CTA).
template <class OpT, int B, int U, int VB>
__global__ void __launch_bounds__(B, 1) rd_cluster_kernel(const KArgs args) {
  using Acc = typename OpT::Acc;
  __shared__ Acc smem[32];
  __shared__ __align__(16) Slot cpart;
  Acc a = vector_body<OpT, B, U, VB>(args, smem);
  if (threadIdx.x == 0) cpart = OpT::pack(a);
  cluster_sync();
  if (cluster_ctarank() == 0 && threadIdx.x < 32) {
    const unsigned G = cluster_nctarank();
    const int ln = threadIdx.x & 31;
    Slot mine{0, 0};
    if ((unsigned)ln < G) mine = dsmem_load_slot(&cpart, (unsigned)ln);
    Acc b = OpT::identity();
    for (unsigned j = 0; j < G; ++j) {
      const Slot q{shfl_idx_u64(mine.a, (int)j), shfl_idx_u64(mine.b, (int)j)};
      b = OpT::combine(b, OpT::unpack(q));
    }
    finish_warp0<OpT>(b, args);
  }
  cluster_sync();   // the other CTAs' shared memory stays alive until rank 0 has read it
}

// PAPER.md Listing "Unrolling the step 1", transcribed: work-item
// g reads the F CONSECUTIVE elements iPos..iPos+F-1, iPos = g*F + k*GS*F.
// The listing's algebraic mask (i<len)*x is replaced by predication
// with the op's identity (the mask reads out of bounds and is not an identity
// for x/min/max or for inf/NaN). Used for the F-sweep ablation.
template <class OpT, int B, int F>
__global__ void __launch_bounds__(B) rd_paper_kernel(const KArgs args) {
  using T = typename OpT::T;
  using Acc = typename OpT::Acc;
  __shared__ Acc smem[32];
  Acc acc = OpT::identity();
  const uint64_t gid = (uint64_t)blockIdx.x * B + threadIdx.x;
  const uint64_t gs = (uint64_t)gridDim.x * B;
  const T* x = reinterpret_cast<const T*>(args.x);
  const uint64_t n = args.n;
  pdl_wait();
  for (uint64_t pos = gid * F; pos < n; pos += gs * F) {
    T v[F];
#pragma unroll
    for (int k = 0; k < F; ++k) v[k] = (pos + k < n) ? __ldg(x + pos + k) : T{};
    if constexpr (Blocked<OpT>::value) {   // the F elements as one tree (FloatSum)
#pragma unroll
      for (int k = 0; k < F; ++k) v[k] = (pos + k < n) ? v[k] : (T)(-0.0);
      add_blocks<OpT, F>(acc, v);
    } else {
#pragma unroll
      for (int k = 0; k < F; ++k)
        if (pos + k < n) acc = fold_at<OpT>(acc, v[k], pos + k);
    }
  }
  acc = block_reduce<OpT, B>(acc, smem);
  __syncthreads();
  grid_combine<OpT, B>(acc, args, smem);
}

// ------------------------------------------------------ record combine (N4)
// Folds records in index order with one thread (count is the number of ranks
// or chunks: small); checks every tag.
template <class OpT>
__global__ void rd_combine_kernel(const rd_record* recs, int count, uint32_t tag, void* out,
                                  rd_record* rec_out, int* d_status) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  using Acc = typename OpT::Acc;
  Acc a;
  uint64_t n;
  bool bad;
  fold_records_warp<OpT>(count, tag, [&](int r, uint32_t* t, uint64_t* rn, uint64_t* a0, uint64_t* a1) {
    const ulonglong2 h = __ldcg(reinterpret_cast<const ulonglong2*>(recs + r));       // {tag|status, n}
    const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(recs + r) + 1);   // acc[0..1]
    *t = (uint32_t)h.x;
    *rn = h.y;
    *a0 = v.x;
    *a1 = v.y;
  }, &a, &n, &bad);
  if (threadIdx.x != 0) return;
  if (bad && d_status) *d_status = (int)RD_ERR_MISMATCH;
  if (out) {
    if (n == 0 || bad) OpT::store_empty(out);
    else OpT::store(a, out);
  }
  if (rec_out) {
    Slot s = OpT::pack(a);
    rec_out->tag = tag;
    rec_out->status = bad ? (uint32_t)RD_ERR_MISMATCH : 0u;
    rec_out->n = n;
    rec_out->acc[0] = s.a;
    rec_out->acc[1] = s.b;
  }
}

}  // namespace rd
