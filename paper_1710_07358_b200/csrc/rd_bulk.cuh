// rd_bulk.cuh -- the bulk-copy pipeline variant of Step 1 (the
// "optional TMA or cp.async.bulk shared-memory staging pipeline" of the north
// star).
//
// One persistent CTA per SM = 1 producer warp + CW consumer warps.
//  producer (one elected lane): takes the next CHUNK of the 16-byte-aligned
//    body from a global counter (dynamic scheduling: faster SMs take more
//    chunks, which removes the static partition's tail), and streams it into
//    a STAGES-deep shared-memory ring with cp.async.bulk (UBLKCP), one
//    mbarrier per stage carrying the transaction bytes.
//  consumers: wait on the stage's mbarrier, LDS.128 their fixed slice of the
//    stage, fold into lane accumulators, release the stage. Float + and x
//    (whose bits depend on the evaluation order): at the end of a chunk the
//    CTA reduces the chunk to ONE partial, stored at partials[chunk] -- so the
//    result does not depend on which CTA took which chunk: the reduction tree
//    is fixed by n and the base alignment alone (deterministic, like the
//    vector variant). Order-free ops (integers, float min/max, arg ops; any
//    order gives the same result): the lanes run on across chunks (arg ops
//    fold each chunk's lane bests into a per-thread running best with global
//    indices), one partial per CTA at the end -- no per-chunk block
//    reduction, and the last CTA folds gridDim.x slots, not nchunks.
//  last CTA (atomic ticket): folds the slots in index order plus the
//    head/tail stragglers, writes the result, resets ticket and counter.
// In-flight bytes per SM are STAGES * STAGE_BYTES of shared memory (up to
// 192 KB) instead of registers.
#pragma once
#include "rd_kernels.cuh"

namespace rd {

// Releasing a ring stage: the consumers' generic-proxy READS of the stage are
// ordered before the producer's next async-proxy WRITE (cp.async.bulk) by the
// mbarrier alone -- arrive (release) on EMPTY, the producer's try_wait
// (acquire), then the copy -- as in CUTLASS's consumer_release for TMA-load
// pipelines (a proxy fence is needed for generic WRITES read by the async
// proxy, e.g. before a TMA store). The fence.proxy.async that used to precede
// the arrive cost 1.2-2.3% on the ALU-heavier ops and 5.5% on the exact sum
// (an A/B of builds, profiles/ab/r01_ab_release_fence.jsonl); define
// RD_RELEASE_PROXY_FENCE to restore it.
#ifdef RD_RELEASE_PROXY_FENCE
#define RD_RELEASE_FENCE() asm volatile("fence.proxy.async.shared::cta;" ::: "memory")
#else
#define RD_RELEASE_FENCE() ((void)0)
#endif

// Releasing a stage: every consumer thread arrives on the stage's EMPTY
// barrier itself (count 32 * CW), after reading the stage and its metadata,
// so each reader's own arrive (release) orders its reads before the
// producer's next write into the stage -- the form compute-sanitizer's
// racecheck follows (0 hazards; lane 0 arriving for its warp after
// __syncwarp, count CW, is correct too but racecheck does not see it as
// ordering the other lanes' reads). An A/B of both (profiles/ab/
// r02_ab_arrive_all.jsonl) shows no throughput difference;
// RD_ARRIVE_WARP restores the per-warp arrive.
#ifndef RD_ARRIVE_WARP
#define RD_EMPTY_COUNT(CW) (32 * (CW))
#define RD_RELEASE_STAGE(bar) \
  do {                        \
    __syncwarp();             \
    RD_RELEASE_FENCE();       \
    mbar_arrive(bar);         \
  } while (0)
#else
#define RD_EMPTY_COUNT(CW) (CW)
#define RD_RELEASE_STAGE(bar)        \
  do {                               \
    __syncwarp();                    \
    if ((threadIdx.x & 31) == 0) {   \
      RD_RELEASE_FENCE();            \
      mbar_arrive(bar);              \
    }                                \
  } while (0)
#endif

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "RD_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra RD_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int STAGES, int STAGE_BYTES, int CW>
struct BulkSmem {
  static constexpr int kRing = STAGES * STAGE_BYTES;
  static constexpr int kBytes = kRing + 2048;   // ring + barriers + stage metadata + partials (< 1 KB)
};

template <class OpT, int STAGES, int STAGE_BYTES, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1) rd_bulk_kernel(const KArgs args) {
  using T = typename OpT::T;
  using Acc = typename OpT::Acc;
  constexpr int CT = 32 * CW;                          // consumer threads
  constexpr int L = 16 / (int)sizeof(T);               // lanes per 16-byte vector
  constexpr int PER_THREAD = STAGE_BYTES / (16 * CT);  // LDS.128 per thread per stage
  static_assert(STAGE_BYTES % (16 * CT) == 0, "stage must split evenly over consumer threads");
  constexpr int B = 32 * (CW + 1);
#ifdef RD_BULK_CHUNK_PARTIALS
  constexpr bool kCtaPartial = false;   // (A/B builds) a fixed-tree partial per chunk for every op
#else
  constexpr bool kCtaPartial = OrderFree<OpT>::value;
#endif

  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* st_off = empty + STAGES;                  // body byte offset of each stage
  int32_t* st_chunk = reinterpret_cast<int32_t*>(st_off + STAGES);
  uint32_t* st_bytes = reinterpret_cast<uint32_t*>(st_chunk + STAGES);
  uint32_t* st_last = st_bytes + STAGES;
  Acc* wpart = reinterpret_cast<Acc*>(reinterpret_cast<uintptr_t>(st_last + STAGES + 3) & ~(uintptr_t)15);  // [2][CW]
  __shared__ Acc red[32];

  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], RD_EMPTY_COUNT(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const unsigned char* body = args.x + args.head * sizeof(T);
  const uint64_t body_bytes = args.nvec * 16;
  constexpr bool kPacked = RD_PACKED_SUM && PackedSum32<OpT>::value;
  Acc cta_part = OpT::identity();   // kPacked: the CTA's partial, in thread 0
  pdl_wait();
  if (threadIdx.x == 0) RD_TL(0);

  if (warp == CW) {
    // ---------------------------------------------------------------- producer
    if (ln == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      // the first chunk is static (no atomic on the critical path at start);
      // later claims come from the counter, offset by the grid, and the next
      // claim is issued before the current chunk is streamed (latency hidden)
      uint32_t c = blockIdx.x;
      uint32_t next = atomicAdd(args.work, 1u) + gridDim.x;
      for (;; c = next, next = atomicAdd(args.work, 1u) + gridDim.x) {
        if (c >= args.nchunks) {
          RD_TL(3);
          mbar_wait(&empty[stage], phase ^ 1);
          st_chunk[stage] = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        uint64_t cbeg, clen;
        chunk_range(args, c, body_bytes, &cbeg, &clen);
        const uint64_t cend = cbeg + clen;
        for (uint64_t off = cbeg; off < cend; off += STAGE_BYTES) {
          const uint32_t bytes = (uint32_t)min((uint64_t)STAGE_BYTES, cend - off);
          mbar_wait(&empty[stage], phase ^ 1);
          st_chunk[stage] = (int32_t)c;
          st_off[stage] = off;
          st_bytes[stage] = bytes;
          st_last[stage] = (off + bytes == cend);
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(ring + (size_t)stage * STAGE_BYTES, body + off, bytes, &full[stage], pol);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- consumers
    const int t = threadIdx.x;  // 0 .. CT-1
    using LO = LaneOps<OpT>;
    typename LO::Lane acc[L];
    Acc run = OpT::identity();   // indexed order-free ops: this thread's best over its finished chunks
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] = LO::identity();
    int stage = 0;
    uint32_t phase = 0, nchunk_local = 0;
    uint32_t cstage = 0;   // stage number within the current chunk
    const uint32_t ring_addr = smem_addr(ring);
#ifdef RD_TIMELINE
    bool first = true;
#endif
    for (;;) {
      mbar_wait(&full[stage], phase);
#ifdef RD_TIMELINE
      if (first && t == 0) RD_TL(1);
      first = false;
#endif
      const int32_t c = st_chunk[stage];
      if (c < 0) {
        if (t == 0) RD_TL(2);
        break;
      }
      const uint32_t bytes = st_bytes[stage];
      const uint32_t last = st_last[stage];
      const uint32_t base = ring_addr + stage * STAGE_BYTES;
      const uint32_t step0 = cstage * PER_THREAD;   // steps grow with the element index
      if (bytes == STAGE_BYTES) {
        uint4 v[PER_THREAD];
#pragma unroll
        for (int k = 0; k < PER_THREAD; ++k) v[k] = lds128(base + (k * CT + t) * 16);
        T xs[PER_THREAD][L];
#pragma unroll
        for (int k = 0; k < PER_THREAD; ++k) {
          Vec<16> w{{v[k].x, v[k].y, v[k].z, v[k].w}};
#pragma unroll
          for (int l = 0; l < L; ++l) xs[k][l] = lane<T, 16>(w, l);
        }
        LO::fold_vecs(acc, xs, step0);
      } else if constexpr (Blocked<OpT>::value) {
        // a short stage (the chunk's last): missing vectors are the identity
        // -0.0, so the block tree is the same as for a full stage
        T xs[PER_THREAD][L];
#pragma unroll
        for (int k = 0; k < PER_THREAD; ++k) {
          const uint32_t off = (k * CT + t) * 16;
          uint4 q = make_uint4(0, 0, 0, 0);
          if (off < bytes) q = lds128(base + off);
          Vec<16> w{{q.x, q.y, q.z, q.w}};
#pragma unroll
          for (int l = 0; l < L; ++l) xs[k][l] = off < bytes ? lane<T, 16>(w, l) : (T)(-0.0);
        }
        LO::fold_vecs(acc, xs, step0);
      } else {
#pragma unroll
        for (int k = 0; k < PER_THREAD; ++k) {
          const uint32_t off = (k * CT + t) * 16;
          if (off < bytes) {
            uint4 q = lds128(base + off);
            Vec<16> w{{q.x, q.y, q.z, q.w}};
            T xs[L];
#pragma unroll
            for (int l = 0; l < L; ++l) xs[l] = lane<T, 16>(w, l);
            LO::fold_vec(acc, xs, step0 + k);
          }
        }
      }
      // release the stage: this thread's reads of the ring (and of the stage
      // metadata) are ordered before the producer's next cp.async.bulk write
      // into it by its mbarrier arrive (release; RD_RELEASE_FENCE)
      RD_RELEASE_STAGE(&empty[stage]);
      ++cstage;
      if (kCtaPartial) {
        if (last) {
          if constexpr (OpT::kIndexed) {
            // the chunk's lane bests with their global indices into the running best
            uint64_t coff = 0, clen = 0;
            chunk_range(args, (uint32_t)c, body_bytes, &coff, &clen);
            const uint64_t e_chunk = args.head + coff / sizeof(T);
            run = OpT::combine(run, LO::finish(acc, [&](uint32_t st, uint32_t ln) {
              return e_chunk + ((uint64_t)(st / PER_THREAD) * (STAGE_BYTES / 16) + (st % PER_THREAD) * CT + t) * L + ln;
            }));
#pragma unroll
            for (int l = 0; l < L; ++l) acc[l] = LO::identity();
          }
          cstage = 0;
        }
      } else if (last) {
        // the chunk's partial: fixed tree over (thread, lane) -> independent of the schedule
        uint64_t coff = 0, clen = 0;
        if constexpr (OpT::kIndexed) chunk_range(args, (uint32_t)c, body_bytes, &coff, &clen);
        const uint64_t e_chunk = args.head + coff / sizeof(T);
        Acc a = LO::finish(acc, [&](uint32_t st, uint32_t ln) {
          return e_chunk + ((uint64_t)(st / PER_THREAD) * (STAGE_BYTES / 16) + (st % PER_THREAD) * CT + t) * L + ln;
        });
        a = OpT::warp_reduce(a);
        Acc* wp = wpart + (nchunk_local & 1) * CW;
        if (ln == 0) wp[warp] = a;
        named_sync(1, CT);
        if (warp == 0) {
          Acc b = (ln < CW) ? wp[ln] : OpT::identity();
          b = OpT::warp_reduce(b);
          if (ln == 0) {
            Slot s = OpT::pack(b);
            __stcg(reinterpret_cast<ulonglong2*>(args.partials + c), make_ulonglong2(s.a, s.b));
          }
        }
        ++nchunk_local;
        cstage = 0;
#pragma unroll
        for (int l = 0; l < L; ++l) acc[l] = LO::identity();
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (kCtaPartial) {
      // order-free ops: the CTA's one partial (identity if it took no chunk)
      Acc a;
      if constexpr (OpT::kIndexed) a = run;
      else a = LO::finish(acc, [](uint32_t, uint32_t) { return (uint64_t)0; });
      a = OpT::warp_reduce(a);
      if (ln == 0) wpart[warp] = a;
      named_sync(1, CT);
      if (warp == 0) {
        Acc b = (ln < CW) ? wpart[ln] : OpT::identity();
        b = OpT::warp_reduce(b);
        if (ln == 0) {
          if constexpr (kPacked) {
            cta_part = b;
          } else {
            Slot s = OpT::pack(b);
            __stcg(reinterpret_cast<ulonglong2*>(args.partials + blockIdx.x), make_ulonglong2(s.a, s.b));
          }
        }
      }
    }
  }
  // ------------------------------------------------------------------ grid combine
  pdl_trigger();
  __syncthreads();
  if constexpr (kPacked) {
    // 32-bit integer +: the total from the arrival atomic itself (no slots)
    __shared__ unsigned s_done;
    __shared__ uint32_t s_total;
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      s_done = packed_arrive<true>(args.ticket, cta_part, &tot);
      s_total = tot;
      if (s_done) *args.work = 0u;
      RD_TL(4);
    }
    __syncthreads();
    if (!s_done) return;
    if (threadIdx.x < 32) {   // warp 0: the total + the head / tail stragglers (< 4 each)
      Acc b = threadIdx.x == 0 ? (Acc)s_total : OpT::identity();
      if (threadIdx.x < args.head) b = fold_at<OpT>(b, ldg_scalar<T>(args.x + threadIdx.x * sizeof(T)), threadIdx.x);
      if (threadIdx.x < args.tail)
        b = fold_at<OpT>(b, ldg_scalar<T>(args.x + (args.tail_start + threadIdx.x) * sizeof(T)),
                         args.tail_start + threadIdx.x);
      b = OpT::warp_reduce(b);
      finish_warp0<OpT>(b, args);
    }
    if (threadIdx.x == 0) RD_TL(7);
    return;
  }
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    // release this CTA's chunk partials (all stored by this thread), acquire the others'
    const unsigned tk = ticket_acq_rel(args.ticket);
    s_last = (tk == gridDim.x - 1);
    RD_TL(4);
  }
  __syncthreads();
  if (!s_last) return;
  Acc b = fold_slots<OpT, B, 16>(args.partials, kCtaPartial ? gridDim.x : args.nchunks);
  if (threadIdx.x == 0) RD_TL(5);
  if (threadIdx.x < args.head) b = fold_at<OpT>(b, ldg_scalar<T>(args.x + threadIdx.x * sizeof(T)), threadIdx.x);
  if (threadIdx.x < args.tail)
    b = fold_at<OpT>(b, ldg_scalar<T>(args.x + (args.tail_start + threadIdx.x) * sizeof(T)),
                     args.tail_start + threadIdx.x);
  b = block_reduce<OpT, B>(b, red);
  if (threadIdx.x == 0) {
    RD_TL(6);
    *args.ticket = 0u;
    *args.work = 0u;
  }
  if (threadIdx.x < 32) finish_warp0<OpT>(b, args);
  if (threadIdx.x == 0) RD_TL(7);
}

}  // namespace rd
