/*
 * b200reduce.h -- C ABI of the B200-native (sm_100a) reduction library.
 *
 * The operation (§1.1 "Problem Definition"):
 *   "Given a set X with n values, X = {x_0, x_1, ..., x_{n-1}}, compute
 *    x_0 (x) x_1 (x) ... (x) x_{n-1}. The associative operator (x) ... can be
 *    (but is not limited to) any one of the set {+, x, AND, OR, XOR, ..., max, min}."
 * evaluated in any order, which associativity and commutativity allow
 * (P:42-50); the result for an empty X is the initial accumulator of
 * Algorithm 1 "Summation(A)" (`accumulator <- 0`; INFINITY for min,
 * Listing 1 ln041).
 *
 * The GPU structure follows the two-stage reduction with the
 * paper's unrolled persistent-thread Step 1, re-designed for
 * sm_100a: one single-pass launch whose grid-level combine ("Stage 2")
 * is done by the last CTA to finish, through an atomic ticket.
 *
 * Conventions for every entry point
 *  - All functions return rd_status; no C++ exception crosses the ABI.
 *  - Arguments are validated synchronously BEFORE anything is enqueued; a call
 *    that returns an error enqueued nothing and left every output untouched.
 *  - Device entry points are asynchronous and stream-ordered on `stream`
 *    (a cudaStream_t; NULL = the legacy default stream). They never
 *    synchronise the host and are capturable in CUDA graphs once the
 *    per-(device, stream) workspace exists (it is created by the first call
 *    on that stream, outside capture). A captured graph keeps the capture
 *    stream's workspace: do not replay it concurrently with other calls that
 *    use that workspace (eager calls on the capture stream, or another graph
 *    captured on the same stream) -- they would share one ticket.
 *  - Element-aligned base pointers are required (x % sizeof(dtype) == 0,
 *    else RD_ERR_MISALIGNED); any element offset is valid.
 *  - Bitwise ops (AND/OR/XOR) on float dtypes -> RD_ERR_UNSUPPORTED.
 *  - n == 0 writes the empty result (table below) and returns RD_OK.
 *  - For RD_ARGMIN / RD_ARGMAX every `out` below points to an rd_arg_result
 *    (8-byte aligned) instead of one element.
 *
 * Results:
 *  - integers: + and x wrap modulo 2^w; min/max signed for int32/int64,
 *    unsigned for uint32; AND/OR/XOR on raw bits. Bit-exact for any order.
 *  - float min/max: IEEE 754-2019 minimum/maximum (NaN propagates as a quiet
 *    NaN, -0.0 < +0.0). Bit-exact.
 *  - float +: blocked pairwise summation in a fixed order -- each thread sums
 *    the <= 32 elements it loads per iteration as a balanced tree in the
 *    input precision and adds the block sums into a wide accumulator (fp64
 *    for fp32 data, double-double for fp64 data), in which every later
 *    combine happens; one rounding at the end. For EVERY input whose partial
 *    sums stay finite (e.g. sum|x_i| <= the dtype's largest finite value):
 *    |result - exact| <= 3.01 * eps(dtype) * sum|x_i|, inside the north-star
 *    bound 4 * eps * sum|x_i| (R6). A zero sum is -0.0 iff every
 *    x_i is -0.0; empty -> +0.0.
 *  - float x: fp32 accumulates in fp64, fp64 in double-double, then one
 *    rounding; |result - exact| <= 4 * eps(dtype) * |exact| when no partial
 *    product over/underflows.
 *  - float exact sum (RD_SUM_EXACT): the real sum rounded once -- the same
 *    bits for every grid, variant, base alignment, shard split and GPU count.
 *  - Determinism: identical (x, n, base alignment, dtype, op, device) give
 *    identical bits (no float atomics; every combine is in a fixed order).
 *
 *  empty results:   +   x    min          max          and   or  xor   (+ compensated / exact: as +)
 *      int32        0   1    INT32_MAX    INT32_MIN    -1    0   0
 *      uint32       0   1    UINT32_MAX   0            ~0u   0   0
 *      int64        0   1    INT64_MAX    INT64_MIN    -1    0   0
 *      float32/64  +0.0 1.0  +inf         -inf         (unsupported)
 */
#ifndef B200REDUCE_H
#define B200REDUCE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { RD_INT32 = 0, RD_UINT32 = 1, RD_INT64 = 2, RD_FLOAT32 = 3, RD_FLOAT64 = 4 } rd_dtype;
typedef enum {
  RD_SUM = 0, RD_PROD = 1, RD_MIN = 2, RD_MAX = 3, RD_AND = 4, RD_OR = 5, RD_XOR = 6,
  /* (value, smallest index) of the min / max -- the paper's
   * consumers are shortest paths and golden-section search.
   * `out` points to an rd_arg_result. NaN anywhere: value NaN, index of the
   * first NaN; -0.0 ranks below +0.0; empty: identity value, index -1. */
  RD_ARGMIN = 7, RD_ARGMAX = 8,
  /* compensated sum (P:50 fn 3, "double precision ... or
   * ... Kahan"): fp32 accumulates in fp64, fp64 in double-double (TwoSum per
   * term), so the result is the exact sum rounded once except in near-tie
   * cases -- in practice independent of order, grid and GPU count.
   * |result - exact| <= 0.5 ulp(result) + d * u_acc * sum|x_i| for every
   * input with finite partial sums, d < 2^21 the depth of the kernels' wide
   * chains (R16), u_acc = 2^-53 (fp32 data) / ~2^-104 (fp64 data).
   * Integers: identical to RD_SUM. */
  RD_SUM_COMPENSATED = 9,
  /* SURVEY §8(f) f2, reproducible: the EXACT sum rounded once (round to
   * nearest, ties to even) -- DESIGN.md reading R17. P:50 fn 2: the real sum
   * "is always the same, no matter the order the terms are added"; this is
   * that sum, so the bits do not depend on the grid, variant, base alignment
   * or number of GPUs. Any NaN, or +inf with -inf -> NaN; else +-inf if any;
   * a finite exact sum past the dtype's range -> +-inf; an exact zero is -0.0
   * iff every term is -0.0. Floats: reduce, rd_reduce_ex (vector / bulk),
   * reduce_multi, reduce_fused, reduce_host and reduce_exact_partial /
   * rd_combine_exact_records (the 32-byte rd_record cannot carry an exact
   * partial, so reduce_partial and rd_combine_records return
   * RD_ERR_UNSUPPORTED for float dtypes).
   * Throughput depends on the data, never the result: near the plain sum's
   * when the terms' exponents cluster (uniform / normal data), about half of
   * it when they spread over ~80 binades (binned extraction),
   * lowest for fp64 terms spread over hundreds of binades.
   * Integers: identical to RD_SUM everywhere. */
  RD_SUM_EXACT = 10
} rd_op;

/* Output of RD_ARGMIN / RD_ARGMAX (16 bytes, 8-byte aligned). */
typedef struct rd_arg_result {
  uint64_t value;   /* the element's bits in the low sizeof(dtype) bytes (little endian) */
  int64_t index;    /* smallest index attaining it; -1 for n == 0 */
} rd_arg_result;
typedef enum {
  RD_OK = 0,
  RD_ERR_INVALID_ARG = 1,  /* NULL where a buffer is needed, unknown enum, bad config  */
  RD_ERR_UNSUPPORTED = 2,  /* bitwise op on a float dtype; a configuration with no
                              compiled kernel; an exact float sum into a 32-byte record */
  RD_ERR_MISALIGNED = 3,   /* base pointer not aligned to sizeof(dtype)                */
  RD_ERR_CUDA = 4,         /* CUDA launch / allocation / copy failure (rd_last_error)  */
  RD_ERR_NCCL = 5,         /* NCCL failure (rd_last_error)                             */
  RD_ERR_MISMATCH = 6,     /* ranks or records disagree on dtype/op                    */
  RD_ERR_TIMEOUT = 7       /* fused exchange: a peer's record never arrived (~seconds) */
} rd_status;

/* A CUDA stream handle; identical to cudaStream_t / CUstream. */
typedef struct CUstream_st* rd_stream_t;

/*
 * rd_record -- the un-narrowed partial result of one block of X.
 * 32 bytes, plain data, device- or host-resident. Partials are what the
 * two-stage structure passes between its stages (the |SM|-sized "result"
 * vector of P:143/P:174); here they are what shards exchange.
 *   tag    = 0x52440000 | dtype << 8 | op      (0 marks "no record")
 *   status = 0 (reserved)
 *   n      = number of elements the partial covers
 *   acc    = the accumulator bits (integer value; fp32 + and x: double
 *            bits; fp64 + and x: double-double hi, lo;
 *            float min/max: order-preserving key and the max |x| bit pattern;
 *            argmin/argmax: order key and the index WITHIN the block, which
 *            rd_combine_records shifts by the n of the records before it)
 */
typedef struct rd_record {
  uint32_t tag;
  uint32_t status;
  uint64_t n;
  uint64_t acc[2];
} rd_record;

/*
 * rd_exact_record -- the exact partial sum of one block of float X
 * (RD_SUM_EXACT): a fixed-point integer sum_k word[k] * 2^(32k) in units of
 * the dtype's smallest subnormal (2^-149 for float32, 2^-1074 for float64),
 * words carried to digits in [0, 2^32) except the signed top word
 * word[nwords-1]; nwords = 12 (float32) / 68 (float64), the rest zero.
 *   flags = 1 NaN seen | 2 +inf seen | 4 -inf seen | 8 some term is not -0.0
 * 608 bytes, plain data, 16-byte aligned when allocated so. Adding the words
 * of two records is the exact sum of the two blocks (any order).
 */
#define RD_EXACT_MAX_WORDS 72
typedef struct rd_exact_record {
  uint32_t tag;
  uint32_t status;
  uint64_t n;
  uint32_t flags;
  uint32_t nwords;
  uint64_t reserved;
  int64_t word[RD_EXACT_MAX_WORDS];
} rd_exact_record;

/* ------------------------------------------------------------------ reduce
 * reduce -- out[0] = x_0 (x) ... (x) x_{n-1} on one GPU.
 *   x      device pointer to n contiguous elements of `dtype` (caller-owned,
 *          read-only, any element-aligned offset).
 *   n      element count, 0 <= n < 2^40.
 *   out    device pointer to ONE element of `dtype` (caller-owned, written).
 *   stream launch stream.
 * One kernel launch (a single-pass persistent grid).
 * Errors: INVALID_ARG (x NULL with n > 0, out NULL, bad enum), UNSUPPORTED,
 * MISALIGNED (x or out), CUDA. */
rd_status reduce(const void* x, size_t n, rd_dtype dtype, rd_op op, void* out, rd_stream_t stream);

/* reduce_partial -- like reduce, but writes the un-narrowed partial of
 * x[0..n) as one rd_record at device pointer `rec` (8-byte aligned).
 * Used to split one logical reduction across shards, chunks or GPUs. */
rd_status reduce_partial(const void* x, size_t n, rd_dtype dtype, rd_op op, rd_record* rec,
                         rd_stream_t stream);

/* rd_combine_records -- fold `count` device records in INDEX ORDER (rank or
 * chunk order, so the result is deterministic) and write the narrowed value
 * to device `out` (one element; may be NULL) and/or the folded record to
 * device `rec_out` (may be NULL). If any record's tag differs from
 * (dtype, op), *d_status (a device int, may be NULL) is set to
 * RD_ERR_MISMATCH and `out` receives the empty result.
 * The "second stage" of P:180 applied across blocks held by different
 * owners. One warp: records are loaded 32 at a time and folded sequentially.
 * Errors: INVALID_ARG (recs NULL with count > 0, count < 0, both outputs
 * NULL), MISALIGNED (recs not 16-byte aligned), UNSUPPORTED, CUDA. */
rd_status rd_combine_records(const rd_record* recs, int count, rd_dtype dtype, rd_op op,
                             void* out, rd_record* rec_out, int* d_status, rd_stream_t stream);

/* reduce_exact_partial -- the exact partial of float x[0..n) (RD_SUM_EXACT)
 * as one rd_exact_record at device pointer `rec` (8-byte aligned).
 * Errors: as reduce_partial; UNSUPPORTED for integer dtypes (use
 * reduce_partial with RD_SUM, which is exact). */
rd_status reduce_exact_partial(const void* x, size_t n, rd_dtype dtype, rd_exact_record* rec,
                               rd_stream_t stream);

/* rd_combine_exact_records -- add `count` device exact records (float
 * dtype) and write the once-rounded value to device `out` (may be NULL)
 * and/or the summed record to device `rec_out` (may be NULL). A record whose
 * tag or nwords differs sets *d_status (device int, may be NULL) to
 * RD_ERR_MISMATCH and `out` receives +0.0. One CTA. Errors: INVALID_ARG,
 * MISALIGNED (recs not 16-byte aligned), UNSUPPORTED (integer dtype), CUDA. */
rd_status rd_combine_exact_records(const rd_exact_record* recs, int count, rd_dtype dtype, void* out,
                                   rd_exact_record* rec_out, int* d_status, rd_stream_t stream);

/* reduce_host -- end-to-end reduction of a HOST array (pinned or pageable)
 * on the current device: chunks are copied host->device on a copy stream,
 * overlapped with reduce_partial on a compute stream (double-buffered), the
 * chunk records are combined in chunk order, and the result is copied back
 * to host `out_host` (one element). Synchronous: returns when *out_host is
 * written. Device staging buffers are library-owned (freed by
 * rd_release_workspaces). Errors: as reduce, plus CUDA. */
rd_status reduce_host(const void* x_host, size_t n, rd_dtype dtype, rd_op op, void* out_host);

/* ------------------------------------------------------------ multi-GPU
 * One process per GPU. Rank r holds the r-th contiguous block of the
 * logical array (rd_shard_range gives the canonical split). reduce_multi
 * reduces the local block to a record, all-gathers the W records over NCCL
 * (NVLink/NVSwitch), and folds them in RANK ORDER on every rank, so every
 * rank gets the bitwise-identical result in its device `out`. n_local may
 * differ across ranks and may be 0. Stream-ordered; a dtype/op disagreement
 * between ranks is reported by the next rd_comm_check (all ranks see it). */
typedef struct rd_comm* rd_comm_t;
typedef struct { char internal[128]; } rd_unique_id;

rd_status rd_get_unique_id(rd_unique_id* id);                  /* wraps ncclGetUniqueId */
rd_status rd_comm_init(rd_comm_t* comm, int nranks, int rank, const rd_unique_id* id, int device);
rd_status rd_comm_destroy(rd_comm_t comm);
rd_status reduce_multi(const void* x_local, size_t n_local, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, rd_comm_t comm);
/* Synchronises `stream`; returns RD_ERR_MISMATCH if any reduce_multi on this
 * comm since the previous check saw records that disagree, and clears it. */
rd_status rd_comm_check(rd_comm_t comm, rd_stream_t stream);
/* Canonical contiguous split: rank r gets [begin, begin+count) with
 * count = n/W + (r < n%W). Pure host function. */
rd_status rd_shard_range(uint64_t n, int nranks, int rank, uint64_t* begin, uint64_t* count);

/* ------------------------------------------- fused multi-GPU
 * reduce_fused -- the sharded reduction with the exchange step INSIDE the
 * reduce kernel: the last CTA of rank r stores its rd_record into slot r of
 * every rank's mailbox over NVLink (peer stores to CUDA-IPC-mapped device
 * memory) as self-validating "LL" words -- each 8-byte store carries 4
 * payload bytes and the call's 32-bit epoch, so no fence or release is
 * needed: a reader polls until every word carries the epoch -- waits for the
 * W records of this call in its own mailbox and folds them in rank order.
 * One kernel launch per rank; no NCCL call, no host synchronisation. Same
 * results and contract as reduce_multi (bitwise-identical on all ranks).
 * Every rank's record starts with the same 32-byte header {tag, 0, n} (exact
 * sums add their words after it), so ranks that disagree on dtype or op --
 * plain or exact -- report RD_ERR_MISMATCH, not a timeout.
 *
 * Setup (collective, every rank in the same order):
 *   rd_fused_create(&f, nranks, rank, device, handle)   allocates this rank's
 *       mailbox and writes its 64-byte IPC handle to host `handle`;
 *   exchange the nranks handles (e.g. an all-gather over the process group);
 *   rd_fused_connect(f, handles)                         opens the peers'.
 * Single-process use (several virtual ranks, one or more devices):
 *   rd_fused_mailbox(f, &ptr) and rd_fused_connect_local(f, ptrs) with the
 *   nranks mailbox device pointers instead of IPC handles; peer access from
 *   this rank's device to every other mailbox's device is enabled there
 *   (RD_ERR_UNSUPPORTED if the devices cannot access each other).
 * rd_comm_init / rd_fused_create / rd_fused_connect* leave the caller's
 * current device unchanged and synchronise no other stream.
 * Every rank must call reduce_fused the same number of times in the same
 * order (epochs are counted on the device, in each rank's mailbox, so the
 * call can be captured in a CUDA graph and replayed); nranks <= 32. A peer that
 * never arrives makes the kernel give up after ~4 s with RD_ERR_TIMEOUT
 * (reported by rd_fused_check) instead of hanging. */
typedef struct rd_fused* rd_fused_t;
rd_status rd_fused_create(rd_fused_t* f, int nranks, int rank, int device, void* ipc_handle_out);
rd_status rd_fused_connect(rd_fused_t f, const void* ipc_handles);
rd_status rd_fused_mailbox(rd_fused_t f, void** mailbox);
rd_status rd_fused_connect_local(rd_fused_t f, void* const* mailboxes);
rd_status reduce_fused(const void* x_local, size_t n_local, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, rd_fused_t f);
/* Synchronises `stream`; returns the first RD_ERR_MISMATCH / RD_ERR_TIMEOUT
 * seen by reduce_fused on this communicator since the last check, and clears it. */
rd_status rd_fused_check(rd_fused_t f, rd_stream_t stream);
rd_status rd_fused_destroy(rd_fused_t f);

/* ---------------------------------------------------------------- helpers */
/* Host copy of the empty result (table above) into host_out (one element;
 * an rd_arg_result with index -1 for RD_ARGMIN / RD_ARGMAX). */
rd_status rd_identity(rd_dtype dtype, rd_op op, void* host_out);
/* Frees the cached per-(device, stream) workspaces and reduce_host buffers.
 * Must not race with in-flight calls. */
rd_status rd_release_workspaces(void);
const char* rd_status_string(rd_status s);
/* Thread-local detail string for the last error on the calling thread. */
const char* rd_last_error(void);

/* ---------------------------------------------------- explicit launch control
 * rd_reduce_ex -- reduce with an explicit kernel configuration, for the
 * loads-in-flight ablation (the B200 form of PAPER.md Table 2)
 * and for tests that force grid shapes. Any field 0 = the planner's choice.
 *   variant   RD_VARIANT_AUTO, RD_VARIANT_VECTOR (grid-stride vector loads),
 *             RD_VARIANT_PAPER (PAPER.md Listing "Unrolling the step 1",
 *             F consecutive elements per work-item per iteration,
 *             bounds handled by predication instead of the (i<len)*x mask),
 *             RD_VARIANT_BULK (cp.async.bulk shared-memory ring, dynamic
 *             chunk scheduling, per-chunk partials: still deterministic),
 *             RD_VARIANT_CLUSTER (the vector kernel's body on a grid that is
 *             one thread-block cluster of 1..16 CTAs, the CTA partials
 *             combined over distributed shared memory: AUTO's choice for
 *             small inputs that need 2..16 CTAs)
 *   vec_bytes 4, 8, 16 or 32 bytes per load (VECTOR variant);
 *             bytes per ring stage (BULK variant)
 *   unroll    loads in flight per thread per iteration (U; the paper's F);
 *             ring stages (BULK variant)
 *   grid      CTAs (clamped to [1, 4096]; [1, 16] for the CLUSTER variant)
 * RD_SUM_EXACT on floats has one compiled kernel per variant (vector and
 * cluster: 32-byte loads, U = 6; bulk: the default ring with 16 consumer
 * warps): only variant and grid may be chosen.
 * The chosen configuration is written to *info (may be NULL).
 * Configurations without a compiled kernel return RD_ERR_UNSUPPORTED. */
enum { RD_VARIANT_AUTO = 0, RD_VARIANT_VECTOR = 1, RD_VARIANT_PAPER = 2, RD_VARIANT_BULK = 3,
       RD_VARIANT_CLUSTER = 4 };
typedef struct { int32_t variant, vec_bytes, unroll, block, grid, reserved[3]; } rd_config;
typedef struct {
  int32_t variant, vec_bytes, unroll, block, grid, regs_per_thread, ctas_per_sm, reserved;
  uint64_t head, nvec, tail;
} rd_launch_info;
rd_status rd_reduce_ex(const void* x, size_t n, rd_dtype dtype, rd_op op, void* out,
                       rd_stream_t stream, const rd_config* cfg, rd_launch_info* info);

#ifdef __cplusplus
}
#endif
#endif /* B200REDUCE_H */
