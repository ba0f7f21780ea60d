// rd_internal.h -- host-side pieces shared by the library's translation units
// (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "b200reduce.h"

namespace rd {

// Tuning knobs are for measurement builds only (`python -m
// paper_1710_07358_b200.build --tuning` defines RD_TUNING and writes
// build/tuning/libb200reduce.so). The shipped library reads no environment
// variable: its results are a function of the call's arguments alone.
#ifdef RD_TUNING
inline const char* tune_env(const char* name) { return std::getenv(name); }
#else
inline const char* tune_env(const char*) { return nullptr; }
#endif

// thread-local detail for rd_last_error()
void set_error(const std::string& msg);
rd_status cuda_fail(cudaError_t e, const char* what);

// argument checks shared by every entry point (synchronous, enqueue nothing)
rd_status check_dtype_op(int dtype, int op);
int dtype_size(int dtype);
bool is_arg_op(int op);
bool is_exact_float(int dtype, int op);   // RD_SUM_EXACT on float32/float64
int out_size(int dtype, int op);   // bytes of one result: element, or rd_arg_result

struct Mailbox;
// mode 2 (fused exchange) parameters
struct FusedArgs {
  Mailbox* const* peers;   // device array of nranks mailbox pointers
  Mailbox* self;
  int* err;
  int nranks, rank;
};

// Plan + launch one reduction of x[0..n) (a0-a7). mode 0 writes one element
// to `out`, mode 1 writes one rd_record to `rec`, mode 2 exchanges records
// through the mailboxes of `fused` and writes the folded result to `out`.
rd_status launch_reduce(const void* x, size_t n, int dtype, int op, int mode, void* out,
                        rd_record* rec, cudaStream_t stream, const rd_config* cfg,
                        rd_launch_info* info, const FusedArgs* fused = nullptr);

// RD_SUM_EXACT on floats (rd_exact.cuh): mode 0 -> one element at `out`,
// mode 1 -> one rd_exact_record at `xrec`, mode 2 -> the fused exchange of
// `fused` (exact records in LL form); and the exact-record combine.
rd_status launch_exact(const void* x, size_t n, int dtype, int mode, void* out, rd_exact_record* xrec,
                       cudaStream_t stream, const rd_config* cfg, rd_launch_info* info,
                       const FusedArgs* fused = nullptr);
rd_status launch_exact_combine(const rd_exact_record* recs, int count, int dtype, void* out,
                               rd_exact_record* rec_out, int* d_status, cudaStream_t stream);

// Launch the record-combine kernel (N4).
rd_status launch_combine(const rd_record* recs, int count, int dtype, int op, void* out,
                         rd_record* rec_out, int* d_status, cudaStream_t stream);

// load every default kernel up front (see rd_api.cu)
rd_status preload_default_kernels(int dev);

// per-(device) cleanup hooks of the other translation units
void release_host_pipelines();

}  // namespace rd
