/* examples/reduce_example.c -- calling the library from plain C (C99).
 *
 *   gcc -std=c99 -O2 examples/reduce_example.c -Iinclude \
 *       -Lpaper_1710_07358_b200 -lb200reduce -Wl,-rpath,$PWD/paper_1710_07358_b200 \
 *       -L/usr/local/cuda/lib64 -lcudart -o reduce_example
 *   ./reduce_example [log2n]
 *
 * Reduces n float32 ones on the GPU (sum must be n exactly for n <= 2^24),
 * the paper's absorption example with the exact sum (two halves as exact
 * records, combined), and times back-to-back reduce() calls (host + device)
 * with CUDA events. */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>

#include "b200reduce.h"

#define CK(x) do { rd_status s_ = (x); if (s_ != RD_OK) { \
  fprintf(stderr, "%s: %s (%s)\n", #x, rd_status_string(s_), rd_last_error()); return 1; } } while (0)

int main(int argc, char** argv) {
  int log2n = argc > 1 ? atoi(argv[1]) : 24;
  size_t n = (size_t)1 << log2n;
  float* x = NULL;
  float* out = NULL;
  if (cudaMalloc((void**)&x, n * sizeof(float)) != cudaSuccess) return 2;
  if (cudaMalloc((void**)&out, sizeof(float)) != cudaSuccess) return 2;
  float* h = (float*)malloc(n * sizeof(float));
  for (size_t i = 0; i < n; ++i) h[i] = 1.0f;
  cudaMemcpy(x, h, n * sizeof(float), cudaMemcpyHostToDevice);
  free(h);

  CK(reduce(x, n, RD_FLOAT32, RD_SUM, out, NULL));
  float s = 0.0f;
  cudaMemcpy(&s, out, sizeof(float), cudaMemcpyDeviceToHost);
  printf("sum of %zu ones = %.1f\n", n, s);
  if (n <= (1u << 24) && s != (float)n) { fprintf(stderr, "wrong sum\n"); return 1; }

  rd_arg_result am;
  rd_arg_result* d_am = NULL;
  cudaMalloc((void**)&d_am, sizeof(rd_arg_result));
  CK(reduce(x, n, RD_FLOAT32, RD_ARGMAX, d_am, NULL));
  cudaMemcpy(&am, d_am, sizeof am, cudaMemcpyDeviceToHost);
  printf("argmax index = %lld (lowest of the ties)\n", (long long)am.index);
  if (am.index != 0) { fprintf(stderr, "wrong argmax\n"); return 1; }

  /* PAPER.md P:50 fn 2: 1.5 + 4^50 - 4^50 is 0 or 1.5 by evaluation order;
   * RD_SUM_EXACT returns the real sum, 1.5, whatever the split or order */
  float terms[3] = {4.0f * 0x1p98f, 1.5f, -4.0f * 0x1p98f};
  float* d_t = NULL;
  rd_exact_record* d_rec = NULL;
  cudaMalloc((void**)&d_t, sizeof terms);
  cudaMalloc((void**)&d_rec, 2 * sizeof(rd_exact_record));
  cudaMemcpy(d_t, terms, sizeof terms, cudaMemcpyHostToDevice);
  CK(reduce_exact_partial(d_t, 1, RD_FLOAT32, d_rec, NULL));          /* block [0, 1) */
  CK(reduce_exact_partial(d_t + 1, 2, RD_FLOAT32, d_rec + 1, NULL));  /* block [1, 3) */
  CK(rd_combine_exact_records(d_rec, 2, RD_FLOAT32, out, NULL, NULL, NULL));
  float e = 0.0f;
  cudaMemcpy(&e, out, sizeof e, cudaMemcpyDeviceToHost);
  printf("exact sum of {4^50, 1.5, -4^50} = %.1f\n", e);
  if (e != 1.5f) { fprintf(stderr, "wrong exact sum\n"); return 1; }
  cudaFree(d_t);
  cudaFree(d_rec);

  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int K = 200;
  for (int i = 0; i < 10; ++i) CK(reduce(x, n, RD_FLOAT32, RD_SUM, out, NULL));
  cudaEventRecord(a, NULL);
  for (int i = 0; i < K; ++i) CK(reduce(x, n, RD_FLOAT32, RD_SUM, out, NULL));
  cudaEventRecord(b, NULL);
  cudaEventSynchronize(b);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, a, b);
  printf("n=2^%d: %.2f us per back-to-back reduce() from C, %.1f GB/s\n", log2n, 1e3 * ms / K,
         (double)n * 4 * K / (ms * 1e-3) / 1e9);
  cudaFree(x);
  cudaFree(out);
  cudaFree(d_am);
  return 0;
}
