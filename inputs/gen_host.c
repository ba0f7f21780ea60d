/*
 * inputs/gen_host.c -- host twin of the seeded input generator (gen.h).
 * Holds no reduction arithmetic; see gen.h.
 */
#include "gen.h"
#include <stddef.h>

/* Fill out[0..count) with elements offset .. offset+count-1 of the workload
 * (global indices, so shards of one logical array are generated independently).
 * Returns 0, or -1 for an unsupported (dtype, workload). */
int in_fill_host(void* out, uint64_t count, int dtype, int workload, uint64_t seed,
                 uint64_t offset, uint64_t n_total) {
  const int s = gen_dtype_size(dtype);
  unsigned char* p = (unsigned char*)out;
  if (s == 0) return -1;
  for (uint64_t j = 0; j < count; ++j) {
    if (gen_element(dtype, workload, seed, offset + j, n_total, p + j * (uint64_t)s) != 0) return -1;
  }
  return 0;
}

void in_planted_positions(uint64_t seed, uint64_t n_total, uint64_t* p_max, uint64_t* p_min) {
  gen_planted_positions(seed, n_total, p_max, p_min);
}
