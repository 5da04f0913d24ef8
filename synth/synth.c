/* Host generator (OpenMP). See synth.h for the definition. */
#include "synth.h"
#include <stdint.h>

/* Fill `count` matrices b = b0 .. b0+count-1 (seed = seed0 + b) of order n,
 * row-major with leading dimension ld, matrix stride `stride` elements. */
void synth_fill_host(int64_t n, int64_t b0, int64_t count, uint64_t seed0, uint64_t tag,
                     char uplo, int diag, double* out, int64_t ld, int64_t stride) {
  #pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < count; ++b) {
    for (int64_t i = 0; i < n; ++i) {
      uint64_t key = synth_key(seed0 + (uint64_t)(b0 + b), tag);
      double* row = out + b * stride + i * ld;
      for (int64_t j = 0; j < n; ++j) row[j] = synth_entry(key, n, i, j, uplo, diag);
    }
  }
}

/* One column j of matrix b (for sampled checks without materialising). */
void synth_column_host(int64_t n, int64_t b, uint64_t seed0, uint64_t tag, char uplo, int diag,
                       int64_t j, double* out) {
  uint64_t key = synth_key(seed0 + (uint64_t)b, tag);
  for (int64_t i = 0; i < n; ++i) out[i] = synth_entry(key, n, i, j, uplo, diag);
}
