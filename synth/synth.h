/* synth.h — counter-based seeded input generator shared by tests and bench.
 *
 * This module holds NO arithmetic of the inversion method: it only turns
 * (seed, tag, matrix, i, j) into the fp64 entries of the synthetic workloads
 * described in BASELINE.json configs.
 * The host version (synth.c) and the device twin (synth_cuda.cu) implement the
 * same integer hash and the same IEEE operations, so they agree bit for bit.
 *
 *   K(seed, tag)       = mix64(mix64(seed ^ G) ^ tag)
 *   h(K, idx, stream)  = mix64(K + (2*idx + stream + 1) * G)      (mod 2^64)
 *   u                  = (h >> 11) * 2^-53                       in [0, 1)
 *   off-diagonal       = (2u - 1) / n                              "uniform [-1,1]/n"
 *   diagonal SIGNED    = (1 + u) * (top bit of h(K, idx, 1) ? -1 : +1)
 *   diagonal POS       = 1 + u                                     "uniform [1,2]"
 *   diagonal ONE       = 1.0                                       (unit factors)
 * idx = i*n + j.  Matrix b of a batch uses seed = seed0 + b ("one seed per batch
 * index", C10).  The unreferenced triangle is written as 0.0 ("upper part zero").
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#define SYNTH_G 0x9E3779B97F4A7C15ULL

enum { SYNTH_DIAG_SIGNED = 0, SYNTH_DIAG_POS = 1, SYNTH_DIAG_ONE = 2 };

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

SYNTH_HD uint64_t synth_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
SYNTH_HD uint64_t synth_key(uint64_t seed, uint64_t tag) {
  return synth_mix64(synth_mix64(seed ^ SYNTH_G) ^ tag);
}
SYNTH_HD uint64_t synth_hash(uint64_t key, uint64_t idx, uint64_t stream) {
  return synth_mix64(key + (2ULL * idx + stream + 1ULL) * SYNTH_G);
}
SYNTH_HD double synth_u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* Entry (i, j) of an n x n triangular matrix; uplo 'L' or 'U'. */
SYNTH_HD double synth_entry(uint64_t key, int64_t n, int64_t i, int64_t j, char uplo, int diag) {
  int in_tri = (uplo == 'L') ? (i >= j) : (i <= j);
  if (!in_tri) return 0.0;
  uint64_t idx = (uint64_t)i * (uint64_t)n + (uint64_t)j;
  if (i != j) {
    double u = synth_u01(synth_hash(key, idx, 0));
    double t = 2.0 * u - 1.0; /* exact: u has 53 bits, |2u-1| < 1 */
    return t / (double)n;
  }
  if (diag == SYNTH_DIAG_ONE) return 1.0;
  double d = 1.0 + synth_u01(synth_hash(key, idx, 0));
  if (diag == SYNTH_DIAG_SIGNED && (synth_hash(key, idx, 1) >> 63)) d = -d;
  return d;
}
#endif
