// strassen.cu — Strassen's 7-product recursion for the dense block products of the
// recursive split (NEXT row f3): the paper's fast multiplication of the
// full x full products P_FF inside P_TF (Eq. PTFmbk).
//
// strassen_acc computes C = beta C + alpha A B for square h x h operands with `levels`
// levels of the recursion over the DMMA GEMM engine (gemm.cu): per level the 10 operand
// sums (one pass over each operand's four quadrants) and the 4 output combinations (one
// pass over M1..M7) run in mix_kernel (HBM-bound), the 7 half-size products recurse (level 0: one DMMA GEMM with alpha / beta).  The
// products of the recursion are summed in FP64, so its error is normwise (it grows with
// the levels, Higham's bound) where the DMMA GEMM's is componentwise: DESIGN.md §11 keeps
// or drops it on the measured floored-relative error and time of whole inversions.
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

#include <cstdlib>

namespace trinv {

// Several combinations of the same inputs in ONE pass: out_o = beta out_o + sum_i c[o][i] in_i
// for up to 7 inputs and 5 outputs (the 5 operand sums of A from its 4 quadrants, likewise for
// B, and the 4 output quadrants from M1..M7): 33 instead of 50 quadrant-sized HBM transfers
// per Strassen level (round 2; the first version ran 14 two-input passes).
struct Mix {
  const double* in[7];
  int64_t ldin[7];
  double* out[5];
  int64_t ldout[5];
  double c[5][7];
  int nin, nout;
};
template <int NIN, int NOUT>
__global__ void __launch_bounds__(256) mix_kernel(int64_t rows, int64_t cols, double beta, const Mix m) {
  pdl_trigger_early();
  pdl_wait();
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    for (int64_t j = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); j < cols;
         j += 2 * (int64_t)gridDim.x * blockDim.x) {
      double2 v[NIN];
#pragma unroll
      for (int q = 0; q < NIN; ++q) v[q] = __ldcs(reinterpret_cast<const double2*>(m.in[q] + i * m.ldin[q] + j));
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        double2* dst = reinterpret_cast<double2*>(m.out[o] + i * m.ldout[o] + j);
        double2 acc = make_double2(0.0, 0.0);
        if (beta != 0.0) {
          acc = *dst;
          acc.x *= beta;
          acc.y *= beta;
        }
#pragma unroll
        for (int q = 0; q < NIN; ++q) {
          if (m.c[o][q] != 0.0) {
            acc.x = fma(m.c[o][q], v[q].x, acc.x);
            acc.y = fma(m.c[o][q], v[q].y, acc.y);
          }
        }
        *dst = acc;
      }
    }
  }
}

// The same combinations as two-input geam passes (TRINV_STRASSEN_SUMS=geam: the operand sums;
// experiment for the concurrency finding of DESIGN.md §9b)
static cudaError_t mix_geam(int64_t n, double beta, const Mix& m, cudaStream_t s, int64_t* launches) {
  for (int o = 0; o < m.nout; ++o) {
    bool first = true;
    for (int q = 0; q < m.nin; ++q) {
      if (m.c[o][q] == 0.0) continue;
      cudaError_t e;
      if (first && beta == 0.0)
        e = launch_geam(n, n, m.c[o][q], m.in[q], m.ldin[q], 0.0, m.in[q], m.ldin[q], m.out[o], m.ldout[o], s, launches);
      else if (first)
        e = launch_geam(n, n, m.c[o][q], m.in[q], m.ldin[q], beta, m.out[o], m.ldout[o], m.out[o], m.ldout[o], s, launches);
      else
        e = launch_geam(n, n, 1.0, m.out[o], m.ldout[o], m.c[o][q], m.in[q], m.ldin[q], m.out[o], m.ldout[o], s, launches);
      if (e != cudaSuccess) return e;
      first = false;
    }
  }
  return cudaSuccess;
}
static bool sums_by_geam() {
  static const bool on = [] { const char* e = std::getenv("TRINV_STRASSEN_SUMS"); return e && e[0] == 'g'; }();
  return on;
}

template <int NIN, int NOUT>
static cudaError_t mix(int64_t n, double beta, const Mix& m, cudaStream_t s, int64_t* launches) {
  if (NIN == 4 && sums_by_geam()) return mix_geam(n, beta, m, s, launches);
  prefer_l1_once<mix_kernel<NIN, NOUT>>();
  const int threads = 256;
  const int64_t bx = (n / 2 + threads - 1) / threads;
  const dim3 grid((unsigned)(bx < 8 ? bx : 8), (unsigned)(n < 65535 ? n : 65535));
  const cudaError_t e = launch_k(mix_kernel<NIN, NOUT>, grid, dim3(threads), 0, s, n, n, beta, m);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

static int64_t even_up2(int64_t x) { return (x + 1) & ~int64_t(1); }
static size_t aup(size_t x) { return (x + 255) & ~size_t(255); }

// A level is applied only while its half-size products keep q >= min_q (the library passes
// min_h / 2: 2048 by default): below that the DMMA GEMM of the products loses more than the
// 1/8 of the flops a level saves (config 2's 1024-size products: 5.56 -> 6.75 ms;
// profiles/r02_strassen_inversion.txt).
static bool strassen_level_ok(int64_t h, int levels, int64_t min_q) {
  return levels > 0 && h % 4 == 0 && h / 2 >= min_q;
}

constexpr int STRASSEN_TEMPS = 17;  // 5 operand sums of A, 5 of B, M1..M7

size_t strassen_ws_bytes(int64_t h, int levels, int64_t min_q) {
  if (!strassen_level_ok(h, levels, min_q)) return 0;
  const int64_t q = h / 2;
  return STRASSEN_TEMPS * aup((size_t)q * even_up2(q) * sizeof(double)) + strassen_ws_bytes(q, levels - 1, min_q);
}

cudaError_t strassen_acc(int64_t h, double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double beta, double* C, int64_t ldc, int levels, int64_t min_q, void* ws, cudaStream_t s,
                         int64_t* launches) {
  if (!strassen_level_ok(h, levels, min_q)) {  // one DMMA GEMM
    GemmArgs g{};
    g.M = h; g.N = h; g.K = h; g.batch = 1;
    g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
    g.alpha = alpha; g.beta = beta; g.triA = TRI_NONE; g.triB = TRI_NONE;
    return launch_gemm(g, s, launches);
  }
  const int64_t q = h / 2, lq = even_up2(q);
  const size_t slot = aup((size_t)q * lq * sizeof(double));
  char* w = static_cast<char*>(ws);
  auto buf = [&](int k) { return reinterpret_cast<double*>(w + k * slot); };
  double *SA1 = buf(0), *SA2 = buf(1), *SA5 = buf(2), *SA6 = buf(3), *SA7 = buf(4);
  double *SB1 = buf(5), *SB3 = buf(6), *SB4 = buf(7), *SB6 = buf(8), *SB7 = buf(9);
  double* M[7];
  for (int k = 0; k < 7; ++k) M[k] = buf(10 + k);
  void* inner = w + STRASSEN_TEMPS * slot;
  const double *A11 = A, *A12 = A + q, *A21 = A + q * lda, *A22 = A + q * lda + q;
  const double *B11 = B, *B12 = B + q, *B21 = B + q * ldb, *B22 = B + q * ldb + q;
  double *C11 = C, *C12 = C + q, *C21 = C + q * ldc, *C22 = C + q * ldc + q;
  cudaError_t e = cudaSuccess;
#define S_TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  // operand sums, one pass per operand: inputs (X11, X12, X21, X22)
  Mix ma{};
  ma.nin = 4; ma.nout = 5;
  const double* ain[4] = {A11, A12, A21, A22};
  double* aout[5] = {SA1, SA2, SA5, SA6, SA7};
  const double ac[5][4] = {{1, 0, 0, 1},    // A11 + A22  (M1)
                           {0, 0, 1, 1},    // A21 + A22  (M2)
                           {1, 1, 0, 0},    // A11 + A12  (M5)
                           {-1, 0, 1, 0},   // A21 - A11  (M6)
                           {0, 1, 0, -1}};  // A12 - A22  (M7)
  Mix mb = ma;
  const double* bin[4] = {B11, B12, B21, B22};
  double* bout[5] = {SB1, SB3, SB4, SB6, SB7};
  const double bc[5][4] = {{1, 0, 0, 1},    // B11 + B22  (M1)
                           {0, 1, 0, -1},   // B12 - B22  (M3)
                           {-1, 0, 1, 0},   // B21 - B11  (M4)
                           {1, 1, 0, 0},    // B11 + B12  (M6)
                           {0, 0, 1, 1}};   // B21 + B22  (M7)
  for (int i = 0; i < 4; ++i) {
    ma.in[i] = ain[i]; ma.ldin[i] = lda;
    mb.in[i] = bin[i]; mb.ldin[i] = ldb;
  }
  for (int o = 0; o < 5; ++o) {
    ma.out[o] = aout[o]; ma.ldout[o] = lq;
    mb.out[o] = bout[o]; mb.ldout[o] = lq;
    for (int i = 0; i < 4; ++i) { ma.c[o][i] = ac[o][i]; mb.c[o][i] = bc[o][i]; }
  }
  S_TRY((mix<4, 5>(q, 0.0, ma, s, launches)));
  S_TRY((mix<4, 5>(q, 0.0, mb, s, launches)));
  auto prod = [&](const double* X, int64_t lx, const double* Y, int64_t ly, double* Z) {
    return strassen_acc(q, 1.0, X, lx, Y, ly, 0.0, Z, lq, levels - 1, min_q, inner, s, launches);
  };
  S_TRY(prod(SA1, lq, SB1, lq, M[0]));   // M1 = (A11 + A22)(B11 + B22)
  S_TRY(prod(SA2, lq, B11, ldb, M[1]));  // M2 = (A21 + A22) B11
  S_TRY(prod(A11, lda, SB3, lq, M[2]));  // M3 = A11 (B12 - B22)
  S_TRY(prod(A22, lda, SB4, lq, M[3]));  // M4 = A22 (B21 - B11)
  S_TRY(prod(SA5, lq, B22, ldb, M[4]));  // M5 = (A11 + A12) B22
  S_TRY(prod(SA6, lq, SB6, lq, M[5]));   // M6 = (A21 - A11)(B11 + B12)
  S_TRY(prod(SA7, lq, SB7, lq, M[6]));   // M7 = (A12 - A22)(B21 + B22)
  // C11 = beta C11 + alpha (M1 + M4 - M5 + M7), C12 = .. (M3 + M5), C21 = .. (M2 + M4),
  // C22 = .. (M1 - M2 + M3 + M6): one pass over M1..M7
  Mix mc{};
  mc.nin = 7; mc.nout = 4;
  double* cout[4] = {C11, C12, C21, C22};
  const double cc[4][7] = {{1, 0, 0, 1, -1, 0, 1},
                           {0, 0, 1, 0, 1, 0, 0},
                           {0, 1, 0, 1, 0, 0, 0},
                           {1, -1, 1, 0, 0, 1, 0}};
  for (int i = 0; i < 7; ++i) { mc.in[i] = M[i]; mc.ldin[i] = lq; }
  for (int o = 0; o < 4; ++o) {
    mc.out[o] = cout[o]; mc.ldout[o] = ldc;
    for (int i = 0; i < 7; ++i) mc.c[o][i] = alpha * cc[o][i];
  }
  S_TRY((mix<7, 4>(q, beta, mc, s, launches)));
#undef S_TRY
  return cudaSuccess;
}

}  // namespace trinv
