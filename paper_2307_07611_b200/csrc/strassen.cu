// strassen.cu — Strassen's 7-product recursion for the dense block products of the
// recursive split (NEXT row f3): the paper's fast multiplication of the
// full x full products P_FF inside P_TF (Eq. PTFmbk).
//
// strassen_acc computes C = beta C + alpha A B for square h x h operands with `levels`
// levels of the recursion over the DMMA GEMM engine (gemm.cu): per level the 10 operand
// sums and the 4 output combinations are single fused passes (lincomb_kernel, HBM-bound),
// the 7 half-size products recurse (level 0: one DMMA GEMM with alpha / beta).  The
// products of the recursion are summed in FP64, so its error is normwise (it grows with
// the levels, Higham's bound) where the DMMA GEMM's is componentwise: DESIGN.md §11 keeps
// or drops it on the measured floored-relative error and time of whole inversions.
#include <cuda_runtime.h>

#include <initializer_list>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

struct LinComb {
  const double* x[4];
  int64_t ld[4];
  double c[4];
  int k;
};

// C[i][j] = beta C[i][j] + sum_t c_t X_t[i][j]  (beta == 0: C not read).  One column pair per
// thread, rows over blockIdx.y: 0.5 of HBM on a 2048^2 combination incl. the launch ramp
// (profiles/r02_ncu_lincomb_v1.txt); a one-CTA-per-row variant with 4 pairs per thread took
// 31 instead of 18 us (config 3: 11 -> 21 ms) and was reverted.
__global__ void lincomb_kernel(int64_t rows, int64_t cols, double beta, double* C, int64_t ldc, const LinComb t) {
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    for (int64_t j = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); j < cols;
         j += 2 * (int64_t)gridDim.x * blockDim.x) {
      double2 acc = beta == 0.0 ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(C + i * ldc + j);
      if (beta != 0.0 && beta != 1.0) { acc.x *= beta; acc.y *= beta; }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < t.k) {
          const double2 v = *reinterpret_cast<const double2*>(t.x[q] + i * t.ld[q] + j);
          acc.x = fma(t.c[q], v.x, acc.x);
          acc.y = fma(t.c[q], v.y, acc.y);
        }
      }
      *reinterpret_cast<double2*>(C + i * ldc + j) = acc;
    }
  }
}

static cudaError_t lincomb(int64_t n, double beta, double* C, int64_t ldc, std::initializer_list<const double*> xs,
                           std::initializer_list<int64_t> lds, std::initializer_list<double> cs, cudaStream_t s,
                           int64_t* launches) {
  LinComb t{};
  t.k = 0;
  auto xi = xs.begin();
  auto li = lds.begin();
  auto ci = cs.begin();
  for (; xi != xs.end(); ++xi, ++li, ++ci, ++t.k) {
    t.x[t.k] = *xi;
    t.ld[t.k] = *li;
    t.c[t.k] = *ci;
  }
  const int threads = 256;
  const int64_t bx = (n / 2 + threads - 1) / threads;
  const dim3 grid((unsigned)(bx < 8 ? bx : 8), (unsigned)(n < 65535 ? n : 65535));
  const cudaError_t e = launch_k(lincomb_kernel, grid, dim3(threads), 0, s, n, n, beta, C, ldc, t);
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

size_t strassen_ws_bytes(int64_t h, int levels, int64_t min_q) {
  if (!strassen_level_ok(h, levels, min_q)) return 0;
  const int64_t q = h / 2;
  return 9 * aup((size_t)q * even_up2(q) * sizeof(double)) + strassen_ws_bytes(q, levels - 1, min_q);
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
  double* SA = reinterpret_cast<double*>(w);
  double* SB = reinterpret_cast<double*>(w + slot);
  double* M[7];
  for (int k = 0; k < 7; ++k) M[k] = reinterpret_cast<double*>(w + (2 + k) * slot);
  void* inner = w + 9 * slot;
  const double *A11 = A, *A12 = A + q, *A21 = A + q * lda, *A22 = A + q * lda + q;
  const double *B11 = B, *B12 = B + q, *B21 = B + q * ldb, *B22 = B + q * ldb + q;
  double *C11 = C, *C12 = C + q, *C21 = C + q * ldc, *C22 = C + q * ldc + q;
  cudaError_t e = cudaSuccess;
#define S_TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  auto prod = [&](const double* X, int64_t lx, const double* Y, int64_t ly, double* Z) {
    return strassen_acc(q, 1.0, X, lx, Y, ly, 0.0, Z, lq, levels - 1, min_q, inner, s, launches);
  };
  // M1 = (A11 + A22)(B11 + B22)
  S_TRY(lincomb(q, 0.0, SA, lq, {A11, A22}, {lda, lda}, {1.0, 1.0}, s, launches));
  S_TRY(lincomb(q, 0.0, SB, lq, {B11, B22}, {ldb, ldb}, {1.0, 1.0}, s, launches));
  S_TRY(prod(SA, lq, SB, lq, M[0]));
  // M2 = (A21 + A22) B11
  S_TRY(lincomb(q, 0.0, SA, lq, {A21, A22}, {lda, lda}, {1.0, 1.0}, s, launches));
  S_TRY(prod(SA, lq, B11, ldb, M[1]));
  // M3 = A11 (B12 - B22)
  S_TRY(lincomb(q, 0.0, SB, lq, {B12, B22}, {ldb, ldb}, {1.0, -1.0}, s, launches));
  S_TRY(prod(A11, lda, SB, lq, M[2]));
  // M4 = A22 (B21 - B11)
  S_TRY(lincomb(q, 0.0, SB, lq, {B21, B11}, {ldb, ldb}, {1.0, -1.0}, s, launches));
  S_TRY(prod(A22, lda, SB, lq, M[3]));
  // M5 = (A11 + A12) B22
  S_TRY(lincomb(q, 0.0, SA, lq, {A11, A12}, {lda, lda}, {1.0, 1.0}, s, launches));
  S_TRY(prod(SA, lq, B22, ldb, M[4]));
  // M6 = (A21 - A11)(B11 + B12)
  S_TRY(lincomb(q, 0.0, SA, lq, {A21, A11}, {lda, lda}, {1.0, -1.0}, s, launches));
  S_TRY(lincomb(q, 0.0, SB, lq, {B11, B12}, {ldb, ldb}, {1.0, 1.0}, s, launches));
  S_TRY(prod(SA, lq, SB, lq, M[5]));
  // M7 = (A12 - A22)(B21 + B22)
  S_TRY(lincomb(q, 0.0, SA, lq, {A12, A22}, {lda, lda}, {1.0, -1.0}, s, launches));
  S_TRY(lincomb(q, 0.0, SB, lq, {B21, B22}, {ldb, ldb}, {1.0, 1.0}, s, launches));
  S_TRY(prod(SA, lq, SB, lq, M[6]));
  // C11 += M1 + M4 - M5 + M7, C12 += M3 + M5, C21 += M2 + M4, C22 += M1 - M2 + M3 + M6 (x alpha)
  S_TRY(lincomb(q, beta, C11, ldc, {M[0], M[3], M[4], M[6]}, {lq, lq, lq, lq}, {alpha, alpha, -alpha, alpha}, s,
                launches));
  S_TRY(lincomb(q, beta, C12, ldc, {M[2], M[4]}, {lq, lq}, {alpha, alpha}, s, launches));
  S_TRY(lincomb(q, beta, C21, ldc, {M[1], M[3]}, {lq, lq}, {alpha, alpha}, s, launches));
  S_TRY(lincomb(q, beta, C22, ldc, {M[0], M[1], M[2], M[5]}, {lq, lq, lq, lq}, {alpha, -alpha, alpha, alpha}, s,
                launches));
#undef S_TRY
  return cudaSuccess;
}

}  // namespace trinv
