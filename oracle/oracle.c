/* oracle.c — plain, slow, obviously-correct CPU reference for the FP64
 * triangular-inverse hot path of arXiv 2307.07611.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2307_07611_b200/csrc); neither includes the other.
 *
 * Arithmetic: IEEE fp64, compiled with -O2 -ffp-contract=off (no FMA
 * contraction), true division, sums with the index ascending.  Every routine
 * cites the passage of /root/reference/PAPER.md (P:line) it writes out.
 * Storage: row-major, element (i, j) at M[i*ld + j]; 0-based indices.
 *
 * Pins (tests/test_oracle_pins.py): the paper's 4x4 worked example,
 * Hopscotch listing and count, Cor. 2 integer closure
 * checked by exact integer L*X = I, unit-bidiagonal closed form s^(i-j),
 * all-ones triangle, identity/diagonal/2x2 closed forms, power-of-two scaling,
 * the printed 5x5 factors of §6.1, and brute force (pathsum)
 * against the recurrences for n <= 12.  No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define AT(M, ld, i, j) ((M)[(int64_t)(i) * (ld) + (j)])

#include <omp.h>
/* Thread count of the OpenMP loops below (bench.py's 1-thread cpu_baseline figure);
 * not arithmetic: every routine computes the same bits at any thread count. */
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_max_threads(void) { return omp_get_max_threads(); }

/* ---------------------------------------------------------------------------
 * CRIT (Algorithm 3) for an upper-triangular R, exactly as listed:
 *   for i = 1..n:  S(i,i) = 1/R(i,i)
 *                  for j = i+1..n:  S(i,j) = -S(i,i:j-1) . R(i:j-1,j) / R(j,j)
 * With unit != 0 this is CRIT* (Algorithm 2): S(i,i) = 1 and no
 * division; the j = i+1 entry, left unassigned by the listing's "j = i+2"
 * loop start, is the j = i+1 term of the same recurrence, S(i,i+1) = -T(i,i+1)
 * (reading C3).  The stored diagonal is not read when unit != 0.
 * Rows are independent ("every single element ... totally independent").
 * The strictly lower triangle of S is written as +0.0 (Eq. 6 "0, otherwise").
 * ------------------------------------------------------------------------- */
void oracle_crit_upper(int64_t n, const double* R, int64_t ldr, double* S, int64_t lds, int unit) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < i; ++j) AT(S, lds, i, j) = 0.0;
    AT(S, lds, i, i) = unit ? 1.0 : 1.0 / AT(R, ldr, i, i);
    for (int64_t j = i + 1; j < n; ++j) {
      double dot = 0.0;
      for (int64_t k = i; k < j; ++k) dot += AT(S, lds, i, k) * AT(R, ldr, k, j);
      AT(S, lds, i, j) = unit ? -dot : -dot / AT(R, ldr, j, j);
    }
  }
}

/* Lower-triangular L via the transpose ("For the lower triangle matrix,
 * we just consider the transpose operator"): X = (CRIT(L^T))^T.  Row i of
 * CRIT(L^T) is column i of X, so with R(a,b) = L(b,a):
 *   X(i,i) = 1/L(i,i);  X(j,i) = -( sum_{k=i}^{j-1} X(k,i) L(j,k) ) / L(j,j),  j > i.
 * This is forward substitution for L x = e_i (the recurrence of P:243). */
void oracle_crit_lower(int64_t n, const double* L, int64_t ldl, double* X, int64_t ldx, int unit) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < i; ++j) AT(X, ldx, j, i) = 0.0;
    AT(X, ldx, i, i) = unit ? 1.0 : 1.0 / AT(L, ldl, i, i);
    for (int64_t j = i + 1; j < n; ++j) {
      double dot = 0.0;
      for (int64_t k = i; k < j; ++k) dot += AT(X, ldx, k, i) * AT(L, ldl, j, k);
      AT(X, ldx, j, i) = unit ? -dot : -dot / AT(L, ldl, j, j);
    }
  }
}

/* Batched lower inverses: the lower definition applied per matrix. */
void oracle_crit_lower_batched(int64_t n, int64_t batch, const double* A, int64_t lda, int64_t sA,
                               double* X, int64_t ldx, int64_t sX, int unit) {
  #pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < batch; ++b) {
    const double* L = A + b * sA;
    double* Y = X + b * sX;
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t j = 0; j < i; ++j) AT(Y, ldx, j, i) = 0.0;
      AT(Y, ldx, i, i) = unit ? 1.0 : 1.0 / AT(L, lda, i, i);
      for (int64_t j = i + 1; j < n; ++j) {
        double dot = 0.0;
        for (int64_t k = i; k < j; ++k) dot += AT(Y, ldx, k, i) * AT(L, lda, j, k);
        AT(Y, ldx, j, i) = unit ? -dot : -dot / AT(L, lda, j, j);
      }
    }
  }
}

void oracle_crit_upper_batched(int64_t n, int64_t batch, const double* A, int64_t lda, int64_t sA,
                               double* X, int64_t ldx, int64_t sX, int unit) {
  for (int64_t b = 0; b < batch; ++b)
    oracle_crit_upper(n, A + b * sA, lda, X + b * sX, ldx, unit);
}

/* Column j of L^{-1}: forward substitution L x = e_j (same arithmetic, same
 * order as oracle_crit_lower column j, so bitwise equal to it).  Used for the
 * 64 sampled columns at large n.  x has length n. */
void oracle_lower_column(int64_t n, const double* L, int64_t ldl, int unit, int64_t j, double* x) {
  for (int64_t i = 0; i < j; ++i) x[i] = 0.0;
  x[j] = unit ? 1.0 : 1.0 / AT(L, ldl, j, j);
  for (int64_t i = j + 1; i < n; ++i) {
    double dot = 0.0;
    for (int64_t k = j; k < i; ++k) dot += x[k] * AT(L, ldl, i, k);
    x[i] = unit ? -dot : -dot / AT(L, ldl, i, i);
  }
}

/* Column j of U^{-1}: back substitution U x = e_j,
 *   x_j = 1/U_jj;  x_i = -( sum_{k=i+1}^{j} U_ik x_k ) / U_ii,  i = j-1 .. 0.
 * This is the definition of the inverse column (U x = e_j); it is a different
 * summation than CRIT's row recurrence (which solves S U = I), so it also
 * serves as an independent cross-check of oracle_crit_upper. */
void oracle_upper_column(int64_t n, const double* U, int64_t ldu, int unit, int64_t j, double* x) {
  for (int64_t i = j + 1; i < n; ++i) x[i] = 0.0;
  x[j] = unit ? 1.0 : 1.0 / AT(U, ldu, j, j);
  for (int64_t i = j - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int64_t k = i + 1; k <= j; ++k) dot += AT(U, ldu, i, k) * x[k];
    x[i] = unit ? -dot : -dot / AT(U, ldu, i, i);
  }
}

/* Many sampled columns in parallel.  cols[c] is the column index; the result
 * for cols[c] goes to out[c*n .. c*n+n-1]. uplo 'L' or 'U'. */
void oracle_columns(char uplo, int64_t n, const double* T, int64_t ld, int unit,
                    int64_t ncols, const int64_t* cols, double* out) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < ncols; ++c) {
    if (uplo == 'L') oracle_lower_column(n, T, ld, unit, cols[c], out + c * n);
    else oracle_upper_column(n, T, ld, unit, cols[c], out + c * n);
  }
}

/* Column j of A^{-1} = U^{-1} L^{-1} (SKUL: "S K = A^{-1}", with
 * S = U^{-1}, K = L^{-1}): y = L^{-1} e_j by forward substitution, then
 * x = U^{-1} y by back substitution (x_i = (y_i - sum_{k>i} U_ik x_k)/U_ii). */
void oracle_lu_column(int64_t n, const double* L, int64_t ldl, int unitL,
                      const double* U, int64_t ldu, int unitU, int64_t j, double* x, double* y) {
  oracle_lower_column(n, L, ldl, unitL, j, y);
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t k = i + 1; k < n; ++k) s -= AT(U, ldu, i, k) * x[k];
    x[i] = unitU ? s : s / AT(U, ldu, i, i);
  }
}

void oracle_lu_columns(int64_t n, const double* L, int64_t ldl, int unitL,
                       const double* U, int64_t ldu, int unitU,
                       int64_t ncols, const int64_t* cols, double* out) {
  #pragma omp parallel
  {
    double* y = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    #pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < ncols; ++c)
      oracle_lu_column(n, L, ldl, unitL, U, ldu, unitU, cols[c], out + c * n, y);
    free(y);
  }
}

/* ---------------------------------------------------------------------------
 * Brute-force Theorem 1 (Eq. TMatrixInversecombinatorixFormula),
 * generalised to a non-unit upper R by the decomposition R = D T of P:353
 * (D = diag(R), T = D^{-1} R unit upper), so R^{-1} = T^{-1} D^{-1}:
 *   S_ij = sum over sequences <i = a_1 < a_2 < ... < a_l = j> of H(i,j)
 *          (-1)^(l-1) prod_{t=1}^{l-1} T_{a_t, a_{t+1}},   S_ii = 1,
 *   (R^{-1})_ij = S_ij / R_jj.
 * H(i,j) is enumerated as the subsets of the interior {i+1..j-1} (Def. 1 read
 * as "all subsets of the interior", C17) in ascending bitmask order;
 * |H(i,j)| = 2^(j-i-1) (Prop. 1).  Exponential: n <= 24 only.
 * T_ab is formed as R_ab / R_aa (one IEEE division per factor).  unit != 0:
 * D = I and the stored diagonal is not read.
 * ------------------------------------------------------------------------- */
int oracle_pathsum_upper(int64_t n, const double* R, int64_t ldr, double* X, int64_t ldx, int unit) {
  if (n > 24) return -1;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) AT(X, ldx, i, j) = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i; j < n; ++j) {
      double s;
      if (j == i) {
        s = 1.0;
      } else {
        int64_t m = j - i - 1;               /* interior size */
        s = 0.0;
        for (uint64_t mask = 0; mask < (1ULL << m); ++mask) {
          double prod = 1.0;
          int64_t len = 1, a = i;            /* sequence starts at i */
          for (int64_t t = 0; t < m; ++t) {
            if (mask & (1ULL << t)) {
              int64_t nxt = i + 1 + t;
              double Tab = unit ? AT(R, ldr, a, nxt) : AT(R, ldr, a, nxt) / AT(R, ldr, a, a);
              prod = prod * Tab;
              a = nxt; ++len;
            }
          }
          double Taj = unit ? AT(R, ldr, a, j) : AT(R, ldr, a, j) / AT(R, ldr, a, a);
          prod = prod * Taj; ++len;          /* l = len elements */
          s += ((len - 1) % 2) ? -prod : prod; /* (-1)^(l-1) */
        }
      }
      AT(X, ldx, i, j) = unit ? s : s / AT(R, ldr, j, j);
    }
  }
  return 0;
}

/* Transposed form for lower L: X = (pathsum(L^T))^T. */
int oracle_pathsum_lower(int64_t n, const double* L, int64_t ldl, double* X, int64_t ldx, int unit) {
  if (n > 24) return -1;
  double* Lt = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  double* Xt = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) Lt[i * n + j] = AT(L, ldl, j, i);
  int rc = oracle_pathsum_upper(n, Lt, n, Xt, n, unit);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) AT(X, ldx, i, j) = Xt[j * n + i];
  free(Lt); free(Xt);
  return rc;
}

/* ---------------------------------------------------------------------------
 * SKUL (Algorithm 5) written out in the paper's order and notation,
 * 0-based: Crout factorisation A = L U (U_ii = 1) with the inverse factors
 * S = U^{-1} (by CRIT*, row recurrence) and K = L^{-1} computed online, and
 * finally K <- K D (D = diag(1/L_ii)).  S K = A^{-1}.  No pivoting
 * (the paper has none); returns 1 + i at the first zero L_ii, 0 otherwise.
 * All outputs are n x n row-major with leading dimension n.  The listing's
 * "S_{1,2} = -U_{1,2}" line is the l = 1, i = 1 instance of the S update and is
 * realised by running that update for i = 1 as well (reading C3 of DESIGN.md).
 * ------------------------------------------------------------------------- */
int oracle_skul(int64_t n, const double* A, double* L, double* U, double* S, double* K) {
  const int64_t N = n;
  double* D = (double*)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
  for (int64_t k = 0; k < N * N; ++k) { L[k] = 0.0; U[k] = 0.0; S[k] = 0.0; K[k] = 0.0; }
  int info = 0;
  for (int64_t i = 0; i < N; ++i) {                       /* for i = 1..n */
    L[i * N + 0] = A[i * N + 0];                          /*   L_{i,1} = A_{i,1} */
    U[i * N + i] = 1.0; S[i * N + i] = 1.0; K[i * N + i] = 1.0;
  }
  if (N == 0) { free(D); return 0; }
  if (L[0] == 0.0) info = 1;
  for (int64_t j = 1; j < N; ++j) U[0 * N + j] = A[0 * N + j] / L[0];  /* U_{1,j} = A_{1,j}/L_{1,1} */
  D[0] = 1.0 / L[0];
  if (N > 1) S[0 * N + 1] = -U[0 * N + 1];                 /* S_{1,2} = -U_{1,2} */
  for (int64_t i = 1; i < N; ++i) {                        /* for i = 2..n */
    for (int64_t j = 1; j <= i; ++j) {                     /*   L_{i,j} = A_{i,j} - L_{i,1:j-1} . U_{1:j-1,j} */
      double dot = 0.0;
      for (int64_t p = 0; p < j; ++p) dot += L[i * N + p] * U[p * N + j];
      L[i * N + j] = A[i * N + j] - dot;
    }
    if (L[i * N + i] == 0.0 && !info) info = (int)(i + 1);
    D[i] = 1.0 / L[i * N + i];                             /*   D_{i,i} = 1/L_{i,i} */
    for (int64_t j = 0; j < i; ++j) {                      /*   K_{i,j} = -L_{i,1:i} . K_{1:i,j} D_{i,i} */
      double dot = 0.0;
      for (int64_t p = 0; p <= i; ++p) dot += L[i * N + p] * K[p * N + j];
      K[i * N + j] = -dot * D[i];
    }
    for (int64_t j = i + 1; j < N; ++j) {                  /*   U_{i,j} = (A_{i,j} - L_{i,1:i-1} . U_{1:i-1,j}) / L_{i,i} */
      double dot = 0.0;
      for (int64_t p = 0; p < i; ++p) dot += L[i * N + p] * U[p * N + j];
      U[i * N + j] = (A[i * N + j] - dot) / L[i * N + i];
    }
    if (i < N - 1) {                                       /*   S_{l,i+1} = -S_{l,l:i} . U_{l:i,i+1}, l = 1..i */
      for (int64_t l = 0; l <= i; ++l) {
        double dot = 0.0;
        for (int64_t p = l; p <= i; ++p) dot += S[l * N + p] * U[p * N + i + 1];
        S[l * N + i + 1] = -dot;
      }
    }
  }
  for (int64_t i = 0; i < N; ++i)                          /* K <- K D */
    for (int64_t j = 0; j < N; ++j) K[i * N + j] *= D[j];
  free(D);
  return info;
}
