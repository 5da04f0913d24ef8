/*
 * trinv.h — C ABI of the B200-native FP64 triangular-inverse library
 * (hot path of arXiv 2307.07611, "fast inversion" of triangular matrices).
 *
 * Citations are to /root/reference/PAPER.md lines (P:NNN) with the section,
 * equation or algorithm they fall in; DESIGN.md lists the readings used where
 * the paper is silent (C1..C21 there).
 *
 * Conventions for every entry point
 *  - All matrices are IEEE fp64, ROW-MAJOR: element (i, j) of a matrix with
 *    leading dimension ld lives at ptr[i*ld + j], 0 <= i, j < n, ld >= n.
 *  - Matrix pointers (A, X, L, U, workspace) are DEVICE pointers; `stream`
 *    is a cudaStream_t (0 = legacy default stream).  Every call only ENQUEUES
 *    work on `stream` and returns; completion is observed through the stream.
 *  - Ownership: the caller allocates and frees every buffer.  The library
 *    never allocates device memory on the call path and keeps no pointer after
 *    returning (with the default product engine; the opt-in INT8 engine keeps a
 *    per-device guard scratch, see trinv_set_product_engine).  Buffers must
 *    stay alive until the enqueued work completes.
 *  - Only the referenced triangle of an input is used (the other triangle may
 *    hold anything, including NaN; it may be loaded but never enters the
 *    arithmetic).  With diag == TRINV_UNIT the stored diagonal is not used and
 *    is taken as 1 (CRIT*, Alg. 2).
 *  - Outputs are FULL matrices: the triangle opposite to the inverse's is
 *    written as +0.0 (Thm 1 "0, otherwise"; Eq. defT).
 *  - Synchronous errors (returned before anything is enqueued): see
 *    trinv_status_t.  n == 0 (or batch == 0) is a no-op returning TRINV_OK.
 *  - Asynchronous numerical status: an exact zero on a referenced diagonal
 *    ("If R_jj = 0 stop", P:713-714 / P:731-732) is reported through d_info
 *    (device int32, may be NULL) as 1 + the smallest such row index, 0 if
 *    none (LAPACK trtri convention).  The output of a singular input is
 *    unspecified (Inf/NaN).  NaN/Inf inputs propagate.  No host sync occurs
 *    (with the default product engine; the opt-in INT8 engine's scaling guard
 *    synchronises once per call, see trinv_set_product_engine).
 *  - Entry points are re-entrant and thread-safe; they may be called on any
 *    device (the current device is used).
 *  - Concurrency note (round 2, profiles/r02_strassen_concurrency.txt): two
 *    calls that take a Strassen path (trinv_lower / trinv_upper with n >=
 *    16384 at the default trinv_set_strassen threshold; inv_from_lu /
 *    inv_general with n >= 8192; trinv_gemm_strassen) running at the same time
 *    on different streams produced occasional wrong tiles until the library's
 *    element-wise kernels were given the maximum-L1 carve-out preference; with
 *    it the reproducer shows no error (tests/test_gpu_concurrency.py), but the
 *    root cause is not established, so the library itself never overlaps its
 *    Strassen work with other work, and callers who need certainty can
 *    serialise such calls or turn Strassen off (trinv_set_strassen(0)).
 */
#ifndef TRINV_H
#define TRINV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TRINV_OK = 0,
  TRINV_INVALID_ARG = 1,          /* n<0, ld<n, batch<0, stride too small, NULL with n>0, bad op/uplo */
  TRINV_ALIASING = 2,             /* input and output ranges overlap (non-batched calls) */
  TRINV_WORKSPACE_TOO_SMALL = 3,  /* ws_bytes < trinv_workspace_bytes(...) */
  TRINV_CUDA_ERROR = 4,           /* a CUDA launch or API call failed; see trinv_last_cuda_error() */
  TRINV_NOT_SUPPORTED = 5         /* request outside the implemented envelope (e.g. batched n > 128) */
} trinv_status_t;

typedef enum { TRINV_NON_UNIT = 0, TRINV_UNIT = 1 } trinv_diag_t;

/* Device workspace (bytes) needed by trinv_lower ('L'), trinv_upper ('U') or
 * inv_from_lu ('G') for order n.  A / X are the matrices that will be passed
 * (only their addresses' 16-byte alignment is inspected; NULL means
 * "aligned") with leading dimensions lda / ldx: an odd leading dimension or a
 * misaligned pointer makes the call stage that matrix through the workspace.
 * For 'G', A = L factor, X = output; the U factor is assumed laid out like L.
 * 'F' = lu_crout (A, X ignored), 'A' = inv_general (A = input, X = output).
 * Returns 0 for n <= 0 or an unknown op. */
size_t trinv_workspace_bytes(char op, int64_t n, const void* A, int64_t lda, const void* X, int64_t ldx);

/* X = L^{-1} for a non-singular LOWER-triangular L (n x n).
 * Method: COMBRIT with beta = 2 (Alg. 1), i.e.
 * the recursive split inv([A 0; C B]) = [A^{-1} 0; -B^{-1} C A^{-1}  B^{-1}]
 * (the transpose of P:1066-1069), bottom-up over levels; 32-wide diagonal
 * leaves are inverted in shared memory by the column recurrence of the proof
 * of Thm 1 (CRIT, Alg. 3); the off-diagonal products
 * run on the FP64 tensor cores (DMMA) fed by TMA.
 *   A, lda : input (device, read-only), only the lower triangle is used.
 *   X, ldx : output (device), full n x n written; must not overlap A
 *            (TRINV_ALIASING).
 *   ws     : device workspace of ws_bytes >= trinv_workspace_bytes('L', ...);
 *            may be NULL when that size is 0.
 *   d_info : device int32 or NULL (see above). */
trinv_status_t trinv_lower(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                           trinv_diag_t diag, void* ws, size_t ws_bytes, int32_t* d_info,
                           void* stream);

/* X = U^{-1} for a non-singular UPPER-triangular U; the mirror image of
 * trinv_lower: inv([A B; 0 C]) = [A^{-1}  -A^{-1} B C^{-1}; 0 C^{-1}]
 * (P:1066-1069).  Same arguments and rules as trinv_lower (op 'U'). */
trinv_status_t trinv_upper(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                           trinv_diag_t diag, void* ws, size_t ws_bytes, int32_t* d_info,
                           void* stream);

/* Batched small inverses: for b in [0, batch): X_b = T_b^{-1}, T_b at
 * A + b*strideA (leading dim lda), X_b at X + b*strideX (leading dim ldx).
 * uplo 'L' or 'U'; 1 <= n <= 128 (TRINV_NOT_SUPPORTED above).  Lane j computes
 * column j by the recurrence of P:243 (CRIT for the upper case) in
 * registers, one warp per matrix for n <= 32.  Orders 33..128 run one CTA per
 * matrix: 32-wide leaves by that recurrence, then the beta = 2 merges of
 * Alg. 1 on the FP64 tensor cores from shared memory.  For n = 32
 * with even lda/ldx/strides and 16-byte aligned pointers the referenced
 * triangle is staged in shared memory by 2-D TMA (cp.async.bulk.tensor);
 * other layouts use plain coalesced loads.
 * X == A exactly (in-place, same ld and stride) is allowed; any other overlap
 * is undefined.  strideA >= n*lda and strideX >= n*ldx are required.
 * d_info: NULL or device int32[batch], one status per matrix. */
trinv_status_t trinv_batched(char uplo, int64_t n, int64_t batch, const double* A, int64_t lda,
                             int64_t strideA, double* X, int64_t ldx, int64_t strideX,
                             trinv_diag_t diag, int32_t* d_info, void* stream);

/* Batched inverses of HOST-resident matrices (the end-to-end path): A_host and
 * X_host are host pointers to contiguous [batch][n][n] row-major arrays
 * (page-locked memory is required for the copies to overlap; pageable memory
 * works but serialises).  The batch is processed in chunks of `chunk` matrices
 * (0 = default 4096) cycling through TRINV_HOST_SLOTS device slots carved from
 * `ws`: the host->device copy of chunk i+1, the in-place inversion of chunk i
 * (trinv_batched) and the device->host copy of chunk i-1 run concurrently on
 * two internal copy streams and `stream`, ordered by events.  The call only
 * enqueues; when `stream` reaches the work enqueued by this call, every X_host
 * row is written.  X_host may equal A_host.  ws_bytes >=
 * trinv_batched_host_workspace_bytes(n, chunk); d_info as for trinv_batched
 * (device int32[batch] or NULL).  n <= 128. */
#define TRINV_HOST_SLOTS 4
size_t trinv_batched_host_workspace_bytes(int64_t n, int64_t chunk);
trinv_status_t trinv_batched_host(char uplo, int64_t n, int64_t batch, const double* A_host, double* X_host,
                                  trinv_diag_t diag, int64_t chunk, void* ws, size_t ws_bytes, int32_t* d_info,
                                  void* stream);

/* General inverse from triangular factors, X = (L U)^{-1} = U^{-1} L^{-1}
 * (SKUL, "S K = A^{-1}" with S = U^{-1}, K = L^{-1}): L^{-1} and
 * U^{-1} by the two calls above, then the upper x lower product
 * X_ij = sum_{k >= max(i,j)} (U^{-1})_ik (L^{-1})_kj  (P_UL) on the
 * DMMA engine (with the opt-in INT8 CRT engine and n >= its block threshold: the
 * diagonal terms in one elementwise pass and the strictly triangular product on the
 * INT8 tensor cores).  Lf (lower, ldl) and Uf (upper, ldu) are read-only; X
 * (ldx) must not overlap either (TRINV_ALIASING).  diagL / diagU select unit
 * factors (the paper's Crout makes U unit; BASELINE config 4 makes L
 * unit).  ws_bytes >= trinv_workspace_bytes('G', n, Lf, ldl, X, ldx).
 * d_info reports a zero diagonal of L first (1+i), then of U (n+1+i). */
trinv_status_t inv_from_lu(int64_t n, const double* Lf, int64_t ldl, const double* Uf, int64_t ldu,
                           double* X, int64_t ldx, trinv_diag_t diagL, trinv_diag_t diagU,
                           void* ws, size_t ws_bytes, int32_t* d_info, void* stream);

/* ---- NEXT row f2: general inverse from A ---------------------------
 * Crout factorisation without pivoting, A = L U with L lower (diagonal kept) and
 * U UNIT upper — the convention of the paper's SKUL (Alg. 5, "U_ii <- 1",
 * L_ij = A_ij - L_i,1:j-1 U_1:j-1,j, U_ij = (A_ij - L_i,1:i-1 U_1:i-1,j)/L_ii).
 * In place, packed: on return the lower triangle with the diagonal holds L and the
 * strict upper triangle holds U.  Blocked right-looking recursion: diagonal blocks
 * <= 128 in registers of one CTA, off-diagonal blocks U12 = L11^-1 A12 and L21 = A21 U11^-1
 * through the triangular inverses above and the DMMA engine, Schur complement on
 * the DMMA engine (with the opt-in INT8 engine, inv_general's own recursion routes its
 * products of blocks >= 2048 through it).  As in the paper there is no pivoting: the leading principal
 * minors must be non-zero; an exact zero pivot k sets d_info = 1 + k (output then
 * unspecified).  A: device, 16-byte aligned with even lda when n > 128
 * (TRINV_NOT_SUPPORTED otherwise).  ws_bytes >= trinv_workspace_bytes('F', n, ...). */
trinv_status_t lu_crout(int64_t n, double* A, int64_t lda, void* ws, size_t ws_bytes, int32_t* d_info,
                        void* stream);

/* X = A^{-1} for a general non-singular A with non-zero leading principal minors:
 * a Crout recursion on a copy of A that builds K = L^{-1} and S = U^{-1} alongside the
 * factors (the merges of the recursive split reuse the diagonal-block inverses), then
 * X = S K — SKUL's S K = A^{-1}.  Independent product pairs run on a second
 * stream forked from and joined to `stream`.  A is read-only (any layout); X must not
 * overlap A.  2 n^3 flops.
 * ws_bytes >= trinv_workspace_bytes('A', n, A, lda, X, ldx). */
trinv_status_t inv_general(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx, void* ws,
                           size_t ws_bytes, int32_t* d_info, void* stream);

/* The DMMA product engine as a batched GEMM: for g < batch,
 *   C_g = alpha * A_g B_g + beta * C_g,
 * A_g = A + g*strideA (M x K, lda), B_g = B + g*strideB (K x N, ldb), C_g = C +
 * g*strideC (M x N, ldc), all row-major fp64 on the device.  structA = 'L' / 'U'
 * declares A[i][k] = 0 for k > i / k < i (triangular structure anchored at its
 * top-left corner; the structurally zero blocks are skipped and the zeros inside
 * the diagonal tiles must be stored); structB = 'L' / 'U' declares B[k][j] = 0
 * for k < j / k > j; at most one operand may be structured; 'N' = dense.
 * A and B must be 16-byte aligned with even lda/ldb/strides (TRINV_NOT_SUPPORTED
 * otherwise); C must not overlap A or B.  K >= 1 (K = 0: TRINV_NOT_SUPPORTED). */
trinv_status_t trinv_gemm(int64_t M, int64_t N, int64_t K, int64_t batch, double alpha, const double* A,
                          int64_t lda, int64_t strideA, char structA, const double* B, int64_t ldb, int64_t strideB,
                          char structB, double beta, double* C, int64_t ldc, int64_t strideC, void* stream);

/* ---- NEXT row f4: COMBRIT block size beta ------------------------------------------
 * trinv_lower / trinv_upper use beta = 2.  trinv_tri_ex selects the block count of
 * the TOP level of Alg. 1: beta = 2 (same as trinv_lower/upper) or
 * beta = 4 (n = 4m, m = 32 * 2^k; the four diagonal blocks by the beta = 2 levels,
 * then B_ij = iD_ii A_ij, the block Thm 1 inverse of the unit block
 * triangle (via the recurrence of its proof) and iA_ij = iB_ij iD_jj
 * (P:452), all on the DMMA engine).  Other n with beta = 4: TRINV_NOT_SUPPORTED.
 * ws_bytes >= trinv_tri_ex_workspace_bytes(beta, n); A, X 16-byte aligned with
 * even leading dimensions for beta = 4. */
size_t trinv_tri_ex_workspace_bytes(int beta, int64_t n);
trinv_status_t trinv_tri_ex(char uplo, int beta, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                            trinv_diag_t diag, void* ws, size_t ws_bytes, int32_t* d_info, void* stream);

/* ---- NEXT row f3: Strassen inside the inversion ------------------------------------------
 * The paper's P_TF recursion (Eq. PTFmbk): a triangle-times-full product of order
 * 2h splits into four half-size triangle-times-full products and two full-times-full ones,
 * the latter by Strassen's 7-product recursion.  With levels > 0 (and
 * the DMMA engine) the single top merge of trinv_lower / trinv_upper (n = 2b, h = b/2 >=
 * min_h, h % 4 == 0) and the U^-1 L^-1 product of inv_from_lu (n % 8 == 0, n/2 >= min_h)
 * run by quadrants with up to `levels` Strassen levels in their dense h^3 products (a level
 * only while its half-size products are >= 2048); all other products are unchanged.
 * Default: levels 2, min_h 4096 (measured faster at equal floored error);
 * levels 0 = off.  levels 0..3, min_h >= 64, else TRINV_INVALID_ARG.  Strassen's error is
 * normwise: with it the DMMA path is no longer exactly invariant under power-of-two row /
 * column scalings for n >= 16384 (set levels 0 for that).  Process-wide; TRINV_STRASSEN=<levels> sets it before the first call.
 * Changes trinv_workspace_bytes ('L', 'U', 'G'): query it after.  DESIGN.md §11 has the
 * measured time and error that decide the default. */
trinv_status_t trinv_set_strassen(int levels, int64_t min_h);
int trinv_get_strassen(void);

/* NEXT row f3, standalone: C = A B for dense n x n (n % 4 == 0) with ONE level of Strassen's
 * 7-product recursion over the DMMA GEMM (the same routine the inversion uses above).
 * ws_bytes >= trinv_strassen_workspace_bytes(n); A, B, C 16-byte aligned with even ld
 * (TRINV_NOT_SUPPORTED otherwise). */
size_t trinv_strassen_workspace_bytes(int64_t n);
trinv_status_t trinv_gemm_strassen(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                   int64_t ldc, void* ws, size_t ws_bytes, void* stream);

/* Opt-in FP64-emulated product (Ozaki-II): C = alpha A B + beta C with the
 * products on the INT8 tensor cores (tcgen05 kind::i8) by modular arithmetic: operands
 * scaled row- / column-wise by powers of two to P-bit integers (P = 55 at K = 16384), 16
 * int8 products modulo 16 pairwise coprime moduli <= 256 and a CRT reconstruction of the
 * integer product as the centred fraction C' / M in 96-bit fixed point (error < 2^-85 M,
 * then FP64 roundings of 2^-53 relative).  The error is normwise (2^-P of the row / column
 * maxima), not componentwise as on DMMA.  A row of A or column of B holding NaN / Inf makes
 * that row / column of C NaN.  Row-major device matrices; structA / structB as in
 * trinv_gemm (one triangular operand at most, or 'U' x 'L').  Envelope: M % 128 == 0,
 * N % 256 == 0, K % 128 == 0, K <= 65536, else TRINV_NOT_SUPPORTED.  `digits` must be 0
 * (the digit-splitting variant was retired: TRINV_NOT_SUPPORTED otherwise).
 * ws: device scratch of trinv_gemm_oz_workspace_bytes(M, N, K, 0) bytes. */
size_t trinv_gemm_oz_workspace_bytes(int64_t M, int64_t N, int64_t K, int digits);
trinv_status_t trinv_gemm_oz(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                             char structA, const double* B, int64_t ldb, char structB, double beta, double* C,
                             int64_t ldc, int digits, void* ws, size_t ws_bytes, void* stream);

/* Product engine for the level products of trinv_lower / trinv_upper (and the
 * triangular inverses inside inv_from_lu, its U^-1 L^-1 product and the LU products of
 * inv_general): engine 0 (default) = FP64 DMMA (mma.sync) for every product, the engine
 * BJ.north_star names; 2 = opt-in FP64 emulation on the INT8 tensor cores (the modular
 * engine above) for every product whose blocks are >= min_block (>= 256; default 2048) and
 * whose shapes fit its envelope, all other products on DMMA.  Any other engine value:
 * TRINV_INVALID_ARG; `digits` is ignored.  Engine 2 runs a scaling guard per call: the
 * exact spread of the row- and column-maximum exponents of the input's referenced entries
 * (a unit diagonal counted as 1, its stored value not read) is computed on the device;
 * above 8 binades, or with any NaN / Inf entry, the call runs every product on DMMA.  The
 * guard costs one read of the input and ONE HOST SYNCHRONISATION per call (an event,
 * resolved when the first INT8 product is reached), a one-time 64-byte pinned host
 * allocation per thread and device and a per-device device scratch of 2 n doubles that
 * grows with n (allocated outside the workspace).  Under stream capture the guard cannot
 * run and the captured call uses DMMA.  Process-wide; the environment variable
 * TRINV_PRODUCTS=dmma|int8crt selects the engine before the first call.  Changing it
 * changes trinv_workspace_bytes ('L', 'U', 'G', 'A', 'F'): query the workspace after. */
trinv_status_t trinv_set_product_engine(int engine, int digits, int64_t min_block);
int trinv_get_product_engine(void);

/* The scaling guard of the INT8 engine on its own (for callers composing products
 * themselves, e.g. the multi-rank split): 1 when the row- and column-maximum exponents
 * of the n x n matrix A (device, ld lda; uplo 'L' / 'U' = only that triangle is read,
 * 'N' = all of it; diag = TRINV_UNIT: the stored diagonal is not read and counts as 1)
 * span at most 8 binades and every referenced entry is finite; 0 otherwise, and 0 when
 * `stream` is capturing (the check cannot run); -TRINV_INVALID_ARG / -TRINV_CUDA_ERROR
 * on error.  Waits for the check on `stream`. */
int trinv_int8_scaling_ok(int64_t n, const double* A, int64_t lda, char uplo, trinv_diag_t diag, void* stream);

/* Diagnostic (bench.py's roofline denominator, not a product path): the FP64 tensor-core
 * ceiling measured live — a register-only loop of mma.sync m8n8k4 f64 (DMMA.8x8x4, 512
 * flop per warp instruction) on 2 CTAs x 8 warps per SM, grown until one launch lasts
 * about ms_target milliseconds — in TFLOP/s at the current clocks.  SYNCHRONISES `stream`.
 * Returns a negative value on a CUDA error. */
double trinv_probe_dmma_tflops(double ms_target, void* stream);

/* Static description of a status code. */
const char* trinv_status_string(trinv_status_t s);

/* The last CUDA error code seen by this thread's calls (0 if none). */
int trinv_last_cuda_error(void);

/* Library version string, e.g. "trinv-b200 0.1 sm_100a". */
const char* trinv_version(void);

/* Observability: number of kernel launches enqueued by this thread's calls
 * since the last reset (used by bench.py for its "gpu_launches" count). */
int64_t trinv_launch_count(void);
void trinv_reset_launch_count(void);

/* Observability: per-launch device timing.  Between trinv_profile_begin() and
 * trinv_profile_end() every kernel this thread enqueues is bracketed by CUDA
 * events recorded on its stream (small overhead; for measurement runs only).
 * trinv_profile_read(kind, ...) synchronises those events and returns, for
 * kind 0 (leaf / batched kernels), 1 (DMMA product kernels), 2 (opt-in INT8
 * engine: the tensor-core GEMM kernel of the CRT engine; bytes = int8 operations)
 * or 3 (the CRT engine's scaling, residue
 * and reconstruction kernels; flops = 0), the device milliseconds covered by those
 * launches (the union of their intervals: launches on two streams may overlap), the
 * number of timed scopes and the ALGORITHMIC flops and bytes of those launches
 * (n^3/3 per leaf; triangular-aware products; leaf bytes
 * = referenced triangle in + full matrix out).
 * Any output pointer may be NULL.  Returns a trinv_status_t value. */
void trinv_profile_begin(void);
void trinv_profile_end(void);
int trinv_profile_read(int kind, double* ms, int64_t* launches, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* TRINV_H */
