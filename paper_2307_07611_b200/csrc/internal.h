// internal.h — launchers shared between the kernel translation units and the
// C-ABI driver (trinv.cu).  Not part of the public ABI (include/trinv.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <utility>
#include <atomic>
#include <cstdint>
#include <cstdlib>

namespace trinv {

// Cached per-device SM count (host).
inline int device_sms() {
  static std::atomic<int> cache[64];
  int d = 0;
  cudaGetDevice(&d);
  d &= 63;
  int v = cache[d].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device.
template <auto Kernel>
inline void set_smem_once(int bytes) {
  static std::atomic<uint64_t> done{0};
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
  }
}

// Element-wise kernels without shared memory (Strassen's combination passes, geam, zero and
// copy passes) prefer the maximum L1 carve-out, once per kernel and device.  Round 2 finding
// (DESIGN.md §9b): with the default carve-out, two Strassen products on concurrent streams
// occasionally produced a wrong tile in a DMMA GEMM that shared its SMs with the other
// stream's element-wise CTAs; with this preference those CTAs no longer share an SM with
// the GEMMs' shared-memory-heavy CTAs and the reproducer (tools/strassen_concurrency.py)
// shows no error.  TRINV_ELEM_CARVEOUT=-1 restores the default (experiments).
template <auto Kernel>
inline void prefer_l1_once() {
  static std::atomic<uint64_t> done{0};
  static const int pref = [] { const char* e = std::getenv("TRINV_ELEM_CARVEOUT"); return e ? atoi(e) : 0; }();
  if (pref < 0) return;
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(Kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pref);
    done.fetch_or(bit, std::memory_order_release);
  }
}

// ---- leaf / batched kernels (leaf.cu) ------------------------------------------
struct LeafArgs {
  const double* A;
  int64_t lda, sA;
  double* X;
  int64_t ldx, sX;
  int64_t batch;    // number of matrices
  int n;            // order of matrices 0..batch-2
  int n_last;       // order of the last matrix (ragged leaf); == n for uniform batches
  int unit;         // 1: unit diagonal (not read)
  int32_t* info;    // NULL, per-matrix [batch], or a single accumulator
  int info_mode;    // 0 none, 1 per matrix, 2 single min-nonzero of (info_off + b*info_stride + i + 1)
  int64_t info_stride, info_off;
};
// Returns cudaError_t of the launch.  uplo 'L' or 'U'.  The TMA-staged path is
// taken when every address and size it moves is 16-byte aligned.
cudaError_t launch_leaf(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches);

// ---- batched 64 x 64, one warp per matrix, TMA-staged triangle (leaf64.cu) -------
// Taken for n == n_last == 64 with even ld / strides and 16-byte aligned pointers.
bool leaf64_tma_ok(const LeafArgs& a);
cudaError_t launch_leaf64_tma(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches);

// ---- whole-block inverses of order <= BLK_MAX, one CTA per block (blk.cu) --------
// Same LeafArgs contract (any ld / alignment; X == A allowed); a.n, a.n_last <= BLK_MAX.
constexpr int BLK_MAX = 128;
cudaError_t launch_blk(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches);

// ---- DMMA GEMM engine (gemm.cu) ---------------------------------------------------
enum GemmMode : int {
  MODE_LOWER_1 = 0,  // W   = C . A^{-1}          (C from input, A^{-1} lower from X)
  MODE_LOWER_2 = 1,  // X21 = -B^{-1} . W         (B^{-1} lower from X), mirror X12 := 0
  MODE_UPPER_1 = 2,  // W   = A^{-1} . B          (A^{-1} upper from X, B from input)
  MODE_UPPER_2 = 3,  // X12 = -W . C^{-1}         (C^{-1} upper from X), mirror X21 := 0
  MODE_UL = 4        // X   = U^{-1} . L^{-1}     (k >= max(i, j))
};

struct MatRef {
  const double* ptr;
  int64_t rows, cols, ld;  // bounds (elements) and leading dimension
};

struct LevelArgs {
  int mode;
  int64_t n;   // matrix order
  int64_t b;   // level block size (size of the first half of every merge); == n for UL
  int64_t merges;
  MatRef opA, opB;  // operand matrices (TMA-read)
  double* out;      // output matrix (row-major, ldo)
  int64_t ldo, out_rows, out_cols;
  double* mir;      // matrix whose mirrored tile is zero-filled (LOWER_2/UPPER_2), else NULL
  int64_t ldm;
  double alpha;
  // split-K (launch_level sets these): NULL / 0 = one CTA per output tile.  Else every tile's
  // K range is cut into chunks of kchunk; chunk c of a tile adds its partial product to the
  // tile after chunk c-1 has (a per-tile semaphore in sync[1..], a ticket counter in sync[0]
  // hands out work units in order): deterministic summation order.
  int* sync;        // LEVEL_SYNC_BYTES of device scratch (caller-provided), or NULL
  int32_t kchunk;
  // split_mode 2 ("fix-up"): no chunk waits.  Every chunk stores alpha * its partial in
  // partial[unit]; a per-tile arrival counter (sync[1 + tile], left at 0 again) elects the
  // last chunk to finish, which sums the tile's partials in chunk order into the output.
  int32_t split_mode;
  double* partial;  // LEVEL_PARTIAL_BYTES of device scratch, or NULL
  // stream-K launches of the mid-size levels (gemm.cu dmma_sk_level_kernel): SK_FLAG_INTS flags,
  // zero before the call's first level (left zero by every launch), and SK_PARTIAL_BYTES of
  // per-CTA partial tiles; NULL = one CTA per tile.
  int* sk_flags;
  double* sk_partial;
};
constexpr int SK_FLAG_INTS = 512;
constexpr size_t SK_PARTIAL_BYTES = (size_t)160 * 128 * 128 * sizeof(double);
constexpr size_t LEVEL_PARTIAL_BYTES = (size_t)48 << 20;  // split-K fix-up partial tiles
constexpr size_t LEVEL_SYNC_BYTES = 65536;  // split-K: ticket + tile semaphores; fused: tickets + W-tile flags
constexpr int LEVEL_TICKETS = 64;            // fused launches: one ticket per level of a call
constexpr int LEVEL_FLAG_MAX = 16384 - LEVEL_TICKETS;
// Both products of a level in one launch (gemm.cu FusedTraits): l1 = W = first product, l2 =
// second; l1.sync = the call's LEVEL_SYNC_BYTES, zeroed once per call; epoch in 1..63.
bool level_split_fixup();
bool level_sk_enabled();  // TRINV_SK=1: stream-K launches of the mid-size levels (opt-in)
// Level chain (gemm.cu): the lowest levels that run 32x32 tiles, all their products in one
// persistent dependency-driven launch.  ph[0..nphase) = [W, X21] per level, W by position
// (first products: out = W with ld = the widest chained level, out_rows = n; second products
// read W through a map of n rows); counters: nphase * cstride ints of device scratch.
bool level_chain_enabled();
bool level_uses_t32(const LevelArgs& a);
cudaError_t launch_level_chain(const LevelArgs* ph, int nphase, int* counters, int cstride, cudaStream_t s,
                               int64_t* launches);
bool level_fusable(const LevelArgs& l1);
cudaError_t launch_level_fused(const LevelArgs& l1, const LevelArgs& l2, int epoch, cudaStream_t s,
                               int64_t* launches);
cudaError_t launch_level(const LevelArgs& a, cudaStream_t s, int64_t* launches);

// General batched GEMM on the same engine: for g < batch,
//   C_g = alpha * A_g B_g + beta * C_g,  A_g: M x K (lda, stride sA), B_g: K x N (ldb, sB), C_g: M x N (ldc, sC),
// row-major.  triA / triB declare a triangular operand whose structurally zero
// blocks are skipped (A lower: A[i][k] = 0 for k > i; A upper: k < i; B lower:
// B[k][j] = 0 for k < j; B upper: k > j); its diagonal tiles must hold explicit
// zeros in the other triangle.  A, B 16-byte aligned with even ld / stride.
// C must not overlap A or B.
enum TriKind : int { TRI_NONE = 0, TRI_LOWER = 1, TRI_UPPER = 2 };
struct GemmArgs {
  int64_t M, N, K, batch;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  double alpha, beta;
  int triA, triB;
};
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s, int64_t* launches);

// ---- FP64 products on the INT8 tensor cores by modular arithmetic / CRT (oz2.cu) ----
bool oz2_supported(int64_t M, int64_t N, int64_t K);
size_t oz2_workspace_bytes(int64_t M, int64_t N, int64_t K);
// strict: bit 0 / bit 1 = the diagonal (k == i of A, k == j of B) is read as zero.
// skip: bit 0 / bit 1 = A / B already split into ws by launch_oz2_prepare.
cudaError_t launch_oz2_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                            int64_t ldb, int triB, double* C, int64_t ldc, double alpha, double beta, void* ws,
                            cudaStream_t st, int64_t* launches, int strict = 0, int skip = 0);
// The operand splits of launch_oz2_gemm alone (which: 1 = A, 2 = B), same workspace layout.
cudaError_t launch_oz2_prepare(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA,
                               const double* B, int64_t ldb, int triB, void* ws, cudaStream_t st, int which,
                               int64_t* launches, int strict = 0);
// X = S K (S upper, K lower, order n) on the modular engine with the diagonals split off:
// X = D_S D_K + D_S N_K + N_S D_K (one elementwise pass, exact up to one rounding) plus the
// product of the strictly triangular parts N_S N_K (row / column scales set by the
// off-diagonal entries alone).  ws: oz2_workspace_bytes(n, n, n).
cudaError_t launch_oz2_ul(int64_t n, const double* S, int64_t lds, const double* K, int64_t ldk, double* X,
                          int64_t ldx, void* ws, cudaStream_t st, int64_t* launches);

// ---- Crout factorisation of a diagonal block of order <= LU_MAX (lu.cu) -------
constexpr int LU_MAX = 128;
// Reads the block from W (ldw), writes the packed factors to F (ldf); F may equal W.
cudaError_t launch_lu_leaf(const double* W, int64_t ldw, double* F, int64_t ldf, int n, int32_t* info,
                           int64_t info_off, cudaStream_t s, int64_t* launches);
double gemm_flops(const GemmArgs& a);
cudaError_t launch_geam(int64_t rows, int64_t cols, double alpha, const double* A, int64_t lda, double beta,
                        const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s, int64_t* launches);
// p[i*ld + j] = +0.0 for i < rows, j < cols.
cudaError_t launch_zero_2d(double* p, int64_t ld, int64_t rows, int64_t cols, cudaStream_t s, int64_t* launches);
cudaError_t launch_copy_2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                           cudaStream_t s, int64_t* launches);

// ---- Strassen's recursion for dense square block products (strassen.cu, NEXT f3) ------
// C = beta C + alpha A B (h x h, row-major, 16-byte aligned, even ld) with `levels` levels of
// Strassen's 7 products over the DMMA GEMM; a level is applied while h % 4 == 0 and its
// products are >= min_q (else one GEMM).
size_t strassen_ws_bytes(int64_t h, int levels, int64_t min_q);
cudaError_t strassen_acc(int64_t h, double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double beta, double* C, int64_t ldc, int levels, int64_t min_q, void* ws, cudaStream_t s,
                         int64_t* launches);

// Programmatic dependent launch: launch `k` on `s` with the programmatic stream
// serialization attribute when pdl_enabled() (default on, TRINV_PDL=0 off), so that its launch
// overlaps the previous kernel's drain; `k` must call pdl_wait() before touching global memory
// the previous kernel produces or consumes (every launch_k kernel does so first).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Host helper: encode a 2-D FP64 tensor map (cuTensorMapEncodeTiled through the
// runtime's driver entry point).  Returns false on failure.
bool encode_map(CUtensorMap* m, const MatRef& r, int box_cols, int box_rows, bool swizzle128);
// General FP64 tiled map (no swizzle, zero OOB fill): dims[0] innermost, strides in bytes for dims 1..rank-1.
bool encode_map_nd(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box);

// Optional per-launch timing (trinv_profile_* in include/trinv.h): when enabled on
// this thread, every launch is bracketed by CUDA events on its stream.
// KIND_OZ: INT8 tensor-core products (oz.cu: the whole product; oz2.cu: the GEMM kernel);
// flops = FP64-equivalent, bytes = int8 ops.  KIND_OZAUX: oz2.cu's scaling / residue /
// reconstruction kernels; bytes = their algorithmic HBM bytes.
enum LaunchKind : int { KIND_LEAF = 0, KIND_DMMA = 1, KIND_OZ = 2, KIND_OZAUX = 3, KIND_COUNT = 4 };
struct ProfileScope {
  ProfileScope(int kind, double flops, double bytes, cudaStream_t s);
  ~ProfileScope();
  void* rec;
  cudaStream_t stream_ = nullptr;
};

}  // namespace trinv
