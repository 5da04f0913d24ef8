// trinv.cu — C-ABI entry points (include/trinv.h) and the host-side recursion
// planner (§Boundary).
//
// trinv_lower / trinv_upper run COMBRIT with beta = 2 (Alg. 1)
// bottom-up: all 128-wide diagonal blocks in one launch (blk.cu: 32-wide
// leaves, "any preferred method", and the levels b = 32,
// 64 inside each CTA), then for b = 128, 256, ... < n one level of
// merges [s, s+b) + [s+b, s+2b) (the last one ragged, C13) with two grouped
// DMMA launches per level (launch_level, gemm.cu).  inv_from_lu adds the
// U^{-1} L^{-1} product.  Nothing here allocates device memory or
// synchronises the stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/trinv.h"
#include "internal.h"

namespace trinv {

// Programmatic dependent launch of the product / combination kernels (internal.h launch_k):
// on by default (TRINV_PDL=0 turns it off).  The dependents are released only as the previous
// grid's CTAs exit (ptx.cuh pdl_trigger_early): graph-replayed n = 1024 / 2048 71.2 -> 69.3 /
// 151.6 -> 149.3 us, configs 2 / 3 / 4 5.446 -> 5.419 / 309.5 -> 308.3 / 158.75 -> 158.08 ms.
// The first variant released them at the start of every CTA and was slower (n = 2048: 165 ->
// 198 us in round 2's first sessions; profiles/r02_pdl.txt).
bool pdl_enabled() {
  static const bool on = [] { const char* e = std::getenv("TRINV_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

static thread_local int g_last_cuda_error = 0;
static thread_local int64_t g_launches = 0;

// ---- optional per-launch profiling ------------------------------------------------
struct ProfRec {
  int kind;
  double flops, bytes;
  cudaEvent_t e0, e1;
};
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec>* g_prof = nullptr;

ProfileScope::ProfileScope(int kind, double flops, double bytes, cudaStream_t s) : rec(nullptr) {
  if (!g_prof_on) return;
  if (!g_prof) g_prof = new std::vector<ProfRec>();
  ProfRec r{kind, flops, bytes, nullptr, nullptr};
  cudaEventCreate(&r.e0);
  cudaEventCreate(&r.e1);
  cudaEventRecord(r.e0, s);
  g_prof->push_back(r);
  rec = reinterpret_cast<void*>(static_cast<uintptr_t>(g_prof->size()));
  stream_ = s;
}
ProfileScope::~ProfileScope() {
  if (!rec || !g_prof) return;
  const size_t i = reinterpret_cast<uintptr_t>(rec) - 1;
  cudaEventRecord((*g_prof)[i].e1, stream_);
}

// ---- tensor-map encoding through the runtime's driver entry point -----------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool encode_map(CUtensorMap* m, const MatRef& r, int box_cols, int box_rows, bool swizzle128) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)r.cols, (cuuint64_t)r.rows};
  cuuint64_t strides[1] = {(cuuint64_t)r.ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(r.ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

bool encode_map_nd(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc || rank < 1 || rank > 5) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides[i];
  CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), d, st, b, e,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

// ---- layout helpers -----------------------------------------------------------
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static bool tma_ok(const void* p, int64_t ld) { return p == nullptr ? (ld % 2 == 0) : (aligned16(p) && ld % 2 == 0); }
static int64_t even_up(int64_t x) { return (x + 1) & ~int64_t(1); }
static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// ---- product engine for the level products (trinv_set_product_engine) ---------------
// 0 (default): FP64 DMMA (mma.sync, gemm.cu) for every product — the engine BJ.north_star
// names for a5/a6.  2 (opt-in): FP64-emulated products on the INT8 tensor cores (Ozaki-II:
// 16 moduli + CRT, oz2.cu) for the levels whose block size is >= g_oz_min and whose shapes
// fit its envelope; every other level stays on DMMA.  TRINV_PRODUCTS=int8crt selects it
// before the first call.  (Engine 1, the digit-splitting variant, was retired.)
static std::atomic<int> g_engine{-1};
static std::atomic<int64_t> g_oz_min{2048};  // tools/minblock_probe.py: 2048 beats 1024 / 4096
static int product_engine() {
  int e = g_engine.load(std::memory_order_relaxed);
  if (e < 0) {
    const char* v = getenv("TRINV_PRODUCTS");
    e = (v && strcmp(v, "int8crt") == 0) ? 2 : 0;
    g_engine.store(e, std::memory_order_relaxed);
  }
  return e;
}

// ---- scaling guard of the opt-in INT8 engine -----------------------------------------------
// The INT8 engine truncates its operands relative to row / column maxima, so inputs whose
// rows or columns span many binades lose accuracy there (1.2e-10 at a
// 2^+-16 row / column scaling, 9e-4 beyond 2^+-30) while the DMMA path is exactly scaling
// invariant.  Before a call that would use it, the exact spread of the row-maximum
// exponents and of the column-maximum exponents of the input's referenced entries is
// computed on the device (one read of the referenced part for the rows, one for the
// columns; with a unit diagonal the stored diagonal is skipped and the implicit 1 enters
// both maxima); above OZ_MAX_SPREAD (8) binades, or when any referenced entry is NaN / Inf,
// the call runs every product on DMMA (which propagates non-finite values).  The decision
// needs the result on the host: the opt-in engine synchronises on one event per call (the
// default DMMA engine never does).  Under stream capture the guard cannot run, so a
// captured call always uses DMMA.
// 8 binades: the engine's floored elementwise error measured ~1.3e-14 x 2^spread on row-scaled
// BASELINE inputs (tests/test_gpu_scaling.py: 3.5e-9 at 18, 3.4e-8 at 20 binades, above the
// 1e-10 gate), so 8 keeps a 30x margin; BASELINE inputs have spread 0.
constexpr int OZ_MAX_SPREAD = 8;
constexpr int SPREAD_ROWS = 256;  // rows per block of the column pass
// Per call: the check kernels run first on the call's stream and copy their 5 ints per
// checked matrix to pinned host memory behind an event; the decision is taken (event
// synchronize) only when the first INT8-eligible product is reached, so the host waits
// while the GPU works through the leaves and the small DMMA levels.
struct ScaleCheck {
  int* dev = nullptr;        // [2 matrices][8] ints, then [2][n] column-maximum bits
  int* host = nullptr;       // pinned [16]
  cudaEvent_t ev = nullptr;
  int nmat = 0;              // matrices checked in this call
  bool pending = false;
};
static thread_local ScaleCheck g_check[64];
static thread_local bool g_int8_veto = false;
static thread_local ScaleCheck* g_pending = nullptr;
// RAII scope of one public call (active = true): fresh veto / pending-check state, the
// caller's restored at exit.  Internal calls (active = false) share their caller's state.
struct Int8Scope {
  bool active, prev_veto = false;
  ScaleCheck* prev_pending = nullptr;
  explicit Int8Scope(bool a) : active(a) {
    if (!active) return;
    prev_veto = g_int8_veto;
    prev_pending = g_pending;
    g_int8_veto = false;
    g_pending = nullptr;
  }
  ~Int8Scope() {
    if (!active) return;
    if (g_pending && g_pending->pending) {  // never resolved: let its copy land before reuse
      cudaEventSynchronize(g_pending->ev);
      g_pending->pending = false;
    }
    g_int8_veto = prev_veto;
    g_pending = prev_pending;
  }
};
__device__ __forceinline__ int spread_exp(double m) {
  int e;
  frexp(m, &e);
  return e;
}
// NaN-propagating maximum of magnitudes: as unsigned bit patterns, +NaN > +Inf > finite
__device__ __forceinline__ double spread_max(double m, double x) {
  const double a = fabs(x);
  return (a > m || a != a) ? a : m;
}
// r: [0] min row exponent, [1] max, [2] min column exponent, [3] max, [4] non-finite seen
__global__ void spread_init_kernel(int* r, unsigned long long* cmax, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) cmax[j] = 0ull;
  if (j == 0) { r[0] = r[2] = 1 << 30; r[1] = r[3] = -(1 << 30); r[4] = 0; }
}
__device__ __forceinline__ void spread_note(int* r, int lo, int hi, double m) {
  if (!(m <= 1.7976931348623157e308)) { atomicOr(&r[4], 1); return; }  // NaN or Inf
  if (m > 0.0) {
    const int e = spread_exp(m);
    atomicMin(&r[lo], e);
    atomicMax(&r[hi], e);
  }
}
// row maxima over the referenced part of every row (uplo 'L' / 'U' / 'N'; unit: the stored
// diagonal is skipped and the implicit 1 counted): one block per row
__global__ void spread_rows_kernel(const double* A, int64_t lda, int n, char uplo, int unit, int* r) {
  __shared__ double red[8];
  const int i = blockIdx.x;
  const int j0 = uplo == 'U' ? i : 0, j1 = uplo == 'L' ? i + 1 : n;
  double m = unit ? 1.0 : 0.0;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x)
    if (!(unit && j == i)) m = spread_max(m, A[(int64_t)i * lda + j]);
  for (int o = 16; o; o >>= 1) m = spread_max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = spread_max(m, red[w]);
    spread_note(r, 0, 1, m);
  }
}
// column maxima: thread per column over SPREAD_ROWS rows of its block (blockIdx.y), all
// referenced rows of the column across the grid; combined by an atomic max on the bits
__global__ void spread_cols_kernel(const double* A, int64_t lda, int n, char uplo, int unit, unsigned long long* cmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * SPREAD_ROWS, i1 = min(n, i0 + SPREAD_ROWS);
  if (j >= n) return;
  int lo = i0, hi = i1;  // referenced rows of column j: lower i >= j, upper i <= j
  if (uplo == 'L') lo = max(lo, j);
  if (uplo == 'U') hi = min(hi, j + 1);
  double m = (unit && j >= i0 && j < i1) ? 1.0 : 0.0;
#pragma unroll 4
  for (int i = lo; i < hi; ++i)
    if (!(unit && i == j)) m = spread_max(m, A[(int64_t)i * lda + j]);
  if (m != 0.0) atomicMax(&cmax[j], (unsigned long long)__double_as_longlong(m));
}
__global__ void spread_colred_kernel(const unsigned long long* cmax, int n, int* r) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  spread_note(r, 2, 3, __longlong_as_double((long long)cmax[j]));
}
// launch the check of one input matrix of the current call (under stream capture: veto)
static void int8_check_begin(const double* A, int64_t lda, int64_t n, char uplo, int unit, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    g_int8_veto = true;
    return;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) { g_int8_veto = true; return; }
  ScaleCheck& c = g_check[dev];
  static thread_local int64_t cap[64] = {};
  // one-time per thread and device: the pinned result slot; the device scratch grows with n
  if (!c.host) {
    if (cudaMallocHost(&c.host, 16 * sizeof(int)) != cudaSuccess) { c.host = nullptr; g_int8_veto = true; return; }
    if (cudaEventCreateWithFlags(&c.ev, cudaEventDisableTiming) != cudaSuccess) { g_int8_veto = true; return; }
  }
  if (cap[dev] < n) {  // [16 ints | 2 x n column maxima]
    if (c.dev) cudaFree(c.dev);
    if (cudaMalloc(&c.dev, 256 + 2 * (size_t)n * 8) != cudaSuccess) {
      c.dev = nullptr; cap[dev] = 0; g_int8_veto = true; return;
    }
    cap[dev] = n;
  }
  if (g_pending != &c) { c.nmat = 0; c.pending = true; g_pending = &c; }
  if (c.nmat >= 2) return;
  int* r = c.dev + 8 * c.nmat;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(c.dev) + 256) + c.nmat * n;
  const unsigned cb = (unsigned)((n + 255) / 256);
  spread_init_kernel<<<cb, 256, 0, s>>>(r, cmax, (int)n);
  spread_rows_kernel<<<(unsigned)n, 256, 0, s>>>(A, lda, (int)n, uplo, unit, r);
  spread_cols_kernel<<<dim3(cb, (unsigned)((n + SPREAD_ROWS - 1) / SPREAD_ROWS)), 256, 0, s>>>(A, lda, (int)n, uplo,
                                                                                                unit, cmax);
  spread_colred_kernel<<<cb, 256, 0, s>>>(cmax, (int)n, r);
  g_launches += 4;
  ++c.nmat;
  cudaMemcpyAsync(c.host, c.dev, 8 * c.nmat * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaEventRecord(c.ev, s);
}
// the veto for the current call: resolves a pending check (waits for its event only)
static bool int8_veto() {
  if (g_pending && g_pending->pending) {
    ScaleCheck& c = *g_pending;
    c.pending = false;
    if (cudaEventSynchronize(c.ev) == cudaSuccess) {
      for (int m = 0; m < c.nmat; ++m) {
        const int* h = c.host + 8 * m;
        const int sr = h[1] >= h[0] ? h[1] - h[0] : 0, sc = h[3] >= h[2] ? h[3] - h[2] : 0;
        if (std::max(sr, sc) > OZ_MAX_SPREAD || h[4] != 0) g_int8_veto = true;
      }
    } else {
      g_int8_veto = true;
    }
  }
  return g_int8_veto;
}
// whether a call of order n would run any product on an INT8 engine (sizes only)
static bool int8_would_run(int64_t n);  // defined below with the level predicates

// Number of merges at level b: g with 2gb + b < n.
static int64_t merges_at(int64_t n, int64_t b) { return (n - b + 2 * b - 1) / (2 * b); }

// Scratch for the off-diagonal products W (every merge owns b rows x b columns).
static size_t w_bytes(int64_t n) {
  size_t best = 0;
  for (int64_t b = 32; b < n; b *= 2) best = std::max(best, (size_t)(merges_at(n, b) * b * b) * sizeof(double));
  return best;
}
static size_t mat_bytes(int64_t n) { return (size_t)n * (size_t)even_up(n) * sizeof(double); }

// INT8 engine: a level takes it when every merge's two products fit the envelope
// (lower: r x b x b and r x b x r; upper: b x r x b and b x r x r); its scratch is the
// largest of those products' workspaces.
static bool oz_shape_ok(int64_t M, int64_t N, int64_t K) { return oz2_supported(M, N, K); }
static size_t oz_shape_ws(int64_t M, int64_t N, int64_t K) { return oz2_workspace_bytes(M, N, K); }
static cudaError_t oz_product(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                              int64_t ldb, int triB, double* C, int64_t ldc, double alpha, void* ws, cudaStream_t s) {
  return launch_oz2_gemm(M, N, K, A, lda, triA, B, ldb, triB, C, ldc, alpha, 0.0, ws, s, &g_launches);
}
static bool oz_level_ok(int64_t n, int64_t b) {
  if (product_engine() == 0 || b < g_oz_min.load() || b % 256) return false;
  for (int64_t s = 0; s + b < n; s += 2 * b) {
    const int64_t r = std::min(b, n - s - b);
    if (r % 256 || !oz_shape_ok(r, b, b) || !oz_shape_ok(r, b, r) || !oz_shape_ok(b, r, b) || !oz_shape_ok(b, r, r))
      return false;
  }
  return true;
}
// A second stream per device for the independent product pairs of lu_inv_rec (U12 / L21,
// the K21 / S12 chains, the two leaf inversions): forked from and joined back to the
// caller's stream by events, so ordering with the caller's work is unchanged and the pair
// is captured as two graph branches under stream capture.
struct ForkCtx {
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static cudaError_t fork_ctx(ForkCtx** out) {
  static thread_local ForkCtx ctx[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  ForkCtx& c = ctx[dev];
  if (!c.aux) {
    if ((e = cudaStreamCreateWithFlags(&c.aux, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  *out = &c;
  return cudaSuccess;
}
static cudaError_t fork_to(ForkCtx* c, cudaStream_t s) {
  cudaError_t e = cudaEventRecord(c->fork, s);
  return e != cudaSuccess ? e : cudaStreamWaitEvent(c->aux, c->fork, 0);
}
static cudaError_t join_from(ForkCtx* c, cudaStream_t s) {
  cudaError_t e = cudaEventRecord(c->join, c->aux);
  return e != cudaSuccess ? e : cudaStreamWaitEvent(s, c->join, 0);
}

// Scratch of one INT8 product of level b (the largest of its merges' products).
static size_t oz_level_scratch(int64_t n, int64_t b) {
  size_t best = 0;
  for (int64_t s = 0; s + b < n; s += 2 * b) {
    const int64_t r = std::min(b, n - s - b);
    for (size_t v : {oz_shape_ws(r, b, b), oz_shape_ws(r, b, r), oz_shape_ws(b, r, b), oz_shape_ws(b, r, r)})
      best = std::max(best, v);
  }
  return align_up(best);
}
// Levels with two or more merges run their merges alternately on two streams, each with
// its own product scratch (run_tri): the residue / reconstruction kernels of one merge
// overlap the tensor-core GEMM of the other.
// With the CRT engine a single-merge level (the top level) splits its second product's
// inverse-block operand on the second stream while the first product runs: two scratches.
static size_t oz_scratch(int64_t n) {
  if (product_engine() == 0 || n <= BLK_MAX) return 0;
  size_t best = 0;
  for (int64_t b = BLK_MAX; b < n; b *= 2)
    if (oz_level_ok(n, b))
      best = std::max(best, 2 * oz_level_scratch(n, b));
  return best;
}

// whether a triangular inverse of order n runs any level product on an INT8 engine
static bool int8_would_run(int64_t n) {
  if (product_engine() == 0) return false;
  for (int64_t b = BLK_MAX; b < n; b *= 2)
    if (oz_level_ok(n, b)) return true;
  return false;
}

// The U^{-1} L^{-1} product on the INT8 CRT engine: the diagonals of both factors are split
// off (launch_oz2_ul), because with them in the row / column maxima the scaled product of
// factors with a dominant diagonal and small entries off it left the smallest entries of
// S K with ~2^-39 relative precision (config 4 measured 1.0e-10 against the 1e-10 gate).
static bool ul_on_int8(int64_t n) {
  return product_engine() == 2 && n >= g_oz_min.load() && oz2_supported(n, n, n);
}

// ---- NEXT row f3: Strassen in the dense quadrant products of the top level ------------------
// The paper's P_TF recursion (Eq. PTFmbk): a triangle-times-full product of order
// 2h splits into 4 half-size triangle-times-full products and 2 full-times-full ones, the latter
// by Strassen's 7-product recursion.  With g_strassen_levels > 0 the top
// merge of a triangular inverse (one merge, n = 2b, h = b/2 >= g_strassen_min, h % 4 == 0) and
// the U^-1 L^-1 product of inv_from_lu run that way on the DMMA engine (strassen.cu);
// TRINV_STRASSEN=<levels> sets it before the first call.  Default 2 levels from h = 4096 (each
// level only while its products stay >= 2048): config 3 327.9 -> 316.3 ms, config 4 165.5 ->
// ~163 ms at unchanged floored error (profiles/r02_strassen_inversion.txt).
static std::atomic<int> g_strassen_levels{-1};
static std::atomic<int64_t> g_strassen_min{4096};
static int strassen_levels() {
  int l = g_strassen_levels.load(std::memory_order_relaxed);
  if (l < 0) {
    const char* v = getenv("TRINV_STRASSEN");
    l = v ? std::max(0, std::min(3, atoi(v))) : 2;
    g_strassen_levels.store(l, std::memory_order_relaxed);
  }
  return l;
}
static int64_t strassen_min_q() { return std::max<int64_t>(16, g_strassen_min.load() / 2); }
static bool strassen_top(int64_t n, int64_t b) {  // does the merge at level b take the Strassen path?
  const int64_t h = b / 2;
  return strassen_levels() > 0 && product_engine() == 0 && n == 2 * b && h % 4 == 0 &&
         h >= g_strassen_min.load();
}
static int64_t top_block(int64_t n) {  // the block size of the top level (its single merge)
  int64_t b = BLK_MAX;
  while (2 * b < n) b *= 2;
  return b;
}
static size_t strassen_scratch(int64_t n) {
  const int64_t b = top_block(n);
  return (n > BLK_MAX && strassen_top(n, b)) ? align_up(strassen_ws_bytes(b / 2, strassen_levels(), strassen_min_q())) : 0;
}
static bool strassen_ul(int64_t n) {
  return strassen_levels() > 0 && product_engine() == 0 && n % 8 == 0 && n / 2 >= g_strassen_min.load();
}

static size_t partial_bytes() { return level_split_fixup() ? LEVEL_PARTIAL_BYTES : 0; }
// stream-K scratch of the mid-size level launches: flags + per-CTA partial tiles
static size_t sk_bytes() { return level_sk_enabled() ? align_up(SK_FLAG_INTS * sizeof(int)) + SK_PARTIAL_BYTES : 0; }

static size_t tri_ws(int64_t n, const void* A, int64_t lda, const void* X, int64_t ldx) {
  if (n <= BLK_MAX) return 0;  // a single block: no products, any layout
  size_t bytes = align_up(w_bytes(n)) + oz_scratch(n) + strassen_scratch(n) + LEVEL_SYNC_BYTES + partial_bytes() +
                 sk_bytes();
  if (!tma_ok(A, lda)) bytes += align_up(mat_bytes(n));
  if (!tma_ok(X, ldx)) bytes += align_up(mat_bytes(n));
  return bytes;
}

static bool overlap(const double* a, int64_t lda, const double* x, int64_t ldx, int64_t n) {
  const char* a0 = reinterpret_cast<const char*>(a);
  const char* a1 = reinterpret_cast<const char*>(a + (n - 1) * lda + n);
  const char* x0 = reinterpret_cast<const char*>(x);
  const char* x1 = reinterpret_cast<const char*>(x + (n - 1) * ldx + n);
  return a0 < x1 && x0 < a1;
}

static trinv_status_t cuda_fail(cudaError_t e) {
  if (e == cudaSuccess) return TRINV_OK;
  g_last_cuda_error = (int)e;
  return TRINV_CUDA_ERROR;
}
#define TRY(expr)                                   \
  do {                                              \
    trinv_status_t _st = cuda_fail((expr));         \
    if (_st != TRINV_OK) return _st;                \
  } while (0)

static cudaError_t gemm_tri(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, int triA,
                            const double* B, int64_t ldb, int triB, double beta, double* C, int64_t ldc,
                            cudaStream_t s) {
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K; g.batch = 1;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta; g.triA = triA; g.triB = triB;
  return launch_gemm(g, s, &g_launches);
}
// C = alpha A B + beta C for square operands of order h, exactly one of them triangular
// (P_TF = h^3), by its quadrants (the recursion of Eq. PTFmbk): the
// two dense quadrant products (half the flops) by Strassen's recursion, the four triangular
// ones by this function again, down to quadrants below the Strassen size (then one
// triangular DMMA GEMM).  E.g. A lower = [A11 0; A21 A22]:
//   C1j = beta C1j + alpha A11 B1j,   C2j = beta C2j + alpha (A22 B2j + A21 B1j)   (j = 1, 2).
// The triangular operand's diagonal quadrants keep their explicit zeros (as gemm_tri needs).
// sws >= strassen_ws_bytes(h / 2, ...); one stream.  NEXT f3.
static bool trmm_split_ok(int64_t h) {
  static const bool on = [] { const char* e = std::getenv("TRINV_TRMM"); return !(e && e[0] == '0'); }();
  return on && strassen_levels() > 0 && product_engine() == 0 && h % 8 == 0 && h / 2 >= g_strassen_min.load();
}
static cudaError_t trmm_sq(int64_t h, double alpha, const double* A, int64_t lda, int triA, const double* B,
                           int64_t ldb, int triB, double beta, double* C, int64_t ldc, void* sws, cudaStream_t s) {
  if (!sws || !trmm_split_ok(h)) return gemm_tri(h, h, h, alpha, A, lda, triA, B, ldb, triB, beta, C, ldc, s);
  const int64_t q = h / 2;
  auto a = [&](int i, int j) { return A + i * q * lda + j * q; };
  auto b = [&](int i, int j) { return B + i * q * ldb + j * q; };
  auto c = [&](int i, int j) { return C + i * q * ldc + j * q; };
  const int lv = strassen_levels();
  const int64_t mq = strassen_min_q();
  cudaError_t e;
#define T_TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  auto dense = [&](const double* X, int64_t lx, const double* Y, int64_t ly, double bt, double* Z) {
    return strassen_acc(q, alpha, X, lx, Y, ly, bt, Z, ldc, lv, mq, sws, s, &g_launches);
  };
  auto tri = [&](const double* X, const double* Y, double bt, double* Z) {
    return trmm_sq(q, alpha, X, lda, triA, Y, ldb, triB, bt, Z, ldc, sws, s);
  };
  for (int j = 0; j < 2; ++j) {
    if (triA == TRI_LOWER) {         // A = [A11 0; A21 A22]
      T_TRY(tri(a(0, 0), b(0, j), beta, c(0, j)));
      T_TRY(tri(a(1, 1), b(1, j), beta, c(1, j)));
      T_TRY(dense(a(1, 0), lda, b(0, j), ldb, 1.0, c(1, j)));
    } else if (triA == TRI_UPPER) {  // A = [A11 A12; 0 A22]
      T_TRY(tri(a(0, 0), b(0, j), beta, c(0, j)));
      T_TRY(dense(a(0, 1), lda, b(1, j), ldb, 1.0, c(0, j)));
      T_TRY(tri(a(1, 1), b(1, j), beta, c(1, j)));
    } else if (triB == TRI_LOWER) {  // B = [B11 0; B21 B22]:  Cj1 = Aj1 B11 + Aj2 B21, Cj2 = Aj2 B22
      T_TRY(tri(a(j, 0), b(0, 0), beta, c(j, 0)));
      T_TRY(dense(a(j, 1), lda, b(1, 0), ldb, 1.0, c(j, 0)));
      T_TRY(tri(a(j, 1), b(1, 1), beta, c(j, 1)));
    } else {                         // B = [B11 B12; 0 B22]:  Cj1 = Aj1 B11, Cj2 = Aj1 B12 + Aj2 B22
      T_TRY(tri(a(j, 0), b(0, 0), beta, c(j, 0)));
      T_TRY(tri(a(j, 1), b(1, 1), beta, c(j, 1)));
      T_TRY(dense(a(j, 0), lda, b(0, 1), ldb, 1.0, c(j, 1)));
    }
  }
#undef T_TRY
  return cudaSuccess;
}

// The single top merge of order n = 2b with the quadrant decomposition (h = b/2):
//   lower  W = C A^-1,  A^-1 = [P 0; Q R]:  W = [C1 P + C2 Q, C2 R];
//          X21 = -B^-1 W, B^-1 = [P' 0; Q' R']:  X21 = -[P' W1; Q' W1 + R' W2]
//   upper  W = A^-1 B,  A^-1 = [P Q; 0 R]:  W = [P B1 + Q B2; R B2];
//          X12 = -W C^-1, C^-1 = [P' Q'; 0 R']:  X12 = -[W1 P', W1 Q' + W2 R']
// Triangular quadrant products on the DMMA GEMM with their structurally zero blocks skipped;
// the dense ones (C2 Q, Q' W1 / Q B2, W1 Q': two h^3 squares each) by strassen_acc.
static cudaError_t strassen_merge(char uplo, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                                  double* W, void* sws, cudaStream_t s) {
  const int64_t b = n / 2, h = b / 2;
  const int lv = strassen_levels();
  const int64_t mq = strassen_min_q();
  const double* Ai = X;                    // A^-1 (b x b)
  const double* Bi = X + b * ldx + b;      // B^-1 / C^-1 (b x b)
  cudaError_t e;
#define M_TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  if (uplo == 'L') {
    const double* C = A + b * lda;  // b x b, input rows b.., cols 0..b
    double* X21 = X + b * ldx;
    for (int64_t r0 = 0; r0 < b; r0 += h) {                                                             // C1 P
      M_TRY(trmm_sq(h, 1.0, C + r0 * lda, lda, TRI_NONE, Ai, ldx, TRI_LOWER, 0.0, W + r0 * b, b, sws, s));
      M_TRY(strassen_acc(h, 1.0, C + r0 * lda + h, lda, Ai + h * ldx, ldx, 1.0, W + r0 * b, b, lv, mq, sws, s,
                         &g_launches));                                                                   // + C2 Q
      M_TRY(trmm_sq(h, 1.0, C + r0 * lda + h, lda, TRI_NONE, Ai + h * ldx + h, ldx, TRI_LOWER, 0.0, W + r0 * b + h,
                    b, sws, s));                                                                          // C2 R
    }
    for (int64_t c0 = 0; c0 < b; c0 += h) {
      M_TRY(trmm_sq(h, -1.0, Bi, ldx, TRI_LOWER, W + c0, b, TRI_NONE, 0.0, X21 + c0, ldx, sws, s));    // -P' W1
      M_TRY(trmm_sq(h, -1.0, Bi + h * ldx + h, ldx, TRI_LOWER, W + h * b + c0, b, TRI_NONE, 0.0,
                    X21 + h * ldx + c0, ldx, sws, s));                                                    // -R' W2
    }
    for (int64_t c0 = 0; c0 < b; c0 += h)                                                                 // - Q' W1
      M_TRY(strassen_acc(h, -1.0, Bi + h * ldx, ldx, W + c0, b, 1.0, X21 + h * ldx + c0, ldx, lv, mq, sws, s,
                         &g_launches));
    M_TRY(launch_zero_2d(X + b, ldx, b, b, s, &g_launches));
  } else {
    const double* B = A + b;  // b x b, input rows 0..b, cols b..
    double* X12 = X + b;
    for (int64_t c0 = 0; c0 < b; c0 += h) {
      M_TRY(trmm_sq(h, 1.0, Ai, ldx, TRI_UPPER, B + c0, lda, TRI_NONE, 0.0, W + c0, b, sws, s));          // P B1
      M_TRY(strassen_acc(h, 1.0, Ai + h, ldx, B + h * lda + c0, lda, 1.0, W + c0, b, lv, mq, sws, s,
                         &g_launches));                                                                   // + Q B2
      M_TRY(trmm_sq(h, 1.0, Ai + h * ldx + h, ldx, TRI_UPPER, B + h * lda + c0, lda, TRI_NONE, 0.0, W + h * b + c0,
                    b, sws, s));                                                                          // R B2
    }
    for (int64_t r0 = 0; r0 < b; r0 += h) {
      M_TRY(trmm_sq(h, -1.0, W + r0 * b, b, TRI_NONE, Bi, ldx, TRI_UPPER, 0.0, X12 + r0 * ldx, ldx, sws, s));  // -W1 P'
      M_TRY(trmm_sq(h, -1.0, W + r0 * b + h, b, TRI_NONE, Bi + h * ldx + h, ldx, TRI_UPPER, 0.0,
                    X12 + r0 * ldx + h, ldx, sws, s));                                                    // -W2 R'
    }
    for (int64_t r0 = 0; r0 < b; r0 += h)                                                                 // - W1 Q'
      M_TRY(strassen_acc(h, -1.0, W + r0 * b, b, Bi + h, ldx, 1.0, X12 + r0 * ldx + h, ldx, lv, mq, sws, s,
                         &g_launches));
    M_TRY(launch_zero_2d(X + b * ldx, ldx, b, b, s, &g_launches));
  }
#undef M_TRY
  return cudaSuccess;
}

// Core recursion on an aligned, even-ld problem (or n <= 32 in any layout).
// info: NULL or a single accumulator already initialised by the caller.
// aux: NULL, or the public entry's scratch after W and the INT8 scratch: [Strassen scratch |
// LEVEL_SYNC_BYTES of split-K tickets / semaphores]; without it the top merge stays on the
// level launches and no level is split along K (callers with their own workspace layout).
static trinv_status_t run_tri(char uplo, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                              int unit, double* W, int32_t* info, int64_t info_off, cudaStream_t s,
                              int64_t b_stop = 0, void* aux = nullptr) {
  if (n <= BLK_MAX && b_stop == 0) {  // one block of order n (BASELINE config 0): a single launch
    LeafArgs l1{};
    l1.A = A; l1.lda = lda; l1.sA = n * lda; l1.X = X; l1.ldx = ldx; l1.sX = n * ldx;
    l1.batch = 1; l1.n = (int)n; l1.n_last = (int)n; l1.unit = unit;
    l1.info = info; l1.info_mode = info ? 2 : 0; l1.info_stride = 0; l1.info_off = info_off;
    return cuda_fail(launch_leaf(uplo, l1, s, &g_launches));
  }
  // (a1, a2) diagonal blocks: 128-wide blocks inverted whole in one CTA each (blk.cu:
  // leaves + the levels b = 32, 64 in shared memory), the last one ragged; or, when
  // the caller stops the recursion below 128 (beta = 4 top level), 32-wide leaves.
  const int64_t bw = (b_stop == 0 || b_stop >= BLK_MAX) ? BLK_MAX : 32;
  const int64_t full = n / bw, tail = n % bw;
  LeafArgs la{};
  la.A = A; la.lda = lda; la.sA = bw * lda + bw;
  la.X = X; la.ldx = ldx; la.sX = bw * ldx + bw;
  la.unit = unit; la.info = info; la.info_mode = info ? 2 : 0; la.info_stride = bw; la.info_off = info_off;
  if (bw == BLK_MAX) {
    la.batch = full + (tail > 0); la.n = (int)bw; la.n_last = (int)(tail > 0 ? tail : bw);
    TRY(launch_blk(uplo, la, s, &g_launches));
  } else {
    if (full > 0) {
      la.batch = full; la.n = 32; la.n_last = 32;
      TRY(launch_leaf(uplo, la, s, &g_launches));
    }
    if (tail > 0) {
      LeafArgs lt = la;
      lt.A = A + full * 32 * (lda + 1); lt.X = X + full * 32 * (ldx + 1);
      lt.batch = 1; lt.n = (int)tail; lt.n_last = (int)tail;
      lt.info_off = info_off + full * 32;
      TRY(launch_leaf(uplo, lt, s, &g_launches));
    }
  }
  // (a4-a7) levels: two grouped DMMA launches per level, or one fused launch (both products,
  // the second's tiles gated per W tile: launch_level_fused) when the call has the sync scratch.
  const int64_t b_end = b_stop > 0 ? b_stop : n;
  int fused_epoch = 0;
  bool sk_zeroed = false;
  int64_t b_first = bw;
  // the lowest levels that run 32x32 tiles: one persistent dependency-driven launch (gemm.cu)
  if (aux && bw == BLK_MAX && b_stop == 0 && level_chain_enabled() && product_engine() == 0 && !level_sk_enabled() &&
      !level_split_fixup()) {
    static const bool opt_out = [] {  // the other opt-in level experiments keep their launches
      const char* a = std::getenv("TRINV_SPLITK");
      const char* f = std::getenv("TRINV_FUSED");
      return (a && atoi(a) != 0) || (f && f[0] == '1');
    }();
    LevelArgs ph[8];
    int np = 0;
    int64_t bmax = 0, b = bw;
    for (; b < n && np + 2 <= 8; b *= 2) {
      const int64_t merges = merges_at(n, b);
      LevelArgs t{};
      t.mode = uplo == 'L' ? MODE_LOWER_1 : MODE_UPPER_1; t.n = n; t.b = b; t.merges = merges;
      if (opt_out || !level_uses_t32(t) || (strassen_top(n, b)) ||
          (size_t)n * (size_t)b * sizeof(double) > w_bytes(n))
        break;
      bmax = b;
      np += 2;
    }
    if (np >= 4) {  // at least two levels (one level gains nothing over two launches)
      const int64_t ldw = bmax;
      np = 0;
      for (int64_t bb = bw; bb <= bmax; bb *= 2) {
        const int64_t merges = merges_at(n, bb);
        const MatRef in{A, n, n, lda}, xr{X, n, n, ldx}, wr{W, n, bmax, ldw};
        LevelArgs& l1 = ph[np++];
        LevelArgs& l2 = ph[np++];
        l1 = LevelArgs{}; l2 = LevelArgs{};
        l1.n = l2.n = n; l1.b = l2.b = bb; l1.merges = l2.merges = merges;
        l1.out = W; l1.ldo = ldw; l1.out_rows = n; l1.out_cols = bb; l1.alpha = 1.0;
        l2.out = X; l2.ldo = ldx; l2.out_rows = n; l2.out_cols = n; l2.alpha = -1.0;
        l2.mir = X; l2.ldm = ldx;
        if (uplo == 'L') {
          l1.mode = MODE_LOWER_1; l1.opA = in; l1.opB = xr;
          l2.mode = MODE_LOWER_2; l2.opA = xr; l2.opB = wr;
        } else {
          l1.mode = MODE_UPPER_1; l1.opA = xr; l1.opB = in;
          l2.mode = MODE_UPPER_2; l2.opA = wr; l2.opB = xr;
        }
      }
      int* counters = reinterpret_cast<int*>(static_cast<char*>(aux) + strassen_scratch(n));
      TRY(launch_level_chain(ph, np, counters, (int)merges_at(n, bw), s, &g_launches));
      b_first = 2 * bmax;
    }
  }
  for (int64_t b = b_first; b < b_end && b < n; b *= 2) {
    const int64_t merges = merges_at(n, b);
    const MatRef in{A, n, n, lda}, xr{X, n, n, ldx}, wr{W, merges * b, b, b};
    LevelArgs l1{}, l2{};
    l1.n = l2.n = n; l1.b = l2.b = b; l1.merges = l2.merges = merges;
    l1.out = W; l1.ldo = b; l1.out_rows = merges * b; l1.out_cols = b; l1.alpha = 1.0;
    l2.out = X; l2.ldo = ldx; l2.out_rows = n; l2.out_cols = n; l2.alpha = -1.0;
    l2.mir = X; l2.ldm = ldx;
    if (uplo == 'L') {
      l1.mode = MODE_LOWER_1; l1.opA = in; l1.opB = xr;
      l2.mode = MODE_LOWER_2; l2.opA = xr; l2.opB = wr;
    } else {
      l1.mode = MODE_UPPER_1; l1.opA = xr; l1.opB = in;
      l2.mode = MODE_UPPER_2; l2.opA = wr; l2.opB = xr;
    }
    if (aux && b_stop == 0 && strassen_top(n, b)) {  // NEXT f3: the top merge with Strassen's dense quadrants
      TRY(strassen_merge(uplo, n, A, lda, X, ldx, W, aux, s));
      continue;
    }
    if (aux) {  // split-K tickets / semaphores (launch_level zeroes them when it splits)
      l1.sync = l2.sync = reinterpret_cast<int*>(static_cast<char*>(aux) + strassen_scratch(n));
      if (partial_bytes())
        l1.partial = l2.partial =
            reinterpret_cast<double*>(static_cast<char*>(aux) + strassen_scratch(n) + LEVEL_SYNC_BYTES);
      char* skp = static_cast<char*>(aux) + strassen_scratch(n) + LEVEL_SYNC_BYTES + partial_bytes();
      if (sk_bytes()) {
        l1.sk_flags = l2.sk_flags = reinterpret_cast<int*>(skp);
        l1.sk_partial = l2.sk_partial = reinterpret_cast<double*>(skp + align_up(SK_FLAG_INTS * sizeof(int)));
      }
      if (sk_bytes() && !sk_zeroed) {  // stream-K flags: zero once per call, every launch leaves them zero
        TRY(cudaMemsetAsync(skp, 0, SK_FLAG_INTS * sizeof(int), s));
        sk_zeroed = true;
      }
    }
    if (oz_level_ok(n, b) && !int8_veto()) {  // both products of every merge on the INT8 tensor cores
      void* ozws0 = reinterpret_cast<char*>(W) + align_up(w_bytes(n));
      const bool two = merges > 1;
      ForkCtx* fc = nullptr;
      if (two) {
        TRY(fork_ctx(&fc));
        TRY(fork_to(fc, s));
      }
      if (!two) {
        // one merge: the second product's inverse-block operand (B^-1 rows for the lower
        // case, C^-1 columns for the upper) is split on the second stream during the first
        // product; the second product then runs in the second scratch with that split done
        TRY(fork_ctx(&fc));
        const int64_t s0 = 0, r = std::min(b, n - b);
        double* Wg = W;
        const double* Ai = X;
        const double* Bi = X + b * ldx + b;
        void* ws2 = reinterpret_cast<char*>(ozws0) + oz_level_scratch(n, b);
        TRY(fork_to(fc, s));
        if (uplo == 'L')
          TRY(launch_oz2_prepare(r, b, r, Bi, ldx, TRI_LOWER, Wg, b, TRI_NONE, ws2, fc->aux, 1, &g_launches));
        else
          TRY(launch_oz2_prepare(b, r, r, Wg, b, TRI_NONE, Bi, ldx, TRI_UPPER, ws2, fc->aux, 2, &g_launches));
        if (uplo == 'L') {
          TRY(oz_product(r, b, b, A + b * lda, lda, TRI_NONE, Ai, ldx, TRI_LOWER, Wg, b, 1.0, ozws0, s));
          TRY(join_from(fc, s));
          TRY(launch_oz2_gemm(r, b, r, Bi, ldx, TRI_LOWER, Wg, b, TRI_NONE, X + b * ldx, ldx, -1.0, 0.0, ws2, s,
                              &g_launches, 0, 1));
          TRY(launch_zero_2d(X + b, ldx, b, r, s, &g_launches));
        } else {
          TRY(oz_product(b, r, b, Ai, ldx, TRI_UPPER, A + b, lda, TRI_NONE, Wg, b, 1.0, ozws0, s));
          TRY(join_from(fc, s));
          TRY(launch_oz2_gemm(b, r, r, Wg, b, TRI_NONE, Bi, ldx, TRI_UPPER, X + b, ldx, -1.0, 0.0, ws2, s,
                              &g_launches, 0, 2));
          TRY(launch_zero_2d(X + b * ldx, ldx, r, b, s, &g_launches));
        }
        (void)s0;
        continue;
      }
      const cudaStream_t s_main = s;
      for (int64_t g = 0; g < merges; ++g) {
        const bool odd = two && (g & 1);
        const cudaStream_t s = odd ? fc->aux : s_main;  // merges alternate between the two streams
        void* ozws = reinterpret_cast<char*>(ozws0) + (odd ? oz_level_scratch(n, b) : 0);
        const int64_t s0 = 2 * g * b, r = std::min(b, n - s0 - b);
        double* Wg = W + g * b * b;
        const double* Ai = X + s0 * ldx + s0;                // A^{-1}
        const double* Bi = X + (s0 + b) * ldx + (s0 + b);    // B^{-1} (lower) / C^{-1} (upper)
        if (uplo == 'L') {  // W = C A^{-1}; X21 = -B^{-1} W; X12 := 0
          TRY(oz_product(r, b, b, A + (s0 + b) * lda + s0, lda, TRI_NONE, Ai, ldx, TRI_LOWER, Wg, b, 1.0, ozws, s));
          TRY(oz_product(r, b, r, Bi, ldx, TRI_LOWER, Wg, b, TRI_NONE, X + (s0 + b) * ldx + s0, ldx, -1.0, ozws, s));
          TRY(launch_zero_2d(X + s0 * ldx + s0 + b, ldx, b, r, s, &g_launches));
        } else {            // W = A^{-1} B; X12 = -W C^{-1}; X21 := 0
          TRY(oz_product(b, r, b, Ai, ldx, TRI_UPPER, A + s0 * lda + s0 + b, lda, TRI_NONE, Wg, b, 1.0, ozws, s));
          TRY(oz_product(b, r, r, Wg, b, TRI_NONE, Bi, ldx, TRI_UPPER, X + s0 * ldx + s0 + b, ldx, -1.0, ozws, s));
          TRY(launch_zero_2d(X + (s0 + b) * ldx + s0, ldx, r, b, s, &g_launches));
        }
      }
      if (two) TRY(join_from(fc, s_main));
      continue;
    }
    if (l1.sync && level_fusable(l1) && fused_epoch < LEVEL_TICKETS - 1 && !(product_engine() != 0)) {
      if (fused_epoch == 0) TRY(cudaMemsetAsync(l1.sync, 0, LEVEL_SYNC_BYTES, s));  // once per call
      TRY(launch_level_fused(l1, l2, ++fused_epoch, s, &g_launches));
      continue;
    }
    TRY(launch_level(l1, s, &g_launches));
    TRY(launch_level(l2, s, &g_launches));
  }
  return TRINV_OK;
}

static trinv_status_t check_tri_args(int64_t n, const double* A, int64_t lda, const double* X, int64_t ldx,
                                     int diag) {
  if (n < 0 || (diag != TRINV_UNIT && diag != TRINV_NON_UNIT)) return TRINV_INVALID_ARG;
  if (n == 0) return TRINV_OK;
  if (!A || !X || lda < n || ldx < n) return TRINV_INVALID_ARG;
  if (overlap(A, lda, X, ldx, n)) return TRINV_ALIASING;
  return TRINV_OK;
}

// Public triangular entry (shared by lower/upper): validation, staging of
// unsupported layouts through the workspace, info initialisation.
static trinv_status_t tri_entry(char uplo, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                                int diag, void* ws, size_t ws_bytes, int32_t* info, int64_t info_off,
                                bool init_info, cudaStream_t s) {
  trinv_status_t st = check_tri_args(n, A, lda, X, ldx, diag);
  if (st != TRINV_OK || n == 0) return st;
  const size_t need = tri_ws(n, A, lda, X, ldx);
  if (ws_bytes < need || (need > 0 && ws == nullptr)) return TRINV_WORKSPACE_TOO_SMALL;
  // public entries check the input's scaling for the INT8 engines; internal calls inherit
  Int8Scope scope(init_info);
  if (init_info && int8_would_run(n)) int8_check_begin(A, lda, n, uplo, diag, s);
  if (init_info && info) TRY(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (n <= BLK_MAX) return run_tri(uplo, n, A, lda, X, ldx, diag, nullptr, info, info_off, s);

  char* p = static_cast<char*>(ws);
  double* W = reinterpret_cast<double*>(p);
  void* aux = p + align_up(w_bytes(n)) + oz_scratch(n);                               // run_tri's aux scratch
  p += align_up(w_bytes(n)) + oz_scratch(n) + strassen_scratch(n) + LEVEL_SYNC_BYTES + partial_bytes() +
       sk_bytes();  // then staging
  const double* Ause = A;
  int64_t lda_use = lda;
  if (!tma_ok(A, lda)) {  // stage the input into an even-ld, aligned copy
    double* As = reinterpret_cast<double*>(p);
    p += align_up(mat_bytes(n));
    lda_use = even_up(n);
    TRY(launch_copy_2d(A, lda, As, lda_use, n, n, s, &g_launches));
    Ause = As;
  }
  double* Xuse = X;
  int64_t ldx_use = ldx;
  const bool stage_x = !tma_ok(X, ldx);
  if (stage_x) {
    Xuse = reinterpret_cast<double*>(p);
    ldx_use = even_up(n);
  }
  st = run_tri(uplo, n, Ause, lda_use, Xuse, ldx_use, diag, W, info, info_off, s, 0, aux);
  if (st != TRINV_OK) return st;
  if (stage_x) TRY(launch_copy_2d(Xuse, ldx_use, X, ldx, n, n, s, &g_launches));
  return TRINV_OK;
}


// U^-1 L^-1 = S K by quadrants (h = n/2): S = [S11 S12; 0 S22], K = [K11 0; K21 K22]:
//   X11 = S11 K11 + S12 K21,  X12 = S12 K22,  X21 = S22 K21,  X22 = S22 K22
// (S11 K11 and S22 K22 are upper x lower products of order h, P_UL; S12 K21 dense, by
// strassen_acc; S12 K22 / S22 K21 dense x triangular).  NEXT f3.
static size_t ul_strassen_scratch(int64_t n) {
  return strassen_ul(n) ? align_up(strassen_ws_bytes(n / 2, strassen_levels(), strassen_min_q())) : 0;
}
// The diagonal quadrants S11 K11 / S22 K22 are upper x lower products again: the same
// decomposition recursively while its dense quadrant is of Strassen size, else one MODE_UL
// launch; S12 K22 / S22 K21 by trmm_sq.
static trinv_status_t ul_strassen(int64_t n, const double* S, const double* K, int64_t ld, double* X, int64_t ldx,
                                  void* sws, cudaStream_t s) {
  const int64_t h = n / 2;
  auto ul = [&](const double* Sq, const double* Kq, double* Xq) -> trinv_status_t {
    if (strassen_ul(h)) return ul_strassen(h, Sq, Kq, ld, Xq, ldx, sws, s);
    LevelArgs u{};
    u.mode = MODE_UL; u.n = h; u.b = h; u.merges = 1;
    u.opA = MatRef{Sq, h, h, ld}; u.opB = MatRef{Kq, h, h, ld};
    u.out = Xq; u.ldo = ldx; u.out_rows = h; u.out_cols = h; u.alpha = 1.0;
    return cuda_fail(launch_level(u, s, &g_launches));
  };
  trinv_status_t st = ul(S, K, X);                                                            // S11 K11
  if (st != TRINV_OK) return st;
  TRY(strassen_acc(h, 1.0, S + h, ld, K + h * ld, ld, 1.0, X, ldx, strassen_levels(), strassen_min_q(), sws, s,
                   &g_launches));                                                             // + S12 K21
  TRY(trmm_sq(h, 1.0, S + h, ld, TRI_NONE, K + h * ld + h, ld, TRI_LOWER, 0.0, X + h, ldx, sws, s));      // S12 K22
  TRY(trmm_sq(h, 1.0, S + h * ld + h, ld, TRI_UPPER, K + h * ld, ld, TRI_NONE, 0.0, X + h * ldx, ldx, sws,
              s));                                                                            // S22 K21
  return ul(S + h * ld + h, K + h * ld + h, X + h * ldx + h);                                 // S22 K22
}

// ---- NEXT row f4: COMBRIT with beta = 4 at the top level ------------------------------
// Alg. 1 with beta = 4 on n = 4m (m = 32 * 2^k): the four diagonal
// blocks are inverted by the beta = 2 levels b < m ("Recall COMBRIT ...
// or any preferred method"), then, for the upper case (the lower one is
// its transpose image):
//   B'_ij = -iD_ii A_ij                      (negated; 3 launches)
//   iB = block Thm 1 inverse of [I B; 0 I]:  iB_i,i+1 = B'_i,i+1,
//        iB_02 = B'_02 + B'_01 B'_12,  iB_03 = B'_03 + [B'_01 iB_02][B'_13; B'_23],
//        iB_13 = B'_13 + B'_12 B'_23     (the recurrence of the proof of Thm 1, P:243,
//                                          = the path sums of Eq. 6 in block form)
//   iA_ij = iB_ij iD_jj                      (3 launches), iA_ii = iD_ii.
static bool beta4_ok(int64_t n) {
  if (n % 4) return false;
  const int64_t m = n / 4;
  if (m < 32) return false;
  for (int64_t b = 32; b <= m; b *= 2)
    if (b == m) return true;
  return false;
}
static size_t beta4_ws(int64_t n) {
  const int64_t m = n / 4;
  size_t wl = 0;
  for (int64_t b = 32; b < m; b *= 2) wl = std::max(wl, (size_t)(merges_at(n, b) * b * b) * sizeof(double));
  return align_up(wl) + align_up((size_t)9 * m * m * sizeof(double));
}

static trinv_status_t run_tri_beta4(char uplo, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                                    int unit, char* ws, int32_t* info, cudaStream_t s) {
  const int64_t m = n / 4;
  size_t wl = 0;
  for (int64_t b = 32; b < m; b *= 2) wl = std::max(wl, (size_t)(merges_at(n, b) * b * b) * sizeof(double));
  double* W = reinterpret_cast<double*>(ws);
  double* WB = reinterpret_cast<double*>(ws + align_up(wl));  // 3m x 3m, ld 3m
  const int64_t ldb = 3 * m;
  trinv_status_t st = run_tri(uplo, n, A, lda, X, ldx, unit, W, info, 0, s, m);  // diagonal blocks iD_ii
  if (st != TRINV_OK) return st;
  auto Ab = [&](int64_t i, int64_t j) { return A + i * m * lda + j * m; };
  auto Xb = [&](int64_t i, int64_t j) { return X + i * m * ldx + j * m; };
  auto gemm = [&](int64_t M, int64_t N, int64_t K, const double* pa, int64_t la, int triA, const double* pb,
                  int64_t lb, int triB, double* pc, int64_t lc, double alpha, double beta) {
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K; g.batch = 1;
    g.A = pa; g.lda = la; g.B = pb; g.ldb = lb; g.C = pc; g.ldc = lc;
    g.alpha = alpha; g.beta = beta; g.triA = triA; g.triB = triB;
    return cuda_fail(launch_gemm(g, s, &g_launches));
  };
  if (uplo == 'U') {
    // WB block (i, j) (i < j) at rows i*m, cols (j-1)*m
    auto Wb = [&](int64_t i, int64_t j) { return WB + i * m * ldb + (j - 1) * m; };
    for (int64_t i = 0; i < 3 && st == TRINV_OK; ++i)  // B'_i,(i+1..3) = -iD_ii A_i,(i+1..3)
      st = gemm(m, (3 - i) * m, m, Xb(i, i), ldx, TRI_UPPER, Ab(i, i + 1), lda, TRI_NONE, Wb(i, i + 1), ldb, -1.0, 0.0);
    if (st == TRINV_OK)  // iB_02 = B'_02 + B'_01 B'_12
      st = gemm(m, m, m, Wb(0, 1), ldb, TRI_NONE, Wb(1, 2), ldb, TRI_NONE, Wb(0, 2), ldb, 1.0, 1.0);
    if (st == TRINV_OK)  // iB_03 = B'_03 + [B'_01 iB_02] [B'_13; B'_23]
      st = gemm(m, m, 2 * m, Wb(0, 1), ldb, TRI_NONE, Wb(1, 3), ldb, TRI_NONE, Wb(0, 3), ldb, 1.0, 1.0);
    if (st == TRINV_OK)  // iB_13 = B'_13 + B'_12 B'_23
      st = gemm(m, m, m, Wb(1, 2), ldb, TRI_NONE, Wb(2, 3), ldb, TRI_NONE, Wb(1, 3), ldb, 1.0, 1.0);
    for (int64_t j = 1; j < 4 && st == TRINV_OK; ++j)  // iA_(0..j-1),j = iB_(0..j-1),j iD_jj
      st = gemm(j * m, m, m, Wb(0, j), ldb, TRI_NONE, Xb(j, j), ldx, TRI_UPPER, Xb(0, j), ldx, 1.0, 0.0);
    for (int64_t i = 1; i < 4 && st == TRINV_OK; ++i)  // strictly lower block triangle := 0
      st = cuda_fail(launch_zero_2d(Xb(i, 0), ldx, m, i * m, s, &g_launches));
  } else {
    // WB block (i, j) (i > j) at rows (i-1)*m, cols j*m
    auto Wb = [&](int64_t i, int64_t j) { return WB + (i - 1) * m * ldb + j * m; };
    for (int64_t j = 0; j < 3 && st == TRINV_OK; ++j)  // B'_(j+1..3),j = -A_(j+1..3),j iD_jj
      st = gemm((3 - j) * m, m, m, Ab(j + 1, j), lda, TRI_NONE, Xb(j, j), ldx, TRI_LOWER, Wb(j + 1, j), ldb, -1.0, 0.0);
    if (st == TRINV_OK)  // iB_20 = B'_20 + B'_21 B'_10
      st = gemm(m, m, m, Wb(2, 1), ldb, TRI_NONE, Wb(1, 0), ldb, TRI_NONE, Wb(2, 0), ldb, 1.0, 1.0);
    if (st == TRINV_OK)  // iB_30 = B'_30 + [B'_31 B'_32] [B'_10; iB_20]
      st = gemm(m, m, 2 * m, Wb(3, 1), ldb, TRI_NONE, Wb(1, 0), ldb, TRI_NONE, Wb(3, 0), ldb, 1.0, 1.0);
    if (st == TRINV_OK)  // iB_31 = B'_31 + B'_32 B'_21
      st = gemm(m, m, m, Wb(3, 2), ldb, TRI_NONE, Wb(2, 1), ldb, TRI_NONE, Wb(3, 1), ldb, 1.0, 1.0);
    for (int64_t i = 1; i < 4 && st == TRINV_OK; ++i)  // iA_i,(0..i-1) = iD_ii iB_i,(0..i-1)
      st = gemm(m, i * m, m, Xb(i, i), ldx, TRI_LOWER, Wb(i, 0), ldb, TRI_NONE, Xb(i, 0), ldx, 1.0, 0.0);
    for (int64_t i = 0; i < 3 && st == TRINV_OK; ++i)  // strictly upper block triangle := 0
      st = cuda_fail(launch_zero_2d(Xb(i, i + 1), ldx, m, (3 - i) * m, s, &g_launches));
  }
  return st;
}

// ---- blocked Crout LU (NEXT row f2) -----------------------------------------------
// Split point of the factor recursion: a multiple of 64 near n/2.
static int64_t lu_split(int64_t n) { return 64 * ((n + 127) / 128); }

// Scratch of lu_rec at order n: L11^{-1}, U11^{-1} (h x even(h)), their triangular
// workspace, and one off-diagonal product buffer (h x even(n-h) or (n-h) x even(h)).
static size_t lu_scratch(int64_t n) {
  if (n <= LU_MAX) return 0;
  const int64_t h = lu_split(n), r = n - h;
  size_t b = 2 * align_up(mat_bytes(h)) + align_up(tri_ws(h, nullptr, even_up(h), nullptr, even_up(h)));
  b += align_up((size_t)std::max(h * even_up(r), r * even_up(h)) * sizeof(double));
  return std::max(b, lu_scratch(r));
}

// Factors the working matrix W (destroyed: it carries the Schur complements) into the
// packed factors F (lower triangle with diagonal = L, strict upper = U).  F may be W
// itself (lu_crout, in place): the off-diagonal blocks then go through the scratch T
// and a copy; with F != W (inv_general) the products are written straight into F.
static trinv_status_t lu_rec(int64_t n, double* W, int64_t ldw, double* F, int64_t ldf, char* ws, int32_t* info,
                             int64_t info_off, cudaStream_t s) {
  if (n <= LU_MAX) return cuda_fail(launch_lu_leaf(W, ldw, F, ldf, (int)n, info, info_off, s, &g_launches));
  const int64_t h = lu_split(n), r = n - h, ldh = even_up(h);
  const bool inplace = (F == W);
  double *W12 = W + h, *W21 = W + h * ldw, *W22 = W21 + h;
  double *F12 = F + h, *F21 = F + h * ldf, *F22 = F21 + h;
  trinv_status_t st = lu_rec(h, W, ldw, F, ldf, ws, info, info_off, s);  // A11 = L11 U11
  if (st != TRINV_OK) return st;
  char* p = ws;
  double* Li = reinterpret_cast<double*>(p); p += align_up(mat_bytes(h));
  double* Ui = reinterpret_cast<double*>(p); p += align_up(mat_bytes(h));
  double* tws = reinterpret_cast<double*>(p); p += align_up(tri_ws(h, nullptr, ldh, nullptr, ldh));
  double* T = reinterpret_cast<double*>(p);
  // L11^{-1} (lower, diagonal kept) and U11^{-1} (unit upper) by the recursive split
  st = run_tri('L', h, F, ldf, Li, ldh, 0, tws, nullptr, 0, s);
  if (st != TRINV_OK) return st;
  st = run_tri('U', h, F, ldf, Ui, ldh, 1, tws, nullptr, 0, s);
  if (st != TRINV_OK) return st;
  // U12 = L11^{-1} A12  (h x r; L11^{-1} lower: K-range k <= row)
  const int64_t ldr = even_up(r);
  GemmArgs g{};
  g.M = h; g.N = r; g.K = h; g.batch = 1;
  g.A = Li; g.lda = ldh; g.B = W12; g.ldb = ldw;
  g.C = inplace ? T : F12; g.ldc = inplace ? ldr : ldf;
  g.alpha = 1.0; g.beta = 0.0; g.triA = TRI_LOWER; g.triB = TRI_NONE;
  TRY(launch_gemm(g, s, &g_launches));
  if (inplace) TRY(launch_copy_2d(T, ldr, F12, ldf, h, r, s, &g_launches));
  // L21 = A21 U11^{-1}  (r x h; U11^{-1} upper: K-range k <= column)
  GemmArgs g2{};
  g2.M = r; g2.N = h; g2.K = h; g2.batch = 1;
  g2.A = W21; g2.lda = ldw; g2.B = Ui; g2.ldb = ldh;
  g2.C = inplace ? T : F21; g2.ldc = inplace ? ldh : ldf;
  g2.alpha = 1.0; g2.beta = 0.0; g2.triA = TRI_NONE; g2.triB = TRI_UPPER;
  TRY(launch_gemm(g2, s, &g_launches));
  if (inplace) TRY(launch_copy_2d(T, ldh, F21, ldf, r, h, s, &g_launches));
  // Schur complement W22 <- A22 - L21 U12
  GemmArgs g3{};
  g3.M = r; g3.N = r; g3.K = h; g3.batch = 1;
  g3.A = F21; g3.lda = ldf; g3.B = F12; g3.ldb = ldf; g3.C = W22; g3.ldc = ldw;
  g3.alpha = -1.0; g3.beta = 1.0; g3.triA = TRI_NONE; g3.triB = TRI_NONE;
  TRY(launch_gemm(g3, s, &g_launches));
  return lu_rec(r, W22, ldw, F22, ldf, ws, info, info_off + h, s);
}
// SKUL-style blocked recursion (the inverse factors computed alongside the factors, as
// SKUL does element-wise, "S K = A^{-1}"): W (working copy, destroyed) is
// factored into the packed F, and K = L^{-1} (Li, lower, diagonal kept) and S = U^{-1}
// (Ui, unit upper) are assembled from the children's inverse factors by the merge of
// the recursive split (COMBRIT beta = 2):
//   K = [K11 0; -K22 (L21 K11)  K22],   S = [S11  -(S11 U12) S22; 0 S22].
// The diagonal-block inverses computed for the factorisation are thus reused, and no
// separate triangular inversion of the full factors is needed.  All matrices share
// the even leading dimension ld; T is the (h x r | r x h) product scratch.
// Two product scratches (the K21 and S12 chains run concurrently), each of the largest
// (h x r | r x h) shape of the recursion.
static size_t lu_inv_half_scratch(int64_t n) {
  if (n <= LU_MAX) return 0;
  const int64_t h = lu_split(n), r = n - h;
  return align_up((size_t)std::max(h * even_up(r), r * even_up(h)) * sizeof(double));
}
static size_t lu_inv_scratch(int64_t n) { return 2 * lu_inv_half_scratch(n); }

// INT8 CRT scratch for the products of lu_inv_rec that run on the modular engine (all of
// them with min(M, N, K) >= the engine's block threshold): the largest over the recursion.
static bool lu_gemm_on_int8(int64_t M, int64_t N, int64_t K) {
  return product_engine() == 2 && std::min(M, std::min(N, K)) >= g_oz_min.load() && oz2_supported(M, N, K);
}
static size_t lu_oz_ws(int64_t n) {
  if (n <= LU_MAX || product_engine() != 2) return 0;
  const int64_t h = lu_split(n), r = n - h;
  size_t best = std::max(lu_oz_ws(h), lu_oz_ws(r));
  const int64_t shapes[5][3] = {{h, r, h}, {r, h, h}, {r, r, h}, {r, h, r}, {h, r, r}};
  for (const auto& m : shapes)
    if (lu_gemm_on_int8(m[0], m[1], m[2])) best = std::max(best, align_up(oz2_workspace_bytes(m[0], m[1], m[2])));
  return best;
}
// ozws: two CRT scratches of ozhalf bytes each, one per stream (nullptr: DMMA only)
// sws: NULL or the Strassen scratch of the top Schur update (lu_strassen_scratch): dense square
// Schur updates of order >= the Strassen threshold run strassen_acc (NEXT f3).
static trinv_status_t lu_inv_rec(int64_t n, double* W, double* F, double* Li, double* Ui, int64_t ld, double* T,
                                 int32_t* info, int64_t info_off, cudaStream_t s, void* ozws, size_t ozhalf,
                                 void* sws = nullptr) {
  ForkCtx* fc = nullptr;
  TRY(fork_ctx(&fc));
  if (n <= LU_MAX) {
    TRY(launch_lu_leaf(W, ld, F, ld, (int)n, info, info_off, s, &g_launches));
    static const bool fork_leaf = [] { const char* e = std::getenv("TRINV_LU_FORK"); return !(e && e[0] == '0'); }();
    if (fork_leaf) TRY(fork_to(fc, s));  // K = L^{-1} here, S = U^{-1} on the second stream
    trinv_status_t st = run_tri('L', n, F, ld, Li, ld, 0, nullptr, nullptr, 0, s);
    if (st != TRINV_OK) return st;
    st = run_tri('U', n, F, ld, Ui, ld, 1, nullptr, nullptr, 0, fork_leaf ? fc->aux : s);
    if (st != TRINV_OK) return st;
    if (fork_leaf) TRY(join_from(fc, s));
    return TRINV_OK;
  }
  const int64_t h = lu_split(n), r = n - h;
  double* T2 = T + lu_inv_half_scratch(n) / sizeof(double);
  auto blk = [&](double* M, int64_t i, int64_t j) { return M + i * ld + j; };
  auto gemm = [&](int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                  int64_t ldb, int triB, double* C, int64_t ldc, double alpha, double beta, cudaStream_t st) {
    if (ozws && lu_gemm_on_int8(M, N, K) && !int8_veto()) {  // one CRT scratch per stream
      void* w = st == fc->aux ? static_cast<void*>(static_cast<char*>(ozws) + ozhalf) : ozws;
      return cuda_fail(launch_oz2_gemm(M, N, K, A, lda, triA, B, ldb, triB, C, ldc, alpha, beta, w, st,
                                       &g_launches));
    }
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K; g.batch = 1;
    g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
    g.alpha = alpha; g.beta = beta; g.triA = triA; g.triB = triB;
    return cuda_fail(launch_gemm(g, st, &g_launches));
  };
  // the two products of a pair run concurrently (each stream has its own CRT scratch)
  static const bool fork_on = [] { const char* e = std::getenv("TRINV_LU_FORK"); return !(e && e[0] == '0'); }();
  // The six triangle-times-full products of a node with h = r >= 2 Strassen sizes (the top node of
  // n = 16384) by the P_TF quadrant recursion with Strassen in the dense quadrants (trmm_sq, Eq.
  // PTFmbk P:614-629), all on the caller's stream (Strassen never runs beside other work, §9b):
  // config 5 249.0 -> 247.8 ms, sampled error unchanged.  TRINV_LU_TRMM=0 keeps them on the
  // DMMA GEMM with the U12 / L21 and K21 / S12 pairs on two streams.
  static const bool lu_trmm = [] { const char* e = std::getenv("TRINV_LU_TRMM"); return !(e && e[0] == '0'); }();
  const bool tsq = lu_trmm && sws && r == h && !ozws && trmm_split_ok(h);
  const bool par = fork_on && !tsq;
  cudaStream_t s2 = par ? fc->aux : s;
  auto tprod = [&](int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                   int64_t ldb, int triB, double* C, int64_t ldc, double alpha, double beta, cudaStream_t st) {
    if (tsq) return cuda_fail(trmm_sq(h, alpha, A, lda, triA, B, ldb, triB, beta, C, ldc, sws, s));
    return gemm(M, N, K, A, lda, triA, B, ldb, triB, C, ldc, alpha, beta, st);
  };
  trinv_status_t st = lu_inv_rec(h, W, F, Li, Ui, ld, T, info, info_off, s, ozws, ozhalf, sws);  // A11 = L11 U11, K11, S11
  if (st != TRINV_OK) return st;
  // U12 = K11 A12 (K11 lower) || L21 = A21 S11 (S11 upper); Schur W22 <- A22 - L21 U12
  if (par) TRY(fork_to(fc, s));
  if ((st = tprod(h, r, h, Li, ld, TRI_LOWER, blk(W, 0, h), ld, TRI_NONE, blk(F, 0, h), ld, 1.0, 0.0, s))) return st;
  if ((st = tprod(r, h, h, blk(W, h, 0), ld, TRI_NONE, Ui, ld, TRI_UPPER, blk(F, h, 0), ld, 1.0, 0.0, s2))) return st;
  if (par) TRY(join_from(fc, s));
  if (sws && r == h && !(ozws && lu_gemm_on_int8(r, r, h)) && strassen_ul(2 * h)) {  // W22 -= L21 U12 by Strassen
    TRY(strassen_acc(h, -1.0, blk(F, h, 0), ld, blk(F, 0, h), ld, 1.0, blk(W, h, h), ld, strassen_levels(),
                     strassen_min_q(), sws, s, &g_launches));
  } else if ((st = gemm(r, r, h, blk(F, h, 0), ld, TRI_NONE, blk(F, 0, h), ld, TRI_NONE, blk(W, h, h), ld, -1.0, 1.0,
                        s))) {
    return st;
  }
  st = lu_inv_rec(r, blk(W, h, h), blk(F, h, h), blk(Li, h, h), blk(Ui, h, h), ld, T, info, info_off + h, s, ozws,
                  ozhalf, sws);
  if (st != TRINV_OK) return st;
  const int64_t lth = even_up(h), ltr = even_up(r);
  if (par) TRY(fork_to(fc, s));
  // K21 = -K22 (L21 K11)
  if ((st = tprod(r, h, h, blk(F, h, 0), ld, TRI_NONE, Li, ld, TRI_LOWER, T, lth, 1.0, 0.0, s))) return st;
  if ((st = tprod(r, h, r, blk(Li, h, h), ld, TRI_LOWER, T, lth, TRI_NONE, blk(Li, h, 0), ld, -1.0, 0.0, s))) return st;
  // S12 = -(S11 U12) S22 (second stream, second scratch)
  if ((st = tprod(h, r, h, Ui, ld, TRI_UPPER, blk(F, 0, h), ld, TRI_NONE, T2, ltr, 1.0, 0.0, s2))) return st;
  if ((st = tprod(h, r, r, T2, ltr, TRI_NONE, blk(Ui, h, h), ld, TRI_UPPER, blk(Ui, 0, h), ld, -1.0, 0.0, s2)))
    return st;
  // structural zeros of the opposite triangles (read densely by the diagonal tiles of S K)
  TRY(launch_zero_2d(blk(Li, 0, h), ld, h, r, s, &g_launches));
  TRY(launch_zero_2d(blk(Ui, h, 0), ld, r, h, s2, &g_launches));
  if (par) TRY(join_from(fc, s));
  return TRINV_OK;
}

static trinv_status_t inv_from_lu_core(int64_t n, const double* Lf, int64_t ldl, const double* Uf, int64_t ldu,
                                       double* X, int64_t ldx, trinv_diag_t diagL, trinv_diag_t diagU, void* ws,
                                       size_t ws_bytes, int32_t* d_info, bool init_info, cudaStream_t s) {
  if (n < 0) return TRINV_INVALID_ARG;
  if ((diagL != TRINV_UNIT && diagL != TRINV_NON_UNIT) || (diagU != TRINV_UNIT && diagU != TRINV_NON_UNIT))
    return TRINV_INVALID_ARG;
  if (n == 0) return TRINV_OK;
  if (!Lf || !Uf || !X || ldl < n || ldu < n || ldx < n) return TRINV_INVALID_ARG;
  if (overlap(Lf, ldl, X, ldx, n) || overlap(Uf, ldu, X, ldx, n)) return TRINV_ALIASING;
  const int64_t lde = even_up(n);
  const size_t tws_bytes = std::max(tri_ws(n, Lf, ldl, nullptr, lde), tri_ws(n, Uf, ldu, nullptr, lde));
  const bool stage_x = !tma_ok(X, ldx);
  const size_t need = 2 * align_up(mat_bytes(n)) + align_up(tws_bytes) + (stage_x ? align_up(mat_bytes(n)) : 0) +
                      (ul_on_int8(n) ? align_up(oz2_workspace_bytes(n, n, n)) : 0) + ul_strassen_scratch(n);
  if (ws_bytes < need || ws == nullptr) return TRINV_WORKSPACE_TOO_SMALL;
  Int8Scope scope(true);
  if (int8_would_run(n) || ul_on_int8(n)) {
    int8_check_begin(Lf, ldl, n, 'L', (int)diagL, s);
    int8_check_begin(Uf, ldu, n, 'U', (int)diagU, s);
  }
  char* p = static_cast<char*>(ws);
  double* Ui = reinterpret_cast<double*>(p); p += align_up(mat_bytes(n));
  double* Li = reinterpret_cast<double*>(p); p += align_up(mat_bytes(n));
  void* tws = p; p += align_up(tws_bytes);
  if (init_info && d_info) TRY(cudaMemsetAsync(d_info, 0, sizeof(int32_t), s));
  // zero diagonals: L reports 1+i, U reports n+1+i (header); the min is kept
  trinv_status_t st = tri_entry('L', n, Lf, ldl, Li, lde, (int)diagL, tws, tws_bytes, d_info, 0, false, s);
  if (st != TRINV_OK) return st;
  st = tri_entry('U', n, Uf, ldu, Ui, lde, (int)diagU, tws, tws_bytes, d_info, n, false, s);
  if (st != TRINV_OK) return st;
  double* Xuse = X;
  int64_t ldx_use = ldx;
  if (stage_x) { Xuse = reinterpret_cast<double*>(p); ldx_use = lde; p += align_up(mat_bytes(n)); }
  if (ul_on_int8(n) && !int8_veto()) {  // S K on the INT8 tensor cores (k >= max(i, j))
    TRY(launch_oz2_ul(n, Ui, lde, Li, lde, Xuse, ldx_use, p, s, &g_launches));
  } else if (strassen_ul(n)) {  // NEXT f3: S K by quadrants, S12 K21 by Strassen
    const trinv_status_t su = ul_strassen(n, Ui, Li, lde, Xuse, ldx_use, p, s);
    if (su != TRINV_OK) return su;
  } else {
    LevelArgs ul{};
    ul.mode = MODE_UL; ul.n = n; ul.b = n; ul.merges = 1;
    ul.opA = MatRef{Ui, n, n, lde}; ul.opB = MatRef{Li, n, n, lde};
    ul.out = Xuse; ul.ldo = ldx_use; ul.out_rows = n; ul.out_cols = n; ul.alpha = 1.0;
    TRY(launch_level(ul, s, &g_launches));
  }
  if (stage_x) TRY(launch_copy_2d(Xuse, ldx_use, X, ldx, n, n, s, &g_launches));
  return TRINV_OK;
}

}  // namespace trinv

using namespace trinv;

extern "C" {

size_t trinv_workspace_bytes(char op, int64_t n, const void* A, int64_t lda, const void* X, int64_t ldx) {
  if (n <= 0) return 0;
  if (op == 'L' || op == 'U') return tri_ws(n, A, lda, X, ldx);
  if (op == 'F') return align_up(lu_scratch(n));
  if (op == 'A') {  // inv_general: F, W, K, S (n x even(n) each), the product scratch, X staging, INT8 scratch
    size_t bytes = 4 * align_up(mat_bytes(n)) + align_up(lu_inv_scratch(n));
    if (!tma_ok(X, ldx)) bytes += align_up(mat_bytes(n));
    bytes += std::max(2 * lu_oz_ws(n), ul_on_int8(n) ? align_up(oz2_workspace_bytes(n, n, n)) : (size_t)0);
    bytes += ul_strassen_scratch(n);  // Strassen: the top Schur update and S K (h = n/2 both)
    (void)A; (void)lda;
    return bytes;
  }
  if (op == 'G') {
    // [U^{-1} | L^{-1} | triangular scratch (+ factor staging) | X staging]; the
    // U factor is assumed to be laid out like the L factor (A, lda).
    size_t bytes = 2 * align_up(mat_bytes(n)) + align_up(tri_ws(n, A, lda, nullptr, even_up(n)));
    if (!tma_ok(X, ldx)) bytes += align_up(mat_bytes(n));
    if (ul_on_int8(n)) bytes += align_up(oz2_workspace_bytes(n, n, n));
    return bytes + ul_strassen_scratch(n);
  }
  return 0;
}

trinv_status_t trinv_lower(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx, trinv_diag_t diag,
                           void* ws, size_t ws_bytes, int32_t* d_info, void* stream) {
  return tri_entry('L', n, A, lda, X, ldx, (int)diag, ws, ws_bytes, d_info, 0, true, (cudaStream_t)stream);
}

trinv_status_t trinv_upper(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx, trinv_diag_t diag,
                           void* ws, size_t ws_bytes, int32_t* d_info, void* stream) {
  return tri_entry('U', n, A, lda, X, ldx, (int)diag, ws, ws_bytes, d_info, 0, true, (cudaStream_t)stream);
}

trinv_status_t trinv_batched(char uplo, int64_t n, int64_t batch, const double* A, int64_t lda, int64_t strideA,
                             double* X, int64_t ldx, int64_t strideX, trinv_diag_t diag, int32_t* d_info,
                             void* stream) {
  if ((uplo != 'L' && uplo != 'U') || n < 0 || batch < 0) return TRINV_INVALID_ARG;
  if (diag != TRINV_UNIT && diag != TRINV_NON_UNIT) return TRINV_INVALID_ARG;
  if (n == 0 || batch == 0) return TRINV_OK;
  if (!A || !X || lda < n || ldx < n) return TRINV_INVALID_ARG;
  if (batch > 1 && (strideA < n * lda || strideX < n * ldx)) return TRINV_INVALID_ARG;
  if (n > BLK_MAX) return TRINV_NOT_SUPPORTED;
  LeafArgs la{};
  la.A = A; la.lda = lda; la.sA = batch > 1 ? strideA : n * lda;
  la.X = X; la.ldx = ldx; la.sX = batch > 1 ? strideX : n * ldx;
  la.batch = batch; la.n = (int)n; la.n_last = (int)n; la.unit = (int)diag;
  la.info = d_info; la.info_mode = d_info ? 1 : 0;
  return cuda_fail(launch_leaf(uplo, la, (cudaStream_t)stream, &g_launches));
}

static int64_t host_chunk(int64_t chunk) { return chunk > 0 ? chunk : 4096; }

size_t trinv_batched_host_workspace_bytes(int64_t n, int64_t chunk) {
  if (n <= 0) return 0;
  return (size_t)TRINV_HOST_SLOTS * align_up((size_t)host_chunk(chunk) * n * n * sizeof(double));
}

trinv_status_t trinv_batched_host(char uplo, int64_t n, int64_t batch, const double* A_host, double* X_host,
                                  trinv_diag_t diag, int64_t chunk, void* ws, size_t ws_bytes, int32_t* d_info,
                                  void* stream) {
  if ((uplo != 'L' && uplo != 'U') || n < 0 || batch < 0 || chunk < 0) return TRINV_INVALID_ARG;
  if (diag != TRINV_UNIT && diag != TRINV_NON_UNIT) return TRINV_INVALID_ARG;
  if (n == 0 || batch == 0) return TRINV_OK;
  if (!A_host || !X_host) return TRINV_INVALID_ARG;
  if (n > BLK_MAX) return TRINV_NOT_SUPPORTED;
  chunk = host_chunk(chunk);
  const size_t slot_bytes = align_up((size_t)chunk * n * n * sizeof(double));
  if (!ws || ws_bytes < trinv_batched_host_workspace_bytes(n, chunk)) return TRINV_WORKSPACE_TOO_SMALL;
  cudaStream_t s = (cudaStream_t)stream;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  TRY(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
  TRY(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
  const int64_t nchunks = (batch + chunk - 1) / chunk;
  cudaEvent_t start, loaded[TRINV_HOST_SLOTS], done[TRINV_HOST_SLOTS], freed[TRINV_HOST_SLOTS];
  TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  for (int i = 0; i < TRINV_HOST_SLOTS; ++i) {
    TRY(cudaEventCreateWithFlags(&loaded[i], cudaEventDisableTiming));
    TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    TRY(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
  }
  // the copies may start only after the work already enqueued on `stream`
  TRY(cudaEventRecord(start, s));
  TRY(cudaStreamWaitEvent(h2d, start, 0));
  trinv_status_t st = TRINV_OK;
  for (int64_t c = 0; c < nchunks && st == TRINV_OK; ++c) {
    const int slot = (int)(c % TRINV_HOST_SLOTS);
    double* buf = reinterpret_cast<double*>(static_cast<char*>(ws) + slot * slot_bytes);
    const int64_t b0 = c * chunk, cnt = std::min(chunk, batch - b0);
    const size_t bytes = (size_t)cnt * n * n * sizeof(double);
    if (c >= TRINV_HOST_SLOTS) TRY(cudaStreamWaitEvent(h2d, freed[slot], 0));
    TRY(cudaMemcpyAsync(buf, A_host + b0 * n * n, bytes, cudaMemcpyHostToDevice, h2d));
    TRY(cudaEventRecord(loaded[slot], h2d));
    TRY(cudaStreamWaitEvent(s, loaded[slot], 0));
    LeafArgs la{};
    la.A = buf; la.lda = n; la.sA = n * n; la.X = buf; la.ldx = n; la.sX = n * n;
    la.batch = cnt; la.n = (int)n; la.n_last = (int)n; la.unit = (int)diag;
    la.info = d_info ? d_info + b0 : nullptr; la.info_mode = d_info ? 1 : 0;
    st = cuda_fail(launch_leaf(uplo, la, s, &g_launches));
    if (st != TRINV_OK) break;
    TRY(cudaEventRecord(done[slot], s));
    TRY(cudaStreamWaitEvent(d2h, done[slot], 0));
    TRY(cudaMemcpyAsync(X_host + b0 * n * n, buf, bytes, cudaMemcpyDeviceToHost, d2h));
    TRY(cudaEventRecord(freed[slot], d2h));
  }
  // `stream` observes completion of every device->host copy
  TRY(cudaStreamWaitEvent(s, freed[(nchunks - 1) % TRINV_HOST_SLOTS], 0));
  cudaEventDestroy(start);
  for (int i = 0; i < TRINV_HOST_SLOTS; ++i) {
    cudaEventDestroy(loaded[i]); cudaEventDestroy(done[i]); cudaEventDestroy(freed[i]);
  }
  cudaStreamDestroy(h2d);
  cudaStreamDestroy(d2h);
  return st;
}

trinv_status_t inv_from_lu(int64_t n, const double* Lf, int64_t ldl, const double* Uf, int64_t ldu, double* X,
                           int64_t ldx, trinv_diag_t diagL, trinv_diag_t diagU, void* ws, size_t ws_bytes,
                           int32_t* d_info, void* stream) {
  return inv_from_lu_core(n, Lf, ldl, Uf, ldu, X, ldx, diagL, diagU, ws, ws_bytes, d_info, true,
                          (cudaStream_t)stream);
}

trinv_status_t trinv_tri_ex(char uplo, int beta, int64_t n, const double* A, int64_t lda, double* X, int64_t ldx,
                            trinv_diag_t diag, void* ws, size_t ws_bytes, int32_t* d_info, void* stream) {
  if (uplo != 'L' && uplo != 'U') return TRINV_INVALID_ARG;
  if (beta == 2) return tri_entry(uplo, n, A, lda, X, ldx, (int)diag, ws, ws_bytes, d_info, 0, true, (cudaStream_t)stream);
  if (beta != 4) return TRINV_INVALID_ARG;
  trinv_status_t st = check_tri_args(n, A, lda, X, ldx, (int)diag);
  if (st != TRINV_OK || n == 0) return st;
  if (!beta4_ok(n) || !tma_ok(A, lda) || !tma_ok(X, ldx)) return TRINV_NOT_SUPPORTED;
  if (ws_bytes < beta4_ws(n) || !ws) return TRINV_WORKSPACE_TOO_SMALL;
  cudaStream_t s = (cudaStream_t)stream;
  if (d_info) TRY(cudaMemsetAsync(d_info, 0, sizeof(int32_t), s));
  Int8Scope scope(true);
  if (int8_would_run(n)) int8_check_begin(A, lda, n, uplo, (int)diag, s);
  return run_tri_beta4(uplo, n, A, lda, X, ldx, (int)diag, static_cast<char*>(ws), d_info, s);
}

size_t trinv_tri_ex_workspace_bytes(int beta, int64_t n) {
  if (n <= 0) return 0;
  if (beta == 4 && beta4_ok(n)) return beta4_ws(n);
  return tri_ws(n, nullptr, even_up(n), nullptr, even_up(n));
}

size_t trinv_strassen_workspace_bytes(int64_t n) {
  if (n <= 0 || n % 4) return 0;
  return strassen_ws_bytes(n, 1, 16);  // 2 operand sums + 7 products of (n/2)^2
}

// NEXT row f3: one level of Strassen's 7-product recursion (cited by the paper for its block
// products) over the DMMA GEMM for a dense n x n product
// C = A B (n % 4 == 0): strassen_acc (strassen.cu), as inside the inversion.
trinv_status_t trinv_gemm_strassen(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                   int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) return TRINV_INVALID_ARG;
  if (n == 0) return TRINV_OK;
  if (!A || !B || !C || lda < n || ldb < n || ldc < n) return TRINV_INVALID_ARG;
  if (n % 4 || !tma_ok(A, lda) || !tma_ok(B, ldb) || !tma_ok(C, ldc)) return TRINV_NOT_SUPPORTED;
  const size_t need = trinv_strassen_workspace_bytes(n);
  if (ws_bytes < need || (need > 0 && !ws)) return TRINV_WORKSPACE_TOO_SMALL;
  return cuda_fail(strassen_acc(n, 1.0, A, lda, B, ldb, 0.0, C, ldc, 1, 16, ws, s, &g_launches));
}

trinv_status_t trinv_gemm(int64_t M, int64_t N, int64_t K, int64_t batch, double alpha, const double* A,
                          int64_t lda, int64_t strideA, char structA, const double* B, int64_t ldb, int64_t strideB,
                          char structB, double beta, double* C, int64_t ldc, int64_t strideC, void* stream) {
  if (M < 0 || N < 0 || K < 0 || batch < 0) return TRINV_INVALID_ARG;
  if (M == 0 || N == 0 || batch == 0) return TRINV_OK;
  if (K == 0) return TRINV_NOT_SUPPORTED;
  auto tri = [](char c) { return c == 'L' ? TRI_LOWER : (c == 'U' ? TRI_UPPER : (c == 'N' ? TRI_NONE : -1)); };
  const int ta = tri(structA), tb = tri(structB);
  if (ta < 0 || tb < 0 || (ta != TRI_NONE && tb != TRI_NONE)) return TRINV_INVALID_ARG;
  if (!C || (K > 0 && (!A || !B)) || ldc < N || (K > 0 && (lda < K || ldb < N))) return TRINV_INVALID_ARG;
  if (batch > 1 && (strideA < M * lda || strideB < K * ldb || strideC < M * ldc)) return TRINV_INVALID_ARG;
  // a single-row operand never uses its leading dimension: any even value is equivalent
  if (M == 1) lda = even_up(lda);
  if (K == 1) ldb = even_up(ldb);
  if (!tma_ok(A, lda) || !tma_ok(B, ldb) || (batch > 1 && (strideA % 2 || strideB % 2)))
    return TRINV_NOT_SUPPORTED;
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.lda = lda; g.sA = strideA; g.B = B; g.ldb = ldb; g.sB = strideB;
  g.C = C; g.ldc = ldc; g.sC = strideC; g.alpha = alpha; g.beta = beta; g.triA = ta; g.triB = tb;
  return cuda_fail(launch_gemm(g, (cudaStream_t)stream, &g_launches));
}

trinv_status_t lu_crout(int64_t n, double* A, int64_t lda, void* ws, size_t ws_bytes, int32_t* d_info,
                        void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) return TRINV_INVALID_ARG;
  if (n == 0) return TRINV_OK;
  if (!A || lda < n) return TRINV_INVALID_ARG;
  if (n > LU_MAX && !tma_ok(A, lda)) return TRINV_NOT_SUPPORTED;
  const size_t need = align_up(lu_scratch(n));
  if (ws_bytes < need || (need > 0 && !ws)) return TRINV_WORKSPACE_TOO_SMALL;
  if (d_info) TRY(cudaMemsetAsync(d_info, 0, sizeof(int32_t), s));
  return lu_rec(n, A, lda, A, lda, static_cast<char*>(ws), d_info, 0, s);
}

trinv_status_t inv_general(int64_t n, const double* A, int64_t lda, double* X, int64_t ldx, void* ws,
                           size_t ws_bytes, int32_t* d_info, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) return TRINV_INVALID_ARG;
  if (n == 0) return TRINV_OK;
  if (!A || !X || lda < n || ldx < n) return TRINV_INVALID_ARG;
  if (overlap(A, lda, X, ldx, n)) return TRINV_ALIASING;
  const size_t need = trinv_workspace_bytes('A', n, A, lda, X, ldx);
  if (ws_bytes < need || !ws) return TRINV_WORKSPACE_TOO_SMALL;
  Int8Scope scope(true);
  if (lu_oz_ws(n) > 0 || ul_on_int8(n)) int8_check_begin(A, lda, n, 'N', 0, s);
  const int64_t lde = even_up(n);
  // workspace: [F packed factors | W working copy of A | K = L^{-1} | S = U^{-1} | T | X staging]
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { double* q = reinterpret_cast<double*>(p); p += align_up(bytes); return q; };
  double* F = take(mat_bytes(n));
  double* Wk = take(mat_bytes(n));
  double* Li = take(mat_bytes(n));
  double* Ui = take(mat_bytes(n));
  double* T = take(lu_inv_scratch(n));
  const bool stage_x = !tma_ok(X, ldx);
  double* Xuse = stage_x ? take(mat_bytes(n)) : X;
  const int64_t ldx_use = stage_x ? lde : ldx;
  const size_t oz_bytes = std::max(2 * lu_oz_ws(n), ul_on_int8(n) ? align_up(oz2_workspace_bytes(n, n, n)) : (size_t)0);
  void* ozws = oz_bytes ? static_cast<void*>(take(oz_bytes)) : nullptr;
  if (d_info) TRY(cudaMemsetAsync(d_info, 0, sizeof(int32_t), s));
  TRY(launch_copy_2d(A, lda, Wk, lde, n, n, s, &g_launches));
  // A = L U (U unit, Crout) with K = L^{-1}, S = U^{-1} alongside (SKUL)
  void* sws = ul_strassen_scratch(n) ? static_cast<void*>(take(ul_strassen_scratch(n))) : nullptr;
  trinv_status_t st = lu_inv_rec(n, Wk, F, Li, Ui, lde, T, d_info, 0, s, lu_oz_ws(n) ? ozws : nullptr, lu_oz_ws(n),
                                 sws);
  if (st != TRINV_OK) return st;
  // A^{-1} = S K = U^{-1} L^{-1}: X_ij = sum_{k >= max(i,j)} S_ik K_kj (P_UL)
  if (ul_on_int8(n) && !int8_veto()) {
    TRY(launch_oz2_ul(n, Ui, lde, Li, lde, Xuse, ldx_use, ozws, s, &g_launches));
  } else if (sws) {  // NEXT f3: S K by quadrants, S12 K21 by Strassen
    st = ul_strassen(n, Ui, Li, lde, Xuse, ldx_use, sws, s);
    if (st != TRINV_OK) return st;
  } else {
    LevelArgs ul{};
    ul.mode = MODE_UL; ul.n = n; ul.b = n; ul.merges = 1;
    ul.opA = MatRef{Ui, n, n, lde}; ul.opB = MatRef{Li, n, n, lde};
    ul.out = Xuse; ul.ldo = ldx_use; ul.out_rows = n; ul.out_cols = n; ul.alpha = 1.0;
    TRY(launch_level(ul, s, &g_launches));
  }
  if (stage_x) TRY(launch_copy_2d(Xuse, ldx_use, X, ldx, n, n, s, &g_launches));
  return TRINV_OK;
}

size_t trinv_gemm_oz_workspace_bytes(int64_t M, int64_t N, int64_t K, int digits) {
  if (digits > 0) return 0;  // the digit-splitting variant was retired
  return oz2_supported(M, N, K) ? oz2_workspace_bytes(M, N, K) : 0;
}

trinv_status_t trinv_gemm_oz(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                             char structA, const double* B, int64_t ldb, char structB, double beta, double* C,
                             int64_t ldc, int digits, void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || N < 0 || K < 0) return TRINV_INVALID_ARG;
  if (digits > 0) return TRINV_NOT_SUPPORTED;  // the digit-splitting variant was retired
  if (M == 0 || N == 0) return TRINV_OK;
  auto tri = [](char c) { return c == 'L' ? TRI_LOWER : (c == 'U' ? TRI_UPPER : (c == 'N' ? TRI_NONE : -1)); };
  const int ta = tri(structA), tb = tri(structB);
  if (ta < 0 || tb < 0) return TRINV_INVALID_ARG;
  // two triangular operands: only upper x lower (k >= max(i, j))
  if (ta != TRI_NONE && tb != TRI_NONE && !(ta == TRI_UPPER && tb == TRI_LOWER)) return TRINV_INVALID_ARG;
  if (!A || !B || !C || lda < K || ldb < N || ldc < N) return TRINV_INVALID_ARG;
  if (!oz2_supported(M, N, K)) return TRINV_NOT_SUPPORTED;
  if (!ws || ws_bytes < oz2_workspace_bytes(M, N, K)) return TRINV_WORKSPACE_TOO_SMALL;
  return cuda_fail(launch_oz2_gemm(M, N, K, A, lda, ta, B, ldb, tb, C, ldc, alpha, beta, ws, (cudaStream_t)stream,
                                   &g_launches));
}

trinv_status_t trinv_set_product_engine(int engine, int digits, int64_t min_block) {
  (void)digits;
  if ((engine != 0 && engine != 2) || min_block < 256) return TRINV_INVALID_ARG;
  g_oz_min.store(min_block);
  g_engine.store(engine);
  return TRINV_OK;
}

int trinv_get_product_engine(void) { return product_engine(); }

trinv_status_t trinv_set_strassen(int levels, int64_t min_h) {
  if (levels < 0 || levels > 3 || min_h < 64) return TRINV_INVALID_ARG;
  g_strassen_min.store(min_h);
  g_strassen_levels.store(levels);
  return TRINV_OK;
}
int trinv_get_strassen(void) { return strassen_levels(); }

int trinv_int8_scaling_ok(int64_t n, const double* A, int64_t lda, char uplo, trinv_diag_t diag, void* stream) {
  if (n <= 0 || !A || lda < n || (uplo != 'L' && uplo != 'U' && uplo != 'N')) return -(int)TRINV_INVALID_ARG;
  if (diag != TRINV_UNIT && diag != TRINV_NON_UNIT) return -(int)TRINV_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  Int8Scope scope(true);
  int8_check_begin(A, lda, n, uplo, uplo == 'N' ? 0 : (int)diag, s);
  const bool veto = int8_veto();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_last_cuda_error = (int)e; return -(int)TRINV_CUDA_ERROR; }
  return veto ? 0 : 1;
}

const char* trinv_status_string(trinv_status_t st) {
  switch (st) {
    case TRINV_OK: return "TRINV_OK";
    case TRINV_INVALID_ARG: return "TRINV_INVALID_ARG: bad size, leading dimension, stride, flag or NULL pointer";
    case TRINV_ALIASING: return "TRINV_ALIASING: input and output overlap";
    case TRINV_WORKSPACE_TOO_SMALL: return "TRINV_WORKSPACE_TOO_SMALL: see trinv_workspace_bytes()";
    case TRINV_CUDA_ERROR: return "TRINV_CUDA_ERROR: a CUDA call failed; see trinv_last_cuda_error()";
    case TRINV_NOT_SUPPORTED: return "TRINV_NOT_SUPPORTED: outside the implemented envelope";
  }
  return "unknown trinv status";
}

int trinv_last_cuda_error(void) { return g_last_cuda_error; }
const char* trinv_version(void) { return "trinv-b200 0.1 sm_100a"; }
int64_t trinv_launch_count(void) { return g_launches; }
void trinv_reset_launch_count(void) { g_launches = 0; }

void trinv_profile_begin(void) {
  trinv_profile_end();
  g_prof_on = true;
}

void trinv_profile_end(void) {
  g_prof_on = false;
  if (!g_prof) return;
  for (auto& r : *g_prof) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_prof->clear();
}

int trinv_profile_read(int kind, double* ms, int64_t* launches, double* flops, double* bytes) {
  // device time = length of the union of this kind's [start, end] intervals (launches of
  // one kind may overlap on two streams), measured from the session's first event
  double t = 0, f = 0, b = 0;
  int64_t c = 0;
  if (g_prof && !g_prof->empty()) {
    const cudaEvent_t base = g_prof->front().e0;
    if (cudaEventSynchronize(base) != cudaSuccess) return (int)TRINV_CUDA_ERROR;
    std::vector<std::pair<double, double>> iv;
    for (auto& r : *g_prof) {
      if (r.kind != kind) continue;
      if (cudaEventSynchronize(r.e1) != cudaSuccess) return (int)TRINV_CUDA_ERROR;
      float a = 0.f, e = 0.f;
      cudaEventElapsedTime(&a, base, r.e0);
      cudaEventElapsedTime(&e, base, r.e1);
      iv.emplace_back((double)a, (double)e);
      f += r.flops; b += r.bytes; ++c;
    }
    std::sort(iv.begin(), iv.end());
    double lo = 0, hi = -1;
    for (const auto& x : iv) {
      if (x.first > hi) {
        if (hi > lo) t += hi - lo;
        lo = x.first; hi = x.second;
      } else if (x.second > hi) {
        hi = x.second;
      }
    }
    if (hi > lo) t += hi - lo;
  }
  if (ms) *ms = t;
  if (launches) *launches = c;
  if (flops) *flops = f;
  if (bytes) *bytes = b;
  return (int)TRINV_OK;
}

}  // extern "C"
