// gemm.cu — FP64 tensor-core (DMMA) product engine: the off-diagonal products
// of the recursive split and a
// general batched GEMM with triangular-operand K-ranges used by the NEXT rows
// (LU / general inverse, COMBRIT beta = 4, Strassen experiment).
//
// Level launches (launch_level): one launch covers every merge of one recursion
// level (COMBRIT with beta = 2, Alg. 1: the n/(2b) merges of a level
// are independent).  Per merge at offset s with halves b and r:
//   lower  inv([A 0; C B]) = [A^{-1} 0; -B^{-1} C A^{-1}  B^{-1}]
//     MODE_LOWER_1:  W   = C . A^{-1}       tile (I,J): k in [J*BN, b)       (A^{-1} lower)
//     MODE_LOWER_2:  X21 = -B^{-1} . W      tile (I,J): k in [0, (I+1)*BM)   (B^{-1} lower)
//   upper  inv([A B; 0 C]) = [A^{-1}  -A^{-1} B C^{-1}; 0 C^{-1}]
//     MODE_UPPER_1:  W   = A^{-1} . B       tile (I,J): k in [I*BM, b)
//     MODE_UPPER_2:  X12 = -W . C^{-1}      tile (I,J): k in [0, (J+1)*BN)
//   general from factors (SKUL S K = A^{-1}; P_UL)
//     MODE_UL:       X = U^{-1} . L^{-1}    tile (I,J): k in [max(I*BM, J*BN), n)
// The K-ranges skip the structurally-zero blocks of the triangular operand
// (P_TF = m^3); diagonal tiles are multiplied densely on the
// explicit zeros written by the previous level.  LOWER_2 / UPPER_2 also write
// +0.0 over the mirrored tile of the opposite triangle (row a7).
//
// Engine: CTA tile BM x BN, K-step BK = 16, STAGES-deep smem ring filled by
// TMA (cp.async.bulk.tensor) from a producer warp through full/empty
// mbarriers; WM x WN consumer warps issue mma.sync.m8n8k4.f64 (DMMA.8x8x4).
// Shared-memory layout for the m8n8k4 fragments, whose 64-bit loads are served
// per half-warp (16 lanes = 128 B must cover the 32 banks once): A tile = BK/4
// boxes of [BM rows][4 k], B tile = BN/4 boxes of [BK rows][4 n]; each
// half-warp fragment load reads 128 contiguous bytes (measured best of three
// layouts, profiles/r01_gemm_variants.txt).  Out-of-range rows / columns are
// zero-filled by TMA and clipped at the store.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

constexpr int BK = 16;
#ifndef LEVEL_GROUP
#define LEVEL_GROUP 12  // K-classes per raster group of the level launches
#endif

// One output tile: where its operands come from and its K-range.  Only o_row /
// o_col / g stay live across the main loop; everything else of the epilogue is
// read from the kernel parameters (constant bank), which keeps the 128x128 tile
// within the 168-register cap of a 9-warp CTA without spills.
struct TileJob {
  int32_t a_row, a_col;  // A-operand: rows a_row.., columns a_col + k
  int32_t b_row, b_col;  // B-operand: rows b_row + k, columns b_col..
  int32_t ga, gb;        // 3rd TMA coordinate (batch) of A / B (3-D maps only)
  int32_t k_begin, k_end;
  int32_t o_row, o_col, g;  // output tile origin (and batch index)
  int32_t m_row, m_col;     // mirror tile origin (zero fill, level modes 2), or -1
  int32_t sem, chunk;       // split-K: the tile's semaphore index and this unit's K chunk (sem -1: unsplit)
  int32_t nch, unit0;       // split-K: chunks of the tile, unit index of its chunk 0
  int32_t lg, li, lj;       // level launches: merge and tile indices
  int32_t phase;            // fused level launches: 0 = first product (W), 1 = second
  bool valid;
};

template <int BM, int BN, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int kConsumerWarps = WM * WN;
  static constexpr int kThreads = (kConsumerWarps + 1) * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BK * BN * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of 8x8");
  static_assert(BM % BK == 0 && BN % BK == 0, "BK must divide BM and BN");
};

// ---------------------------------------------------------------------------
// Level launches: tile mapping (grid order = longest K first, so the hardware
// block scheduler approximates a longest-processing-time schedule) + epilogue.
struct LevelTraits {
  using Params = LevelArgs;
  template <int BM, int BN>
  static __host__ __device__ __forceinline__ TileJob job(const LevelArgs& p, int64_t t) {
    TileJob j{};
    const int64_t b = p.b, n = p.n, merges = p.merges;
    const int64_t TMmax = (b + BM - 1) / BM, TNmax = (b + BN - 1) / BN;
    int64_t g = 0, I = 0, J = 0;
    // Tiles are ordered by their K-class (the tile index the K-range depends on), longest K
    // first (an LPT schedule under the in-order CTA dispatch), and within a class group of
    // LEVEL_GROUP classes the free index is the outer loop: a wave of ~148 CTAs then reads
    // ~LEVEL_GROUP + 148 / LEVEL_GROUP operand panels instead of ~149 (grouped raster, L2
    // reuse; the top-level TRMM of config 3 moved 124 GB of DRAM with the class-major order).
    const bool cls_is_j = p.mode == MODE_LOWER_1 || p.mode == MODE_UPPER_2;
    const int64_t Tc = cls_is_j ? TNmax : TMmax, Tf = cls_is_j ? TMmax : TNmax;
    int64_t chunk = -1;
    // K-length of a class (split-K levels have full merges, r = b)
    auto cls_len = [&](int64_t cc) -> int64_t {
      switch (p.mode) {
        case MODE_LOWER_1: return b - cc * BN;
        case MODE_UPPER_1: return b - cc * BM;
        case MODE_LOWER_2: return (cc + 1) * BM < b ? (cc + 1) * BM : b;
        default: return (cc + 1) * BN < b ? (cc + 1) * BN : b;
      }
    };
    if (p.kchunk > 0) {  // split-K: classes in dispatch order, each tile's chunks consecutive
      const int64_t kc = p.kchunk;
      int64_t c = 0, cc = 0, nc = 1, rem = t;
      for (; c < Tc; ++c) {
        cc = (p.mode == MODE_LOWER_2 || p.mode == MODE_UPPER_2) ? Tc - 1 - c : c;
        nc = (cls_len(cc) + kc - 1) / kc;
        const int64_t cnt = merges * Tf * nc;
        if (rem < cnt) break;
        rem -= cnt;
      }
      const int64_t tl = rem / nc;
      chunk = rem % nc;
      j.nch = (int32_t)nc;
      j.unit0 = (int32_t)(t - chunk);
      g = tl / Tf;
      const int64_t f = tl % Tf;
      if (cls_is_j) { J = cc; I = f; } else { I = cc; J = f; }
      j.sem = (int32_t)((g * Tc + cc) * Tf + f);
    } else if (p.mode != MODE_UL) {
      // small levels (operands L2-resident) keep the exact class-major LPT order (G = 1)
      const int64_t G = b >= 8192 ? LEVEL_GROUP : 1;
      const int64_t per_cls = merges * Tf, cg = t / (per_cls * G);
      const int64_t gsz = Tc - cg * G < G ? Tc - cg * G : G;
      const int64_t local = t - cg * per_cls * G;
      g = local / (Tf * gsz);
      const int64_t l2 = local % (Tf * gsz);
      const int64_t f = l2 / gsz, c = cg * G + l2 % gsz;
      // ascending class = longest K first for LOWER_1 (k >= J) / UPPER_1 (k >= I); LOWER_2 /
      // UPPER_2 have k < (I+1) / (J+1): descending
      const int64_t cc = (p.mode == MODE_LOWER_2 || p.mode == MODE_UPPER_2) ? Tc - 1 - c : c;
      if (cls_is_j) { J = cc; I = f; } else { I = cc; J = f; }
    }
    switch (p.mode) {
      case MODE_LOWER_1: case MODE_LOWER_2: case MODE_UPPER_1: case MODE_UPPER_2: break;
      default: {  // MODE_UL: max(I, J) ascending
        int64_t m = (int64_t)sqrt((double)t);
        while (m * m > t) --m;
        while ((m + 1) * (m + 1) <= t) ++m;
        const int64_t q = t - m * m;
        if (q <= m) { I = m; J = q; } else { I = q - m - 1; J = m; }
      } break;
    }
    const int64_t s = 2 * g * b;
    const int64_t r = (p.mode == MODE_UL) ? n : (n - s - b < b ? n - s - b : b);  // second half
    j.valid = true;
    j.m_row = j.m_col = -1;
    j.g = 0; j.ga = j.gb = 0;
    const int32_t sem = p.kchunk > 0 ? j.sem : -1;
    switch (p.mode) {
      case MODE_LOWER_1:
        j.valid = I * BM < r;
        j.a_row = (int32_t)(s + b + I * BM); j.a_col = (int32_t)s;
        j.b_row = (int32_t)s; j.b_col = (int32_t)(s + J * BN);
        j.o_row = (int32_t)(g * b + I * BM); j.o_col = (int32_t)(J * BN);
        j.k_begin = (int32_t)(J * BN); j.k_end = (int32_t)b;
        break;
      case MODE_LOWER_2:
        j.valid = I * BM < r;
        j.a_row = (int32_t)(s + b + I * BM); j.a_col = (int32_t)(s + b);
        j.b_row = (int32_t)(g * b); j.b_col = (int32_t)(J * BN);
        j.o_row = (int32_t)(s + b + I * BM); j.o_col = (int32_t)(s + J * BN);
        j.m_row = (int32_t)(s + J * BN); j.m_col = (int32_t)(s + b + I * BM);
        j.k_begin = 0; j.k_end = (int32_t)((I + 1) * BM < r ? (I + 1) * BM : r);
        break;
      case MODE_UPPER_1:
        j.valid = J * BN < r;
        j.a_row = (int32_t)(s + I * BM); j.a_col = (int32_t)s;
        j.b_row = (int32_t)s; j.b_col = (int32_t)(s + b + J * BN);
        j.o_row = (int32_t)(g * b + I * BM); j.o_col = (int32_t)(J * BN);
        j.k_begin = (int32_t)(I * BM); j.k_end = (int32_t)b;
        break;
      case MODE_UPPER_2:
        j.valid = J * BN < r;
        j.a_row = (int32_t)(g * b + I * BM); j.a_col = 0;
        j.b_row = (int32_t)(s + b); j.b_col = (int32_t)(s + b + J * BN);
        j.o_row = (int32_t)(s + I * BM); j.o_col = (int32_t)(s + b + J * BN);
        j.m_row = (int32_t)(s + b + J * BN); j.m_col = (int32_t)(s + I * BM);
        j.k_begin = 0; j.k_end = (int32_t)((J + 1) * BN < r ? (J + 1) * BN : r);
        break;
      default:
        j.a_row = (int32_t)(I * BM); j.a_col = 0;
        j.b_row = 0; j.b_col = (int32_t)(J * BN);
        j.o_row = (int32_t)(I * BM); j.o_col = (int32_t)(J * BN);
        j.k_begin = (int32_t)((I * BM > J * BN) ? I * BM : J * BN); j.k_end = (int32_t)n;
        break;
    }
    j.sem = sem;
    j.chunk = (int32_t)(chunk < 0 ? 0 : chunk);
    j.lg = (int32_t)g; j.li = (int32_t)I; j.lj = (int32_t)J; j.phase = 0;
    if (sem >= 0) {  // this unit's K chunk of the tile's range
      const int32_t kb = j.k_begin + j.chunk * p.kchunk;
      j.k_end = kb + p.kchunk < j.k_end ? kb + p.kchunk : j.k_end;
      j.k_begin = kb;
    }
    return j;
  }
  static __device__ __forceinline__ int* sync(const LevelArgs& p) { return p.kchunk > 0 ? p.sync : nullptr; }
  static constexpr bool kFused = false;
  static __device__ __forceinline__ void wait_k(const LevelArgs&, const TileJob&, int32_t, int32_t) {}
  static __device__ __forceinline__ int split_mode(const LevelArgs& p) { return p.split_mode; }
  static __device__ __forceinline__ double* partial(const LevelArgs& p) { return p.partial; }
  static __device__ __forceinline__ double* out(const LevelArgs& p, const TileJob& j) {
    return p.out + (int64_t)j.o_row * p.ldo + j.o_col;
  }
  static __device__ __forceinline__ int64_t ldo(const LevelArgs& p) { return p.ldo; }
  static __device__ __forceinline__ int64_t rows_left(const LevelArgs& p, const TileJob& j) { return p.out_rows - j.o_row; }
  static __device__ __forceinline__ int64_t cols_left(const LevelArgs& p, const TileJob& j) { return p.out_cols - j.o_col; }
  static __device__ __forceinline__ double alpha(const LevelArgs& p) { return p.alpha; }
  static __device__ __forceinline__ double beta(const LevelArgs&) { return 0.0; }
  static __device__ __forceinline__ double* mir(const LevelArgs& p) { return p.mir; }
  static __device__ __forceinline__ int64_t ldm(const LevelArgs& p) { return p.ldm; }
  static __device__ __forceinline__ int64_t n(const LevelArgs& p) { return p.n; }
};

// General batched GEMM: tiles g outer, then I, J (K-range classes of a
// triangular operand ordered longest first).
struct GemmTraits {
  using Params = GemmArgs;
  template <int BM, int BN>
  static __device__ __forceinline__ TileJob job(const GemmArgs& p, int64_t t) {
    TileJob j{};
    const int64_t TM = (p.M + BM - 1) / BM, TN = (p.N + BN - 1) / BN;
    const int64_t per = TM * TN;
    const int64_t g = t / per, rem = t % per;
    int64_t I, J;
    if (p.triA != TRI_NONE) {  // class = I (its K-range)
      I = rem / TN; J = rem % TN;
      if (p.triA == TRI_LOWER) I = TM - 1 - I;  // long K (large I) first
    } else {
      J = rem / TM; I = rem % TM;
      if (p.triB == TRI_UPPER) J = TN - 1 - J;  // long K (large J) first
    }
    int64_t kb = 0, ke = p.K;
    if (p.triA == TRI_LOWER) ke = ke < (I + 1) * BM ? ke : (I + 1) * BM;  // A[i][k] = 0 for k > i
    if (p.triA == TRI_UPPER) kb = kb > I * BM ? kb : I * BM;              // A[i][k] = 0 for k < i
    if (p.triB == TRI_LOWER) kb = kb > J * BN ? kb : J * BN;              // B[k][j] = 0 for k < j
    if (p.triB == TRI_UPPER) ke = ke < (J + 1) * BN ? ke : (J + 1) * BN;  // B[k][j] = 0 for k > j
    j.valid = true;
    j.a_row = (int32_t)(I * BM); j.a_col = 0;
    j.b_row = 0; j.b_col = (int32_t)(J * BN);
    j.ga = j.gb = j.g = (int32_t)g;
    j.k_begin = (int32_t)kb; j.k_end = (int32_t)(ke > kb ? ke : kb);
    j.o_row = (int32_t)(I * BM); j.o_col = (int32_t)(J * BN);
    j.m_row = j.m_col = -1;
    j.sem = -1; j.chunk = 0;
    return j;
  }
  static __device__ __forceinline__ double* out(const GemmArgs& p, const TileJob& j) {
    return p.C + (int64_t)j.g * p.sC + (int64_t)j.o_row * p.ldc + j.o_col;
  }
  static __device__ __forceinline__ int64_t ldo(const GemmArgs& p) { return p.ldc; }
  static __device__ __forceinline__ int64_t rows_left(const GemmArgs& p, const TileJob& j) { return p.M - j.o_row; }
  static __device__ __forceinline__ int64_t cols_left(const GemmArgs& p, const TileJob& j) { return p.N - j.o_col; }
  static __device__ __forceinline__ double alpha(const GemmArgs& p) { return p.alpha; }
  static __device__ __forceinline__ double beta(const GemmArgs& p) { return p.beta; }
  static __device__ __forceinline__ double* mir(const GemmArgs&) { return nullptr; }
  static __device__ __forceinline__ int64_t ldm(const GemmArgs&) { return 0; }
  static __device__ __forceinline__ int64_t n(const GemmArgs&) { return 0; }
  static __device__ __forceinline__ int* sync(const GemmArgs&) { return nullptr; }
  static constexpr bool kFused = false;
  static __device__ __forceinline__ void wait_k(const GemmArgs&, const TileJob&, int32_t, int32_t) {}
  static __device__ __forceinline__ int split_mode(const GemmArgs&) { return 0; }
  static __device__ __forceinline__ double* partial(const GemmArgs&) { return nullptr; }
};

// ---------------------------------------------------------------------------
// Fused level launches: both products of one level in ONE launch.  Work units are the
// first product's tiles (W, longest K first) followed by the second product's tiles, handed
// out by an in-order ticket (a unit is given to a CTA only after every earlier unit has a
// running CTA, so no unit waits on an unscheduled one).  A W tile publishes a per-tile flag
// (= the launch's epoch) after its stores; the producer warp of a second-product tile waits
// for the flag of each W tile its K range enters before issuing the TMA loads of that K
// block, so second-product tiles start while the first product drains.
struct FusedArgs {
  LevelArgs p[2];
  int64_t units1;  // tiles of the first product
  int* ticket;     // zeroed once per call
  int* flags;      // per W tile of merge g, tile (I, J): (g TM + I) TN + J
  int32_t epoch;   // flag value meaning "stored" (unique per fused launch of the call)
};
struct FusedTraits {
  using Params = FusedArgs;
  static constexpr bool kFused = true;
  template <int BM, int BN>
  static __device__ __forceinline__ TileJob job(const FusedArgs& p, int64_t t) {
    const int ph = t < p.units1 ? 0 : 1;
    TileJob j = LevelTraits::template job<BM, BN>(p.p[ph], ph ? t - p.units1 : t);
    j.phase = ph;
    return j;
  }
  static __device__ __forceinline__ const LevelArgs& L(const FusedArgs& p, const TileJob& j) { return p.p[j.phase]; }
  static __device__ __forceinline__ double* out(const FusedArgs& p, const TileJob& j) { return LevelTraits::out(L(p, j), j); }
  static __device__ __forceinline__ int64_t ldo(const FusedArgs& p) { return p.p[0].ldo; }  // unused: see ldo_j
  static __device__ __forceinline__ int64_t ldo_j(const FusedArgs& p, const TileJob& j) { return L(p, j).ldo; }
  static __device__ __forceinline__ int64_t rows_left(const FusedArgs& p, const TileJob& j) {
    return LevelTraits::rows_left(L(p, j), j);
  }
  static __device__ __forceinline__ int64_t cols_left(const FusedArgs& p, const TileJob& j) {
    return LevelTraits::cols_left(L(p, j), j);
  }
  static __device__ __forceinline__ double alpha_j(const FusedArgs& p, const TileJob& j) { return L(p, j).alpha; }
  static __device__ __forceinline__ double beta(const FusedArgs&) { return 0.0; }
  static __device__ __forceinline__ double* mir_j(const FusedArgs& p, const TileJob& j) { return L(p, j).mir; }
  static __device__ __forceinline__ int64_t ldm_j(const FusedArgs& p, const TileJob& j) { return L(p, j).ldm; }
  static __device__ __forceinline__ int64_t n(const FusedArgs& p) { return p.p[0].n; }
  static __device__ __forceinline__ int* sync(const FusedArgs& p) { return p.ticket; }
  static __device__ __forceinline__ int split_mode(const FusedArgs&) { return 0; }
  static __device__ __forceinline__ double* partial(const FusedArgs&) { return nullptr; }
  // producer of a second-product tile: before the K block at k, wait for the W tile it reads
  template <int T>
  static __device__ __forceinline__ void wait_k(const FusedArgs& p, const TileJob& j, int32_t k, int32_t k_prev) {
    if (j.phase == 0 || (k_prev >= 0 && k / T == k_prev / T)) return;
    const LevelArgs& a = p.p[1];
    const int64_t TMt = (a.b + T - 1) / T;
    const bool lower = a.mode == MODE_LOWER_2;  // W is B (rows k) for lower, A (columns k) for upper
    const int64_t idx = lower ? ((int64_t)j.lg * TMt + k / T) * TMt + j.lj : ((int64_t)j.lg * TMt + j.li) * TMt + k / T;
    const int* f = p.flags + idx;
    int v;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (++spins > (1ll << 30)) __trap();  // a missing flag must fail loudly, not hang the GPU
    } while (v != p.epoch);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> TMA reads
  }
  template <int T>
  static __device__ __forceinline__ int* publish_flag(const FusedArgs& p, const TileJob& j) {
    if (j.phase != 0) return nullptr;
    const int64_t TMt = (p.p[0].b + T - 1) / T;
    return p.flags + ((int64_t)j.lg * TMt + j.li) * TMt + j.lj;
  }
};

// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES, int RANK, typename TR>
__device__ __forceinline__ void run_tile(const CUtensorMap* mapA, const CUtensorMap* mapB,
                                         const typename TR::Params& p, unsigned char* smem_raw) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  // split-K levels take their work unit from an in-order ticket (a unit is handed out only
  // after every earlier unit has a running CTA, so a chunk never waits on an unscheduled one)
  __shared__ int s_unit;
  // PDL: wait for the previous kernel before touching global memory (a no-op without the
  // launch attribute); the next kernel is released as this grid's CTAs exit (pdl_trigger_early
  // is a no-op unless built with -DTRINV_PDL_EARLY)
  pdl_trigger_early();
  pdl_wait();
  int* sync = TR::sync(p);
  if (sync) {
    if (threadIdx.x == 0) s_unit = atomicAdd(sync, 1);
    __syncthreads();
  }
  const TileJob tj = TR::template job<BM, BN>(p, sync ? (int64_t)s_unit : (int64_t)blockIdx.x);
  if constexpr (TR::kFused) {  // the phase's operand maps: [A1, B1, A2, B2]
    mapA += 2 * tj.phase;
    mapB += 2 * tj.phase;
  }
  if (!tj.valid) return;
  // align by offsetting the __shared__ pointer itself (an integer round trip would turn
  // the fragment loads into generic LD instead of LDS)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(base);                              // [STAGES][BK/4][BM][4]
  double* sB = reinterpret_cast<double*>(base + (size_t)STAGES * C::A_BYTES);  // [STAGES][BN/4][BK][4]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (tj.k_end - tj.k_begin + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::kConsumerWarps) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(mapA);
      tma_prefetch_desc(mapB);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        const int use = kt / STAGES;
        if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
        const int32_t k = tj.k_begin + kt * BK;
        if constexpr (TR::kFused) TR::template wait_k<BM>(p, tj, k, kt > 0 ? k - BK : -1);
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        double* sa = sA + (size_t)s * BM * BK;
#pragma unroll
        for (int kb = 0; kb < BK / 4; ++kb) {
          if (RANK == 2)
            tma_load_2d(sa + kb * BM * 4, mapA, tj.a_col + k + 4 * kb, tj.a_row, &full[s]);
          else
            tma_load_3d(sa + kb * BM * 4, mapA, tj.a_col + k + 4 * kb, tj.a_row, tj.ga, &full[s]);
        }
        double* sb = sB + (size_t)s * BK * BN;
#pragma unroll
        for (int nb = 0; nb < BN / 4; ++nb) {
          if (RANK == 2)
            tma_load_2d(sb + nb * BK * 4, mapB, tj.b_col + nb * 4, tj.b_row + k, &full[s]);
          else
            tma_load_3d(sb + nb * BK * 4, mapB, tj.b_col + nb * 4, tj.b_row + k, tj.gb, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  if (tj.m_row >= 0 && tj.chunk == 0) {  // mirror-tile zero fill (row a7): BN rows x BM columns of the opposite triangle
    int64_t ldm;
    double* mir0;
    if constexpr (TR::kFused) { ldm = TR::ldm_j(p, tj); mir0 = TR::mir_j(p, tj); }
    else { ldm = TR::ldm(p); mir0 = TR::mir(p); }
    const int64_t nn = TR::n(p);
    double* mir = mir0 + (int64_t)tj.m_row * ldm + tj.m_col;
    constexpr int PAIRS = BM / 2;
    for (int e = threadIdx.x; e < BN * PAIRS; e += C::kConsumerWarps * 32) {
      const int64_t row = e / PAIRS, col = 2 * (e % PAIRS);
      if (tj.m_row + row < nn) {
        double* q = mir + row * ldm + col;
        if (tj.m_col + col + 1 < nn) *reinterpret_cast<double2*>(q) = make_double2(0.0, 0.0);
        else if (tj.m_col + col < nn) *q = 0.0;
      }
    }
  }

  const int wm = warp / WN, wn = warp % WN;
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int lr = lane >> 2, lc = lane & 3;
  // per-lane fragment offsets (doubles): A[row][k] in box k/4 of [BM][4]; B[k][col] in box col/4 of [BK][4]
  const int a_base = (wm * C::WTM + lr) * 4 + lc;
  const int b_base = ((wn * C::WTN + lr) >> 2) * BK * 4 + lc * 4 + (lr & 3);
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
    const double* a_st = sA + (size_t)s * BM * BK + a_base;
    const double* b_st = sB + (size_t)s * BK * BN + b_base;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) af[mi] = a_st[kk * BM * 4 + mi * 32];
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) bf[ni] = b_st[kk * 16 + ni * 2 * BK * 4];
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue: out = alpha * acc (+ beta * out), clipped ----------------
  double* out = TR::out(p, tj);
  int64_t ldo;
  double alpha;
  if constexpr (TR::kFused) { ldo = TR::ldo_j(p, tj); alpha = TR::alpha_j(p, tj); }
  else { ldo = TR::ldo(p); alpha = TR::alpha(p); }
  const int64_t rows = TR::rows_left(p, tj), cols = TR::cols_left(p, tj);
  double beta = TR::beta(p);
  int* sem = nullptr;
  bool fixup = false;
  fixup = tj.sem >= 0 && TR::split_mode(p) == 2;
  if (fixup) {  // split-K fix-up: store alpha * partial in this unit's slot, the last chunk sums
    constexpr int TS = BM * BN;
    double* slot = TR::partial(p) + (int64_t)(tj.unit0 + tj.chunk) * TS;
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) {
        const int row = wm * C::WTM + mi * 8 + lr, col = wn * C::WTN + ni * 8 + 2 * lc;
        __stcg(reinterpret_cast<double2*>(slot + row * BN + col),
               make_double2(alpha * acc[mi][ni][0], alpha * acc[mi][ni][1]));
      }
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
    __shared__ int s_last;
    int* cnt = sync + 1 + tj.sem;
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(cnt, 1);
      s_last = prev == tj.nch - 1;
      if (s_last) *cnt = 0;  // ready for the next split launch of the call
    }
    asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
    if (!s_last) return;
    __threadfence();  // acquire side: the other chunks' partials are visible (read via L2 below)
    const double* base = TR::partial(p) + (int64_t)tj.unit0 * TS;
#pragma unroll
    for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) {
        const int row = wm * C::WTM + mi * 8 + lr, col = wn * C::WTN + ni * 8 + 2 * lc;
        double2 sum = __ldcg(reinterpret_cast<const double2*>(base + row * BN + col));
        for (int c = 1; c < tj.nch; ++c) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(base + (int64_t)c * TS + row * BN + col));
          sum.x += v.x;
          sum.y += v.y;
        }
        acc[mi][ni][0] = sum.x;
        acc[mi][ni][1] = sum.y;
      }
  }
  const double alpha_out = fixup ? 1.0 : alpha;  // the partials already carry alpha
  if (tj.sem >= 0 && !fixup) {  // split-K: add this chunk's partial after chunk - 1 has stored its sum
    sem = sync + 1 + tj.sem;
    if (tj.chunk > 0) {
      if (lane == 0) {
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(sem) : "memory");
        } while (v < tj.chunk);
      }
      __syncwarp();
      beta = 1.0;
    }
  }
  // 16-byte stores need an even leading dimension and an aligned tile origin
  const bool vec = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && (ldo % 2 == 0);
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi) {
    const int64_t row = wm * C::WTM + mi * 8 + lr;
    if (row >= rows) continue;
    double* orow = out + row * ldo;
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) {
      const int64_t col = wn * C::WTN + ni * 8 + 2 * lc;
      double v0 = alpha_out * acc[mi][ni][0], v1 = alpha_out * acc[mi][ni][1];
      if (col + 1 < cols && vec) {
        if (beta != 0.0) {
          const double2 o = __ldcg(reinterpret_cast<const double2*>(orow + col));
          v0 = fma(beta, o.x, v0);
          v1 = fma(beta, o.y, v1);
        }
        *reinterpret_cast<double2*>(orow + col) = make_double2(v0, v1);
      } else {
        if (col < cols) orow[col] = (beta != 0.0) ? fma(beta, __ldcg(orow + col), v0) : v0;
        if (col + 1 < cols) orow[col + 1] = (beta != 0.0) ? fma(beta, __ldcg(orow + col + 1), v1) : v1;
      }
    }
  }
  if (sem) {  // every consumer warp has stored: release the next chunk
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sem), "r"(tj.chunk + 1) : "memory");
  }
  if constexpr (TR::kFused) {  // a W tile of a fused launch: publish it for the second product
    int* flag = TR::template publish_flag<BM>(p, tj);
    if (flag) {
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(p.epoch) : "memory");
    }
  }
}

template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES>::kThreads, 1)
    dmma_level_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const LevelArgs p) {
  extern __shared__ unsigned char smem_raw[];
  run_tile<BM, BN, WM, WN, STAGES, 2, LevelTraits>(&mapA, &mapB, p, smem_raw);
}
// The same kernel capped at 128 registers: a warp then takes 4096 of its SM sub-partition's
// 16384 registers, so three 5-warp CTAs fit per SM where 131 registers allow two (ncu
// launch__occupancy_limit_registers; the 64x32 tile of the mid-size top levels).
template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __maxnreg__(128)
    dmma_level_kernel_r128(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                           const LevelArgs p) {
  extern __shared__ unsigned char smem_raw[];
  run_tile<BM, BN, WM, WN, STAGES, 2, LevelTraits>(&mapA, &mapB, p, smem_raw);
}

struct FusedMaps {
  CUtensorMap m[4];  // A1, B1, A2, B2
};
template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES>::kThreads, 1)
    dmma_fused_level_kernel(const __grid_constant__ FusedMaps maps, const FusedArgs p) {
  extern __shared__ unsigned char smem_raw[];
  run_tile<BM, BN, WM, WN, STAGES, 2, FusedTraits>(&maps.m[0], &maps.m[1], p, smem_raw);
}

template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES>::kThreads, 1)
    dmma_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const GemmArgs p) {
  extern __shared__ unsigned char smem_raw[];
  run_tile<BM, BN, WM, WN, STAGES, 3, GemmTraits>(&mapA, &mapB, p, smem_raw);
}

// ---------------------------------------------------------------------------
// Stream-K level launches (mid-size levels).  With one CTA per tile a level whose tiles fit
// in one or two waves is as long as its longest-K tile (the triangular K ranges span 1..b/BK
// iterations), and every CTA pays the pipeline fill once per tile.  Here a persistent grid of
// P CTAs splits the level's total K-iterations (sum over its tiles, in the LPT tile order of
// LevelTraits::job, of ceil(K range / BK)) into P contiguous ranges of W iterations: CTA c
// runs [c W, (c+1) W), crossing tile boundaries with one continuous TMA ring.  A tile cut by
// a range boundary is finished by the CTA that ran its first iterations (the "owner", whose
// piece is the last one of its range): the CTAs holding the tile's later iterations run them
// FIRST in their ranges, store the raw partial sum in their slot and release a flag; the
// owner adds the partials in CTA order (a fixed, schedule-determined summation order) and
// stores alpha * sum (+ the mirror-tile zero fill).  Only owners wait, only on higher CTAs,
// whose pieces come first in their ranges: with all P CTAs resident nothing waits long, and
// the last CTA never waits.  Flags are 0 between launches (each owner clears the flags it
// consumed; the call zeroes them once before its first level).
constexpr int SK_MAX_P = 320;
struct SkArgs {
  int32_t W;            // K-iterations per CTA
  int32_t total;        // K-iterations of the level
  int* flags;           // [P]: 1 = CTA c's leading partial is stored
  double* partial;      // [P][BM * BN] raw partial sums
  int32_t t0[SK_MAX_P];    // tile of CTA c's first iteration
  int32_t off0[SK_MAX_P];  // that iteration's index inside the tile
};
template <int BM, int BN>
__host__ __device__ __forceinline__ int32_t sk_nk(const TileJob& j) {
  return j.valid ? (j.k_end - j.k_begin + BK - 1) / BK : 0;
}

template <int BM, int BN, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES>::kThreads, MINB)
    dmma_sk_level_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         const LevelArgs p, const __grid_constant__ SkArgs sk) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  extern __shared__ unsigned char smem_raw[];
  const int c = blockIdx.x;
  const int32_t todo = min(sk.W, sk.total - c * sk.W);
  if (todo <= 0) return;
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(base);                              // [STAGES][BK/4][BM][4]
  double* sB = reinterpret_cast<double*>(base + (size_t)STAGES * C::A_BYTES);  // [STAGES][BN/4][BK][4]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::kConsumerWarps) {
    // ---------------- TMA producer: the CTA's iterations, tile after tile, one ring ----------------
    if (lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      int32_t it = 0, t = sk.t0[c], off = sk.off0[c], rem = todo;
      while (rem > 0) {
        const TileJob tj = LevelTraits::template job<BM, BN>(p, t);
        const int32_t len = min(sk_nk<BM, BN>(tj) - off, rem);
        for (int32_t kt = off; kt < off + len; ++kt, ++it) {
          const int s = it % STAGES;
          const int use = it / STAGES;
          if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
          const int32_t k = tj.k_begin + kt * BK;
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          double* sa = sA + (size_t)s * BM * BK;
#pragma unroll
          for (int kb = 0; kb < BK / 4; ++kb) tma_load_2d(sa + kb * BM * 4, &mapA, tj.a_col + k + 4 * kb, tj.a_row, &full[s]);
          double* sb = sB + (size_t)s * BK * BN;
#pragma unroll
          for (int nb = 0; nb < BN / 4; ++nb) tma_load_2d(sb + nb * BK * 4, &mapB, tj.b_col + nb * 4, tj.b_row + k, &full[s]);
        }
        if (len > 0) rem -= len;
        ++t;
        off = 0;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int wm = warp / WN, wn = warp % WN;
  const int lr = lane >> 2, lc = lane & 3;
  const int a_base = (wm * C::WTM + lr) * 4 + lc;
  const int b_base = ((wn * C::WTN + lr) >> 2) * BK * 4 + lc * 4 + (lr & 3);
  int32_t it = 0, t = sk.t0[c], off = sk.off0[c], rem = todo;
  while (rem > 0) {
    const TileJob tj = LevelTraits::template job<BM, BN>(p, t);
    const int32_t nk = sk_nk<BM, BN>(tj);
    const int32_t len = min(nk - off, rem);
    if (len <= 0) { ++t; off = 0; continue; }
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int32_t kt = 0; kt < len; ++kt, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
      const double* a_st = sA + (size_t)s * BM * BK + a_base;
      const double* b_st = sB + (size_t)s * BK * BN + b_base;
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double af[C::FM], bf[C::FN];
#pragma unroll
        for (int mi = 0; mi < C::FM; ++mi) af[mi] = a_st[kk * BM * 4 + mi * 32];
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) bf[ni] = b_st[kk * 16 + ni * 2 * BK * 4];
#pragma unroll
        for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    constexpr int TS = BM * BN;
    if (off > 0) {
      // a later piece of a tile begun by an earlier CTA (always this CTA's first segment)
      double* slot = sk.partial + (int64_t)c * TS;
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) {
          const int row = wm * C::WTM + mi * 8 + lr, col = wn * C::WTN + ni * 8 + 2 * lc;
          __stcg(reinterpret_cast<double2*>(slot + row * BN + col), make_double2(acc[mi][ni][0], acc[mi][ni][1]));
        }
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sk.flags + c), "r"(1) : "memory");
    } else {
      if (len < nk) {  // owner: add the later pieces, CTA c+1, c+2, ... in order
        int32_t rest = nk - len;
        for (int q = 1; rest > 0; ++q, rest -= sk.W) {
          if (lane == 0) {
            const int* f = sk.flags + c + q;
            int v;
            long long spins = 0;
            do {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
              if (++spins > (1ll << 31)) __trap();  // a missing piece must fail loudly, not hang
            } while (v == 0);
          }
          __syncwarp();
          const double* slot = sk.partial + (int64_t)(c + q) * TS;
#pragma unroll
          for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < C::FN; ++ni) {
              const int row = wm * C::WTM + mi * 8 + lr, col = wn * C::WTN + ni * 8 + 2 * lc;
              const double2 v = __ldcg(reinterpret_cast<const double2*>(slot + row * BN + col));
              acc[mi][ni][0] += v.x;
              acc[mi][ni][1] += v.y;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");  // all warps have read
        if (threadIdx.x == 0) {
          rest = nk - len;
          for (int q = 1; rest > 0; ++q, rest -= sk.W) sk.flags[c + q] = 0;
        }
      }
      if (tj.m_row >= 0) {  // mirror-tile zero fill (row a7)
        double* mir = p.mir + (int64_t)tj.m_row * p.ldm + tj.m_col;
        constexpr int PAIRS = BM / 2;
        for (int e = threadIdx.x; e < BN * PAIRS; e += C::kConsumerWarps * 32) {
          const int64_t row = e / PAIRS, col = 2 * (e % PAIRS);
          if (tj.m_row + row < p.n) {
            double* q = mir + row * p.ldm + col;
            if (tj.m_col + col + 1 < p.n) *reinterpret_cast<double2*>(q) = make_double2(0.0, 0.0);
            else if (tj.m_col + col < p.n) *q = 0.0;
          }
        }
      }
      double* out = LevelTraits::out(p, tj);
      const int64_t rows = LevelTraits::rows_left(p, tj), cols = LevelTraits::cols_left(p, tj);
      const bool vec = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && (p.ldo % 2 == 0);
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) {
        const int64_t row = wm * C::WTM + mi * 8 + lr;
        if (row >= rows) continue;
        double* orow = out + row * p.ldo;
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) {
          const int64_t col = wn * C::WTN + ni * 8 + 2 * lc;
          const double v0 = p.alpha * acc[mi][ni][0], v1 = p.alpha * acc[mi][ni][1];
          if (col + 1 < cols && vec) {
            *reinterpret_cast<double2*>(orow + col) = make_double2(v0, v1);
          } else {
            if (col < cols) orow[col] = v0;
            if (col + 1 < cols) orow[col + 1] = v1;
          }
        }
      }
    }
    rem -= len;
    ++t;
    off = 0;
  }
}

// Host side of the stream-K plan: per-CTA first tile / offset from the same tile map.
template <int BM, int BN, int WM, int WN, int STAGES, int MINB>
static cudaError_t launch_level_sk_cfg(const LevelArgs& a, int ctas_per_sm, int w_min, cudaStream_t s,
                                       int64_t* launches) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  const int64_t tiles = a.merges * ((a.b + BM - 1) / BM) * ((a.b + BN - 1) / BN);
  static thread_local SkArgs sk;  // ~2.6 KB: kept off the stack
  int64_t total = 0;
  for (int64_t t = 0; t < tiles; ++t) total += sk_nk<BM, BN>(LevelTraits::template job<BM, BN>(a, t));
  if (total <= 0) return cudaSuccess;
  constexpr auto k = dmma_sk_level_kernel<BM, BN, WM, WN, STAGES, MINB>;
  set_smem_once<k>((int)C::SMEM);
  // every CTA must be resident (owners wait on later CTAs): at most the occupancy per SM
  static const int occ = [] {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, C::kThreads, C::SMEM) != cudaSuccess) o = 1;
    return o < 1 ? 1 : o;
  }();
  if (ctas_per_sm > occ) ctas_per_sm = occ;
  int64_t P = (int64_t)ctas_per_sm * device_sms();
  if (P > SK_MAX_P) P = SK_MAX_P;
  if (P > (int64_t)(SK_PARTIAL_BYTES / (BM * BN * sizeof(double)))) P = SK_PARTIAL_BYTES / (BM * BN * sizeof(double));
  if (P > (total + w_min - 1) / w_min) P = (total + w_min - 1) / w_min;
  if (P < 1) P = 1;
  const int64_t W = (total + P - 1) / P;
  P = (total + W - 1) / W;
  sk.W = (int32_t)W;
  sk.total = (int32_t)total;
  sk.flags = a.sk_flags;
  sk.partial = a.sk_partial;
  int64_t cum = 0, cta = 0;
  for (int64_t t = 0; t < tiles && cta < P; ++t) {
    const int64_t nk = sk_nk<BM, BN>(LevelTraits::template job<BM, BN>(a, t));
    while (cta < P && cta * W < cum + nk) {  // CTA cta starts inside tile t
      sk.t0[cta] = (int32_t)t;
      sk.off0[cta] = (int32_t)(cta * W - cum);
      ++cta;
    }
    cum += nk;
  }
  CUtensorMap mA, mB;
  if (!encode_map(&mA, a.opA, 4, BM, false)) return cudaErrorInvalidValue;
  if (!encode_map(&mB, a.opB, 4, BK, false)) return cudaErrorInvalidValue;
  const cudaError_t e = launch_k(k, dim3((unsigned)P), dim3(C::kThreads), C::SMEM, s, mA, mB, a, sk);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------
// TRINV_R128 = bit mask of the 128-register level-kernel variants (dmma_level_kernel_r128):
// 1 = 64x64 (default: 3 CTAs / SM instead of 2, n = 8192 5420 -> 5299 us, config 2 5.418 ->
// 5.302 ms, config 4 158.09 -> 157.51 ms), 2 = 64x32 (slower: n = 2048's top level 39.7 -> 48.3
// us), 0 = off; only levels with >= TRINV_R128_WAVES (4) waves of 3 CTAs per SM take it (n = 4096's
// top level, 2.3 waves, measured 765 -> 803 us with it).  profiles/r02_tile_waves.txt
static int r128_mask() {
  static const int m = [] { const char* e = std::getenv("TRINV_R128"); return e ? atoi(e) : 1; }();
  return m;
}

template <int BM, int BN, int WM, int WN, int STAGES>
static cudaError_t launch_level_cfg(const LevelArgs& a, cudaStream_t s, int64_t* launches, int64_t units = 0) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  CUtensorMap mA, mB;
  if (!encode_map(&mA, a.opA, 4, BM, false)) return cudaErrorInvalidValue;
  if (!encode_map(&mB, a.opB, 4, BK, false)) return cudaErrorInvalidValue;
  int64_t tiles;
  if (units > 0) {
    tiles = units;  // split-K work units
  } else if (a.mode == MODE_UL) {
    const int64_t T = (a.n + BM - 1) / BM;
    tiles = T * T;
  } else {
    tiles = a.merges * ((a.b + BM - 1) / BM) * ((a.b + BN - 1) / BN);
  }
  if (tiles <= 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  cudaError_t e;
  bool done = false;
  if constexpr (BM == 64 && (BN == 32 || BN == 64)) {
    // (the 128-register variant only where the level has >= TRINV_R128_WAVES waves of 3 CTAs / SM)
    static const double r128_waves = [] { const char* e = std::getenv("TRINV_R128_WAVES"); return e ? atof(e) : 4.0; }();
    if ((r128_mask() & (BN == 64 ? 1 : 2)) && tiles >= (int64_t)(r128_waves * 3 * device_sms())) {
      constexpr auto k = dmma_level_kernel_r128<BM, BN, WM, WN, STAGES>;
      set_smem_once<k>((int)C::SMEM);
      e = launch_k(k, dim3((unsigned)tiles), dim3(C::kThreads), C::SMEM, s, mA, mB, a);
      done = true;
    }
  }
  if (!done) {
    constexpr auto k = dmma_level_kernel<BM, BN, WM, WN, STAGES>;
    set_smem_once<k>((int)C::SMEM);
    e = launch_k(k, dim3((unsigned)tiles), dim3(C::kThreads), C::SMEM, s, mA, mB, a);
  }
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Both products of one level in one launch (FusedTraits).  ticket / flags: zeroed by the
// caller once per call; `epoch` unique among the fused launches of the call (1, 2, ...).
template <int T, int WM, int WN, int STAGES>
static cudaError_t launch_fused_cfg(const LevelArgs& l1, const LevelArgs& l2, int* ticket, int* flags, int epoch,
                                    cudaStream_t s, int64_t* launches) {
  using C = GemmCfg<T, T, WM, WN, STAGES>;
  FusedMaps maps;
  if (!encode_map(&maps.m[0], l1.opA, 4, T, false) || !encode_map(&maps.m[1], l1.opB, 4, BK, false) ||
      !encode_map(&maps.m[2], l2.opA, 4, T, false) || !encode_map(&maps.m[3], l2.opB, 4, BK, false))
    return cudaErrorInvalidValue;
  const int64_t tiles = l1.merges * ((l1.b + T - 1) / T) * ((l1.b + T - 1) / T);
  FusedArgs f{};
  f.p[0] = l1; f.p[1] = l2;
  f.p[0].kchunk = f.p[1].kchunk = 0;
  f.units1 = tiles;
  f.ticket = ticket;
  f.flags = flags;
  f.epoch = epoch;
  constexpr auto k = dmma_fused_level_kernel<T, T, WM, WN, STAGES>;
  set_smem_once<k>((int)C::SMEM);
  k<<<(unsigned)(2 * tiles), C::kThreads, C::SMEM, s>>>(maps, f);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// Algorithmic flops of one level launch, exploiting the triangular operand
// (P_TF; P_UL): 2 flops per multiply-add that touches
// a non-zero of the triangular factor.
static double level_flops(const LevelArgs& a) {
  if (a.mode == MODE_UL) {
    const double n = (double)a.n;
    return 2.0 * (n * (n + 1) * (2 * n + 1) / 6.0) - n * n;  // sum_{i,j} 2(n - max(i,j)) ~ 2n^3/3
  }
  double f = 0.0;
  for (int64_t g = 0; g < a.merges; ++g) {
    const double b = (double)a.b;
    const int64_t s0 = 2 * g * a.b;
    const double r = (double)(a.n - s0 - a.b < a.b ? a.n - s0 - a.b : a.b);
    const bool first = (a.mode == MODE_LOWER_1 || a.mode == MODE_UPPER_1);
    f += first ? r * b * (b + 1) : b * r * (r + 1);
  }
  return f;
}

// Tile size: the largest of 128 / 64 / 32 (not above `cap`) giving at least two
// CTAs per SM; mid-size problems otherwise leave SMs idle behind a few long
// tiles (profiles/r01_sweep_n.txt).
// 128x128 tiles only when they make at least TRINV_LEVEL_W128 (default 32) waves: the 64x64
// tiles balance the triangular K ranges better (n = 8192: 5553 -> 5305 us, config 3 317.0 ->
// 316.0 ms, config 4 164.2 -> 162.6 ms against the round-1 threshold of 2 waves,
// profiles/r02_tile_waves.txt).
template <typename F>
static int64_t pick_tile(F tiles, int64_t cap) {
  const int sms = device_sms();
  static const double w128 = [] { const char* e = std::getenv("TRINV_LEVEL_W128"); return e ? atof(e) : 32.0; }();
  if (128 <= cap && tiles(128) >= w128 * sms) return 128;
  if (64 <= cap && tiles(64) >= 2 * sms) return 64;
  return cap < 32 ? cap : 32;
}

// Split-K for levels that would underfill the GPU with 64x64 tiles (mid-size orders: at
// n = 2048 the top level had 256 such tiles of K up to 1024, so it runs on 32x32 tiles at
// 63% of the DMMA peak): 64x64 tiles with their K ranges cut into chunks, about 3 work units
// per SM, the chunks of a tile summed in order (LevelArgs::sync).  Full merges only.
// Opt-in (TRINV_SPLITK=1): it measured 1.1-1.8x SLOWER than the unsplit 32x32 tiles at
// n = 1024..8192 (the per-level semaphore memset and the serial chunk epilogues cost more
// than the better tiles gain; profiles/r02_splitk.txt).
static int64_t split_plan(const LevelArgs& a, int64_t& kc, int64_t T) {
  const int sms = device_sms();
  if (!a.sync || a.mode == MODE_UL || a.b < 256 || a.n % (2 * a.b) != 0 || a.b % T) return 0;
  const int64_t Tc = a.b / T, tiles = a.merges * Tc * Tc;
  if ((T == 64 && tiles >= 2 * sms) || 1 + tiles > (int64_t)(LEVEL_SYNC_BYTES / sizeof(int))) return 0;
  auto len = [&](int64_t c) {  // K length of class c (all modes: b - c T or (c + 1) T)
    return (a.mode == MODE_LOWER_1 || a.mode == MODE_UPPER_1) ? a.b - c * T : (c + 1) * T;
  };
  int64_t total = 0;
  for (int64_t c = 0; c < Tc; ++c) total += a.merges * Tc * len(c);
  static const int64_t kc_env = [] { const char* e = std::getenv("TRINV_SPLITK_KC"); return e ? atoll(e) : 0; }();
  kc = kc_env > 0 ? kc_env : (total / (3 * sms) + 63) / 64 * 64;
  if (kc < 64) kc = 64;
  int64_t units = 0;
  for (int64_t c = 0; c < Tc; ++c) units += a.merges * Tc * ((len(c) + kc - 1) / kc);
  return units > tiles ? units : 0;
}

// Stream-K level launches: opt-in (TRINV_SK=1).  Measured slower than one CTA per tile at
// n = 1024..8192 for every tile shape tried (profiles/r02_stream_k.txt): the big-tile CTAs
// reach 80% tensor-pipe activity but the per-SM iteration cost is uneven (active cycles
// max / mean 1.22 at n = 2048's top level), and the small levels lose their parallelism.
bool level_sk_enabled() {
  static const bool on = [] { const char* e = std::getenv("TRINV_SK"); return e && atoi(e) != 0; }();
  return on;
}

bool level_split_fixup() {  // TRINV_SPLITK=2: split-K with the last-chunk fix-up (needs LEVEL_PARTIAL_BYTES)
  static const bool on = [] { const char* e = std::getenv("TRINV_SPLITK"); return e && atoi(e) == 2; }();
  return on;
}

bool level_fusable(const LevelArgs& l1) {
  // opt-in (TRINV_FUSED=1): measured slower (n = 2048 165 -> 217 us, the gated second-product
  // tiles hold SM slots while they wait; profiles/r02_fused_levels.txt)
  static const bool on = [] { const char* e = std::getenv("TRINV_FUSED"); return e && e[0] == '1'; }();
  if (!on || !l1.sync || l1.mode == MODE_UL) return false;
  const int sms = device_sms();
  auto tiles = [&](int64_t T) { const int64_t m = (l1.b + T - 1) / T; return l1.merges * m * m; };
  const int64_t T = pick_tile(tiles, l1.b);
  return T >= 32 && tiles(T) <= (int64_t)LEVEL_FLAG_MAX && tiles(T) < 64 * sms;
}

cudaError_t launch_level_fused(const LevelArgs& l1, const LevelArgs& l2, int epoch, cudaStream_t s,
                               int64_t* launches) {
  ProfileScope prof(KIND_DMMA, level_flops(l1) + level_flops(l2), 0.0, s);
  auto tiles = [&](int64_t T) { const int64_t m = (l1.b + T - 1) / T; return l1.merges * m * m; };
  const int64_t T = pick_tile(tiles, l1.b);
  int* ticket = l1.sync + epoch;           // one ticket per fused launch of the call
  int* flags = l1.sync + LEVEL_TICKETS;    // flags carry the epoch
  if (T >= 128) return launch_fused_cfg<128, 2, 4, 5>(l1, l2, ticket, flags, epoch, s, launches);
  if (T >= 64) return launch_fused_cfg<64, 2, 2, 4>(l1, l2, ticket, flags, epoch, s, launches);
  return launch_fused_cfg<32, 2, 2, 4>(l1, l2, ticket, flags, epoch, s, launches);
}

// ---------------------------------------------------------------------------
// Level chain (opt-in, measured slower): the lowest levels of a recursion (those that would run
// 32x32 tiles) in ONE persistent launch.  Their products are latency-bound (n = 2048: the b = 128..512 levels hold
// 19 us of DMMA work but took 59 us as six launches), so the chain replaces the launch
// boundaries by dataflow: the tiles of all phases [W_l0, X21_l0, W_l1, X21_l1, ...] form one
// list in topological order, CTA c takes tiles c, c + G, c + 2G, ... (G = resident CTAs), and
// before a tile's first TMA load its producer waits for the per-(phase, merge) completion
// counters the tile depends on:
//   W of level l, merge g       <- X21 of level l-1, merges 2g and 2g+1 (A^-1, B^-1 complete)
//   X21 of level l, merge g     <- W of level l, merge g
// (the blocks below the first chained level come from the preceding blk launch).  A finished
// tile bumps its counter after its stores (release: __threadfence, then the atomic); a waiting
// producer acquires, then orders the generic writes before its TMA reads with a proxy fence.
// Every dependency points at an earlier tile of the list and every CTA is resident, so the
// wait always ends.  W is laid out by position (the rows of the merge's second half for the
// lower case, its first half for the upper case, ld = the widest chained level) so that a
// merge's W never overlaps the W of a merge that is not yet complete.
constexpr int CHAIN_MAXP = 8;
struct ChainArgs {
  LevelArgs ph[CHAIN_MAXP];
  int32_t tile0[CHAIN_MAXP + 1];  // first global tile of each phase
  int32_t nphase;
  int32_t cstride;                // counters per phase (>= merges of the first level)
  int* cnt;                       // [nphase][cstride] completion counters, zero at launch
};
struct ChainMaps {
  CUtensorMap m[2 * CHAIN_MAXP];  // per phase: A, B
};

template <int BM, int BN>
__device__ __forceinline__ TileJob chain_job(const ChainArgs& c, int p, int64_t t) {
  const LevelArgs& a = c.ph[p];
  TileJob j = LevelTraits::template job<BM, BN>(a, t);
  const int32_t s = 2 * j.lg * (int32_t)a.b, b = (int32_t)a.b;
  switch (a.mode) {  // W by position (see above)
    case MODE_LOWER_1: j.o_row = s + b + j.li * BM; break;
    case MODE_UPPER_1: j.o_row = s + j.li * BM; break;
    case MODE_LOWER_2: j.b_row = s + b; break;
    default: j.a_row = s + j.li * BM; break;  // MODE_UPPER_2
  }
  return j;
}

__device__ __forceinline__ void chain_wait(const int* ctr, int target) {
  int v;
  long long spins = 0;
  do {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(64);
    if (++spins > (1ll << 28)) __trap();  // a missing tile must fail loudly, not hang the GPU
  } while (true);
}

template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES>::kThreads, 1)
    dmma_chain_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainArgs c) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(base);
  double* sB = reinterpret_cast<double*>(base + (size_t)STAGES * C::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t total = c.tile0[c.nphase];
  if ((int32_t)blockIdx.x >= total) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::kConsumerWarps) {
    // ---------------- producer: dependencies, then the tile's K blocks into the ring ----------------
    if (lane == 0) {
      for (int p = 0; p < c.nphase; ++p) {
        tma_prefetch_desc(&maps.m[2 * p]);
        tma_prefetch_desc(&maps.m[2 * p + 1]);
      }
      int32_t it = 0;
      int p = 0;
      for (int32_t T = blockIdx.x; T < total; T += gridDim.x) {
        while (T >= c.tile0[p + 1]) ++p;
        const TileJob tj = chain_job<BM, BN>(c, p, T - c.tile0[p]);
        if (!tj.valid) continue;
        const LevelArgs& a = c.ph[p];
        if (p & 1) {  // X21 of merge g: its W complete
          const int64_t m = (a.b + BM - 1) / BM;
          chain_wait(c.cnt + (p - 1) * c.cstride + tj.lg, (int)(m * m));
        } else if (p > 0) {  // W of merge g: the level below complete on both halves
          const LevelArgs& q = c.ph[p - 1];
          const int64_t m = (q.b + BM - 1) / BM;
          chain_wait(c.cnt + (p - 1) * c.cstride + 2 * tj.lg, (int)(m * m));
          if (2 * tj.lg + 1 < q.merges) chain_wait(c.cnt + (p - 1) * c.cstride + 2 * tj.lg + 1, (int)(m * m));
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores of other CTAs -> TMA reads
        const CUtensorMap* mA = &maps.m[2 * p];
        const CUtensorMap* mB = &maps.m[2 * p + 1];
        const int nk = (tj.k_end - tj.k_begin + BK - 1) / BK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % STAGES;
          const int use = it / STAGES;
          if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
          const int32_t k = tj.k_begin + kt * BK;
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          double* sa = sA + (size_t)s * BM * BK;
#pragma unroll
          for (int kb = 0; kb < BK / 4; ++kb) tma_load_2d(sa + kb * BM * 4, mA, tj.a_col + k + 4 * kb, tj.a_row, &full[s]);
          double* sb = sB + (size_t)s * BK * BN;
#pragma unroll
          for (int nb = 0; nb < BN / 4; ++nb) tma_load_2d(sb + nb * BK * 4, mB, tj.b_col + nb * 4, tj.b_row + k, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int wm = warp / WN, wn = warp % WN;
  const int lr = lane >> 2, lc = lane & 3;
  const int a_base = (wm * C::WTM + lr) * 4 + lc;
  const int b_base = ((wn * C::WTN + lr) >> 2) * BK * 4 + lc * 4 + (lr & 3);
  int32_t it = 0;
  int p = 0;
  for (int32_t T = blockIdx.x; T < total; T += gridDim.x) {
    while (T >= c.tile0[p + 1]) ++p;
    const TileJob tj = chain_job<BM, BN>(c, p, T - c.tile0[p]);
    const LevelArgs& a = c.ph[p];
    if (tj.valid) {
      if (tj.m_row >= 0) {  // mirror-tile zero fill (row a7)
        double* mir = a.mir + (int64_t)tj.m_row * a.ldm + tj.m_col;
        constexpr int PAIRS = BM / 2;
        for (int e = threadIdx.x; e < BN * PAIRS; e += C::kConsumerWarps * 32) {
          const int64_t row = e / PAIRS, col = 2 * (e % PAIRS);
          if (tj.m_row + row < a.n) {
            double* q = mir + row * a.ldm + col;
            if (tj.m_col + col + 1 < a.n) *reinterpret_cast<double2*>(q) = make_double2(0.0, 0.0);
            else if (tj.m_col + col < a.n) *q = 0.0;
          }
        }
      }
      double acc[C::FM][C::FN][2];
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      const int nk = (tj.k_end - tj.k_begin + BK - 1) / BK;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
        const double* a_st = sA + (size_t)s * BM * BK + a_base;
        const double* b_st = sB + (size_t)s * BK * BN + b_base;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
          double af[C::FM], bf[C::FN];
#pragma unroll
          for (int mi = 0; mi < C::FM; ++mi) af[mi] = a_st[kk * BM * 4 + mi * 32];
#pragma unroll
          for (int ni = 0; ni < C::FN; ++ni) bf[ni] = b_st[kk * 16 + ni * 2 * BK * 4];
#pragma unroll
          for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < C::FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      double* out = a.out + (int64_t)tj.o_row * a.ldo + tj.o_col;
      const int64_t rows = a.out_rows - tj.o_row, cols = a.out_cols - tj.o_col;
      const bool vec = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && (a.ldo % 2 == 0);
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) {
        const int64_t row = wm * C::WTM + mi * 8 + lr;
        if (row >= rows) continue;
        double* orow = out + row * a.ldo;
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) {
          const int64_t col = wn * C::WTN + ni * 8 + 2 * lc;
          const double v0 = a.alpha * acc[mi][ni][0], v1 = a.alpha * acc[mi][ni][1];
          if (col + 1 < cols && vec) {
            *reinterpret_cast<double2*>(orow + col) = make_double2(v0, v1);
          } else {
            if (col < cols) orow[col] = v0;
            if (col + 1 < cols) orow[col + 1] = v1;
          }
        }
      }
    }
    // the tile (valid or not) is complete: release it to the tiles that depend on its merge
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"r"(C::kConsumerWarps * 32) : "memory");
    if (threadIdx.x == 0) atomicAdd(c.cnt + p * c.cstride + tj.lg, 1);
  }
}

// Opt-in (TRINV_CHAIN=1): measured slower than one launch per product (n = 2048: 151 -> 170-228 us
// for 1-6 resident CTAs per SM; the chained levels took 78-90 us against 59 us as six launches;
// profiles/r02_level_chain.txt).  A dependent step inside the persistent grid (poll, proxy fence,
// TMA fill, compute, release) costs more than a graph-replayed launch boundary.
bool level_chain_enabled() {
  static const bool on = [] { const char* e = std::getenv("TRINV_CHAIN"); return e && e[0] == '1'; }();
  return on;
}

// Does the level run 32x32 tiles on the per-launch path (the levels the chain takes over)?
bool level_uses_t32(const LevelArgs& a) {
  if (a.mode == MODE_UL || a.b < 32) return false;
  auto tiles = [&](int64_t T) { const int64_t m = (a.b + T - 1) / T; return a.merges * m * m; };
  static const double w6432 = [] { const char* e = std::getenv("TRINV_T6432_WAVES"); return e ? atof(e) : 3.0; }();
  if (pick_tile(tiles, a.b) != 32) return false;
  if (w6432 > 0 && a.b >= 64 && a.merges * ((a.b + 63) / 64) * ((a.b + 31) / 32) >= (int64_t)(w6432 * device_sms()))
    return false;
  return true;
}

cudaError_t launch_level_chain(const LevelArgs* ph, int nphase, int* counters, int cstride, cudaStream_t s,
                               int64_t* launches) {
  constexpr int BM = 32, BN = 32, WM = 2, WN = 2, STAGES = 4;
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  if (nphase <= 0 || nphase > CHAIN_MAXP) return cudaErrorInvalidValue;
  double fl = 0.0;
  for (int p = 0; p < nphase; ++p) fl += level_flops(ph[p]);
  ProfileScope prof(KIND_DMMA, fl, 0.0, s);
  static thread_local ChainArgs c;
  static thread_local ChainMaps maps;
  c.nphase = nphase;
  c.cstride = cstride;
  c.cnt = counters;
  c.tile0[0] = 0;
  for (int p = 0; p < nphase; ++p) {
    c.ph[p] = ph[p];
    const int64_t m = (ph[p].b + BM - 1) / BM;
    c.tile0[p + 1] = c.tile0[p] + (int32_t)(ph[p].merges * m * m);
    if (!encode_map(&maps.m[2 * p], ph[p].opA, 4, BM, false)) return cudaErrorInvalidValue;
    if (!encode_map(&maps.m[2 * p + 1], ph[p].opB, 4, BK, false)) return cudaErrorInvalidValue;
  }
  constexpr auto k = dmma_chain_kernel<BM, BN, WM, WN, STAGES>;
  set_smem_once<k>((int)C::SMEM);
  static const int occ = [] {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, C::kThreads, C::SMEM) != cudaSuccess) o = 1;
    return o < 1 ? 1 : o;
  }();
  static const int occ_cap = [] { const char* e = std::getenv("TRINV_CHAIN_OCC"); return e ? atoi(e) : 0; }();
  int64_t grid = (int64_t)(occ_cap > 0 && occ_cap < occ ? occ_cap : occ) * device_sms();
  if (grid > c.tile0[nphase]) grid = c.tile0[nphase];
  cudaError_t e = cudaMemsetAsync(counters, 0, (size_t)nphase * cstride * sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = launch_k(k, dim3((unsigned)grid), dim3(C::kThreads), C::SMEM, s, maps, c);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_level(const LevelArgs& a_in, cudaStream_t s, int64_t* launches) {
  LevelArgs a = a_in;
  ProfileScope prof(KIND_DMMA, level_flops(a), 0.0, s);
  a.kchunk = 0;
  // measured slower at every order (profiles/r02_splitk.txt): opt-in experiment, TRINV_SPLITK=1
  static const bool split_on = [] { const char* e = std::getenv("TRINV_SPLITK"); return e && atoi(e) != 0; }();
  static const int64_t split_t = [] { const char* e = std::getenv("TRINV_SPLITK_T"); return e ? atoll(e) : 64; }();
  static const int split_mode = [] { const char* e = std::getenv("TRINV_SPLITK"); return e ? atoi(e) : 0; }();
  int64_t kc = 0;
  int64_t units = split_on ? split_plan(a, kc, split_t == 32 ? 32 : 64) : 0;
  if (units > 0 && split_mode == 2) {  // fix-up mode needs the partial scratch for every unit
    const int64_t T = split_t == 32 ? 32 : 64;
    if (!a.partial || (size_t)units * T * T * sizeof(double) > LEVEL_PARTIAL_BYTES) units = 0;
    a.split_mode = 2;
  }
  if (units > 0) {
    const int64_t T = split_t == 32 ? 32 : 64;
    const int64_t tiles = a.merges * (a.b / T) * (a.b / T);
    cudaError_t e = cudaMemsetAsync(a.sync, 0, (size_t)(1 + tiles) * sizeof(int), s);
    if (e != cudaSuccess) return e;
    a.kchunk = (int32_t)kc;
    if (T == 32) return launch_level_cfg<32, 32, 2, 2, 4>(a, s, launches, units);
    return launch_level_cfg<64, 64, 2, 2, 4>(a, s, launches, units);
  }
  auto tiles = [&](int64_t T) {
    if (a.mode == MODE_UL) { const int64_t m = (a.n + T - 1) / T; return m * m; }
    const int64_t m = (a.b + T - 1) / T;
    return a.merges * m * m;
  };
  // TRINV_LEVEL_TILE = 32 / 64 / 128 forces the tile of the level launches (experiments)
  static const int64_t forced = [] { const char* e = std::getenv("TRINV_LEVEL_TILE"); return e ? atoll(e) : 0; }();
  int64_t t = pick_tile(tiles, a.mode == MODE_UL ? 128 : a.b);
  if (forced >= 32 && forced <= 128 && (a.mode == MODE_UL || forced <= a.b)) t = forced;
  // stream-K for the levels that fit in a few waves of 64x64 tiles (TRINV_SK=0: off;
  // TRINV_SK_TILE 32 / 64, TRINV_SK_CPS CTAs per SM, TRINV_SK_WMIN minimum iterations per CTA,
  // TRINV_SK_WAVES: levels with fewer 64x64 tiles than this many per SM)
  const bool sk_on = level_sk_enabled();
  static const int sk_tile = [] { const char* e = std::getenv("TRINV_SK_TILE"); return e ? atoi(e) : 64; }();
  static const int sk_cps = [] { const char* e = std::getenv("TRINV_SK_CPS"); return e ? atoi(e) : 2; }();
  static const int64_t sk_bmin = [] { const char* e = std::getenv("TRINV_SK_BMIN"); return e ? atoll(e) : 256; }();
  static const int sk_wmin = [] { const char* e = std::getenv("TRINV_SK_WMIN"); return e ? atoi(e) : 8; }();
  static const double sk_waves = [] { const char* e = std::getenv("TRINV_SK_WAVES"); return e ? atof(e) : 8.0; }();
  if (sk_on && a.sk_flags && a.sk_partial && a.mode != MODE_UL && t < 128 && forced == 0 && a.b >= sk_bmin &&
      a.b >= 128 && tiles(64) < (int64_t)(sk_waves * device_sms())) {
    if (sk_tile == 128) return launch_level_sk_cfg<128, 128, 2, 4, 5, 1>(a, 1, sk_wmin, s, launches);
    if (sk_tile == 12864) return launch_level_sk_cfg<128, 64, 4, 2, 4, 1>(a, 1, sk_wmin, s, launches);
    if (sk_tile == 6448) return launch_level_sk_cfg<64, 64, 2, 4, 4, 1>(a, 1, sk_wmin, s, launches);
    return launch_level_sk_cfg<64, 64, 2, 2, 4, 2>(a, sk_cps, sk_wmin, s, launches);
  }
  if (forced == 6432 && a.mode != MODE_UL && a.b >= 64) return launch_level_cfg<64, 32, 2, 2, 4>(a, s, launches);
  if (forced == 3264 && a.mode != MODE_UL && a.b >= 64) return launch_level_cfg<32, 64, 2, 2, 4>(a, s, launches);
  if (forced == 6432 || forced == 3264) t = 32;
  // 64x32 tiles (2x2 warps of 32x16: 6 fragment loads per 8 DMMA instead of 4 per 4) for the
  // levels that would run 32x32 tiles but still have >= TRINV_T6432_WAVES (default 3) waves of
  // 64x32 tiles: n = 2048's top level 88.8 -> 80.8 us (profiles/r02_tile_shapes.txt)
  static const double w6432 = [] { const char* e = std::getenv("TRINV_T6432_WAVES"); return e ? atof(e) : 3.0; }();
  if (t == 32 && forced == 0 && w6432 > 0 && a.mode != MODE_UL && a.b >= 64 &&
      a.merges * ((a.b + 63) / 64) * ((a.b + 31) / 32) >= (int64_t)(w6432 * device_sms()))
    return launch_level_cfg<64, 32, 2, 2, 4>(a, s, launches);
  if (t >= 128) return launch_level_cfg<128, 128, 2, 4, 5>(a, s, launches);
  if (t >= 64) return launch_level_cfg<64, 64, 2, 2, 4>(a, s, launches);
  // 32x32 tiles: 2x2 consumer warps of 16x16.  One warp of 32x32, 1x2 warps of 32x16 and 6
  // stages were measured slower or equal (profiles/r02_t32_layouts.txt).
  return launch_level_cfg<32, 32, 2, 2, 4>(a, s, launches);
}

// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES>
static cudaError_t launch_gemm_cfg(const GemmArgs& a, cudaStream_t s, int64_t* launches) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES>;
  CUtensorMap mA, mB;
  const uint64_t dA[3] = {(uint64_t)a.K, (uint64_t)a.M, (uint64_t)a.batch};
  const uint64_t sAb[2] = {(uint64_t)a.lda * 8, (uint64_t)(a.batch > 1 ? a.sA : a.M * a.lda) * 8};
  const uint32_t bA[3] = {4, (uint32_t)BM, 1};
  const uint64_t dB[3] = {(uint64_t)a.N, (uint64_t)a.K, (uint64_t)a.batch};
  const uint64_t sBb[2] = {(uint64_t)a.ldb * 8, (uint64_t)(a.batch > 1 ? a.sB : a.K * a.ldb) * 8};
  const uint32_t bB[3] = {4, (uint32_t)BK, 1};
  if (!encode_map_nd(&mA, a.A, 3, dA, sAb, bA)) return cudaErrorInvalidValue;
  if (!encode_map_nd(&mB, a.B, 3, dB, sBb, bB)) return cudaErrorInvalidValue;
  const int64_t tiles = a.batch * ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  if (tiles <= 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  constexpr auto k = dmma_gemm_kernel<BM, BN, WM, WN, STAGES>;
  set_smem_once<k>((int)C::SMEM);
  const cudaError_t e = launch_k(k, dim3((unsigned)tiles), dim3(C::kThreads), C::SMEM, s, mA, mB, a);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

double gemm_flops(const GemmArgs& a) {
  // 2 flops per multiply-add with a structurally non-zero element of the triangular operand
  const double M = (double)a.M, N = (double)a.N, K = (double)a.K;
  auto tri_sum = [](double rows, double K) {  // sum_{i < rows} min(i + 1, K)
    const double full = rows < K ? rows : K;
    return full * (full + 1) / 2 + (rows - full) * K;
  };
  double f;
  if (a.triA == TRI_LOWER) f = 2 * N * tri_sum(M, K);
  else if (a.triA == TRI_UPPER) f = 2 * N * (M * K - tri_sum(M, K) + (M < K ? M : K));
  else if (a.triB == TRI_LOWER) f = 2 * M * (N * K - tri_sum(N, K) + (N < K ? N : K));
  else if (a.triB == TRI_UPPER) f = 2 * M * tri_sum(N, K);
  else f = 2 * M * N * K;
  return f * a.batch;
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.M <= 0 || a.N <= 0 || a.batch <= 0) return cudaSuccess;
  ProfileScope prof(KIND_DMMA, gemm_flops(a), 0.0, s);
  // tiles per SM required before a larger tile is taken (experiments: TRINV_GEMM_WAVES)
  static const double waves = [] { const char* e = std::getenv("TRINV_GEMM_WAVES"); return e ? std::atof(e) : 2.0; }();
  auto tiles = [&](int64_t T) { return a.batch * ((a.M + T - 1) / T) * ((a.N + T - 1) / T); };
  // TRINV_GEMM_W128: waves of 128x128 tiles required before they are preferred to 64x64
  // (default 32, as for the level launches: config 4 162.5 -> 161.2 ms, configs 2 / 3
  // unchanged; profiles/r02_pdl.txt)
  static const double w128 = [] { const char* e = std::getenv("TRINV_GEMM_W128"); return e ? atof(e) : 32.0; }();
  int64_t t = 32;
  if (tiles(128) >= (int64_t)(w128 * device_sms())) t = 128;
  else if (tiles(64) >= (int64_t)(waves * device_sms())) t = 64;
  if (t >= 128) return launch_gemm_cfg<128, 128, 2, 4, 5>(a, s, launches);
  if (t >= 64) return launch_gemm_cfg<64, 64, 2, 2, 4>(a, s, launches);
  return launch_gemm_cfg<32, 32, 2, 2, 4>(a, s, launches);
}

// ---------------------------------------------------------------------------
// rows over blockIdx.y (grid-strided), columns over blockIdx.x / threads: no division per entry
__global__ void zero_2d_kernel(double* p, int64_t ld, int64_t rows, int64_t cols) {
  pdl_trigger_early();
  pdl_wait();
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    double* r = p + i * ld;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cols; j += (int64_t)gridDim.x * blockDim.x)
      r[j] = 0.0;
  }
}

// C = alpha A + beta B (rows x cols, row-major, any leading dimensions; C may alias A or B exactly)
__global__ void geam_kernel(int64_t rows, int64_t cols, double alpha, const double* A, int64_t lda, double beta,
                            const double* B, int64_t ldb, double* C, int64_t ldc) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    C[i * ldc + j] = alpha * A[i * lda + j] + beta * B[i * ldb + j];
  }
}

cudaError_t launch_geam(int64_t rows, int64_t cols, double alpha, const double* A, int64_t lda, double beta,
                        const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s, int64_t* launches) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t total = rows * cols;
  const int64_t blocks = (total + 255) / 256;
  const int grid = (int)(blocks < (int64_t)device_sms() * 16 ? blocks : (int64_t)device_sms() * 16);
  prefer_l1_once<geam_kernel>();
  geam_kernel<<<grid, 256, 0, s>>>(rows, cols, alpha, A, lda, beta, B, ldb, C, ldc);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// 2-D copy (device to device) with 16-byte accesses when both rows are 16-byte aligned:
// the staging copies of inv_general / the odd-layout paths run at copy bandwidth (the
// runtime's pitched copy measured 2.0 TB/s on the 2 GB operand of config 5).
__global__ void copy_2d_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                               int64_t rows, int64_t cols, bool vec) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const double* a = src + i * lds;
    double* b = dst + i * ldd;
    if (vec) {
      const int64_t c2 = cols / 2;
      for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c2; j += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<double2*>(b)[j] = reinterpret_cast<const double2*>(a)[j];
      if ((cols & 1) && blockIdx.x == 0 && threadIdx.x == 0) b[cols - 1] = a[cols - 1];
    } else {
      for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cols; j += (int64_t)gridDim.x * blockDim.x)
        b[j] = a[j];
    }
  }
}
cudaError_t launch_copy_2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                           cudaStream_t s, int64_t* launches) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const bool vec = ((lds | ldd) & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t per_row = vec ? (cols / 2 + 255) / 256 : (cols + 255) / 256;
  const unsigned gx = (unsigned)(per_row < 1 ? 1 : (per_row < 8 ? per_row : 8));
  const unsigned gy = (unsigned)(rows < 65535 ? rows : 65535);
  prefer_l1_once<copy_2d_kernel>();
  copy_2d_kernel<<<dim3(gx, gy), 256, 0, s>>>(src, lds, dst, ldd, rows, cols, vec);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_zero_2d(double* p, int64_t ld, int64_t rows, int64_t cols, cudaStream_t s, int64_t* launches) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t gx = std::min<int64_t>((cols + 255) / 256, 64);
  const int64_t gy = std::min<int64_t>(rows, std::max<int64_t>(1, (int64_t)device_sms() * 16 / gx));
  prefer_l1_once<zero_2d_kernel>();
  const cudaError_t e = launch_k(zero_2d_kernel, dim3((unsigned)gx, (unsigned)gy), dim3(256), 0, s, p, ld, rows, cols);
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace trinv
