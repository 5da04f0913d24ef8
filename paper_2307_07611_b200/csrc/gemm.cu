// gemm.cu — the off-diagonal products of the recursive split on the FP64
// tensor cores (DESIGN.md §Kernels "K_trmm").
//
// One launch covers every merge of one recursion level (COMBRIT with
// beta = 2, Alg. 1: the n/(2b) merges of a level are independent,
// P:499-500).  Per merge at offset s with halves b (first) and r (second):
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
// TMA (cp.async.bulk.tensor.2d) from a producer warp through full/empty
// mbarriers; WM x WN consumer warps issue mma.sync.m8n8k4.f64 (DMMA.8x8x4).
// Shared-memory layouts are chosen for the m8n8k4 fragments, whose 64-bit loads
// are served per half-warp (16 lanes = 128 B must cover the 32 banks once):
// A tile = BK/4 boxes of [BM rows][4 k] (32-byte rows), B tile = BN/4 boxes of
// [BK rows][4 n]; each half-warp fragment load then reads 128 contiguous bytes.
// Out-of-range rows / columns (ragged last merge, n not a multiple of the
// tile) are zero-filled by TMA and clipped at the store.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

// Shared-memory layout variants (template parameter LAY):
//   LAY 0: A = one 16-wide box per stage with 128-byte swizzle, B = BN/8 boxes of 8 columns
//   LAY 1: A = BK/4 boxes of 4 columns, B = BN/4 boxes of 4 columns (half-warp conflict-free)
//   LAY 2: A = BK/4 boxes of 4 columns, B = BN/8 boxes of 8 columns
struct TileCoord {
  int64_t a_row, a_col;  // A-operand: rows a_row.., columns a_col + k
  int64_t b_row, b_col;  // B-operand: rows b_row + k, columns b_col..
  int64_t o_row, o_col;  // output tile origin
  int64_t m_row, m_col;  // mirror tile origin (rows BN x cols BM), if any
  int64_t k_begin, k_end;
  bool valid, mirror;
};

template <int BM, int BN, int BK>
__device__ __forceinline__ TileCoord map_tile(const LevelArgs& p, int64_t t) {
  TileCoord c{};
  const int64_t b = p.b, n = p.n, merges = p.merges;
  const int64_t TMmax = (b + BM - 1) / BM, TNmax = (b + BN - 1) / BN;
  int64_t g = 0, I = 0, J = 0;
  c.valid = true;
  c.mirror = false;
  switch (p.mode) {
    case MODE_LOWER_1: {  // longest K first: J ascending
      J = t / (merges * TMmax);
      const int64_t rem = t % (merges * TMmax);
      g = rem / TMmax; I = rem % TMmax;
    } break;
    case MODE_LOWER_2: {  // I descending
      I = TMmax - 1 - t / (merges * TNmax);
      const int64_t rem = t % (merges * TNmax);
      g = rem / TNmax; J = rem % TNmax;
    } break;
    case MODE_UPPER_1: {  // I ascending
      I = t / (merges * TNmax);
      const int64_t rem = t % (merges * TNmax);
      g = rem / TNmax; J = rem % TNmax;
    } break;
    case MODE_UPPER_2: {  // J descending
      J = TNmax - 1 - t / (merges * TMmax);
      const int64_t rem = t % (merges * TMmax);
      g = rem / TMmax; I = rem % TMmax;
    } break;
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
  switch (p.mode) {
    case MODE_LOWER_1:
      c.valid = I * BM < r;
      c.a_row = s + b + I * BM; c.a_col = s;
      c.b_row = s; c.b_col = s + J * BN;
      c.o_row = g * b + I * BM; c.o_col = J * BN;
      c.k_begin = J * BN; c.k_end = b;
      break;
    case MODE_LOWER_2: {
      c.valid = I * BM < r;
      c.a_row = s + b + I * BM; c.a_col = s + b;
      c.b_row = g * b; c.b_col = J * BN;
      c.o_row = s + b + I * BM; c.o_col = s + J * BN;
      c.mirror = true; c.m_row = s + J * BN; c.m_col = s + b + I * BM;
      c.k_begin = 0; c.k_end = (I + 1) * BM < r ? (I + 1) * BM : r;
    } break;
    case MODE_UPPER_1:
      c.valid = J * BN < r;
      c.a_row = s + I * BM; c.a_col = s;
      c.b_row = s; c.b_col = s + b + J * BN;
      c.o_row = g * b + I * BM; c.o_col = J * BN;
      c.k_begin = I * BM; c.k_end = b;
      break;
    case MODE_UPPER_2:
      c.valid = J * BN < r;
      c.a_row = g * b + I * BM; c.a_col = 0;
      c.b_row = s + b; c.b_col = s + b + J * BN;
      c.o_row = s + I * BM; c.o_col = s + b + J * BN;
      c.mirror = true; c.m_row = s + b + J * BN; c.m_col = s + I * BM;
      c.k_begin = 0; c.k_end = (J + 1) * BN < r ? (J + 1) * BN : r;
      break;
    default:
      c.a_row = I * BM; c.a_col = 0;
      c.b_row = 0; c.b_col = J * BN;
      c.o_row = I * BM; c.o_col = J * BN;
      c.k_begin = (I * BM > J * BN) ? I * BM : J * BN; c.k_end = n;
      break;
  }
  return c;
}

template <int BM, int BN, int WM, int WN, int STAGES, int BK = 16, int LAY = 1>
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

template <int BM, int BN, int WM, int WN, int STAGES, int BK, int LAY>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES, BK, LAY>::kThreads, 1)
    dmma_level_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const LevelArgs p) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES, BK, LAY>;
  constexpr int BW = (LAY == 1) ? 4 : 8;  // B box width (columns)
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  double* sA = reinterpret_cast<double*>(base);                              // [STAGES][BK/4][BM][4]
  double* sB = reinterpret_cast<double*>(base + (size_t)STAGES * C::A_BYTES);  // [STAGES][BN/4][BK][4]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const TileCoord tc = map_tile<BM, BN, BK>(p, blockIdx.x);
  if (!tc.valid) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = (tc.k_end - tc.k_begin + BK - 1) / BK;

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
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      for (int64_t kt = 0; kt < nk; ++kt) {
        const int s = (int)(kt % STAGES);
        const int64_t use = kt / STAGES;
        if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int64_t k = tc.k_begin + kt * BK;
        double* sa = sA + (size_t)s * BM * BK;
        if (LAY == 0) {
#pragma unroll
          for (int kb = 0; kb < BK / 16; ++kb)
            tma_load_2d(sa + kb * BM * 16, &mapA, (int32_t)(tc.a_col + k + 16 * kb), (int32_t)tc.a_row, &full[s]);
        } else {
#pragma unroll
          for (int kb = 0; kb < BK / 4; ++kb)
            tma_load_2d(sa + kb * BM * 4, &mapA, (int32_t)(tc.a_col + k + 4 * kb), (int32_t)tc.a_row, &full[s]);
        }
        double* sb = sB + (size_t)s * BK * BN;
#pragma unroll
        for (int nb = 0; nb < BN / BW; ++nb)
          tma_load_2d(sb + nb * BK * BW, &mapB, (int32_t)(tc.b_col + nb * BW), (int32_t)(tc.b_row + k), &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Mirror-tile zero fill (row a7): BN rows x BM columns of the opposite triangle.
  if (tc.mirror) {
    const int ctid = threadIdx.x;
    constexpr int PAIRS = BM / 2;
    for (int e = ctid; e < BN * PAIRS; e += C::kConsumerWarps * 32) {
      const int64_t row = tc.m_row + e / PAIRS, col = tc.m_col + 2 * (e % PAIRS);
      if (row < p.n) {
        double* q = p.mir + row * p.ldm + col;
        if (col + 1 < p.n) *reinterpret_cast<double2*>(q) = make_double2(0.0, 0.0);
        else if (col < p.n) *q = 0.0;
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
  // per-lane fragment offsets (doubles); A[row][k], B[k][col] with k = kk*4 + lc
  const int a_base = (wm * C::WTM + lr) * 4 + lc;                    // LAY 1/2: box k/4 of [BM][4]
  const int b_col = wn * C::WTN + lr;                                  // + ni*8
  const int b_base = (b_col / BW) * BK * BW + lc * BW + (b_col % BW);  // box col/BW of [BK][BW]
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int s = (int)(kt % STAGES);
    mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
    const double* a_st = sA + (size_t)s * BM * BK;
    const double* b_st = sB + (size_t)s * BK * BN + b_base;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi) {
        if (LAY == 0) {  // 16-wide boxes with 128-byte swizzle: chunk (k/2) ^ (row % 8)
          const int row = wm * C::WTM + mi * 8 + lr;
          const int kc = (kk & 3) * 4 + lc;
          const int off = (kk >> 2) * BM * 16 + row * 16 + ((((kc >> 1) ^ (row & 7)) << 1) | (kc & 1));
          af[mi] = a_st[off];
        } else {
          af[mi] = a_st[a_base + kk * BM * 4 + mi * 32];
        }
      }
#pragma unroll
      for (int ni = 0; ni < C::FN; ++ni) bf[ni] = b_st[kk * 4 * BW + (ni * 8 / BW) * BK * BW];
#pragma unroll
      for (int mi = 0; mi < C::FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::FN; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue: alpha * acc -> out (clipped) ----------------
#pragma unroll
  for (int mi = 0; mi < C::FM; ++mi) {
    const int64_t row = tc.o_row + wm * C::WTM + mi * 8 + lr;
    if (row >= p.out_rows) continue;
    double* orow = p.out + row * p.ldo;
#pragma unroll
    for (int ni = 0; ni < C::FN; ++ni) {
      const int64_t col = tc.o_col + wn * C::WTN + ni * 8 + 2 * lc;
      const double v0 = p.alpha * acc[mi][ni][0], v1 = p.alpha * acc[mi][ni][1];
      if (col + 1 < p.out_cols) *reinterpret_cast<double2*>(orow + col) = make_double2(v0, v1);
      else if (col < p.out_cols) orow[col] = v0;
    }
  }
}

// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES, int BK = 16, int LAY = 1>
static cudaError_t launch_cfg(const LevelArgs& a, cudaStream_t s, int64_t* launches) {
  using C = GemmCfg<BM, BN, WM, WN, STAGES, BK, LAY>;
  constexpr int BW = (LAY == 1) ? 4 : 8;
  CUtensorMap mA, mB;
  if (!encode_map(&mA, a.opA, LAY == 0 ? 16 : 4, BM, LAY == 0)) return cudaErrorInvalidValue;
  if (!encode_map(&mB, a.opB, BW, BK, false)) return cudaErrorInvalidValue;
  int64_t tiles;
  if (a.mode == MODE_UL) {
    const int64_t T = (a.n + BM - 1) / BM;
    tiles = T * T;
  } else {
    tiles = a.merges * ((a.b + BM - 1) / BM) * ((a.b + BN - 1) / BN);
  }
  if (tiles <= 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  constexpr auto k = dmma_level_kernel<BM, BN, WM, WN, STAGES, BK, LAY>;
  set_smem_once<k>((int)C::SMEM);
  k<<<(unsigned)tiles, C::kThreads, C::SMEM, s>>>(mA, mB, a);
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

cudaError_t launch_level(const LevelArgs& a, cudaStream_t s, int64_t* launches) {
  ProfileScope prof(KIND_DMMA, level_flops(a), 0.0, s);
  // Tile size per level: the largest of 128 / 64 / 32 (not above b) that still
  // gives at least two CTAs per SM; mid-size levels otherwise leave SMs idle
  // behind a few long triangular tiles (profiles/r01_sweep_n.txt).
  const int sms = device_sms();
  auto tiles = [&](int64_t T) {
    if (a.mode == MODE_UL) { const int64_t m = (a.n + T - 1) / T; return m * m; }
    const int64_t m = (a.b + T - 1) / T;
    return a.merges * m * m;
  };
  int64_t t = 32;
  for (int64_t T : {128, 64}) {
    if ((a.mode == MODE_UL || T <= a.b) && tiles(T) >= 2 * sms) { t = T; break; }
  }
  if (a.mode != MODE_UL && t > a.b) t = a.b;
  if (t >= 128) {
    static const int variant = [] {
      const char* e = getenv("TRINV_GEMM_VARIANT");
      return e ? atoi(e) : 0;
    }();
    // LAY 1 measured best on B200 (config 3: 93.8% vs 92.7% for the swizzled LAY 0,
    // profiles/r01_gemm_variants.txt); the others stay selectable for tuning.
    switch (variant) {
      case 2: return launch_cfg<128, 128, 2, 4, 5, 16, 0>(a, s, launches);
      case 3: return launch_cfg<128, 128, 2, 4, 5, 16, 2>(a, s, launches);
      default: return launch_cfg<128, 128, 2, 4, 5, 16, 1>(a, s, launches);
    }
  }
  if (t >= 64) return launch_cfg<64, 64, 2, 2, 4>(a, s, launches);
  return launch_cfg<32, 32, 2, 2, 4>(a, s, launches);
}

}  // namespace trinv
