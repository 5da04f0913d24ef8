// leaf.cu — 32-wide triangular inverses in shared memory (SURVEY §8(a) rows
// a1, a2, a3; DESIGN.md §Kernels "K_leaf32").
//
// One warp owns one matrix T (n <= 32).  Lane j computes column j of
// X = T^{-1} in 32 FP64 registers by the bordering recurrence of the proof of
// Thm 1, [R v; 0 1]^{-1} = [S  -S v; 0 1], written in its
// right-looking form: solve T x = e_j column-wise,
//     x_k = r_k * acc_k,  acc_i -= T_ik x_k  (i beyond k),   r_k = 1/T_kk,
// which is CRIT (Alg. 3) with the non-unit diagonal handled by
// the reciprocal of R = DT (readings C1/C2/C4).  Entries of
// different columns are independent: the 32 lanes never
// exchange data; T is read from shared memory as warp-wide broadcasts.
//
// HBM staging (a3): every warp runs its own NS-deep ring of smem slots filled
// by 2-D TMA (cp.async.bulk.tensor) with only the referenced triangle, each
// slot completing on its own mbarrier (see leaf32_tma_kernel).  Orders below
// 32 and odd layouts use the plain-load kernel (leaf_plain_kernel).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <utility>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

constexpr int LEAF = 32;

// Zero-diagonal report, "min over non-zero" on a single accumulator.
__device__ __forceinline__ void info_min_nonzero(int32_t* p, int32_t v) {
  int32_t old = *reinterpret_cast<volatile int32_t*>(p);
  while (old == 0 || v < old) {
    int32_t prev = atomicCAS(p, old, v);
    if (prev == old) break;
    old = prev;
  }
}

// T: 32x32 row-major slot (row stride 32).  On return x[i] = X(i, lane).
template <bool UPPER>
__device__ __forceinline__ void leaf_compute(double* T, int n, int unit, int lane, double (&x)[LEAF],
                                             bool& singular, int& first_zero) {
  double d = T[lane * (LEAF + 1)];
  const bool zero = (!unit) && lane < n && d == 0.0;
  const unsigned zmask = __ballot_sync(0xffffffffu, zero);
  singular = zmask != 0;
  first_zero = singular ? __ffs(zmask) - 1 : -1;
  const double r = unit ? 1.0 : 1.0 / d;  // IEEE division: X_jj == 1/T_jj bitwise (C4)
  __syncwarp();
  T[lane * (LEAF + 1)] = r;  // the diagonal slot now holds r_i (broadcast below)
  __syncwarp();
#pragma unroll
  for (int i = 0; i < LEAF; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
  if (!UPPER) {
#pragma unroll
    for (int k = 0; k < LEAF; ++k) {
      if (k < n) {
        const double xk = x[k] * T[k * (LEAF + 1)];
        x[k] = xk;
#pragma unroll
        for (int i = k + 1; i < LEAF; ++i) x[i] = fma(-T[i * LEAF + k], xk, x[i]);
      }
    }
  } else {
#pragma unroll
    for (int k = LEAF - 1; k >= 0; --k) {
      if (k < n) {
        const double xk = x[k] * T[k * (LEAF + 1)];
        x[k] = xk;
#pragma unroll
        for (int i = 0; i < k; ++i) x[i] = fma(-T[i * LEAF + k], xk, x[i]);
      }
    }
  }
}

__device__ __forceinline__ void leaf_report(const LeafArgs& a, int64_t b, int lane, bool singular,
                                            int first_zero) {
  if (a.info_mode == 1) {
    if (lane == 0) a.info[b] = singular ? first_zero + 1 : 0;
  } else if (a.info_mode == 2 && singular && lane == 0) {
    info_min_nonzero(a.info, static_cast<int32_t>(a.info_off + b * a.info_stride + first_zero + 1));
  }
}

// ---------------------------------------------------------------------------
// Triangle-only staging (n = 32).  Each slot holds the referenced triangle as 32/BR
// bands of BR rows, each loaded by one 2-D TMA box (cp.async.bulk.tensor over a 3-D view
// [batch][32 rows][32 cols] of the input): lower band b = rows BR b .. BR b + BR-1 x
// cols 0 .. BR (b+1) - 1; upper band b = the same rows x cols BR b .. 31.  BR = 16 (the
// default): 768 doubles (6 KiB) per matrix in two TMA instructions; BR = 8 / 4 read
// 640 / 576 doubles (4.5 KiB, 9% above the 528 referenced) in 4 / 8 instructions but
// measured 4% / 8% slower (profiles/r01_leaf_variants.txt).  The inverse leaves the
// registers through coalesced 256-byte row stores, so a slot is free again as soon as
// the warp has read it; the next load is issued before the stores.
//
// The upper case runs the lower recurrence on T' = J U J (J = index reversal,
// T'_ik = U_{31-i,31-k}): X' = J U^{-1} J, lane j then holds column 31-j of
// U^{-1}.  One straight-line code path, no per-step branches.
template <int BR>
struct Band {
  static constexpr int NBAND = 32 / BR;
  static constexpr int SLOT = BR * BR * NBAND * (NBAND + 1) / 2;  // doubles per slot
  // lower: band b = rows [BR b, BR b + BR), cols [0, BR (b + 1))
  static __host__ __device__ constexpr int loff(int b) { return BR * BR * b * (b + 1) / 2; }
  static __host__ __device__ constexpr int lidx(int i, int k) {
    return loff(i / BR) + (i - BR * (i / BR)) * BR * (i / BR + 1) + k;
  }
  // upper: band b = rows [BR b, BR b + BR), cols [BR b, 32)
  static __host__ __device__ constexpr int uoff(int b) { return BR * (32 * b - BR * b * (b - 1) / 2); }
  static __host__ __device__ constexpr int uidx(int i, int k) {
    return uoff(i / BR) + (i - BR * (i / BR)) * (32 - BR * (i / BR)) + (k - BR * (i / BR));
  }
};
static_assert(Band<16>::SLOT == 768 && Band<8>::SLOT == 640 && Band<4>::SLOT == 576, "band slots");
static_assert(Band<4>::uoff(8) == 576 && Band<8>::uoff(4) == 640, "upper band offsets");
template <int BR>
struct BandMaps {
  CUtensorMap m[Band<BR>::NBAND];  // m[w - 1]: box BR rows x BR w columns
};

template <bool UPPER, int BR>
__device__ __forceinline__ double2 tri_pair(const double* T, int i, int k) {  // (T'_ik, T'_i,k+1), k even
  if (!UPPER) return *reinterpret_cast<const double2*>(T + Band<BR>::lidx(i, k));
  const double2 v = *reinterpret_cast<const double2*>(T + Band<BR>::uidx(31 - i, 30 - k));  // U_{r,c}, U_{r,c+1}
  return make_double2(v.y, v.x);
}
template <bool UPPER, int BR>
__device__ __forceinline__ double tri_sub(const double* T, int k) {  // T'_{k+1,k}, k even
  return UPPER ? T[Band<BR>::uidx(30 - k, 31 - k)] : T[Band<BR>::lidx(k + 1, k)];
}
template <bool UPPER, int BR>
__device__ __forceinline__ double tri_diag(const double* T, int i) {  // T_ii, original index
  return UPPER ? T[Band<BR>::uidx(i, i)] : T[Band<BR>::lidx(i, i)];
}

template <bool UPPER, int BR, int K>
__device__ __forceinline__ void leaf32_step(const double* T, const double* rr, double (&x)[LEAF]) {
  const double2 r = *reinterpret_cast<const double2*>(rr + K);
  const double xk = x[K] * r.x;
  x[K] = xk;
  x[K + 1] = fma(-tri_sub<UPPER, BR>(T, K), xk, x[K + 1]);
  const double xk1 = x[K + 1] * r.y;
  x[K + 1] = xk1;
#pragma unroll
  for (int i = K + 2; i < LEAF; ++i) {
    const double2 t = tri_pair<UPPER, BR>(T, i, K);
    x[i] = fma(-t.x, xk, x[i]);
    x[i] = fma(-t.y, xk1, x[i]);
  }
}
template <bool UPPER, int BR, int... P>
__device__ __forceinline__ void leaf32_steps(const double* T, const double* rr, double (&x)[LEAF],
                                             std::integer_sequence<int, P...>) {
  (leaf32_step<UPPER, BR, 2 * P>(T, rr, x), ...);
}

template <bool UPPER, int BR>
__device__ __forceinline__ void leaf32_compute(const double* T, double* rr, int unit, int lane, double (&x)[LEAF],
                                               bool& singular, int& first_zero) {
  const double d = tri_diag<UPPER, BR>(T, lane);
  const bool zero = (!unit) && d == 0.0;
  const unsigned zmask = __ballot_sync(0xffffffffu, zero);
  singular = zmask != 0;
  first_zero = singular ? __ffs(zmask) - 1 : -1;
  rr[UPPER ? LEAF - 1 - lane : lane] = unit ? 1.0 : 1.0 / d;  // r'_k = rr[k] in T' order
  __syncwarp();
#pragma unroll
  for (int i = 0; i < LEAF; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
  // pairs (k, k+1): x_k = r_k acc_k; acc_{k+1} -= T'_{k+1,k} x_k; x_{k+1} = r_{k+1} acc_{k+1};
  // acc_i -= T'_ik x_k + T'_{i,k+1} x_{k+1} (i >= k+2), one 16-byte broadcast per row.
  // Compile-time step indices (template expansion) keep x[] in registers.
  leaf32_steps<UPPER, BR>(T, rr, x, std::make_integer_sequence<int, LEAF / 2>{});
}

// BULK (opt-in TRINV_LEAF_BULK=1..3, measured no faster: profiles/r02_leaf_bulk.txt): the inverse
// leaves through an 8 KiB shared-memory staging buffer per warp and one cp.async.bulk shared ->
// global copy per matrix (contiguous 32x32 outputs only) instead of 32 row stores from registers.
template <bool UPPER, int WARPS, int NS, int BR, bool BULK = false>
__global__ void __launch_bounds__(WARPS * 32, 1)
    leaf32_tma_kernel(const __grid_constant__ BandMaps<BR> maps, const LeafArgs a) {
  using BD = Band<BR>;
  constexpr int SLOT = BD::SLOT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slots = reinterpret_cast<double*>(smem_raw) + (size_t)warp * NS * SLOT;
  double* rr = reinterpret_cast<double*>(smem_raw) + (size_t)WARPS * NS * SLOT + warp * LEAF;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_raw + ((size_t)WARPS * NS * SLOT + WARPS * LEAF) * 8) + warp * NS;
  constexpr size_t STAGE_OFF = (((size_t)WARPS * NS * SLOT + WARPS * LEAF) * 8 + WARPS * NS * 8 + 127) & ~size_t(127);
  double* stage = reinterpret_cast<double*>(smem_raw + STAGE_OFF) + (size_t)warp * LEAF * LEAF;

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= a.batch) return;
  const int64_t count = (a.batch - gw + TW - 1) / TW;

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (lane == 0 && warp == 0)
    for (int w = 0; w < BD::NBAND; ++w) tma_prefetch_desc(&maps.m[w]);
  __syncwarp();

  auto issue_load = [&](int64_t t) {  // lane 0 only
    const int b = (int)(gw + t * TW);
    double* slot = slots + (t % NS) * SLOT;
    uint64_t* bar = &bars[t % NS];
    mbar_arrive_expect_tx(bar, SLOT * 8);
#pragma unroll
    for (int g = 0; g < BD::NBAND; ++g) {
      if (!UPPER) tma_load_3d(slot + BD::loff(g), &maps.m[g], 0, BR * g, b, bar);  // cols 0 .. BR (g+1) - 1
      else tma_load_3d(slot + BD::uoff(g), &maps.m[BD::NBAND - 1 - g], BR * g, BR * g, b, bar);  // cols BR g .. 31
    }
  };

  if (lane == 0)
    for (int64_t t = 0; t < NS && t < count; ++t) issue_load(t);

  for (int64_t t = 0; t < count; ++t) {
    const int64_t b = gw + t * TW;
    double* slot = slots + (t % NS) * SLOT;
    mbar_wait(&bars[t % NS], (uint32_t)((t / NS) & 1));

    double x[LEAF];
    bool singular;
    int first_zero;
    leaf32_compute<UPPER, BR>(slot, rr, a.unit, lane, x, singular, first_zero);
    __syncwarp();  // every lane has finished reading the slot and rr
    if (t + NS < count && lane == 0) {
      fence_proxy_async_smem();
      issue_load(t + NS);
    }
    double* dst = a.X + b * a.sX;
    const int col = UPPER ? LEAF - 1 - lane : lane;
    if constexpr (BULK) {
      if (t > 0) {  // the previous matrix's bulk store has read the staging buffer
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
#pragma unroll
      for (int i = 0; i < LEAF; ++i) {
        const int row = UPPER ? LEAF - 1 - i : i;
        stage[row * LEAF + col] = (i < lane) ? 0.0 : x[i];
      }
      fence_proxy_async_smem();  // generic smem writes -> the bulk copy's reads
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(dst, stage, LEAF * LEAF * 8);
        bulk_commit();
      }
    } else {
#pragma unroll
      for (int i = 0; i < LEAF; ++i) {
        const int row = UPPER ? LEAF - 1 - i : i;
        dst[(int64_t)row * a.ldx + col] = (i < lane) ? 0.0 : x[i];
      }
    }
    leaf_report(a, b, lane, singular, first_zero);
  }
  if constexpr (BULK) {
    if (lane == 0) bulk_wait<0>();  // the last store complete before the CTA's shared memory goes
  }
}

// ---------------------------------------------------------------------------
// n = 32, two matrices per warp (opt-in TRINV_LEAF32=pair, measured slower): half-warp h inverts matrix
// 2p + h, lane c computes columns c and c + 16 of its inverse by the same right-looking
// recurrence (CRIT P:568-581), column c in x[32], column c + 16 in y[16] (its
// rows 16..31; its first 16 steps multiply by x_k = 0 and are skipped, an exact no-op).
// Why: the one-warp-per-matrix kernel above is shared-memory (LSU) bound — every 16-byte
// broadcast of T costs two wavefronts (one per half-warp), both serving the same matrix.
// Here the two half-warps read the same offset of their own matrices' slots, so each
// wavefront serves a different matrix: half the LSU wavefronts per matrix, and 37% fewer
// FP64 instructions (no work on column c + 16's structural zeros).  Stores: one 128-byte
// line per half-warp per instruction (PSTORE: whole 256-byte rows after one shuffle per row).
// Staging as above (16-row TMA bands, 768 doubles per matrix), NS pair-slots per warp, one
// mbarrier per pair-slot.  Measured: l1tex 96% -> 64%, LSU wavefronts 546 -> 292 per matrix,
// FP64 pipe 42% -> 30%, same DRAM bytes, but 0.333 ms against 0.303 ms (the band kernel is
// at 0.95 of the copy bandwidth on the bytes DRAM moves: the LSU was not what bounds it).
template <bool UPPER, int BR, int K>
__device__ __forceinline__ void leaf32p_step(const double* T, const double* rr, double (&x)[LEAF], double (&y)[16]) {
  const double2 r = *reinterpret_cast<const double2*>(rr + K);
  const double sub = tri_sub<UPPER, BR>(T, K);
  const double xk = x[K] * r.x;
  x[K] = xk;
  x[K + 1] = fma(-sub, xk, x[K + 1]);
  const double xk1 = x[K + 1] * r.y;
  x[K + 1] = xk1;
  double yk = 0.0, yk1 = 0.0;
  if constexpr (K >= 16) {
    yk = y[K - 16] * r.x;
    y[K - 16] = yk;
    y[K - 15] = fma(-sub, yk, y[K - 15]);
    yk1 = y[K - 15] * r.y;
    y[K - 15] = yk1;
  }
#pragma unroll
  for (int i = K + 2; i < LEAF; ++i) {
    const double2 t = tri_pair<UPPER, BR>(T, i, K);
    x[i] = fma(-t.x, xk, x[i]);
    x[i] = fma(-t.y, xk1, x[i]);
    if constexpr (K >= 16) {
      y[i - 16] = fma(-t.x, yk, y[i - 16]);
      y[i - 16] = fma(-t.y, yk1, y[i - 16]);
    }
  }
}
template <bool UPPER, int BR, int... P>
__device__ __forceinline__ void leaf32p_steps(const double* T, const double* rr, double (&x)[LEAF], double (&y)[16],
                                              std::integer_sequence<int, P...>) {
  (leaf32p_step<UPPER, BR, 2 * P>(T, rr, x, y), ...);
}

template <bool UPPER, int WARPS, int NS, bool PSTORE>
__global__ void __launch_bounds__(WARPS * 32, 1)
    leaf32_pair_kernel(const __grid_constant__ BandMaps<16> maps, const LeafArgs a) {
  constexpr int BR = 16;
  using BD = Band<BR>;
  constexpr int SLOT = BD::SLOT;  // doubles per matrix
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, c = lane & 15;
  double* slots = reinterpret_cast<double*>(smem_raw) + (size_t)warp * NS * 2 * SLOT;
  double* rr = reinterpret_cast<double*>(smem_raw) + (size_t)WARPS * NS * 2 * SLOT + (warp * 2 + h) * LEAF;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_raw + ((size_t)WARPS * NS * 2 * SLOT + WARPS * 2 * LEAF) * 8) + warp * NS;

  const int64_t npairs = (a.batch + 1) / 2;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= npairs) return;
  const int64_t count = (npairs - gw + TW - 1) / TW;

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (lane == 0 && warp == 0)
    for (int w = 0; w < BD::NBAND; ++w) tma_prefetch_desc(&maps.m[w]);
  __syncwarp();

  auto issue_load = [&](int64_t t) {  // lane 0 only
    const int64_t p = gw + t * TW;
    const int nm = 2 * p + 1 < a.batch ? 2 : 1;
    double* slot = slots + (t % NS) * 2 * SLOT;
    uint64_t* bar = &bars[t % NS];
    mbar_arrive_expect_tx(bar, nm * SLOT * 8);
    for (int m = 0; m < nm; ++m) {
      const int b = (int)(2 * p + m);
#pragma unroll
      for (int g = 0; g < BD::NBAND; ++g) {
        if (!UPPER) tma_load_3d(slot + m * SLOT + BD::loff(g), &maps.m[g], 0, BR * g, b, bar);
        else tma_load_3d(slot + m * SLOT + BD::uoff(g), &maps.m[BD::NBAND - 1 - g], BR * g, BR * g, b, bar);
      }
    }
  };
  if (lane == 0)
    for (int64_t t = 0; t < NS && t < count; ++t) issue_load(t);

  for (int64_t t = 0; t < count; ++t) {
    const int64_t b = 2 * (gw + t * TW) + h;  // this half-warp's matrix
    const bool live = b < a.batch;
    const double* T = slots + (t % NS) * 2 * SLOT + h * SLOT;
    mbar_wait(&bars[t % NS], (uint32_t)((t / NS) & 1));

    // a1: reciprocals of rows c and c + 16 (T' order for the upper case), zero-diagonal mask
    const double d0 = tri_diag<UPPER, BR>(T, c), d1 = tri_diag<UPPER, BR>(T, c + 16);
    const unsigned z0 = __ballot_sync(0xffffffffu, live && !a.unit && d0 == 0.0);
    const unsigned z1 = __ballot_sync(0xffffffffu, live && !a.unit && d1 == 0.0);
    const unsigned zmask = ((z0 >> (16 * h)) & 0xffffu) | (((z1 >> (16 * h)) & 0xffffu) << 16);
    rr[UPPER ? LEAF - 1 - c : c] = a.unit ? 1.0 : 1.0 / d0;  // IEEE division: X_jj == 1/T_jj bitwise (C4)
    rr[UPPER ? 15 - c : c + 16] = a.unit ? 1.0 : 1.0 / d1;
    __syncwarp();
    double x[LEAF], y[16];
#pragma unroll
    for (int i = 0; i < LEAF; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = (i == c) ? 1.0 : 0.0;
    leaf32p_steps<UPPER, BR>(T, rr, x, y, std::make_integer_sequence<int, LEAF / 2>{});
    __syncwarp();  // every lane has finished reading the slot and rr
    if (t + NS < count && lane == 0) {
      fence_proxy_async_smem();
      issue_load(t + NS);
    }
    if (PSTORE) {
      // whole 256-byte rows: one instruction writes row i of matrix 2p (lanes 0-15: columns
      // c, lanes 16-31: columns 16 + c, received from lane c), the next row i of matrix 2p+1
      const int64_t b0 = 2 * (gw + t * TW);
      double* d0p = a.X + b0 * a.sX;
      double* d1p = a.X + (b0 + 1 < a.batch ? b0 + 1 : b0) * a.sX;
      const bool live1 = b0 + 1 < a.batch;
      const int col = UPPER ? LEAF - 1 - lane : lane;  // column of the row this lane writes
#pragma unroll
      for (int i = 0; i < LEAF; ++i) {
        const double xv = (i < c) ? 0.0 : x[i];
        const double yv = (i < 16 + c) ? 0.0 : y[i < 16 ? 0 : i - 16];
        const double other = __shfl_xor_sync(0xffffffffu, h ? xv : yv, 16);  // half 0 gets x of matrix 1, half 1 y of matrix 0
        const int64_t row = (int64_t)(UPPER ? LEAF - 1 - i : i) * a.ldx;
        d0p[row + col] = h ? other : xv;
        if (live1) d1p[row + col] = h ? yv : other;
      }
    } else if (live) {
      double* dst = a.X + b * a.sX;
      const int c0 = UPPER ? LEAF - 1 - c : c, c1 = UPPER ? 15 - c : c + 16;
#pragma unroll
      for (int i = 0; i < LEAF; ++i) {
        const int64_t row = (int64_t)(UPPER ? LEAF - 1 - i : i) * a.ldx;
        dst[row + c0] = (i < c) ? 0.0 : x[i];
        dst[row + c1] = (i < 16 + c) ? 0.0 : y[i < 16 ? 0 : i - 16];
      }
    }
    if (live) {
      if (c == 0) {
        const int fz = zmask ? __ffs(zmask) - 1 : -1;
        if (a.info_mode == 1) a.info[b] = zmask ? fz + 1 : 0;
        else if (a.info_mode == 2 && zmask)
          info_min_nonzero(a.info, static_cast<int32_t>(a.info_off + b * a.info_stride + fz + 1));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// n = 32 with the off-diagonal block on the FP64 tensor cores (opt-in, TRINV_LEAF32=mma;
// measured slower than the band kernel, see launch_leaf).
// The scalar recurrence above reads every T_ik (i > k) once per lane: ~250 16-byte
// shared broadcasts per matrix, which made leaf32_tma_kernel shared-memory (LSU) bound
// (ncu: l1tex 96%).  Here the 32x32 matrix is one beta = 2 merge of Alg. 1
// over two 16-wide diagonal blocks (P:440-452 transposed, = P:1066-1069):
//   1. half-warp h inverts diagonal block h by the same right-looking recurrence of the
//      proof of Thm 1, lane c = column c in 16 registers (lower; the upper
//      case runs CRIT's back substitution, lane c = column c);
//   2. the off-diagonal block by two 16x16x16 products on DMMA from shared memory:
//      lower  W = L21 X11 (X11 lower: tile J reads k >= 8 J), X21 = -X22 W (X22 lower:
//             tile I reads k < 8 I + 8);
//      upper  W = U12 X22 (X22 upper: k < 8 J + 8), X12 = -X11 W (X11 upper: k >= 8 I);
//      24 DMMA.8x8x4 per matrix instead of ~250 broadcasts + ~500 FFMA.
// Staging: the referenced triangle, rows rounded to 16-byte pairs (272 chunks, 4352 B),
// is copied by per-lane cp.async (LDGSTS, bypassing L1) into a slot with row stride 36
// doubles (= 4 mod 16: both m8n8k4 fragment patterns bank-conflict free), NS slots per
// warp, each warp a private ring; the stray element of a pair that falls in the other
// triangle is never read.  Outputs leave from registers: X11 / X22 rows as two 128-byte
// segments per store, the zero block as 16-byte stores, the DMMA tile as 16-byte stores.
constexpr int MS = 36;                  // slot row stride (doubles)
constexpr int MSLOT = 32 * MS;          // doubles per slot (9216 B)
constexpr int MCHUNKS = 272;            // 16-byte chunks of the referenced triangle
constexpr int MCPL = (MCHUNKS + 31) / 32;

__device__ __forceinline__ void cpa16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Pair-chunks of row i: lower c in [0, i/2], upper c in [i/2, 15] (columns 2c, 2c+1).
template <bool UPPER>
__device__ __forceinline__ void mchunk(int q, int& i, int& c) {
  int row = 0, start = 0;
  for (; row < 32; ++row) {
    const int cnt = UPPER ? 16 - row / 2 : row / 2 + 1;
    if (q < start + cnt) break;
    start += cnt;
  }
  i = row;
  c = (UPPER ? row / 2 : 0) + (q - start);
}

// Stage 1 step pair for the lower recurrence (k, k+1) and the upper one (k, k-1).
template <int K, int S = MS>
__device__ __forceinline__ void m_lower_step(const double* T, double (&x)[16]) {
  const double xk = x[K] * T[K * (S + 1)];  // the diagonal slot holds r_K
  x[K] = xk;
  x[K + 1] = fma(-T[(K + 1) * S + K], xk, x[K + 1]);
  const double xk1 = x[K + 1] * T[(K + 1) * (S + 1)];
  x[K + 1] = xk1;
#pragma unroll
  for (int i = K + 2; i < 16; ++i) {
    const double2 t = *reinterpret_cast<const double2*>(T + i * S + K);
    x[i] = fma(-t.x, xk, x[i]);
    x[i] = fma(-t.y, xk1, x[i]);
  }
}
template <int K, int S = MS>
__device__ __forceinline__ void m_upper_step(const double* T, double (&x)[16]) {  // K odd: rows K, K-1
  const double xk = x[K] * T[K * (S + 1)];
  x[K] = xk;
  x[K - 1] = fma(-T[(K - 1) * S + K], xk, x[K - 1]);
  const double xk1 = x[K - 1] * T[(K - 1) * (S + 1)];
  x[K - 1] = xk1;
#pragma unroll
  for (int i = 0; i < K - 1; ++i) {
    const double2 t = *reinterpret_cast<const double2*>(T + i * S + K - 1);  // (T_i,K-1, T_iK)
    x[i] = fma(-t.y, xk, x[i]);
    x[i] = fma(-t.x, xk1, x[i]);
  }
}
template <bool UPPER, int S = MS, int... P>
__device__ __forceinline__ void m_steps(const double* T, double (&x)[16], std::integer_sequence<int, P...>) {
  if constexpr (UPPER) (m_upper_step<15 - 2 * P, S>(T, x), ...);
  else (m_lower_step<2 * P, S>(T, x), ...);
}

// acc[I][J] (8x8 tiles of a 16x16 product) += A[16][16] B[16][16], both in the slot
// (stride MS), K-steps of 4 restricted by the triangular operand (TRI: 0 = B lower,
// tile J needs k >= 8J; 1 = A lower, tile I needs k < 8I+8; 2 = B upper, k < 8J+8;
// 3 = A upper, k >= 8I).
template <int TRI>
__device__ __forceinline__ void m_mma16(double (&acc)[2][2][2], const double* A, const double* B, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int k = 0; k < 16; k += 4) {
    const bool hi = k >= 8;  // second half of the K range
    double a[2], b[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      a[t] = A[(8 * t + lr) * MS + k + lc];
      b[t] = B[(k + lc) * MS + 8 * t + lr];
    }
#pragma unroll
    for (int I = 0; I < 2; ++I)
#pragma unroll
      for (int J = 0; J < 2; ++J) {
        const bool need = TRI == 0 ? (hi || J == 0) : TRI == 1 ? (!hi || I == 1)
                        : TRI == 2 ? (!hi || J == 1) : (hi || I == 0);
        if (need) dmma_8x8x4(acc[I][J][0], acc[I][J][1], a[I], b[J]);
      }
  }
}

// Stage 1 (a1, a2): reciprocals into the diagonal slots, the recurrence of half-warp h on
// its diagonal block, X11 / X22 into the slot (operands of stage 2) and to `dst` (when
// `store`), the zero quadrant to `dst`.  Returns the warp's zero-diagonal mask.
template <bool UPPER>
__device__ __forceinline__ unsigned m_stage1(double* S, const LeafArgs& a, double* dst, bool store, int lane) {
  const int h = lane >> 4, c = lane & 15;
  double* Th = S + 16 * h * (MS + 1);  // diagonal block h
  const double d = Th[c * (MS + 1)];
  const unsigned zmask = __ballot_sync(0xffffffffu, (!a.unit) && d == 0.0);
  const double r = a.unit ? 1.0 : __drcp_rn(d);  // correctly rounded: X_jj == 1/T_jj bitwise (C4)
  __syncwarp();
  Th[c * (MS + 1)] = r;
  __syncwarp();
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (i == c) ? 1.0 : 0.0;
  m_steps<UPPER>(Th, x, std::make_integer_sequence<int, 8>{});
  __syncwarp();  // every lane has read its block before it is overwritten by its inverse
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double v = (UPPER ? i > c : i < c) ? 0.0 : x[i];
    Th[i * MS + c] = v;                                               // operand of stage 2
    if (store) dst[(int64_t)(16 * h + i) * a.ldx + 16 * h + c] = v;   // X11 / X22 rows (a7 inside)
  }
  if (store) {  // the zero quadrant (a7): lower rows 0..15 x cols 16..31, upper rows 16..31 x cols 0..15
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rr = 4 * q + (lane >> 3), cc = 2 * (lane & 7);
      *reinterpret_cast<double2*>(dst + (int64_t)(UPPER ? 16 + rr : rr) * a.ldx + (UPPER ? cc : 16 + cc)) =
          make_double2(0.0, 0.0);
    }
  }
  return zmask;
}
// Stage 2a (a5): W = L21 X11 (upper: U12 X22) into the slot's unreferenced quadrant.
template <bool UPPER>
__device__ __forceinline__ void m_stage2a(double* S, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
  double acc[2][2][2] = {};
  double* W = UPPER ? S + 16 * MS : S + 16;
  if (!UPPER) m_mma16<0>(acc, S + 16 * MS, S, lane);   // W = L21 X11
  else m_mma16<2>(acc, S + 16, S + 16 * MS + 16, lane);  // W = U12 X22
#pragma unroll
  for (int I = 0; I < 2; ++I)
#pragma unroll
    for (int J = 0; J < 2; ++J)
      *reinterpret_cast<double2*>(W + (8 * I + lr) * MS + 8 * J + 2 * lc) = make_double2(acc[I][J][0], acc[I][J][1]);
}
// Stage 2b (a6, a7): X21 = -X22 W (upper: X12 = -X11 W) straight to `dst`.
template <bool UPPER>
__device__ __forceinline__ void m_stage2b(const double* S, const LeafArgs& a, double* dst, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
  double acc[2][2][2] = {};
  const double* W = UPPER ? S + 16 * MS : S + 16;
  if (!UPPER) m_mma16<1>(acc, S + 16 * MS + 16, W, lane);  // X21 = -X22 W
  else m_mma16<3>(acc, S, W, lane);                          // X12 = -X11 W
  double* o = dst + (UPPER ? 16 : 16 * a.ldx);
#pragma unroll
  for (int I = 0; I < 2; ++I)
#pragma unroll
    for (int J = 0; J < 2; ++J)
      *reinterpret_cast<double2*>(o + (int64_t)(8 * I + lr) * a.ldx + 8 * J + 2 * lc) =
          make_double2(-acc[I][J][0], -acc[I][J][1]);
}

// PIPE = false: the three stages of matrix t in order.  PIPE = true (NS >= 3): stage 1 of
// matrix t+1 is interleaved with stage 2 of matrix t in three straight-line segments
// separated by __syncwarp (the recurrence's FP64 chain overlaps the DMMA chain of the
// other matrix; every segment touches two different slots).
template <bool UPPER, int WARPS, int NS, bool PIPE>
__global__ void __launch_bounds__(WARPS * 32, 1) leaf32_mma_kernel(const LeafArgs a) {
  static_assert(!PIPE || NS >= 3, "the pipelined loop keeps two slots live and one loading");
  extern __shared__ __align__(16) double msmem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slots = msmem + (size_t)warp * NS * MSLOT;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= a.batch) return;
  const int64_t count = (a.batch - gw + TW - 1) / TW;

  int soff[MCPL], goff[MCPL];  // this lane's chunks: slot offset, input offset (doubles)
#pragma unroll
  for (int m = 0; m < MCPL; ++m) {
    const int q = lane + 32 * m;
    int i = 0, c = 0;
    if (q < MCHUNKS) mchunk<UPPER>(q, i, c);
    soff[m] = q < MCHUNKS ? i * MS + 2 * c : -1;
    goff[m] = i * (int)a.lda + 2 * c;
  }
  auto issue = [&](int64_t t) {
    if (t < count) {
      const double* src = a.A + (gw + t * TW) * a.sA;
      double* dst = slots + (t % NS) * MSLOT;
#pragma unroll
      for (int m = 0; m < MCPL; ++m)
        if (soff[m] >= 0) cpa16(dst + soff[m], src + goff[m]);
    }
    cpa_commit();  // one group per matrix slot, empty past the end (uniform wait counts)
  };
  auto dst_of = [&](int64_t t) { return a.X + (gw + t * TW) * a.sX; };
#pragma unroll
  for (int t = 0; t < NS - 1; ++t) issue(t);

  if constexpr (!PIPE) {
    for (int64_t t = 0; t < count; ++t) {
      issue(t + NS - 1);
      cpa_wait<NS - 1>();
      __syncwarp();
      double* S = slots + (t % NS) * MSLOT;
      double* dst = dst_of(t);
      const unsigned zmask = m_stage1<UPPER>(S, a, dst, true, lane);
      __syncwarp();
      m_stage2a<UPPER>(S, lane);
      __syncwarp();
      m_stage2b<UPPER>(S, a, dst, lane);
      __syncwarp();  // every lane is done with the slot: the next load may overwrite it
      leaf_report(a, gw + t * TW, lane, zmask != 0, zmask ? __ffs(zmask) - 1 : -1);
    }
  } else {
    // prologue: stage 1 of matrix 0
    cpa_wait<NS - 2>();
    __syncwarp();
    unsigned zm = m_stage1<UPPER>(slots, a, dst_of(0), true, lane);
    __syncwarp();
    for (int64_t t = 0; t < count; ++t) {
      const bool next = t + 1 < count;
      issue(t + NS - 1);          // slot of matrix t-1: free since the end of the last iteration
      cpa_wait<NS - 2>();         // matrix t+1 has landed
      __syncwarp();
      double* S = slots + (t % NS) * MSLOT;
      double* Sn = slots + ((t + 1) % NS) * MSLOT;
      double* dst = dst_of(t);
      // stage 1 of t+1 (on a stale slot past the end: computed, not stored) | stage 2 of t
      m_stage2a<UPPER>(S, lane);
      const unsigned zn = m_stage1<UPPER>(Sn, a, dst_of(next ? t + 1 : t), next, lane);
      __syncwarp();
      m_stage2b<UPPER>(S, a, dst, lane);
      __syncwarp();
      leaf_report(a, gw + t * TW, lane, zm != 0, zm ? __ffs(zm) - 1 : -1);
      zm = zn;
    }
  }
  cpa_wait<0>();
}

template <int W, int NS, bool PIPE = false>
static void launch_mma32(char uplo, const LeafArgs& a, int sms, cudaStream_t s) {
  constexpr size_t smem = (size_t)W * NS * MSLOT * 8;
  const int64_t ctas_needed = (a.batch + W - 1) / W;
  const int grid = (int)(ctas_needed < sms ? ctas_needed : sms);
  if (uplo == 'L') {
    constexpr auto k = leaf32_mma_kernel<false, W, NS, PIPE>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(a);
  } else {
    constexpr auto k = leaf32_mma_kernel<true, W, NS, PIPE>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(a);
  }
}

// ---------------------------------------------------------------------------
// n <= 16 (any layout): a half-warp per matrix, two per warp, lane c = column c of the inverse
// by the same 16-wide recurrence (lower: P:221-247 right-looking; upper: CRIT's back
// substitution), orders below 16 padded with the identity (inv([T 0; 0 I]) =
// [T^-1 0; 0 I], nothing of the padding is stored).  Rows move one per instruction (16 lanes
// x 8 B = one 128-byte line per half-warp); the next pair of matrices is loaded into
// registers while the current pair is inverted.  Round 1 ran these orders through the
// one-warp-per-matrix plain kernel at 0.12 of HBM (n = 16); now 0.61 (5x).
constexpr int HS = 18;  // slot row stride (doubles): 16-byte aligned rows for the pair loads
template <bool UPPER>
__global__ void __launch_bounds__(256) leaf16_kernel(const LeafArgs a) {
  __shared__ __align__(16) double slots[8][2][16 * HS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, c = lane & 15;
  double* T = slots[warp][h];
  const int64_t npairs = (a.batch + 1) / 2;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp, TW = (int64_t)gridDim.x * 8;
  const unsigned hmask = 0xffffu << (16 * h);
  auto load = [&](int64_t pr, double (&v)[16]) {
    const int64_t b = 2 * pr + h;
    const int nb = b >= a.batch ? 0 : (b == a.batch - 1 ? a.n_last : a.n);
    const double* src = a.A + (b < a.batch ? b : 0) * a.sA;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool ref = i < nb && c < nb && (UPPER ? c >= i : c <= i) && !(a.unit && c == i);
      v[i] = ref ? src[(int64_t)i * a.lda + c] : (i == c ? 1.0 : 0.0);
    }
  };
  double v[16];
  if (gw < npairs) load(gw, v);
  for (int64_t pr = gw; pr < npairs; pr += TW) {
    const int64_t b = 2 * pr + h;
    const int nb = b >= a.batch ? 0 : (b == a.batch - 1 ? a.n_last : a.n);
#pragma unroll
    for (int i = 0; i < 16; ++i) T[i * HS + c] = v[i];
    __syncwarp();
    if (pr + TW < npairs) load(pr + TW, v);  // the next pair's rows in flight during the inversion
    const double d = T[c * (HS + 1)];
    const bool zero = c < nb && d == 0.0;
    const unsigned zmask = (__ballot_sync(0xffffffffu, zero) & hmask) >> (16 * h);
    __syncwarp();
    T[c * (HS + 1)] = 1.0 / d;  // IEEE division: X_jj == 1/T_jj bitwise (C4); unit / padding: 1
    __syncwarp();
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (i == c) ? 1.0 : 0.0;
    m_steps<UPPER, HS>(T, x, std::make_integer_sequence<int, 8>{});
    __syncwarp();  // the slot is rewritten by the next pair
    if (b < a.batch) {
      double* dst = a.X + b * a.sX;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nb && c < nb) dst[(int64_t)i * a.ldx + c] = (UPPER ? i > c : i < c) ? 0.0 : x[i];
      if (c == 0) {
        const int fz = zmask ? __ffs(zmask) - 1 : -1;
        if (a.info_mode == 1) a.info[b] = zmask ? fz + 1 : 0;
        else if (a.info_mode == 2 && zmask)
          info_min_nonzero(a.info, static_cast<int32_t>(a.info_off + b * a.info_stride + fz + 1));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// n = 32, four matrices per warp (opt-in TRINV_LEAF32=quad, TRINV_LEAF32_QCFG = warps x slots
// [x CTAs per SM]; measured 8-10% slower than the band kernel, profiles/r02_leaf_quad.txt:
// it cuts the shared wavefronts to 143 per matrix and l1tex to 51%, but with ~255 registers per
// thread and 17.5 KB per quad slot only 4-6 warps fit per SM and it is latency-bound).  Same recurrence as the
// band kernel (proof of Thm 1, right-looking; CRIT P:568-581 for the upper case
// through T' = J U J), but quarter-warp h (lanes 8h .. 8h+7) owns matrix 4g + h and lane
// c of a quarter computes the four columns 2c, 2c+1, 2c+16, 2c+17 of its inverse.
// Why (ncu of the band kernel, profiles/r02_ncu_leaf32_full.txt): one warp per matrix makes
// every T_ik a warp-wide broadcast, and a 16-byte broadcast costs two shared-memory
// wavefronts for 16 useful bytes: 546 wavefronts per matrix plus 64 for the row stores and
// 48 for the TMA fills put l1tex at 96%, so the kernel is bound by the LSU exactly where
// DRAM also saturates (compressing the output's zero triangle cut the DRAM writes by a third
// and did not change the time: profiles/r02_leaf_quad.txt).  Here one 16-byte load serves
// four matrices (the four quarters read the same offset of four regions whose bases differ
// by 32 bytes mod 128: four disjoint bank groups) and each T_ik feeds four columns, so the
// shared traffic per matrix drops ~4x; columns 2c+16, 2c+17 skip the 16 steps in which they
// are structurally zero (31% fewer FP64 instructions than one warp per matrix).  Rows K, K+1
// are stored as soon as step pair K has finalised them (their registers die early).
// Staging: per-lane 16-byte cp.async of the referenced triangle, rows rounded to 16-byte
// pairs (272 chunks, 4352 B per matrix, packed row after row: row i starts at chunk P(i) =
// floor(i/2) floor(i/2 + 1) + (i odd) (floor(i/2) + 1)); the upper case stores T' rows
// (U row 31 - i, pairs in reverse order, the two doubles of a pair swapped on read).
// Stores: per row two 16-byte stores per lane (a quarter writes one 128-byte line).
constexpr int QCH = 272;            // 16-byte chunks of a packed triangle
constexpr int QMAT = 2 * QCH + 4;   // doubles per matrix region: 4384 B = 32 mod 128 (bank shift)
constexpr int QSLOT = 4 * QMAT;     // doubles per quad slot
constexpr int QRR = 36;             // doubles per reciprocal vector (288 B = 32 mod 128)
__host__ __device__ constexpr int qP(int i) { return (i / 2) * (i / 2 + 1) + (i & 1) * (i / 2 + 1); }
static_assert(qP(32) == QCH && (QMAT * 8) % 128 == 32 && (QRR * 8) % 128 == 32, "quad layout");

template <bool UPPER>
__device__ __forceinline__ double2 q_pair(const double* T, int i, int k) {  // (T'_ik, T'_i,k+1), k even
  const double2 v = *reinterpret_cast<const double2*>(T + 2 * qP(i) + k);
  return UPPER ? make_double2(v.y, v.x) : v;
}
template <bool UPPER>
__device__ __forceinline__ double q_elem(const double* T, int i, int k) {  // T'_ik
  return T[2 * qP(i) + (UPPER ? (k ^ 1) : k)];
}

// x0[i] = (X'_{i,2c}, X'_{i,2c+1}), rows 0..31; x1[i-16] = (X'_{i,2c+16}, X'_{i,2c+17}), rows 16..31
// (double2: each pair lives in an aligned register quad, stored by one 16-byte store).
template <int K, int OFF, int N>
__device__ __forceinline__ void q_head(double2 (&x)[N], double2 r, double sub, double2& xk, double2& xk1) {
  double2& u = x[K - OFF];
  double2& v = x[K + 1 - OFF];
  u.x *= r.x;
  u.y *= r.x;
  v.x = fma(-sub, u.x, v.x) * r.y;
  v.y = fma(-sub, u.y, v.y) * r.y;
  xk = u;
  xk1 = v;
}
// Rows K and K+1 of X' are final once the head of step pair K has run: they are stored right
// there (the opposite triangle masked to +0.0, row a7), so their registers die early.
template <bool UPPER, int I>
__device__ __forceinline__ void q_store_row(double* dst, int64_t ldx, int c, double2 (&x0)[32], double2 (&x1)[16]) {
  double2 v = x0[I];
  if (I < 2 * c) v.x = 0.0;
  if (I < 2 * c + 1) v.y = 0.0;
  double2 w = make_double2(0.0, 0.0);
  if constexpr (I >= 16) {
    w = x1[I - 16];
    if (I < 2 * c + 16) w.x = 0.0;
    if (I < 2 * c + 17) w.y = 0.0;
  }
  if (!UPPER) {
    double* row = dst + (int64_t)I * ldx;
    *reinterpret_cast<double2*>(row + 2 * c) = v;
    *reinterpret_cast<double2*>(row + 2 * c + 16) = w;
  } else {  // X = J X' J: T' (i, j) -> (31 - i, 31 - j); columns 30-2c, 31-2c as one pair
    double* row = dst + (int64_t)(LEAF - 1 - I) * ldx;
    *reinterpret_cast<double2*>(row + 30 - 2 * c) = make_double2(v.y, v.x);
    *reinterpret_cast<double2*>(row + 14 - 2 * c) = make_double2(w.y, w.x);
  }
}
template <bool UPPER, int K>
__device__ __forceinline__ void q_step(const double* T, const double* rr, double2 (&x0)[32], double2 (&x1)[16],
                                       double* dst, int64_t ldx, int c, bool live) {
  const double2 r = *reinterpret_cast<const double2*>(rr + K);
  const double sub = q_elem<UPPER>(T, K + 1, K);
  double2 a0, b0, a1, b1;
  q_head<K, 0>(x0, r, sub, a0, b0);
  if constexpr (K >= 16) q_head<K, 16>(x1, r, sub, a1, b1);
#pragma unroll
  for (int i = K + 2; i < LEAF; ++i) {
    const double2 t = q_pair<UPPER>(T, i, K);
    x0[i].x = fma(-t.y, b0.x, fma(-t.x, a0.x, x0[i].x));
    x0[i].y = fma(-t.y, b0.y, fma(-t.x, a0.y, x0[i].y));
    if constexpr (K >= 16) {
      x1[i - 16].x = fma(-t.y, b1.x, fma(-t.x, a1.x, x1[i - 16].x));
      x1[i - 16].y = fma(-t.y, b1.y, fma(-t.x, a1.y, x1[i - 16].y));
    }
  }
  if (live) {
    q_store_row<UPPER, K>(dst, ldx, c, x0, x1);
    q_store_row<UPPER, K + 1>(dst, ldx, c, x0, x1);
  }
}
template <bool UPPER, int... P>
__device__ __forceinline__ void q_steps(const double* T, const double* rr, double2 (&x0)[32], double2 (&x1)[16],
                                        double* dst, int64_t ldx, int c, bool live, std::integer_sequence<int, P...>) {
  (q_step<UPPER, 2 * P>(T, rr, x0, x1, dst, ldx, c, live), ...);
}

template <bool UPPER, int WARPS, int NS>
__global__ void __launch_bounds__(WARPS * 32, 1) leaf32_quad_kernel(const LeafArgs a) {
  extern __shared__ __align__(128) double qsmem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 3, c = lane & 7;
  double* slots = qsmem + (size_t)warp * NS * QSLOT;
  double* rr = qsmem + (size_t)WARPS * NS * QSLOT + (warp * 4 + h) * QRR;
  const int64_t nquads = (a.batch + 3) / 4;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= nquads) return;
  const int64_t count = (nquads - gw + TW - 1) / TW;

  // quarter h copies matrix 4g + h: row i, pair c (every row) and pair c + 8 (rows >= 16)
  auto issue = [&](int64_t t) {
    if (t < count) {
      const int64_t b = 4 * (gw + t * TW) + h;
      if (b < a.batch) {
        // source row pointer walked by +-lda (no per-row offsets held in registers)
        const double* src = a.A + b * a.sA + (UPPER ? (LEAF - 1) * a.lda + 30 - 2 * c : 2 * c);
        const int64_t step = UPPER ? -a.lda : a.lda;
        double* dst = slots + (t % NS) * QSLOT + h * QMAT + 2 * c;
#pragma unroll
        for (int i = 0; i < LEAF; ++i) {
          if (c <= i / 2) cpa16(dst + 2 * qP(i), src);                                         // pair c
          if (i >= 16 && c + 8 <= i / 2) cpa16(dst + 2 * qP(i) + 16, src + (UPPER ? -16 : 16));  // pair c + 8
          src += step;
        }
      }
    }
    cpa_commit();  // one group per slot, empty past the end (uniform wait counts)
  };
#pragma unroll
  for (int t = 0; t < NS - 1; ++t) issue(t);

  for (int64_t t = 0; t < count; ++t) {
    issue(t + NS - 1);
    cpa_wait<NS - 1>();
    __syncwarp();
    const int64_t b = 4 * (gw + t * TW) + h;
    const bool live = b < a.batch;
    const double* T = slots + (t % NS) * QSLOT + h * QMAT;
    // a1: reciprocals of T' rows c + 8m (IEEE division: X_jj == 1/T_jj bitwise, C4)
    unsigned zq = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = c + 8 * m;
      const double d = q_elem<UPPER>(T, j, j);
      const unsigned bal = __ballot_sync(0xffffffffu, live && !a.unit && d == 0.0);
      zq |= ((bal >> (8 * h)) & 0xffu) << (8 * m);
      rr[j] = a.unit ? 1.0 : 1.0 / d;
    }
    __syncwarp();
    double2 x0[32], x1[16];
#pragma unroll
    for (int i = 0; i < LEAF; ++i) x0[i] = make_double2(i == 2 * c ? 1.0 : 0.0, i == 2 * c + 1 ? 1.0 : 0.0);
#pragma unroll
    for (int i = 16; i < LEAF; ++i) x1[i - 16] = make_double2(i == 2 * c + 16 ? 1.0 : 0.0, i == 2 * c + 17 ? 1.0 : 0.0);
    double* dst = a.X + (live ? b : 0) * a.sX;
    q_steps<UPPER>(T, rr, x0, x1, dst, a.ldx, c, live, std::make_integer_sequence<int, LEAF / 2>{});
    __syncwarp();  // every lane is done with the slot and rr: the next loads may overwrite them
    if (live) {
      if (c == 0) {
        const unsigned zmask = UPPER ? __brev(zq) : zq;  // original row order
        const int fz = zmask ? __ffs(zmask) - 1 : -1;
        if (a.info_mode == 1) a.info[b] = zmask ? fz + 1 : 0;
        else if (a.info_mode == 2 && zmask)
          info_min_nonzero(a.info, static_cast<int32_t>(a.info_off + b * a.info_stride + fz + 1));
      }
    }
  }
  cpa_wait<0>();
}

template <int W, int NS, int CPS = 1>  // CPS: CTAs per SM
static void launch_quad(char uplo, const LeafArgs& a, int sms, cudaStream_t s) {
  constexpr size_t smem = ((size_t)W * NS * QSLOT + (size_t)W * 4 * QRR) * 8;
  static_assert(smem * CPS <= 227 * 1024, "quad smem");
  const int64_t ctas_needed = ((a.batch + 3) / 4 + W - 1) / W;
  const int grid = (int)(ctas_needed < (int64_t)sms * CPS ? ctas_needed : (int64_t)sms * CPS);
  if (uplo == 'L') {
    constexpr auto k = leaf32_quad_kernel<false, W, NS>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(a);
  } else {
    constexpr auto k = leaf32_quad_kernel<true, W, NS>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(a);
  }
}

// ---------------------------------------------------------------------------
// Plain-load kernel for any layout (odd n / ld, unaligned pointers): one warp
// per matrix, rows loaded coalesced into a smem slot, result stored directly.
template <bool UPPER>
__global__ void __launch_bounds__(128) leaf_plain_kernel(const LeafArgs a) {
  __shared__ double slots[4][LEAF * LEAF];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* T = slots[warp];
  for (int64_t b = (int64_t)blockIdx.x * 4 + warp; b < a.batch; b += (int64_t)gridDim.x * 4) {
    const int nb = (b == a.batch - 1) ? a.n_last : a.n;
    const double* src = a.A + b * a.sA;
    double v[LEAF];
#pragma unroll
    for (int i = 0; i < LEAF; ++i) v[i] = (i < nb && lane < nb) ? src[(int64_t)i * a.lda + lane] : 0.0;
#pragma unroll
    for (int i = 0; i < LEAF; ++i)
      if (i < nb) T[i * LEAF + lane] = v[i];
    __syncwarp();
    double x[LEAF];
    bool singular;
    int first_zero;
    leaf_compute<UPPER>(T, nb, a.unit, lane, x, singular, first_zero);
    double* dst = a.X + b * a.sX;
#pragma unroll
    for (int i = 0; i < LEAF; ++i) {
      const bool zero = UPPER ? (i > lane) : (i < lane);
      if (i < nb && lane < nb) dst[i * a.ldx + lane] = zero ? 0.0 : x[i];
    }
    leaf_report(a, b, lane, singular, first_zero);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// 3-D view [batch][32 rows][32 cols] of the inputs; box = `rows` rows x `cols` columns x 1 matrix.
static bool encode_batch_map(CUtensorMap* m, const LeafArgs& a, int cols, int rows) {
  const uint64_t dims[3] = {32, 32, (uint64_t)a.batch};
  const uint64_t strides[2] = {(uint64_t)a.lda * 8, (uint64_t)a.sA * 8};
  const uint32_t box[3] = {(uint32_t)cols, (uint32_t)rows, 1};
  return encode_map_nd(m, a.A, 3, dims, strides, box);
}

template <int W, int NS, int BR, bool BULK = false>
static bool launch_band(char uplo, const LeafArgs& a, int sms, cudaStream_t s) {
  BandMaps<BR> maps;
  for (int w = 1; w <= Band<BR>::NBAND; ++w)
    if (!encode_batch_map(&maps.m[w - 1], a, BR * w, BR)) return false;
  constexpr size_t base = ((size_t)W * NS * Band<BR>::SLOT + W * LEAF) * 8 + W * NS * 8;
  constexpr size_t smem = BULK ? ((base + 127) & ~size_t(127)) + (size_t)W * LEAF * LEAF * 8 : base;
  const int64_t ctas_needed = (a.batch + W - 1) / W;
  const int grid = (int)(ctas_needed < sms ? ctas_needed : sms);
  if (uplo == 'L') {
    constexpr auto k = leaf32_tma_kernel<false, W, NS, BR, BULK>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(maps, a);
  } else {
    constexpr auto k = leaf32_tma_kernel<true, W, NS, BR, BULK>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(maps, a);
  }
  return true;
}
template <int W, int NS, bool PSTORE = false>
static bool launch_pair(char uplo, const LeafArgs& a, int sms, cudaStream_t s) {
  BandMaps<16> maps;
  for (int w = 1; w <= 2; ++w)
    if (!encode_batch_map(&maps.m[w - 1], a, 16 * w, 16)) return false;
  constexpr size_t smem = ((size_t)W * NS * 2 * Band<16>::SLOT + W * 2 * LEAF) * 8 + W * NS * 8;
  const int64_t ctas_needed = ((a.batch + 1) / 2 + W - 1) / W;
  const int grid = (int)(ctas_needed < sms ? ctas_needed : sms);
  if (uplo == 'L') {
    constexpr auto k = leaf32_pair_kernel<false, W, NS, PSTORE>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(maps, a);
  } else {
    constexpr auto k = leaf32_pair_kernel<true, W, NS, PSTORE>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(maps, a);
  }
  return true;
}

cudaError_t launch_leaf(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.batch <= 0) return cudaSuccess;
  const int sms = device_sms();
  const bool even = (a.n % 2 == 0) && (a.n_last % 2 == 0) && (a.lda % 2 == 0) && (a.ldx % 2 == 0) &&
                    (a.sA % 2 == 0) && (a.sX % 2 == 0);
  const bool tma = even && aligned16(a.A) && aligned16(a.X);
  // algorithmic work: n^3/3 flops and the referenced triangle in + full matrix out per matrix
  if (a.n > LEAF || a.n_last > LEAF) {
    if (leaf64_tma_ok(a)) return launch_leaf64_tma(uplo, a, s, launches);  // 64: one warp per matrix
    return launch_blk(uplo, a, s, launches);                                // 33..128: one CTA per matrix
  }
  const double nn = (double)a.n;
  ProfileScope prof(KIND_LEAF, a.batch * nn * nn * nn / 3.0, a.batch * (nn * (nn + 1) / 2 + nn * nn) * 8.0, s);
  const bool full32 = a.n == LEAF && a.n_last == LEAF;
  // n = 32, TMA-compatible layout: 8 warps x NS slots per CTA (one CTA per SM), bands of
  // BR rows (profiles/r01_leaf_variants.txt); TRINV_LEAF_BR = 4 / 8 / 16 for experiments
  static const int br = [] { const char* e = std::getenv("TRINV_LEAF_BR"); return e ? std::atoi(e) : 16; }();
  // n = 32 default: the scalar TMA-band kernel, at 0.95 of the copy bandwidth on the bytes
  // DRAM actually moves (128-byte line fills: 6144 B read + 8192 B written per matrix).  The
  // DMMA-merge kernel (TRINV_LEAF32=mma; TRINV_LEAF32_CFG = [1000 pipelined +] warps x slots,
  // default 1063) halves the shared-memory wavefronts but is latency-bound and measured
  // 3-12% slower (profiles/r02_leaf_variants.txt).
  static const bool mma = [] { const char* e = std::getenv("TRINV_LEAF32"); return e && !strcmp(e, "mma"); }();
  static const bool pair = [] { const char* e = std::getenv("TRINV_LEAF32"); return e && !strcmp(e, "pair"); }();
  static const int mcfg = [] { const char* e = std::getenv("TRINV_LEAF32_CFG"); return e ? std::atoi(e) : 1063; }();
  static const int pcfg = [] { const char* e = std::getenv("TRINV_LEAF32_PCFG"); return e ? std::atoi(e) : 82; }();
  bool launched = false;
  static const bool quad = [] { const char* e = std::getenv("TRINV_LEAF32"); return e && !strcmp(e, "quad"); }();
  static const int qcfg = [] { const char* e = std::getenv("TRINV_LEAF32_QCFG"); return e ? std::atoi(e) : 43; }();
  if (quad && tma && full32 && a.batch < (int64_t)1 << 31) {
    switch (qcfg) {
      case 62: launch_quad<6, 2>(uplo, a, sms, s); break;
      case 33: launch_quad<3, 3>(uplo, a, sms, s); break;
      case 42: launch_quad<4, 2>(uplo, a, sms, s); break;
      case 52: launch_quad<5, 2>(uplo, a, sms, s); break;
      case 32: launch_quad<3, 2>(uplo, a, sms, s); break;
      case 24: launch_quad<2, 4>(uplo, a, sms, s); break;
      case 223: launch_quad<2, 2, 3>(uplo, a, sms, s); break;
      case 126: launch_quad<1, 2, 6>(uplo, a, sms, s); break;
      case 322: launch_quad<3, 2, 2>(uplo, a, sms, s); break;
      case 134: launch_quad<1, 3, 4>(uplo, a, sms, s); break;
      default: launch_quad<4, 3>(uplo, a, sms, s); break;
    }
    launched = true;
  }
  // two matrices per warp (TRINV_LEAF32=pair; TRINV_LEAF32_PCFG = [100 full-row stores +] warps x
  // pair-slots): half the LSU wavefronts and 37% fewer FP64 instructions per matrix, yet 10%
  // slower than the band kernel in every shape (profiles/r02_leaf_pair.txt)
  if (pair && br == 16 && tma && full32 && a.batch < (int64_t)1 << 31) {
    switch (pcfg) {
      case 43: launched = launch_pair<4, 3>(uplo, a, sms, s); break;
      case 62: launched = launch_pair<6, 2>(uplo, a, sms, s); break;
      case 44: launched = launch_pair<4, 4>(uplo, a, sms, s); break;
      case 52: launched = launch_pair<5, 2>(uplo, a, sms, s); break;
      case 182: launched = launch_pair<8, 2, true>(uplo, a, sms, s); break;
      case 143: launched = launch_pair<4, 3, true>(uplo, a, sms, s); break;
      default: launched = launch_pair<8, 2>(uplo, a, sms, s); break;
    }
  }
  if (mma && tma && full32 && a.lda * 32 < ((int64_t)1 << 31)) {
    switch (mcfg) {
      case 122: launch_mma32<12, 2>(uplo, a, sms, s); break;
      case 64: launch_mma32<6, 4>(uplo, a, sms, s); break;
      case 62: launch_mma32<6, 2>(uplo, a, sms, s); break;
      case 42: launch_mma32<4, 2>(uplo, a, sms, s); break;
      case 82: launch_mma32<8, 2>(uplo, a, sms, s); break;
      case 1083: launch_mma32<8, 3, true>(uplo, a, sms, s); break;
      case 1064: launch_mma32<6, 4, true>(uplo, a, sms, s); break;
      case 1043: launch_mma32<4, 3, true>(uplo, a, sms, s); break;
      case 83: launch_mma32<8, 3>(uplo, a, sms, s); break;
      default: launch_mma32<6, 3, true>(uplo, a, sms, s); break;
    }
    launched = true;
  }
  if (!launched && tma && full32 && a.batch < (int64_t)1 << 31) {
    static const int bulk = [] { const char* e = std::getenv("TRINV_LEAF_BULK"); return e ? atoi(e) : 0; }();
    const bool contiguous = a.ldx == LEAF && a.sX == LEAF * LEAF;
    if (br == 16 && bulk == 1 && contiguous) launched = launch_band<8, 3, 16, true>(uplo, a, sms, s);
    else if (br == 16 && bulk == 2 && contiguous) launched = launch_band<8, 2, 16, true>(uplo, a, sms, s);
    else if (br == 16 && bulk == 3 && contiguous) launched = launch_band<6, 4, 16, true>(uplo, a, sms, s);
    else if (br == 16) launched = launch_band<8, 3, 16>(uplo, a, sms, s);
    else if (br == 8) launched = launch_band<8, 4, 8>(uplo, a, sms, s);
    else launched = launch_band<8, 4, 4>(uplo, a, sms, s);
  }
  if (!launched && a.n <= 16 && a.n_last <= 16) {  // half-warp per matrix
    const int64_t ctas_needed = ((a.batch + 1) / 2 + 7) / 8;
    const int grid = (int)(ctas_needed < (int64_t)sms * 8 ? ctas_needed : (int64_t)sms * 8);
    if (uplo == 'L') leaf16_kernel<false><<<grid, 256, 0, s>>>(a);
    else leaf16_kernel<true><<<grid, 256, 0, s>>>(a);
    launched = true;
  }
  if (!launched) {
    const int64_t ctas_needed = (a.batch + 3) / 4;
    const int grid = (int)(ctas_needed < (int64_t)sms * 8 ? ctas_needed : (int64_t)sms * 8);
    if (uplo == 'L')
      leaf_plain_kernel<false><<<grid, 128, 0, s>>>(a);
    else
      leaf_plain_kernel<true><<<grid, 128, 0, s>>>(a);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace trinv
