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
// HBM staging (a3): every warp runs its own NS-deep ring of 8 KiB slots.
// Loads are 1-D TMA bulk copies (cp.async.bulk, one per matrix when it is
// contiguous, one per row otherwise) completing on a per-slot mbarrier; the
// inverse is written back into the same slot and stored with a bulk copy
// smem->global.  The slot is reloaded only after that store has read it.
#include <cuda_runtime.h>

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

// Write X into the slot row-major; the opposite triangle as +0.0 (C12).
template <bool UPPER>
__device__ __forceinline__ void leaf_write_slot(double* T, int lane, const double (&x)[LEAF]) {
#pragma unroll
  for (int i = 0; i < LEAF; ++i) {
    const bool zero = UPPER ? (i > lane) : (i < lane);
    T[i * LEAF + lane] = zero ? 0.0 : x[i];
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
// TMA-staged persistent kernel: WARPS warps per CTA, NS slots per warp.
template <bool UPPER, int WARPS, int NS>
__global__ void __launch_bounds__(WARPS * 32, 1) leaf_tma_kernel(const LeafArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slots = reinterpret_cast<double*>(smem_raw) + (size_t)warp * NS * LEAF * LEAF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)WARPS * NS * LEAF * LEAF * 8) + warp * NS;

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= a.batch) return;
  const int64_t count = (a.batch - gw + TW - 1) / TW;

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  auto order = [&](int64_t b) { return (b == a.batch - 1) ? a.n_last : a.n; };
  auto issue_load = [&](int64_t t) {
    const int64_t b = gw + t * TW;
    const int nb = order(b);
    double* slot = slots + (t % NS) * LEAF * LEAF;
    uint64_t* bar = &bars[t % NS];
    const double* src = a.A + b * a.sA;
    if (nb == LEAF && a.lda == LEAF) {
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, LEAF * LEAF * 8);
        bulk_g2s(slot, src, LEAF * LEAF * 8, bar);
      }
    } else {
      if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(nb * nb * 8));
      __syncwarp();
      if (lane < nb) bulk_g2s(slot + lane * LEAF, src + lane * a.lda, (uint32_t)(nb * 8), bar);
    }
  };

  for (int64_t t = 0; t < NS - 1 && t < count; ++t) issue_load(t);

  for (int64_t t = 0; t < count; ++t) {
    const int64_t b = gw + t * TW;
    const int nb = order(b);
    double* slot = slots + (t % NS) * LEAF * LEAF;
    mbar_wait(&bars[t % NS], (uint32_t)((t / NS) & 1));

    double x[LEAF];
    bool singular;
    int first_zero;
    leaf_compute<UPPER>(slot, nb, a.unit, lane, x, singular, first_zero);
    __syncwarp();
    leaf_write_slot<UPPER>(slot, lane, x);
    fence_proxy_async_smem();
    __syncwarp();
    double* dst = a.X + b * a.sX;
    if (nb == LEAF && a.ldx == LEAF) {
      if (lane == 0) bulk_s2g(dst, slot, LEAF * LEAF * 8);
    } else {
      if (lane < nb) bulk_s2g(dst + lane * a.ldx, slot + lane * LEAF, (uint32_t)(nb * 8));
    }
    bulk_commit();
    leaf_report(a, b, lane, singular, first_zero);

    const int64_t tn = t + NS - 1;  // refill the slot used by iteration t-1
    if (tn < count) {
      bulk_wait_read<1>();  // the store issued at t-1 has finished reading its slot
      __syncwarp();
      issue_load(tn);
    }
  }
  bulk_wait<0>();
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
    for (int i = 0; i < nb; ++i)
      if (lane < nb) T[i * LEAF + lane] = src[i * a.lda + lane];
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
constexpr int kWarps = 6, kSlots = 4;
constexpr size_t kTmaSmem = (size_t)kWarps * kSlots * LEAF * LEAF * 8 + kWarps * kSlots * 8;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaError_t launch_leaf(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.batch <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool even = (a.n % 2 == 0) && (a.n_last % 2 == 0) && (a.lda % 2 == 0) && (a.ldx % 2 == 0) &&
                    (a.sA % 2 == 0) && (a.sX % 2 == 0);
  const bool tma = even && aligned16(a.A) && aligned16(a.X);
  // algorithmic work: n^3/3 flops and the referenced triangle in + full matrix out per matrix
  const double nn = (double)a.n;
  ProfileScope prof(KIND_LEAF, a.batch * nn * nn * nn / 3.0, a.batch * (nn * (nn + 1) / 2 + nn * nn) * 8.0, s);
  if (tma) {
    const int64_t ctas_needed = (a.batch + kWarps - 1) / kWarps;
    const int grid = (int)(ctas_needed < sms ? ctas_needed : sms);
    if (uplo == 'L') {
      auto k = leaf_tma_kernel<false, kWarps, kSlots>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
      k<<<grid, kWarps * 32, kTmaSmem, s>>>(a);
    } else {
      auto k = leaf_tma_kernel<true, kWarps, kSlots>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
      k<<<grid, kWarps * 32, kTmaSmem, s>>>(a);
    }
  } else {
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
