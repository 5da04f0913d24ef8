// leaf64.cu — batched 64 x 64 triangular inverses, one warp per matrix, with
// TMA-staged triangle loads (SURVEY §8(a) rows a1-a3 for 64-wide blocks;
// DESIGN.md §8 "leaf64_tma_kernel").
//
// The arithmetic is that of the 32-wide leaf (leaf.cu): the bordering
// recurrence of the proof of Thm 1, [R v; 0 1]^{-1} = [S -Sv; 0 1],
// in its right-looking order x_k = r_k acc_k, acc_i -= T_ik x_k (i > k), with
// r_k = 1/T_kk (CRIT's division, as a correctly rounded reciprocal,
// reading C4).  Columns are independent: lane j owns columns j
// and j + 32 of X, i.e. x0[0..63] (rows of column j) and x1[0..31] (rows 32..63
// of column j + 32, whose rows above 32 are structurally zero), both driven by
// the same shared-memory broadcasts of T.  The upper case runs the same code on
// T' = J U J (J = index reversal), as in leaf.cu.
//
// HBM staging: the referenced triangle arrives as four 16-row bands of widths
// 16/32/48/64 (lower; 64/48/32/16 for upper) by 2-D TMA over a 3-D
// [batch][64][64] view (20 KiB per matrix instead of 32), into an NS-deep ring
// of slots per warp completing on per-slot mbarriers; the full 64 x 64 inverse
// leaves through coalesced 256-byte row stores (opposite triangle +0.0).
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

constexpr int L64N = 64;
constexpr int kSlot64 = 2560;  // doubles per slot: 16 x (16 + 32 + 48 + 64)

// Band layout of a slot.  Lower: band b = rows 16b..16b+15, columns 0..16b+15.
// Upper: band b = rows 16b..16b+15, columns 16b..63.
__host__ __device__ constexpr int lo_off(int b) { return 128 * b * (b + 1); }          // 16 * 16 * (0+1+..+b)
__host__ __device__ constexpr int up_off(int b) { return 16 * (64 * b - 8 * b * (b - 1)); }  // 16 * sum (64 - 16 b')
__device__ __forceinline__ int lidx64(int i, int k) { return lo_off(i >> 4) + (i & 15) * (16 * ((i >> 4) + 1)) + k; }
__device__ __forceinline__ int uidx64(int r, int c) {
  return up_off(r >> 4) + (r & 15) * (64 - 16 * (r >> 4)) + (c - 16 * (r >> 4));
}

template <bool UPPER>
__device__ __forceinline__ double2 tri64_pair(const double* T, int i, int k) {  // (T'_ik, T'_i,k+1), k even
  if (!UPPER) return *reinterpret_cast<const double2*>(T + lidx64(i, k));
  const double2 v = *reinterpret_cast<const double2*>(T + uidx64(63 - i, 62 - k));
  return make_double2(v.y, v.x);
}
template <bool UPPER>
__device__ __forceinline__ double tri64_sub(const double* T, int k) {  // T'_{k+1,k}, k even
  return UPPER ? T[uidx64(62 - k, 63 - k)] : T[lidx64(k + 1, k)];
}
template <bool UPPER>
__device__ __forceinline__ double tri64_diag(const double* T, int i) {  // T_ii, original index
  return UPPER ? T[uidx64(i, i)] : T[lidx64(i, i)];
}

// One paired step (k, k+1) on both columns of the lane: x0 = rows 0..63 of column
// j, x1 = rows 32..63 of column j + 32 (steps k >= 32 only).
template <bool UPPER, int K>
__device__ __forceinline__ void leaf64_step(const double* T, const double* rr, double (&x0)[64], double (&x1)[32]) {
  const double2 r = *reinterpret_cast<const double2*>(rr + K);
  const double t10 = tri64_sub<UPPER>(T, K);
  const double xk = x0[K] * r.x;
  x0[K] = xk;
  x0[K + 1] = fma(-t10, xk, x0[K + 1]);
  const double xk1 = x0[K + 1] * r.y;
  x0[K + 1] = xk1;
  double yk = 0.0, yk1 = 0.0;
  if constexpr (K >= 32) {
    yk = x1[K - 32] * r.x;
    x1[K - 32] = yk;
    x1[K - 31] = fma(-t10, yk, x1[K - 31]);
    yk1 = x1[K - 31] * r.y;
    x1[K - 31] = yk1;
  }
#pragma unroll
  for (int i = K + 2; i < L64N; ++i) {
    const double2 t = tri64_pair<UPPER>(T, i, K);
    x0[i] = fma(-t.x, xk, x0[i]);
    x0[i] = fma(-t.y, xk1, x0[i]);
    if constexpr (K >= 32) {
      x1[i - 32] = fma(-t.x, yk, x1[i - 32]);
      x1[i - 32] = fma(-t.y, yk1, x1[i - 32]);
    }
  }
}
template <bool UPPER, int... P>
__device__ __forceinline__ void leaf64_steps(const double* T, const double* rr, double (&x0)[64], double (&x1)[32],
                                             std::integer_sequence<int, P...>) {
  (leaf64_step<UPPER, 2 * P>(T, rr, x0, x1), ...);
}

template <bool UPPER, int WARPS, int NS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    leaf64_tma_kernel(const __grid_constant__ CUtensorMap m16, const __grid_constant__ CUtensorMap m32,
                      const __grid_constant__ CUtensorMap m48, const __grid_constant__ CUtensorMap m64,
                      const LeafArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slots = reinterpret_cast<double*>(smem_raw) + (size_t)warp * NS * kSlot64;
  double* rr = reinterpret_cast<double*>(smem_raw) + (size_t)WARPS * NS * kSlot64 + warp * L64N;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_raw + ((size_t)WARPS * NS * kSlot64 + WARPS * L64N) * 8) + warp * NS;

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t TW = (int64_t)gridDim.x * WARPS;
  if (gw >= a.batch) return;
  const int64_t count = (a.batch - gw + TW - 1) / TW;

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (lane == 0 && warp == 0) {
    tma_prefetch_desc(&m16);
    tma_prefetch_desc(&m32);
    tma_prefetch_desc(&m48);
    tma_prefetch_desc(&m64);
  }
  __syncwarp();

  auto issue_load = [&](int64_t t) {  // lane 0 only
    const int b = (int)(gw + t * TW);
    double* slot = slots + (t % NS) * kSlot64;
    uint64_t* bar = &bars[t % NS];
    mbar_arrive_expect_tx(bar, kSlot64 * 8);
    if (!UPPER) {
      tma_load_3d(slot + lo_off(0), &m16, 0, 0, b, bar);
      tma_load_3d(slot + lo_off(1), &m32, 0, 16, b, bar);
      tma_load_3d(slot + lo_off(2), &m48, 0, 32, b, bar);
      tma_load_3d(slot + lo_off(3), &m64, 0, 48, b, bar);
    } else {
      tma_load_3d(slot + up_off(0), &m64, 0, 0, b, bar);
      tma_load_3d(slot + up_off(1), &m48, 16, 16, b, bar);
      tma_load_3d(slot + up_off(2), &m32, 32, 32, b, bar);
      tma_load_3d(slot + up_off(3), &m16, 48, 48, b, bar);
    }
  };
  if (lane == 0)
    for (int64_t t = 0; t < NS && t < count; ++t) issue_load(t);

  for (int64_t t = 0; t < count; ++t) {
    const int64_t b = gw + t * TW;
    double* slot = slots + (t % NS) * kSlot64;
    mbar_wait(&bars[t % NS], (uint32_t)((t / NS) & 1));

    // a1: reciprocals of the diagonal (T' order), zero-diagonal report (original index)
    const double d0 = tri64_diag<UPPER>(slot, lane), d1 = tri64_diag<UPPER>(slot, lane + 32);
    const unsigned z0 = __ballot_sync(0xffffffffu, !a.unit && d0 == 0.0);
    const unsigned z1 = __ballot_sync(0xffffffffu, !a.unit && d1 == 0.0);
    const int first_zero = z0 ? __ffs(z0) - 1 : (z1 ? 32 + __ffs(z1) - 1 : -1);
    rr[UPPER ? 63 - lane : lane] = a.unit ? 1.0 : 1.0 / d0;  // IEEE division: X_jj == 1/T_jj bitwise (C4)
    rr[UPPER ? 31 - lane : lane + 32] = a.unit ? 1.0 : 1.0 / d1;
    __syncwarp();

    double x0[64], x1[32];
#pragma unroll
    for (int i = 0; i < 64; ++i) x0[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x1[i] = (i == lane) ? 1.0 : 0.0;
    leaf64_steps<UPPER>(slot, rr, x0, x1, std::make_integer_sequence<int, 32>{});
    __syncwarp();  // every lane has finished reading the slot and rr
    if (t + NS < count && lane == 0) {
      fence_proxy_async_smem();
      issue_load(t + NS);
    }
    // a3/a7: full 64 x 64 inverse, coalesced 256-byte row segments, opposite triangle +0.0
    double* dst = a.X + b * a.sX;
    const int c0 = UPPER ? 63 - lane : lane, c1 = UPPER ? 31 - lane : lane + 32;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const int row = UPPER ? 63 - i : i;
      dst[(int64_t)row * a.ldx + c0] = (i < lane) ? 0.0 : x0[i];
      dst[(int64_t)row * a.ldx + c1] = (i < 32 + lane) ? 0.0 : x1[i >= 32 ? i - 32 : 0];
    }
    if (a.info_mode == 1) {
      if (lane == 0) a.info[b] = first_zero >= 0 ? first_zero + 1 : 0;
    } else if (a.info_mode == 2 && first_zero >= 0 && lane == 0) {
      const int32_t v = static_cast<int32_t>(a.info_off + b * a.info_stride + first_zero + 1);
      int32_t old = *reinterpret_cast<volatile int32_t*>(a.info);
      while (old == 0 || v < old) {
        const int32_t prev = atomicCAS(a.info, old, v);
        if (prev == old) break;
        old = prev;
      }
    }
  }
}

// 3-D view [batch][64 rows][64 cols]; box = 16 rows x `cols` columns x 1 matrix.
static bool encode_map64(CUtensorMap* m, const LeafArgs& a, int cols) {
  const uint64_t dims[3] = {64, 64, (uint64_t)a.batch};
  const uint64_t strides[2] = {(uint64_t)a.lda * 8, (uint64_t)a.sA * 8};
  const uint32_t box[3] = {(uint32_t)cols, 16, 1};
  return encode_map_nd(m, a.A, 3, dims, strides, box);
}

template <int W, int NS>
static cudaError_t launch64(char uplo, const CUtensorMap (&m)[4], const LeafArgs& a, cudaStream_t s) {
  constexpr size_t smem = ((size_t)W * NS * kSlot64 + W * L64N) * 8 + W * NS * 8;
  const int64_t ctas_needed = (a.batch + W - 1) / W;
  const int sms = device_sms();
  const int grid = (int)(ctas_needed < sms ? ctas_needed : sms);
  if (uplo == 'L') {
    constexpr auto k = leaf64_tma_kernel<false, W, NS>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(m[0], m[1], m[2], m[3], a);
  } else {
    constexpr auto k = leaf64_tma_kernel<true, W, NS>;
    set_smem_once<k>((int)smem);
    k<<<grid, W * 32, smem, s>>>(m[0], m[1], m[2], m[3], a);
  }
  return cudaGetLastError();
}

bool leaf64_tma_ok(const LeafArgs& a) {
  const bool even = (a.lda % 2 == 0) && (a.ldx % 2 == 0) && (a.sA % 2 == 0) && (a.sX % 2 == 0);
  // one warp per matrix pays off only for batches that fill the machine; below that the
  // one-CTA-per-matrix kernel (blk.cu) has the lower latency (single matrix: ~9.7 vs ~14 us)
  return a.n == L64N && a.n_last == L64N && even && (reinterpret_cast<uintptr_t>(a.A) & 15u) == 0 &&
         (reinterpret_cast<uintptr_t>(a.X) & 15u) == 0 && a.batch >= 4096 && a.batch < ((int64_t)1 << 31);
}

cudaError_t launch_leaf64_tma(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.batch <= 0) return cudaSuccess;
  CUtensorMap m[4];
  for (int i = 0; i < 4; ++i)
    if (!encode_map64(&m[i], a, 16 * (i + 1))) return cudaErrorInvalidValue;
  const double nn = 64.0;
  ProfileScope prof(KIND_LEAF, a.batch * nn * nn * nn / 3.0, a.batch * (nn * (nn + 1) / 2 + nn * nn) * 8.0, s);
  // 8 warps x 1 slot per CTA (one CTA per SM): measured best of 4x2, 5x2, 6x1, 8x1, 3x3
  // (profiles/r01_sweep_batched.txt)
  const cudaError_t e = launch64<8, 1>(uplo, m, a, s);
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace trinv
