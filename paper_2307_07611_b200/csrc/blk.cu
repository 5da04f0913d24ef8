// blk.cu — whole-block triangular inverses of order <= 128 in one CTA
// (SURVEY §8(a) rows a1, a2, a4-a7 for small orders; DESIGN.md §8 "blk_kernel").
//
// One CTA inverts one lower (or, by index reversal, upper) block T of order
// nb <= NB (NB = 64 or 128) entirely in shared memory, running the same
// COMBRIT beta = 2 recursion as the multi-launch path (Alg. 1) but
// inside the CTA:
//   1. the referenced triangle is loaded (the other triangle written as +0.0,
//      rows / columns nb..NB-1 padded with the identity: inv([T 0; 0 I]) =
//      [T^-1 0; 0 I]);
//   2. each half-warp inverts one 16-wide diagonal block by the bordering
//      recurrence of the proof of Thm 1 in its right-looking order,
//      lane c = column c in 16 registers, x_k = r_k acc_k, acc_i -= T_ik x_k,
//      with r_k = 1/T_kk (CRIT divides; reading C4);
//   3. for b = 16, 32, 64 (< NB) every merge [A 0; C B] of the level is finished
//      by the two products of the block Thm 1 inverse with one path
//      (P:440-452 = P:1066-1069 transposed): W = C A^-1, then X21 = -B^-1 W,
//      on the FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA) from shared
//      memory, each warp owning 16x16 output tiles whose K-range skips the
//      structurally zero blocks of the triangular factor (P_TF);
//   4. the full nb x nb inverse is stored (opposite triangle +0.0, row a7).
// The shared-memory row stride NB+4 (= 4 mod 16 doubles) makes both DMMA
// fragment patterns (8 rows x 4 k, and 4 k x 8 columns) bank-conflict free.
//
// The upper case inverts T' = J U J (J the index reversal, T'_ik =
// U_{nb-1-i, nb-1-k}, lower) and stores X = J T'^-1 J: CRIT for the upper case
// is the mirror image of the lower recurrence.
//
// Used for single matrices of order 33..128 (BASELINE config 0: one launch),
// batched orders 33..128, and the 128-wide diagonal blocks at the bottom of
// the multi-launch recursion (which then starts its levels at b = 128).
#include <cuda_runtime.h>

#include <utility>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

template <int NB>
struct BlkCfg {
  static constexpr int S = NB + 4;   // X row stride (doubles)
  static constexpr int HB = NB / 2;  // rows of the W buffer (all merges of a level stacked)
  static constexpr int WS = HB + 4;  // W row stride
  static constexpr int WARPS = NB / 16;
  static constexpr int THREADS = WARPS * 32;
  static constexpr size_t SMEM = (size_t)(NB * S + HB * WS) * sizeof(double);
};

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }


// Zero-diagonal report, "min over non-zero" on a single accumulator.
__device__ __forceinline__ void blk_info_min_nonzero(int32_t* p, int32_t v) {
  int32_t old = *reinterpret_cast<volatile int32_t*>(p);
  while (old == 0 || v < old) {
    const int32_t prev = atomicCAS(p, old, v);
    if (prev == old) break;
    old = prev;
  }
}

// ---- step 2: 16-wide diagonal blocks, two per warp ------------------------------------
// Half-warp h of warp w owns diagonal block 2w + h (T at smem, row stride S),
// lane c = column c in 16 registers.  Pairs (k, k+1) per step: x_k = r_k acc_k;
// acc_{k+1} -= T_{k+1,k} x_k; x_{k+1} = r_{k+1} acc_{k+1}; acc_i -= T_ik x_k +
// T_{i,k+1} x_{k+1} (i >= k+2), one 16-byte broadcast per row and half-warp.
// Compile-time indices keep x[] in registers.
template <int S, int K>
__device__ __forceinline__ void blk_leaf_step(const double* T, double (&x)[16]) {
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
template <int S, int... P>
__device__ __forceinline__ void blk_leaf_steps(const double* T, double (&x)[16], std::integer_sequence<int, P...>) {
  (blk_leaf_step<S, 2 * P>(T, x), ...);
}

template <int S>
__device__ __forceinline__ void blk_leaf16(double* T, int c) {
  const double r = 1.0 / T[c * (S + 1)];  // IEEE division: X_jj == 1/T_jj bitwise (C4)
  __syncwarp();
  T[c * (S + 1)] = r;
  __syncwarp();
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (i == c) ? 1.0 : 0.0;
  blk_leaf_steps<S>(T, x, std::make_integer_sequence<int, 8>{});
  __syncwarp();  // every lane has read T before the block is overwritten by X
#pragma unroll
  for (int i = 0; i < 16; ++i) T[i * S + c] = (i < c) ? 0.0 : x[i];
}

// ---- step 3: 16x16 warp tile products from shared memory ----------------------------
// acc += A[16 rows][k0..k1) * B[k0..k1)[16 cols]; A, B row-major (strides SA, SB).
// m8n8k4 fragments (row.col): a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c = {C[lane/4][2(lane%4)], C[lane/4][2(lane%4)+1]}.
template <int SA, int SB>
__device__ __forceinline__ void blk_mma16(double (&acc)[2][2][2], const double* A, const double* B, int k0, int k1,
                                          int lane) {
  const int lr = lane >> 2, lc = lane & 3;
  const double* a = A + lr * SA + lc;
  const double* b = B + lc * SB + lr;
#pragma unroll 4
  for (int k = k0; k < k1; k += 4) {
    const double a0 = a[k], a1 = a[8 * SA + k];
    const double b0 = b[k * SB], b1 = b[k * SB + 8];
    dmma_8x8x4(acc[0][0][0], acc[0][0][1], a0, b0);
    dmma_8x8x4(acc[0][1][0], acc[0][1][1], a0, b1);
    dmma_8x8x4(acc[1][0][0], acc[1][0][1], a1, b0);
    dmma_8x8x4(acc[1][1][0], acc[1][1][1], a1, b1);
  }
}
template <int SC>
__device__ __forceinline__ void blk_store16(double* C, const double (&acc)[2][2][2], double alpha, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
      *reinterpret_cast<double2*>(C + (mi * 8 + lr) * SC + ni * 8 + 2 * lc) =
          make_double2(alpha * acc[mi][ni][0], alpha * acc[mi][ni][1]);
}

// One level of merges [s, s+b) + [s+b, s+2b), s = 2 g b, inside the NB block (b a
// template parameter: the tile bookkeeping below is shifts, not divisions).
template <int NB, int b>
__device__ __forceinline__ void blk_level(double* X, double* W, int warp, int lane) {
  using C = BlkCfg<NB>;
  constexpr int S = C::S, WS = C::WS;
  constexpr int tb = b / 16;              // 16-tiles per side of a merge block
  constexpr int m = NB / (2 * b);         // merges of the level
  constexpr int tiles = m * tb * tb;
  // Tiles are dealt to the warps in snake order of decreasing K-range so that the
  // four SM sub-partitions (warps w and w + 4 share one) get equal DMMA work.
  // W_g = C_g A_g^-1: tile (I, J), k in [16 J, b)  (A^-1 lower)
  constexpr int per = m * tb;  // tiles per K-class
  for (int r = 0; r * C::WARPS < tiles; ++r) {
    const int q = r * C::WARPS + ((r & 1) ? C::WARPS - 1 - warp : warp);  // snake deal, longest K first
    if (q >= tiles) continue;
    const int J = q / per, g = (q % per) / tb, I = q % tb;  // K = b - 16 J
    const int s = 2 * g * b;
    double acc[2][2][2] = {};
    blk_mma16<S, S>(acc, X + (s + b + 16 * I) * S + s, X + s * S + s + 16 * J, 16 * J, b, lane);
    blk_store16<WS>(W + (g * b + 16 * I) * WS + 16 * J, acc, 1.0, lane);
  }
  __syncthreads();
  // X21_g = -B_g^-1 W_g: tile (I, J), k in [0, 16 (I + 1))  (B^-1 lower); overwrites C_g
  for (int r = 0; r * C::WARPS < tiles; ++r) {
    const int q = r * C::WARPS + ((r & 1) ? C::WARPS - 1 - warp : warp);
    if (q >= tiles) continue;
    const int I = tb - 1 - q / per, g = (q % per) / tb, J = q % tb;  // K = 16 (I + 1)
    const int s = 2 * g * b;
    double acc[2][2][2] = {};
    blk_mma16<S, WS>(acc, X + (s + b + 16 * I) * S + s + b, W + (g * b) * WS + 16 * J, 0, 16 * (I + 1), lane);
    blk_store16<S>(X + (s + b + 16 * I) * S + s + 16 * J, acc, -1.0, lane);
  }
  __syncthreads();
}


template <int NB, bool UPPER>
__global__ void __launch_bounds__(BlkCfg<NB>::THREADS) blk_kernel(const LeafArgs a) {
  using C = BlkCfg<NB>;
  constexpr int S = C::S, T = C::THREADS;
  extern __shared__ __align__(16) double blk_smem[];
  double* X = blk_smem;           // [NB][S]
  double* W = blk_smem + NB * S;  // [HB][WS]
  __shared__ int zmin;
  __shared__ __align__(8) uint64_t ldbar;  // completion of the row bulk loads
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_trigger_early();  // no-op by default (ptx.cuh): the first level launch is released as the blocks exit
  if (tid == 0) { mbar_init(&ldbar, 1); fence_mbar_init(); }
  uint32_t ldphase = 0;
#ifdef TRINV_BLK_TIMING  // phase timestamps of the first block (latency study only)
  unsigned long long tt[8];
  int nt = 0;
  auto stamp = [&]() { if (tid == 0 && nt < 8) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[nt++])); };
  stamp();
#else
  auto stamp = [&]() {};
#endif
  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    const int nb = (b == a.batch - 1) ? a.n_last : a.n;
    const double* src = a.A + b * a.sA;
    if (tid == 0) zmin = 1 << 30;
    __syncthreads();
    // 1. load the referenced triangle in T' order; the other triangle +0.0, the unit /
    //    padding diagonal 1.0.  Full orders with 16-byte-aligned rows: column pairs as
    //    16-byte loads into registers (all in flight), then 16-byte shared stores; other
    //    layouts: 8-byte cp.async per element.
    const bool vec = nb == NB && (a.lda & 1) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
    if (vec && !UPPER && NB == 64) {  // 16-byte cp.async per referenced pair, diagonal fix-ups after
      constexpr int PAIRS = NB * NB / 2, PER = PAIRS / T;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = tid + q * T, i = e / (NB / 2), k = 2 * (e % (NB / 2));
        if (k <= i) cp_async16(X + i * S + k, src + (int64_t)i * a.lda + k);
        else *reinterpret_cast<double2*>(X + i * S + k) = make_double2(0.0, 0.0);
      }
      cp_async_wait_all();
      __syncthreads();  // every copy has landed
      for (int i = tid; i < NB; i += T) {  // the diagonal pair of an even row, unit diagonals
        if ((i & 1) == 0) X[i * S + i + 1] = 0.0;
        if (a.unit) X[i * S + i] = 1.0;
      }
    } else if (vec && !UPPER) {  // NB = 128: one bulk copy per row (its referenced prefix rounded up to 16 bytes)
      constexpr uint32_t BYTES = 16u * (NB / 2) * (NB / 2 + 1);  // sum_i 16 ceil((i + 1) / 2)
      if (tid == 0) mbar_arrive_expect_tx(&ldbar, BYTES);
      __syncthreads();
      for (int i = tid; i < NB; i += T) bulk_g2s(X + i * S, src + (int64_t)i * a.lda, 16u * (i / 2 + 1), &ldbar);
      for (int e = tid; e < NB * NB / 2; e += T) {  // the rest of each row: +0.0
        const int i = e / (NB / 2), k = 2 * (e % (NB / 2));
        if (k > i) *reinterpret_cast<double2*>(X + i * S + k) = make_double2(0.0, 0.0);
      }
      mbar_wait(&ldbar, ldphase);
      ldphase ^= 1;
      for (int i = tid; i < NB; i += T) {  // the diagonal pair of an even row, unit diagonals
        if ((i & 1) == 0) X[i * S + i + 1] = 0.0;
        if (a.unit) X[i * S + i] = 1.0;
      }
    } else if (vec) {  // upper: 16-byte loads into registers, pairs swapped into T' order
      constexpr int PAIRS = NB * NB / 2, PER = PAIRS / T;
      double2 v[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {  // pair (i, k), (i, k + 1), k even
        const int e = tid + q * T, i = e / (NB / 2), k = 2 * (e % (NB / 2));
        const bool need = k <= i;  // at least (i, k) referenced
        const int64_t off = UPPER ? (int64_t)(NB - 1 - i) * a.lda + (NB - 2 - k) : (int64_t)i * a.lda + k;
        v[q] = need ? *reinterpret_cast<const double2*>(src + off) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = tid + q * T, i = e / (NB / 2), k = 2 * (e % (NB / 2));
        double x0 = UPPER ? v[q].y : v[q].x, x1 = UPPER ? v[q].x : v[q].y;  // T'(i, k), T'(i, k + 1)
        if (k > i) x0 = 0.0;
        if (k + 1 > i) x1 = 0.0;
        if (a.unit && k == i) x0 = 1.0;  // the unit diagonal is not read
        if (a.unit && k + 1 == i) x1 = 1.0;
        *reinterpret_cast<double2*>(X + i * S + k) = make_double2(x0, x1);
      }
    } else {
#pragma unroll 8
      for (int e = tid; e < NB * NB; e += T) {
        const int i = e / NB, k = e % NB;
        if (i < nb && (k < i || (k == i && !a.unit))) {
          const int64_t off = UPPER ? (int64_t)(nb - 1 - i) * a.lda + (nb - 1 - k) : (int64_t)i * a.lda + k;
          cp_async8(X + i * S + k, src + off);
        } else {
          X[i * S + k] = (k == i) ? 1.0 : 0.0;
        }
      }
      cp_async_wait_all();
    }
    __syncthreads();
    stamp();
    if (tid < nb && !a.unit && X[tid * (S + 1)] == 0.0) atomicMin(&zmin, UPPER ? nb - 1 - tid : tid);
    // 2. 16-wide diagonal leaves, two per warp (half-warp h of warp w: block 2w + h)
    if (warp < NB / 32) blk_leaf16<S>(X + (2 * warp + (lane >> 4)) * 16 * (S + 1), lane & 15);
    __syncthreads();
    stamp();
    // 3. merge levels b = 16, 32, ... < NB
    // lower full blocks with 16-byte aligned rows leave by per-row bulk copies; for NB =
    // 128, rows [0, 64) are final before the last level and go out while it runs (for NB =
    // 64 the early half measured slower: the store phase is latency, not volume)
    double* dst = a.X + b * a.sX;
    const bool bulk_out = !UPPER && nb == NB && (a.ldx & 1) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;
    auto store_rows = [&](int r0, int r1) {
      fence_proxy_async_smem();
      __syncthreads();
      for (int i = r0 + tid; i < r1; i += T) bulk_s2g(dst + (int64_t)i * a.ldx, X + i * S, NB * 8);
      bulk_commit();
    };
    blk_level<NB, 16>(X, W, warp, lane);
    stamp();
    blk_level<NB, 32>(X, W, warp, lane);
    stamp();
    if constexpr (NB > 64) {
      if (bulk_out) store_rows(0, NB / 2);
      blk_level<NB, 64>(X, W, warp, lane);
      stamp();
    }
    // 4. store nb x nb (X = J X' J for the upper case): lower full blocks with 16-byte
    //    aligned rows as one bulk copy per row; otherwise column pairs as 16-byte stores
    //    where the destination is aligned
    if (bulk_out) {
      store_rows(NB == 64 ? 0 : NB / 2, NB);
      bulk_wait_read<0>();  // X is reused by the next matrix
    } else {
#pragma unroll 4
    for (int e = tid; e < NB * NB / 2; e += T) {
      const int i = e / (NB / 2), k = 2 * (e % (NB / 2));
      if (i < nb && k < nb) {
        const double2 v = *reinterpret_cast<const double2*>(X + i * S + k);
        const double v0 = v.x, v1 = v.y;
        if (!UPPER) {
          double* q = dst + (int64_t)i * a.ldx + k;
          if (k + 1 < nb && (reinterpret_cast<uintptr_t>(q) & 15u) == 0) {
            *reinterpret_cast<double2*>(q) = make_double2(v0, v1);
          } else {
            q[0] = v0;
            if (k + 1 < nb) q[1] = v1;
          }
        } else {
          double* q = dst + (int64_t)(nb - 1 - i) * a.ldx + (nb - 1 - k);  // column nb-1-k, then nb-2-k
          if (k + 1 < nb && (reinterpret_cast<uintptr_t>(q - 1) & 15u) == 0) {
            *reinterpret_cast<double2*>(q - 1) = make_double2(v1, v0);
          } else {
            q[0] = v0;
            if (k + 1 < nb) q[-1] = v1;
          }
        }
      }
    }
    }
#ifdef TRINV_BLK_TIMING
    __syncthreads();
    stamp();
    if (tid == 0 && blockIdx.x == 0 && b == 0)
      printf("blk<%d> ns: load %llu leaves %llu levels %llu %llu %llu store %llu\n", NB, tt[1] - tt[0], tt[2] - tt[1],
             tt[3] - tt[2], nt > 5 ? tt[4] - tt[3] : 0ull, nt > 6 ? tt[5] - tt[4] : 0ull, tt[nt - 1] - tt[nt - 2]);
#endif
    if (tid == 0) {
      const int z = zmin;
      const bool singular = z < nb;
      if (a.info_mode == 1) a.info[b] = singular ? z + 1 : 0;
      else if (a.info_mode == 2 && singular)
        blk_info_min_nonzero(a.info, static_cast<int32_t>(a.info_off + b * a.info_stride + z + 1));
    }
    __syncthreads();
  }
}

template <int NB>
static cudaError_t launch_blk_nb(char uplo, const LeafArgs& a, cudaStream_t s) {
  using C = BlkCfg<NB>;
  const int per_sm = (int)((227 * 1024) / (C::SMEM + 1024));
  const int64_t cap = (int64_t)device_sms() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(a.batch < cap ? a.batch : cap);
  if (uplo == 'L') {
    constexpr auto k = blk_kernel<NB, false>;
    set_smem_once<k>((int)C::SMEM);
    k<<<grid, C::THREADS, C::SMEM, s>>>(a);
  } else {
    constexpr auto k = blk_kernel<NB, true>;
    set_smem_once<k>((int)C::SMEM);
    k<<<grid, C::THREADS, C::SMEM, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_blk(char uplo, const LeafArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.batch <= 0) return cudaSuccess;
  const int nmax = a.n > a.n_last ? a.n : a.n_last;
  if (nmax > BLK_MAX) return cudaErrorInvalidValue;
  const double nn = (double)a.n;
  ProfileScope prof(KIND_LEAF, a.batch * nn * nn * nn / 3.0, a.batch * (nn * (nn + 1) / 2 + nn * nn) * 8.0, s);
  const cudaError_t e = nmax <= 64 ? launch_blk_nb<64>(uplo, a, s) : launch_blk_nb<128>(uplo, a, s);
  if (e == cudaSuccess && launches) ++*launches;
  return e;
}

}  // namespace trinv
