// oz2.cu — FP64 products on the INT8 tensor cores by modular arithmetic (a
// CRT-based Ozaki-type scheme, "Ozaki scheme II"): the default product engine for
// blocks >= 2048 (DESIGN.md §8 "oz2_gemm_kernel", §11), 16 int8 GEMMs per FP64
// product instead of the 36 digit products of oz.cu.
//
// Scaling.  Row i of A is scaled by 2^(P - e_i), 2^e_i > max_k |a_ik|, and truncated:
// A'_ik = trunc(a_ik 2^(P - e_i)), an exact integer with |A'| < 2^P (a_ik has 53
// significant bits, the scaling is a power of two); columns of B likewise (f_j).
// Then C' = A' B' is an exact integer matrix with |C'| < K 2^(2P).
// Residues.  With 16 pairwise coprime moduli m_i <= 256 (M = prod m_i ~ 2^125.4),
// A'_i = A' mod m_i in [0, m_i) (uint8) and B'_i likewise (K <= 32768) or in the symmetric
// range (int8, larger K), the tensor cores give C'_i = A'_i B'_i exactly in int32 (|.| <=
// 255^2 K or 255 * 128 K, < 2^31), reduced mod m_i by the epilogue.
// Reconstruction.  The CRT sum sum_i C'_i w_i (w_i the CRT basis of M) is congruent to
// C' mod M, i.e. C' / M == sum_i C'_i y_i / m_i (mod 1); as |C'| < M/2 by a margin (P
// chosen from K: 2P + log2 K < log2 M - 1), C' / M is that fraction's representative in
// [-1/2, 1/2), evaluated in 96-bit fixed point (error 2^-85, far below the truncation):
//     (A B)_ij ~= 2^(e_i - P) 2^(f_j - P) C'_ij,
// the only errors being the truncation of the scaled operands (2^-P relative to the
// row / column maxima) and the final rounding to FP64.
//
// The GEMM kernel is the engine of oz.cu (TMA 128B-swizzled K blocks, tcgen05.mma
// kind::i8, two TMEM accumulators) looping over the 16 moduli instead of digit pairs;
// its epilogue writes uint8 residues, and a separate kernel reconstructs C.  Products
// with all dimensions >= 8192 use the CTA-pair variant (tcgen05.mma.cta_group::2 over
// two SMs, M 256 x N 256 tiles).  The scaling and residue kernels split only the K
// range each tile reads of a triangular operand.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

constexpr int OZ2_NMOD = 16;
#ifndef OZ2_GROUP
#define OZ2_GROUP 8
#endif
constexpr int OZ2_TM = 128, OZ2_TN = 256, OZ2_TK = 128, OZ2_STAGES = 4, OZ2_GROUP_M = OZ2_GROUP;
constexpr int OZ2_A_BYTES = OZ2_TM * OZ2_TK, OZ2_B_BYTES = OZ2_TN * OZ2_TK, OZ2_STAGE = OZ2_A_BYTES + OZ2_B_BYTES;
constexpr size_t OZ2_SMEM = (size_t)OZ2_STAGES * OZ2_STAGE + 1024 + 256;
constexpr int OZ2_THREADS = 192;
constexpr int OZ2_CMAX_ROWS = 128;
constexpr int OZ2_U8_MAXK = 32768;  // u8 x u8 products up to this K (255^2 K < 2^31), else u8 x s8
  // rows per block of the column-maximum kernel

// pairwise coprime, <= 256 (symmetric residues fit int8)
__host__ __device__ constexpr int oz2_mod(int i) {
  constexpr int m[OZ2_NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
  return m[i];
}
__host__ __device__ constexpr int oz2_inv(int a, int m) {  // a^-1 mod m (a, m coprime), extended Euclid
  int t = 0, nt = 1, r = m, nr = a % m;
  while (nr != 0) {
    const int q = r / nr;
    const int tt = t - q * nt; t = nt; nt = tt;
    const int rr = r - q * nr; r = nr; nr = rr;
  }
  return t < 0 ? t + m : t;
}

// ---- residues of the scaled operands ------------------------------------------------
// A row / column holding a NaN or Inf gets the exponent OZ2_NONFINITE: its entries are
// split as zeros and the reconstruction writes NaN over that row / column of the product
// (an FP64 product would carry NaN / Inf there: NaN x 0 and Inf x 0 are NaN).
constexpr int OZ2_NONFINITE = 1 << 20;
__device__ __forceinline__ int oz2_exp_above(double m) {
  if (m == 0.0) return 0;
  if (!(m <= 1.7976931348623157e308)) return OZ2_NONFINITE;  // NaN or Inf
  int e;
  frexp(m, &e);
  return e;
}
// maximum of magnitudes that propagates NaN (fmax drops it)
__device__ __forceinline__ double oz2_amax(double m, double x) {
  const double a = fabs(x);
  return (a > m || a != a) ? a : m;
}
// x 2^k: one multiplication by an exact power of two in the normal range (exact unless
// the result is subnormal, then one rounding, as ldexp), else ldexp.
__device__ __forceinline__ double oz2_ldexp(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * __longlong_as_double((long long)(k + 1023) << 52);
  return ldexp(x, k);
}
// Residues of an integer |v| < 2^58 (P <= 58) for all 16 moduli from three chunks of
// u = v + 2^59 (0 < u < 2^60): u = lo + mid 2^20 + hi 2^40, so with c1 = 2^20 mod m,
// c2 = 2^40 mod m, s = lo + c1 mid + c2 hi + D < 2^29 is congruent to v + h (h = floor(m/2),
// D = (h - 2^59) mod m), and (s mod m) - h is the residue of v in [-h, m - 1 - h]:
// [-128, 127] for m = 256, [-(m-1)/2, (m-1)/2] for odd m; its low byte is the int8 residue.
// The A operand takes the plain residue in [0, m - 1] (uint8, h = 0: one instruction less
// per residue): |sum_k a_k b_k| <= 255 * 128 * K < 2^31 for K <= 65536; so does the B
// operand when K <= OZ2_U8_MAXK (255^2 K < 2^31).
struct Oz2Chunks {
  uint32_t lo, mid, hi;
};
__device__ __forceinline__ Oz2Chunks oz2_chunks(int64_t v) {
  const uint64_t u = (uint64_t)(v + (1ll << 59));
  return {(uint32_t)u & 0xFFFFFu, (uint32_t)(u >> 20) & 0xFFFFFu, (uint32_t)(u >> 40)};
}
template <int I, bool Sym>
__device__ __forceinline__ uint32_t oz2_residue(const Oz2Chunks& x) {
  constexpr uint32_t m = (uint32_t)oz2_mod(I), h = Sym ? m / 2 : 0;
  constexpr uint32_t c1 = (uint32_t)((1ull << 20) % m), c2 = (uint32_t)((1ull << 40) % m);
  constexpr uint32_t D = (uint32_t)((h + m - (uint32_t)((1ull << 59) % m)) % m);
  const uint32_t s = x.lo + x.mid * c1 + x.hi * c2 + D;
  return s % m - h;
}
__device__ __forceinline__ uint32_t oz2_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// residues of 4 consecutive values, packed one 32-bit word per modulus plane
template <bool Sym, int... I>
__device__ __forceinline__ void oz2_residues4(const int64_t (&v)[4], uint32_t* out, size_t stride_words,
                                              std::integer_sequence<int, I...>) {
  Oz2Chunks x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = oz2_chunks(v[q]);
  ((out[I * stride_words] = oz2_pack4(oz2_residue<I, Sym>(x[0]), oz2_residue<I, Sym>(x[1]),
                                      oz2_residue<I, Sym>(x[2]), oz2_residue<I, Sym>(x[3]))),
   ...);
}

// The K range the GEMM reads for row i of a triangular A (tile rows of OZ2_TM) or column
// j of a triangular B (tile columns of OZ2_TN), oz2_gemm_kernel's kb..ke: only that range
// is scaled and split (the rest of a triangular operand is zero and never read).
__device__ __forceinline__ void oz2_k_range(int tri, bool is_a, int idx, int K, int& kb, int& ke, int tma = OZ2_TM) {
  const int tile = is_a ? tma : OZ2_TN;
  const bool upto = is_a ? tri == TRI_LOWER : tri == TRI_UPPER;  // k < end of idx's tile
  const bool from = is_a ? tri == TRI_UPPER : tri == TRI_LOWER;  // k >= start of idx's tile
  kb = from ? (idx / tile) * tile : 0;
  ke = upto ? min(K, (idx / tile + 1) * tile) : K;
}
// A operand (rows x K, row-major): one warp per row; exponent e_i of the row maximum;
// each lane converts 4 consecutive entries per step (K % 4 == 0).
__global__ void oz2_split_rows_kernel(const double* A, int64_t lda, int rows, int K, int tri, bool strict, int P,
                                      int tma, int8_t* out, int* expo) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  int kb, ke;
  oz2_k_range(tri, true, warp, K, kb, ke, tma);  // the K range of the GEMM's row tile (tma rows)
  const double* a = A + (int64_t)warp * lda;
  double m = 0.0;
  const int kz = strict ? warp : -1;  // a diagonal read as zero
  const bool vec = (reinterpret_cast<uintptr_t>(a) & 15) == 0;  // kb is a multiple of 128
  if (vec) {
    double m1 = 0.0;
#pragma unroll 4
    for (int k = kb + 2 * lane; k < ke; k += 64) {
      const double2 x = *reinterpret_cast<const double2*>(a + k);
      m = k == kz ? m : oz2_amax(m, x.x);
      m1 = k + 1 == kz ? m1 : oz2_amax(m1, x.y);
    }
    m = oz2_amax(m, m1);
  } else {
#pragma unroll 4
    for (int k = kb + lane; k < ke; k += 32) m = k == kz ? m : oz2_amax(m, a[k]);
  }
  for (int o = 16; o; o >>= 1) m = oz2_amax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int e = oz2_exp_above(m);
  if (lane == 0) expo[warp] = e;
  const size_t sw = (size_t)rows * K / 4;  // plane stride in 32-bit words
  uint32_t* o = reinterpret_cast<uint32_t*>(out) + (size_t)warp * K / 4;
  for (int k = kb + 4 * lane; k < ke; k += 128) {
    double x[4];
    if (vec) {
      const double2 x01 = *reinterpret_cast<const double2*>(a + k), x23 = *reinterpret_cast<const double2*>(a + k + 2);
      x[0] = x01.x; x[1] = x01.y; x[2] = x23.x; x[3] = x23.y;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = a[k + q];
    }
    int64_t v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)  // exact, truncated (a non-finite row is split as zeros)
      v[q] = (k + q == kz || e == OZ2_NONFINITE) ? 0 : (int64_t)oz2_ldexp(x[q], P - e);
    oz2_residues4<false>(v, o + k / 4, sw, std::make_integer_sequence<int, OZ2_NMOD>{});  // uint8 residues
  }
}
__global__ void oz2_colmax_kernel(const double* B, int64_t ldb, int K, int cols, int tri, bool strict,
                                  unsigned long long* maxbits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  int kb, ke;
  oz2_k_range(tri, false, j, K, kb, ke);
  const int k0 = max(kb, (int)blockIdx.y * OZ2_CMAX_ROWS), k1 = min(ke, (int)(blockIdx.y + 1) * OZ2_CMAX_ROWS);
  double m = 0.0;
  const int kz = strict ? j : -1;
  const double* b = B + j;
  int k = k0;
  for (; k + 8 <= k1; k += 8) {  // 8 independent loads in flight per thread
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = b[(int64_t)(k + u) * ldb];
#pragma unroll
    for (int u = 0; u < 8; ++u) m = k + u == kz ? m : oz2_amax(m, x[u]);
  }
  for (; k < k1; ++k) m = k == kz ? m : oz2_amax(m, b[(int64_t)k * ldb]);
  if (k0 < k1) atomicMax(&maxbits[j], (unsigned long long)__double_as_longlong(m));
}
// B operand (K x cols): residues written transposed (cols x K, K-major) through a
// 32 (k) x 32 (j) tile of scaled integers; thread t converts k0 + 4 (t % 8) .. +3 of
// column j0 + t / 8 and stores one 32-bit word per modulus plane.  Tiles outside the
// GEMM's K range (a 32-column tile lies in one OZ2_TN column tile) are skipped.
__global__ void __launch_bounds__(256, 8) oz2_split_cols_kernel(const double* B, int64_t ldb, int K, int cols, int tri,
                                                             bool strict, int P, const unsigned long long* maxbits,
                                                             int* expo, int8_t* out) {
  __shared__ long long tile[32][33];
  const int k0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int jx = j0 + tx;
  const int e = jx < cols ? oz2_exp_above(__longlong_as_double((long long)maxbits[jx])) : 0;
  if (blockIdx.y == 0 && ty == 0 && jx < cols) expo[jx] = e;
  int kb, ke;
  oz2_k_range(tri, false, j0, K, kb, ke);
  if (k0 + 32 <= kb || k0 >= ke) return;
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r;
    tile[r][tx] = (k < K && jx < cols && !(strict && k == jx) && e != OZ2_NONFINITE)
                      ? (long long)oz2_ldexp(B[(int64_t)k * ldb + jx], P - e)
                      : 0;
  }
  __syncthreads();
  const int j = j0 + (threadIdx.x >> 3), kq = 4 * (threadIdx.x & 7), k = k0 + kq;
  if (j < cols && k < K) {
    const int64_t v[4] = {tile[kq][j - j0], tile[kq + 1][j - j0], tile[kq + 2][j - j0], tile[kq + 3][j - j0]};
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + ((size_t)j * K + k) / 4;
    if (K > OZ2_U8_MAXK)
      oz2_residues4<true>(v, o, (size_t)cols * K / 4, std::make_integer_sequence<int, OZ2_NMOD>{});
    else
      oz2_residues4<false>(v, o, (size_t)cols * K / 4, std::make_integer_sequence<int, OZ2_NMOD>{});
  }
}

// ---- the int8 tensor-core engine, one exact product per modulus -----------------------
__device__ __forceinline__ uint64_t oz2_smem_desc(const void* p) {
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

struct Oz2Params {
  int M, N, K;
  int triA, triB;
  uint8_t* R;  // residues [16][M][N]
  int tiles_n;
  int msplit;  // CTAs per output tile, each running OZ2_NMOD / msplit consecutive moduli
};

__global__ void __launch_bounds__(OZ2_THREADS, 1)
    oz2_gemm_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, const Oz2Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;
  unsigned char* sB = base + OZ2_STAGES * OZ2_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + OZ2_STAGES * OZ2_STAGE);
  uint64_t* empty = full + OZ2_STAGES;
  uint64_t* acc_full = empty + OZ2_STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = p.M / OZ2_TM;
  const int t = blockIdx.x / p.msplit;
  const int nmod = OZ2_NMOD / p.msplit, mod0 = (blockIdx.x % p.msplit) * nmod;
  // grouped rasterisation: groups of OZ2_GROUP_M row tiles (dense, or B triangular), or
  // of OZ2_GROUP_M column tiles when only A is triangular (its K-range varies along the
  // rows; measured DRAM reads at n = 32768, profiles/r01_oz2_raster.txt)
  int I, J;
  if (p.triA != TRI_NONE && p.triB == TRI_NONE) {
    const int per_group = OZ2_GROUP_M * tiles_m;
    const int first_n = (t / per_group) * OZ2_GROUP_M;
    const int gsz = min(p.tiles_n - first_n, OZ2_GROUP_M);
    J = first_n + (t % per_group) % gsz;
    I = (t % per_group) / gsz;
  } else {
    const int per_group = OZ2_GROUP_M * p.tiles_n;
    const int first_m = (t / per_group) * OZ2_GROUP_M;
    const int gsz = min(tiles_m - first_m, OZ2_GROUP_M);
    I = first_m + (t % per_group) % gsz;
    J = (t % per_group) / gsz;
  }
  if (p.triA == TRI_LOWER) I = tiles_m - 1 - I;
  if (p.triB == TRI_UPPER) J = p.tiles_n - 1 - J;
  int kb = 0, ke = p.K;
  if (p.triA == TRI_LOWER) ke = min(ke, (I + 1) * OZ2_TM);
  if (p.triA == TRI_UPPER) kb = I * OZ2_TM;
  if (p.triB == TRI_LOWER) kb = max(kb, J * OZ2_TN);  // both triangular (U^-1 L^-1): k >= max(i, j)
  if (p.triB == TRI_UPPER) ke = min(ke, (J + 1) * OZ2_TN);
  const int nkb = ke > kb ? (ke - kb) / OZ2_TK : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ2_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], 4); }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * OZ2_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // TMA producer: moduli, K-blocks
    tma_prefetch_desc(&ma);
    tma_prefetch_desc(&mb);
    int it = 0;
    for (int i = mod0; i < mod0 + nmod; ++i)
      for (int kk = 0; kk < nkb; ++kk, ++it) {
        const int st = it % OZ2_STAGES, use = it / OZ2_STAGES;
        if (use > 0) mbar_wait(&empty[st], (uint32_t)((use - 1) & 1));
        mbar_arrive_expect_tx(&full[st], OZ2_STAGE);
        const int k = kb + kk * OZ2_TK;
        tma_load_2d(sA + st * OZ2_A_BYTES, &ma, k, i * p.M + I * OZ2_TM, &full[st]);
        tma_load_2d(sB + st * OZ2_B_BYTES, &mb, k, i * p.N + J * OZ2_TN, &full[st]);
      }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc =
        (2u << 4) | (p.K > OZ2_U8_MAXK ? 1u << 10 : 0u) | ((uint32_t)(OZ2_TN >> 3) << 17) |
        ((uint32_t)(OZ2_TM >> 4) << 24);  // u8 x u8 (u8 x s8 above OZ2_U8_MAXK) -> s32
    int it = 0;
    for (int i = mod0; i < mod0 + nmod; ++i) {
      const int buf = (i - mod0) & 1, use = (i - mod0) >> 1;
      if (use > 0) {
        mbar_wait(&acc_empty[buf], (uint32_t)((use - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
      const uint32_t tacc = tmem + (uint32_t)(buf * OZ2_TN);
      bool first = true;
      for (int kk = 0; kk < nkb; ++kk, ++it) {
        const int st = it % OZ2_STAGES;
        mbar_wait(&full[st], (uint32_t)((it / OZ2_STAGES) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t da = oz2_smem_desc(sA + st * OZ2_A_BYTES), db = oz2_smem_desc(sB + st * OZ2_B_BYTES);
#pragma unroll
        for (int k = 0; k < OZ2_TK / 32; ++k) {
          const uint32_t acc = first ? 0u : 1u;
          first = false;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tacc),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&empty[st]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&acc_full[buf]))
                   : "memory");
    }
  }
  if (warp >= 2) {  // epilogue: residues C'_i = (A'_i B'_i) mod m_i as uint8
    const int q4 = warp & 3;
    const int row = I * OZ2_TM + q4 * 32 + lane;
    for (int i = mod0; i < mod0 + nmod; ++i) {
      const int buf = (i - mod0) & 1, use = (i - mod0) >> 1;
      mbar_wait(&acc_full[buf], (uint32_t)(use & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int m = oz2_mod(i);
      const double rm = 1.0 / m;
      uint8_t* dst = p.R + ((size_t)i * p.M + row) * p.N + J * OZ2_TN;
#pragma unroll 1
      for (int c = 0; c < OZ2_TN; c += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * OZ2_TN + c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          uint32_t w = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int x = nkb ? (int)v[j + b] : 0;
            int r = x - (int)floor((double)x * rm) * m;  // exact quotient for |x| < 2^31 up to one step
            r += (r < 0) ? m : 0;
            r -= (r >= m) ? m : 0;
            w |= (uint32_t)r << (8 * b);
          }
          packed[j / 4] = w;
        }
        *reinterpret_cast<uint4*>(dst + c) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint4*>(dst + c + 16) = make_uint4(packed[4], packed[5], packed[6], packed[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * OZ2_TN));
}

// ---- CTA-pair variant (cta_group::2): one 256 x 256 tile per cluster of two CTAs ------
// Each CTA of the pair stages its 128 rows of A and its 128 columns of B per K block
// (32 KB per stage instead of 48: 6 stages in the same shared memory, i.e. twice the
// bytes in flight per output row), the leader CTA issues tcgen05.mma.cta_group::2
// (M 256, N 256, K 32) over both CTAs' shared memory, each CTA's TMEM holds its 128
// rows x 256 columns.  Protocol: both producers' TMA complete on the leader's full
// barrier (which the leader arms with both halves' bytes); the leader's commits arrive
// on the empty / acc_full barriers of both CTAs (multicast); both CTAs' epilogue warps
// arrive on the leader's acc_empty barrier (8 arrivals).
#ifndef OZ2P_NSTAGES
#define OZ2P_NSTAGES 6
#endif
constexpr int OZ2P_STAGES = OZ2P_NSTAGES;
#ifndef OZ2P_GROUP
#define OZ2P_GROUP 8  // raster group of the pair kernel (in 256-row / 256-column pair tiles)
#endif
constexpr int OZ2P_A_BYTES = 128 * OZ2_TK, OZ2P_B_BYTES = 128 * OZ2_TK, OZ2P_STAGE = OZ2P_A_BYTES + OZ2P_B_BYTES;
constexpr size_t OZ2P_SMEM = (size_t)OZ2P_STAGES * OZ2P_STAGE + 1024 + 256;

__device__ __forceinline__ uint32_t oz2_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t oz2_leader_addr(const void* p) {  // same smem offset in cluster CTA 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void oz2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ2_THREADS, 1)
    oz2_gemm_pair_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                         const Oz2Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;
  unsigned char* sB = base + OZ2P_STAGES * OZ2P_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + OZ2P_STAGES * OZ2P_STAGE);
  uint64_t* empty = full + OZ2P_STAGES;
  uint64_t* acc_full = empty + OZ2P_STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2], leader's used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = oz2_cluster_rank();
  const int tiles_m = p.M / 256;  // row-pair tiles
  const int t = (blockIdx.x >> 1) / p.msplit;
  const int nmod = OZ2_NMOD / p.msplit, mod0 = ((blockIdx.x >> 1) % p.msplit) * nmod;
  // raster group: 4 pair tiles for dense products, 8 with a triangular operand (r01_oz2_pair.txt)
  const int G = (p.triA == TRI_NONE && p.triB == TRI_NONE) ? 4 : OZ2P_GROUP;
  int I, J;
  if (p.triA != TRI_NONE && p.triB == TRI_NONE) {
    const int per_group = G * tiles_m;
    const int first_n = (t / per_group) * G;
    const int gsz = min(p.tiles_n - first_n, G);
    J = first_n + (t % per_group) % gsz;
    I = (t % per_group) / gsz;
  } else {
    const int per_group = G * p.tiles_n;
    const int first_m = (t / per_group) * G;
    const int gsz = min(tiles_m - first_m, G);
    I = first_m + (t % per_group) % gsz;
    J = (t % per_group) / gsz;
  }
  if (p.triA == TRI_LOWER) I = tiles_m - 1 - I;
  if (p.triB == TRI_UPPER) J = p.tiles_n - 1 - J;
  int kb = 0, ke = p.K;  // K range of the 256-row pair tile
  if (p.triA == TRI_LOWER) ke = min(ke, (I + 1) * 256);
  if (p.triA == TRI_UPPER) kb = I * 256;
  if (p.triB == TRI_LOWER) kb = max(kb, J * OZ2_TN);
  if (p.triB == TRI_UPPER) ke = min(ke, (J + 1) * OZ2_TN);
  const int nkb = ke > kb ? (ke - kb) / OZ2_TK : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ2P_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], 8); }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * OZ2_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  oz2_cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // TMA producer (both CTAs): this CTA's A rows and B columns
    tma_prefetch_desc(&ma);
    tma_prefetch_desc(&mb);
    int it = 0;
    for (int i = mod0; i < mod0 + nmod; ++i)
      for (int kk = 0; kk < nkb; ++kk, ++it) {
        const int st = it % OZ2P_STAGES, use = it / OZ2P_STAGES;
        if (use > 0) mbar_wait(&empty[st], (uint32_t)((use - 1) & 1));
        if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * OZ2P_STAGE);
        const uint32_t fb = oz2_leader_addr(&full[st]);
        const int k = kb + kk * OZ2_TK;
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3}], [%4];\n" ::"r"(smem_u32(sA + st * OZ2P_A_BYTES)),
            "l"(reinterpret_cast<uint64_t>(&ma)), "r"(k), "r"(i * p.M + I * 256 + (int)rank * 128), "r"(fb)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3}], [%4];\n" ::"r"(smem_u32(sB + st * OZ2P_B_BYTES)),
            "l"(reinterpret_cast<uint64_t>(&mb)), "r"(k), "r"(i * p.N + J * OZ2_TN + (int)rank * 128), "r"(fb)
            : "memory");
      }
  } else if (warp == 1 && lane == 0 && rank == 0) {  // MMA issuer (leader CTA)
    const uint32_t idesc =
        (2u << 4) | (p.K > OZ2_U8_MAXK ? 1u << 10 : 0u) | ((uint32_t)(OZ2_TN >> 3) << 17) |
        ((uint32_t)(256 >> 4) << 24);  // u8 x u8 (u8 x s8 above OZ2_U8_MAXK) -> s32
    int it = 0;
    for (int i = mod0; i < mod0 + nmod; ++i) {
      const int buf = (i - mod0) & 1, use = (i - mod0) >> 1;
      if (use > 0) {
        mbar_wait(&acc_empty[buf], (uint32_t)((use - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
      const uint32_t tacc = tmem + (uint32_t)(buf * OZ2_TN);
      bool first = true;
      for (int kk = 0; kk < nkb; ++kk, ++it) {
        const int st = it % OZ2P_STAGES;
        mbar_wait(&full[st], (uint32_t)((it / OZ2P_STAGES) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t da = oz2_smem_desc(sA + st * OZ2P_A_BYTES), db = oz2_smem_desc(sB + st * OZ2P_B_BYTES);
#pragma unroll
        for (int k = 0; k < OZ2_TK / 32; ++k) {
          const uint32_t acc = first ? 0u : 1u;
          first = false;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tacc),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(idesc), "r"(acc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                smem_u32(&empty[st])),
            "h"((uint16_t)3)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              smem_u32(&acc_full[buf])),
          "h"((uint16_t)3)
          : "memory");
    }
  }
  if (warp >= 2) {  // epilogue (both CTAs): this CTA's 128 rows of the pair tile
    const int q4 = warp & 3;
    const int row = I * 256 + (int)rank * 128 + q4 * 32 + lane;
    for (int i = mod0; i < mod0 + nmod; ++i) {
      const int buf = (i - mod0) & 1, use = (i - mod0) >> 1;
      mbar_wait(&acc_full[buf], (uint32_t)(use & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int m = oz2_mod(i);
      const double rm = 1.0 / m;
      uint8_t* dst = p.R + ((size_t)i * p.M + row) * p.N + J * OZ2_TN;
#pragma unroll 1
      for (int c = 0; c < OZ2_TN; c += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * OZ2_TN + c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          uint32_t w = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int x = nkb ? (int)v[j + b] : 0;
            int r = x - (int)floor((double)x * rm) * m;
            r += (r < 0) ? m : 0;
            r -= (r >= m) ? m : 0;
            w |= (uint32_t)r << (8 * b);
          }
          packed[j / 4] = w;
        }
        *reinterpret_cast<uint4*>(dst + c) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint4*>(dst + c + 16) = make_uint4(packed[4], packed[5], packed[6], packed[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                         oz2_leader_addr(&acc_empty[buf]))
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  oz2_cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * OZ2_TN));
}

// ---- reconstruction: C' / M = frac(sum_i c_i y_i / m_i) ----------------------------------
// With M_i = M / m_i and y_i = M_i^-1 mod m_i, sum_i c_i M_i y_i == C' (mod M), so
//     C' / M == sum_i c_i (y_i / m_i)   (mod 1),
// and as |C'| < M/2 by a margin (P from K, oz2_scale_bits) C' / M is the representative of
// that sum in [-1/2, 1/2).  F_i = round(2^96 y_i / m_i) in three 32-bit limbs; the limb sums
// A_l = sum_i c_i F_il (< 2^44, 64-bit IMAD.WIDE accumulators) give the fraction mod 1 as a
// signed 96-bit fixed-point number (the integer part carried out of the top limb is dropped)
// with absolute error < 16 * 255 * 2^-97 < 2^-85, i.e. < 2^41 on C' against the 2^P-sized
// truncation error of the scaled operands.  C' = fraction * M in FP64 (relative 2^-52).
struct Oz2Crt {
  uint32_t f[OZ2_NMOD][3];  // limbs of F_i = round(2^96 y_i / m_i)
  double Md96;              // M 2^-96
};

// 4 consecutive entries of one row per thread (N % 4 == 0): one 32-bit word per plane; the
// moduli are the outer loop so each constant is loaded once for the four entries.
__global__ void oz2_reconstruct_kernel(const uint8_t* R, int M, int N, const int* ea, const int* eb, int P,
                                       double alpha, double beta, double* C, int64_t ldc, const Oz2Crt crt) {
  const int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // index of 4 entries
  if (e4 >= (int64_t)M * N / 4) return;
  const int64_t e = 4 * e4;
  const int i = (int)(e / N), j = (int)(e % N);
  const size_t plane_w = (size_t)M * N / 4;
  const uint32_t* Rw = reinterpret_cast<const uint32_t*>(R) + e4;
  uint32_t w[OZ2_NMOD];
#pragma unroll
  for (int q = 0; q < OZ2_NMOD; ++q) w[q] = Rw[q * plane_w];
  uint64_t a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < OZ2_NMOD; ++q) {
    const uint32_t f0 = crt.f[q][0], f1 = crt.f[q][1], f2 = crt.f[q][2];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t c = __byte_perm(w[q], 0u, 0x4440 + b);
      a0[b] += (uint64_t)c * f0;
      a1[b] += (uint64_t)c * f1;
      a2[b] += (uint64_t)c * f2;
    }
  }
  double* out = C + (int64_t)i * ldc + j;
  const int ei = ea[i] - 2 * P;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint64_t b1 = a1[b] + (a0[b] >> 32), b2 = a2[b] + (b1 >> 32);
    const int64_t hi = (int64_t)(((uint64_t)(uint32_t)b2 << 32) | (uint32_t)b1);  // top 64 of 96 bits, signed
    const double frac96 = fma((double)hi, 4294967296.0, (double)(uint32_t)a0[b]);  // fraction * 2^96
    const bool nonfinite = ea[i] == OZ2_NONFINITE || eb[j + b] == OZ2_NONFINITE;
    const double val =
        nonfinite ? __longlong_as_double(0x7ff8000000000000ll) : oz2_ldexp(frac96 * crt.Md96, ei + eb[j + b]);
    out[b] = beta == 0.0 ? alpha * val : fma(alpha, val, beta * out[b]);
  }
}

static Oz2Crt oz2_crt_constants() {
  Oz2Crt c{};
  unsigned __int128 Mall = 1;
  for (int q = 0; q < OZ2_NMOD; ++q) Mall *= (unsigned)oz2_mod(q);
  for (int q = 0; q < OZ2_NMOD; ++q) {
    const unsigned m = (unsigned)oz2_mod(q);
    const unsigned y = (unsigned)oz2_inv((int)((Mall / m) % m), (int)m);
    const unsigned __int128 F = (((unsigned __int128)y << 96) + m / 2) / m;  // < 2^96 (y < m)
    for (int l = 0; l < 3; ++l) c.f[q][l] = (uint32_t)(F >> (32 * l));
  }
  const double Md = (double)(unsigned long long)(Mall >> 64) * 18446744073709551616.0 + (double)(unsigned long long)Mall;
  c.Md96 = std::ldexp(Md, -96);
  return c;
}

// ---- host -------------------------------------------------------------------------------
// P with K 2^(2P) <= (1 - 2^-10) M / 2: |C'| < K 2^(2P) keeps the centred fraction C' / M
// unambiguous (oz2_reconstruct_kernel); at most 58 (the residue chunks of oz2_chunks).
static int oz2_scale_bits(int64_t K) {
  double lm = 0.0;
  for (int q = 0; q < OZ2_NMOD; ++q) lm += std::log2((double)oz2_mod(q));
  int P = (int)std::floor((lm - 1.0 - 1.5e-3 - std::log2((double)K)) / 2.0);
  return P > 58 ? 58 : P;
}

bool oz2_supported(int64_t M, int64_t N, int64_t K) {
  return M > 0 && N > 0 && K > 0 && M % OZ2_TM == 0 && N % OZ2_TN == 0 && K % OZ2_TK == 0 && K <= 65536 &&
         oz2_scale_bits(K) >= 53 && M * N < ((int64_t)1 << 40);
}

size_t oz2_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al((size_t)OZ2_NMOD * M * K) + al((size_t)OZ2_NMOD * N * K) + al((size_t)OZ2_NMOD * M * N) +
         al((size_t)M * 4) + al((size_t)N * 4) + al((size_t)N * 8);
}

static bool oz2_encode(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) != cudaSuccess) return false;
    fn = reinterpret_cast<EncFn>(q);
  }
  cuuint64_t dims[2] = {cols, rows}, strides[1] = {cols};
  cuuint32_t box[2] = {(cuuint32_t)OZ2_TK, box_rows}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// CTA-pair GEMM (cta_group::2) for products with M % 256 == 0 and all dimensions >=
// pair_min (TRINV_OZ2_PAIR = 0 disables, = <n> sets pair_min; default 8192: the pair
// kernel won at the 8192 and 16384 levels, not at 4096, profiles/r01_oz2_pair.txt)
static bool oz2_use_pair(int64_t M, int64_t N, int64_t K) {
  static const int64_t pair_min = [] {
    const char* e = std::getenv("TRINV_OZ2_PAIR");
    if (!e) return (int64_t)8192;
    const long long v = std::atoll(e);
    return v <= 0 ? (int64_t)1 << 62 : (int64_t)v;
  }();
  return M % 256 == 0 && std::min(M, std::min(N, K)) >= pair_min;
}

// Operand splits on their own (which: 1 = A, 2 = B), into the same workspace layout as
// launch_oz2_gemm, which then skips them (skip = which): lets a caller split an operand
// on another stream while an earlier product runs.
cudaError_t launch_oz2_prepare(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA,
                               const double* B, int64_t ldb, int triB, void* ws, cudaStream_t st, int which,
                               int64_t* launches, int strict) {
  if (!oz2_supported(M, N, K)) return cudaErrorInvalidValue;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* w = static_cast<char*>(ws);
  int8_t* As = reinterpret_cast<int8_t*>(w); w += al((size_t)OZ2_NMOD * M * K);
  int8_t* Bs = reinterpret_cast<int8_t*>(w); w += al((size_t)OZ2_NMOD * N * K);
  w += al((size_t)OZ2_NMOD * M * N);
  int* ea = reinterpret_cast<int*>(w); w += al((size_t)M * 4);
  int* eb = reinterpret_cast<int*>(w); w += al((size_t)N * 4);
  unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(w);
  const int P = oz2_scale_bits(K);
  // algorithmic bytes: the K ranges split (8 B read, 16 B of residues written per entry)
  auto range_sum = [&](int64_t rows, int tile, bool upto, bool from) {
    double sum = 0.0;
    for (int64_t t0 = 0; t0 < rows; t0 += tile) {
      const int64_t r = std::min<int64_t>(tile, rows - t0);
      const int64_t b = from ? t0 : 0, e = upto ? std::min<int64_t>(K, t0 + tile) : K;
      sum += (double)r * (double)std::max<int64_t>(0, e - b);
    }
    return sum;
  };
  const double bytes = ((which & 1) ? 24.0 * range_sum(M, OZ2_TM, triA == TRI_LOWER, triA == TRI_UPPER) : 0.0) +
                       ((which & 2) ? 32.0 * range_sum(N, OZ2_TN, triB == TRI_UPPER, triB == TRI_LOWER) : 0.0);
  ProfileScope aux(KIND_OZAUX, 0.0, bytes, st);
  if (which & 1) {
    prefer_l1_once<oz2_split_rows_kernel>();  // element-wise: no shared memory
    oz2_split_rows_kernel<<<(unsigned)((M * 32 + 255) / 256), 256, 0, st>>>(
        A, lda, (int)M, (int)K, triA, (strict & 1) != 0, P, oz2_use_pair(M, N, K) ? 256 : OZ2_TM, As, ea);
    if (launches) ++*launches;
  }
  if (which & 2) {
    cudaError_t e = cudaMemsetAsync(maxbits, 0, (size_t)N * 8, st);
    if (e != cudaSuccess) return e;
    prefer_l1_once<oz2_colmax_kernel>();
    oz2_colmax_kernel<<<dim3((unsigned)((N + 255) / 256), (unsigned)((K + OZ2_CMAX_ROWS - 1) / OZ2_CMAX_ROWS)), 256, 0,
                        st>>>(B, ldb, (int)K, (int)N, triB, (strict & 2) != 0, maxbits);
    oz2_split_cols_kernel<<<dim3((unsigned)((N + 31) / 32), (unsigned)((K + 31) / 32)), 256, 0, st>>>(
        B, ldb, (int)K, (int)N, triB, (strict & 2) != 0, P, maxbits, eb, Bs);
    if (launches) *launches += 2;
  }
  return cudaGetLastError();
}

cudaError_t launch_oz2_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                            int64_t ldb, int triB, double* C, int64_t ldc, double alpha, double beta, void* ws,
                            cudaStream_t st, int64_t* launches, int strict, int skip) {
  if (!oz2_supported(M, N, K)) return cudaErrorInvalidValue;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* w = static_cast<char*>(ws);
  int8_t* As = reinterpret_cast<int8_t*>(w); w += al((size_t)OZ2_NMOD * M * K);
  int8_t* Bs = reinterpret_cast<int8_t*>(w); w += al((size_t)OZ2_NMOD * N * K);
  uint8_t* Rs = reinterpret_cast<uint8_t*>(w); w += al((size_t)OZ2_NMOD * M * N);
  int* ea = reinterpret_cast<int*>(w); w += al((size_t)M * 4);
  int* eb = reinterpret_cast<int*>(w); w += al((size_t)N * 4);
  unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(w);
  const int P = oz2_scale_bits(K);
  GemmArgs ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.batch = 1; ga.triA = triA; ga.triB = triB;
  double f64 = gemm_flops(ga);
  if (triA == TRI_UPPER && triB == TRI_LOWER) {  // S K with both factors triangular (P_UL)
    const double n = (double)K;
    f64 = 2.0 * (n * (n + 1) * (2 * n + 1) / 6.0) - n * n;
  }
  // algorithmic bytes of the auxiliary kernels: the K ranges split (8 B read, 16 B of
  // residues written per entry; the column maxima re-read B), and per output entry 16 B
  // of residues read, 8 B written (+ 8 B read when beta != 0)
  auto range_sum = [&](int64_t rows, int tile, bool upto, bool from) {
    double s = 0.0;
    for (int64_t t0 = 0; t0 < rows; t0 += tile) {
      const int64_t r = std::min<int64_t>(tile, rows - t0);
      const int64_t b = from ? t0 : 0, e = upto ? std::min<int64_t>(K, t0 + tile) : K;
      s += (double)r * (double)std::max<int64_t>(0, e - b);
    }
    return s;
  };
  const double ea_n = range_sum(M, OZ2_TM, triA == TRI_LOWER, triA == TRI_UPPER);
  const double eb_n = range_sum(N, OZ2_TN, triB == TRI_UPPER, triB == TRI_LOWER);
  const bool pair = oz2_use_pair(M, N, K);
  if ((skip & 3) != 3) {
    const cudaError_t e = launch_oz2_prepare(M, N, K, A, lda, triA, B, ldb, triB, ws, st, 3 & ~skip, nullptr, strict);
    if (e != cudaSuccess) return e;
  }
  (void)ea_n; (void)eb_n;
  (void)maxbits;
  CUtensorMap ma, mb;
  if (!oz2_encode(&ma, As, (uint64_t)K, (uint64_t)OZ2_NMOD * M, OZ2_TM) ||
      !oz2_encode(&mb, Bs, (uint64_t)K, (uint64_t)OZ2_NMOD * N, pair ? 128 : OZ2_TN))
    return cudaErrorInvalidValue;
  Oz2Params p{};
  p.M = (int)M; p.N = (int)N; p.K = (int)K; p.triA = triA; p.triB = triB; p.R = Rs;
  p.tiles_n = (int)(N / OZ2_TN);
  // below ~6 waves of tiles, each tile's moduli are split over 2 or 4 CTAs so the last
  // partial wave is a small fraction (the level-4096 products: 512 tiles on 148 SMs)
  const int64_t ctas = pair ? 2 * (M / 256) * (N / OZ2_TN) : (M / OZ2_TM) * (N / OZ2_TN);
  const int64_t waves6 = 6 * (int64_t)device_sms();
  static const int msplit_env = [] { const char* e = std::getenv("TRINV_OZ2_MSPLIT"); return e ? std::atoi(e) : 0; }();
  p.msplit = ctas >= waves6 ? 1 : (2 * ctas >= waves6 ? 2 : 4);
  if (msplit_env == 1 || msplit_env == 2 || msplit_env == 4 || msplit_env == 8) p.msplit = msplit_env;  // experiments
  {
    ProfileScope prof(KIND_OZ, f64, f64 * OZ2_NMOD, st);  // bytes slot: int8 ops
    if (pair) {
      set_smem_once<oz2_gemm_pair_kernel>((int)OZ2P_SMEM);
      oz2_gemm_pair_kernel<<<(unsigned)(ctas * p.msplit), OZ2_THREADS, OZ2P_SMEM, st>>>(ma, mb, p);
    } else {
      set_smem_once<oz2_gemm_kernel>((int)OZ2_SMEM);
      oz2_gemm_kernel<<<(unsigned)(ctas * p.msplit), OZ2_THREADS, OZ2_SMEM, st>>>(ma, mb, p);
    }
  }
  const int64_t total4 = M * N / 4;
  static const Oz2Crt crt = oz2_crt_constants();
  {
    ProfileScope aux(KIND_OZAUX, 0.0, (double)M * N * (beta == 0.0 ? 24.0 : 32.0), st);
    prefer_l1_once<oz2_reconstruct_kernel>();
    oz2_reconstruct_kernel<<<(unsigned)((total4 + 255) / 256), 256, 0, st>>>(Rs, (int)M, (int)N, ea, eb, P, alpha,
                                                                            beta, C, ldc, crt);
  }
  if (launches) *launches += 2 + ((skip & 1) ? 0 : 1) + ((skip & 2) ? 0 : 2);
  return cudaGetLastError();
}

// X_ij = S_ii K_ij (i >= j), S_ij K_jj (i < j): the terms of S K with a diagonal factor.
// Block: 256 columns x 32 rows, the 256 diagonal entries K_jj staged in shared memory.
__global__ void __launch_bounds__(256) oz2_ul_diag_terms_kernel(int n, const double* S, int64_t lds, const double* K,
                                                                int64_t ldk, double* X, int64_t ldx) {
  __shared__ double kd[256];
  const int j = blockIdx.x * 256 + threadIdx.x;
  kd[threadIdx.x] = j < n ? K[(int64_t)j * ldk + j] : 0.0;
  __syncthreads();
  if (j >= n) return;
  for (int r = 0; r < 32; ++r) {
    const int i = blockIdx.y * 32 + r;
    if (i >= n) break;
    X[(int64_t)i * ldx + j] = i >= j ? S[(int64_t)i * lds + i] * K[(int64_t)i * ldk + j]
                                     : S[(int64_t)i * lds + j] * kd[threadIdx.x];
  }
}

cudaError_t launch_oz2_ul(int64_t n, const double* S, int64_t lds, const double* K, int64_t ldk, double* X,
                          int64_t ldx, void* ws, cudaStream_t st, int64_t* launches) {
  if (!oz2_supported(n, n, n)) return cudaErrorInvalidValue;
  oz2_ul_diag_terms_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)((n + 31) / 32)), 256, 0, st>>>(
      (int)n, S, lds, K, ldk, X, ldx);
  if (launches) *launches += 1;
  return launch_oz2_gemm(n, n, n, S, lds, TRI_UPPER, K, ldk, TRI_LOWER, X, ldx, 1.0, 1.0, ws, st, launches, 3);
}

}  // namespace trinv
