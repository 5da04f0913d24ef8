// oz.cu — FP64 products on the INT8 tensor cores (tcgen05 kind::i8) by exact
// operand splitting (an Ozaki-type scheme); an opt-in engine for the large
// off-diagonal products of the recursive split (the paper
// leaves the block products to "any preferred method", and itself
// uses Strassen).  DESIGN.md §8 "oz_gemm_kernel".
//
// Splitting.  Row i of the A operand is scaled by sigma_i = 2^e_i (the power of two
// just above its largest magnitude, so |a_ik / sigma_i| < 1) and cut into s signed
// 7-bit digits: a_ik / sigma_i = sum_{t=1..s} A_t[i][k] 2^{-7t} + r, |r| < 2^{-7s},
// every step exact in FP64 (y = 128 x, d = trunc(y), x = y - d).  Columns of the
// B operand likewise (tau_j, B_u).  Then
//     (A B)_ij ~= sigma_i tau_j sum_{d=2..s+1} 2^{-7d} G_d[i][j],
//     G_d = sum_{t+u=d} A_t B_u   (exact int32 products on the tensor cores),
// dropping the digit pairs with t + u > s + 1; each G_d is one pass of the K-loop over
// the pairs (t, d - t), accumulated in TMEM, and folded into the FP64 output by the
// epilogue (C = beta C + alpha sum ...).  |G_d| <= (d-1) K 127^2 < 2^31 needs
// (d-1) K < 133152: K <= 16384 at s = 8.
//
// Engine: CTA tile 128 x 256, 128-byte K blocks of both operands (int8, K-major; B
// is stored transposed) staged by 2-D TMA with the 128-byte swizzle into a 4-deep
// ring; one thread issues tcgen05.mma (M = 128, N = 256, K = 32 per instruction)
// into a 256-column TMEM accumulator; the four warps read it back with tcgen05.ld.
// Triangular operands skip their structurally zero K-blocks like the DMMA engine.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace trinv {

constexpr int OZ_TM = 128, OZ_TN = 256, OZ_TK = 128, OZ_STAGES = 4;
#ifndef OZ_GROUP_M
#define OZ_GROUP_M 8
#endif
constexpr int OZ_A_BYTES = OZ_TM * OZ_TK, OZ_B_BYTES = OZ_TN * OZ_TK, OZ_STAGE = OZ_A_BYTES + OZ_B_BYTES;
constexpr size_t OZ_SMEM = (size_t)OZ_STAGES * OZ_STAGE + 1024 + 256;  // ring + alignment + barriers

// ---- splitting ----------------------------------------------------------------
__device__ __forceinline__ int pow2_exponent_above(double m) {  // e with m < 2^e (m >= 0); 0 for m == 0
  if (m == 0.0) return 0;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return e;
}

__device__ __forceinline__ void split_digits(double x, int s, int8_t* out, size_t slice_stride) {
  // x in (-1, 1): s truncated base-128 digits, each step exact
  for (int t = 0; t < s; ++t) {
    const double y = x * 128.0;
    const double d = trunc(y);
    out[t * slice_stride] = (int8_t)(int)d;
    x = y - d;
  }
}

// A operand (rows x K, row-major, lda): one warp per row.
__global__ void oz_split_rows_kernel(const double* A, int64_t lda, int rows, int K, int s, int8_t* out,
                                     double* scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const double* a = A + (int64_t)warp * lda;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = fmax(m, fabs(a[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int e = pow2_exponent_above(m);
  if (lane == 0) scale[warp] = ldexp(1.0, e);
  const size_t ss = (size_t)rows * K;
  for (int k = lane; k < K; k += 32) split_digits(ldexp(a[k], -e), s, out + (size_t)warp * K + k, ss);
}

// B operand (K x cols, row-major, ldb): column maxima, then digits written transposed
// (cols x K, K-major) through a 32 x 32 shared-memory tile.
__global__ void oz_colmax_kernel(const double* B, int64_t ldb, int K, int cols, unsigned long long* maxbits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const int k0 = blockIdx.y * 512, k1 = min(K, k0 + 512);
  double m = 0.0;
  for (int k = k0; k < k1; ++k) m = fmax(m, fabs(B[(int64_t)k * ldb + j]));
  atomicMax(&maxbits[j], (unsigned long long)__double_as_longlong(m));  // order-preserving for m >= 0
}
__global__ void oz_split_cols_kernel(const double* B, int64_t ldb, int K, int cols, int s,
                                     const unsigned long long* maxbits, double* scale, int8_t* out) {
  __shared__ double tile[32][33];
  const int k0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int jx = j0 + threadIdx.x;
  const int e = jx < cols ? pow2_exponent_above(__longlong_as_double((long long)maxbits[jx])) : 0;
  if (blockIdx.y == 0 && threadIdx.y == 0 && jx < cols) scale[jx] = ldexp(1.0, e);
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r;
    tile[r][threadIdx.x] = (k < K && jx < cols) ? ldexp(B[(int64_t)k * ldb + jx], -e) : 0.0;  // exact
  }
  __syncthreads();
  const size_t ss = (size_t)cols * K;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, k = k0 + threadIdx.x;
    if (j < cols && k < K) split_digits(tile[threadIdx.x][r], s, out + (size_t)j * K + k, ss);
  }
}

// ---- the int8 tensor-core engine ------------------------------------------------
__device__ __forceinline__ uint64_t oz_smem_desc(const void* p) {
  // K-major, 128-byte swizzle: 128-byte rows, 8-row groups 1024 bytes apart (SBO); LBO unused
  uint64_t d = (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint32_t oz_idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_TN >> 3) << 17) | ((uint32_t)(OZ_TM >> 4) << 24);
}

struct OzGemmParams {
  int M, N, K, s;
  int triA, triB;           // TriKind of the A / B operand (structurally zero K-blocks skipped)
  const double* sa;         // row scales of A [M]
  const double* sb;         // column scales of B [N]
  double* C;                // FP64 output, row-major
  int64_t ldc;
  double alpha, beta;
  int tiles_n;
};

// Warp roles: 0 = TMA producer (one lane), 1 = MMA issuer (one lane), 2..5 = epilogue
// (warp w reads TMEM lanes 32 (w % 4) .. +31, the quarter it may access).
constexpr int OZ_THREADS = 192;
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                   const OzGemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;
  unsigned char* sB = base + OZ_STAGES * OZ_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + OZ_STAGES * OZ_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* acc_full = empty + OZ_STAGES;  // [2]: two TMEM accumulators (d even / odd)
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Grouped rasterisation for L2 reuse: consecutive CTAs cover OZ_GROUP_M tile rows x
  // ~148/OZ_GROUP_M tile columns, so a wave streams each digit block of A and B from
  // HBM about once (row-major order re-read every B block per wave: 109 GB at n = 8192).
  // A triangular operand then reverses I or J so that long K-ranges start first.
  const int tiles_m = p.M / OZ_TM;
  const int t = blockIdx.x;
  const int per_group = OZ_GROUP_M * p.tiles_n;
  const int first_m = (t / per_group) * OZ_GROUP_M;
  const int gsz = min(tiles_m - first_m, OZ_GROUP_M);
  int I = first_m + (t % per_group) % gsz, J = (t % per_group) / gsz;
  if (p.triA == TRI_LOWER) I = tiles_m - 1 - I;
  if (p.triB == TRI_UPPER) J = p.tiles_n - 1 - J;
  int kb = 0, ke = p.K;
  if (p.triA == TRI_LOWER) ke = min(ke, (I + 1) * OZ_TM);
  if (p.triA == TRI_UPPER) kb = I * OZ_TM;
  if (p.triB == TRI_LOWER) kb = J * OZ_TN;
  if (p.triB == TRI_UPPER) ke = min(ke, (J + 1) * OZ_TN);
  const int nkb = ke > kb ? (ke - kb) / OZ_TK : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // the four epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * OZ_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int S = p.s;

  if (warp == 0 && lane == 0) {  // TMA producer: for d = 2..s+1, pairs (t, d-t), K-blocks
    tma_prefetch_desc(&ma);
    tma_prefetch_desc(&mb);
    int it = 0;
    for (int d = 2; d <= S + 1; ++d)
      for (int ta = 1; ta < d; ++ta)
        for (int kk = 0; kk < nkb; ++kk, ++it) {
          const int st = it % OZ_STAGES, use = it / OZ_STAGES;
          if (use > 0) mbar_wait(&empty[st], (uint32_t)((use - 1) & 1));
          mbar_arrive_expect_tx(&full[st], OZ_STAGE);
          const int k = kb + kk * OZ_TK;
          tma_load_2d(sA + st * OZ_A_BYTES, &ma, k, (ta - 1) * p.M + I * OZ_TM, &full[st]);
          tma_load_2d(sB + st * OZ_B_BYTES, &mb, k, (d - ta - 1) * p.N + J * OZ_TN, &full[st]);
        }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = oz_idesc();
    int it = 0;
    for (int d = 2; d <= S + 1; ++d) {
      const int buf = d & 1, use = (d - 2 - buf) / 2;  // accumulator d % 2, its use-th round
      if (use > 0) {  // the epilogue has drained this accumulator (round use - 1, i.e. d - 2)
        mbar_wait(&acc_empty[buf], (uint32_t)((use - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
      const uint32_t tacc = tmem + (uint32_t)(buf * OZ_TN);
      bool first = true;
      for (int ta = 1; ta < d; ++ta)
        for (int kk = 0; kk < nkb; ++kk, ++it) {
          const int st = it % OZ_STAGES;
          mbar_wait(&full[st], (uint32_t)((it / OZ_STAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint64_t da = oz_smem_desc(sA + st * OZ_A_BYTES), db = oz_smem_desc(sB + st * OZ_B_BYTES);
#pragma unroll
          for (int k = 0; k < OZ_TK / 32; ++k) {
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
  // epilogue: C = beta C + alpha sum_d sigma_i tau_j 2^{-7d} G_d, folded in per d
  if (warp >= 2) {
  const int q4 = warp & 3;  // TMEM lane quarter of this warp
  const int row = I * OZ_TM + q4 * 32 + lane;
  const double srow = p.alpha * p.sa[row];
  double* crow = p.C + (int64_t)row * p.ldc + J * OZ_TN;
  const double* tau = p.sb + J * OZ_TN;
  for (int d = 2; d <= S + 1; ++d) {
    const int buf = d & 1, use = (d - 2 - buf) / 2;
    mbar_wait(&acc_full[buf], (uint32_t)(use & 1));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const double f = srow * ldexp(1.0, -7 * d);
#pragma unroll 1
    for (int c = 0; c < OZ_TN; c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * OZ_TN + c);
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
      if (nkb == 0) {  // empty K-range: the accumulator was never written
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
      double* q = crow + c;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double g0 = (double)(int32_t)v[j] * tau[c + j], g1 = (double)(int32_t)v[j + 1] * tau[c + j + 1];
        double2 o;
        if (d == 2) {
          o = p.beta == 0.0 ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(q + j);
          o.x = p.beta == 0.0 ? f * g0 : fma(f, g0, p.beta * o.x);
          o.y = p.beta == 0.0 ? f * g1 : fma(f, g1, p.beta * o.y);
        } else {
          o = *reinterpret_cast<const double2*>(q + j);
          o.x = fma(f, g0, o.x);
          o.y = fma(f, g1, o.y);
        }
        *reinterpret_cast<double2*>(q + j) = o;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_empty[buf]);
  }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * OZ_TN));
}

// ---- host -------------------------------------------------------------------------
bool oz_supported(int64_t M, int64_t N, int64_t K, int s) {
  return M > 0 && N > 0 && K > 0 && M % OZ_TM == 0 && N % OZ_TN == 0 && K % OZ_TK == 0 && s >= 1 && s <= 10 &&
         (int64_t)s * K * 127 * 127 < ((int64_t)1 << 31);
}

size_t oz_workspace_bytes(int64_t M, int64_t N, int64_t K, int s) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al((size_t)s * M * K) + al((size_t)s * N * K) + al((size_t)M * 8) + 2 * al((size_t)N * 8);
}

static bool encode_i8(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
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
  cuuint32_t box[2] = {(cuuint32_t)OZ_TK, box_rows}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C = alpha A B + beta C (A: M x K, lda; B: K x N, ldb; C: M x N, ldc; all FP64 row-major)
// with s base-128 digits per operand.  ws >= oz_workspace_bytes(M, N, K, s).
cudaError_t launch_oz_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int triA, const double* B,
                           int64_t ldb, int triB, double* C, int64_t ldc, double alpha, double beta, int s, void* ws,
                           cudaStream_t st, int64_t* launches) {
  if (!oz_supported(M, N, K, s)) return cudaErrorInvalidValue;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* w = static_cast<char*>(ws);
  int8_t* As = reinterpret_cast<int8_t*>(w); w += al((size_t)s * M * K);
  int8_t* Bs = reinterpret_cast<int8_t*>(w); w += al((size_t)s * N * K);
  double* sa = reinterpret_cast<double*>(w); w += al((size_t)M * 8);
  double* sb = reinterpret_cast<double*>(w); w += al((size_t)N * 8);
  unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(w);
  // algorithmic work: the FP64 flops of the product (the int8 work is s(s+1)/2 times that)
  GemmArgs ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.batch = 1; ga.triA = triA; ga.triB = triB;
  const double f64 = gemm_flops(ga);
  ProfileScope prof(KIND_OZ, f64, f64 * s * (s + 1) / 2.0, st);  // bytes slot: int8 ops
  oz_split_rows_kernel<<<(unsigned)((M * 32 + 255) / 256), 256, 0, st>>>(A, lda, (int)M, (int)K, s, As, sa);
  cudaError_t e = cudaMemsetAsync(maxbits, 0, (size_t)N * 8, st);
  if (e != cudaSuccess) return e;
  oz_colmax_kernel<<<dim3((unsigned)((N + 255) / 256), (unsigned)((K + 511) / 512)), 256, 0, st>>>(B, ldb, (int)K,
                                                                                                  (int)N, maxbits);
  oz_split_cols_kernel<<<dim3((unsigned)((N + 31) / 32), (unsigned)((K + 31) / 32)), dim3(32, 8), 0, st>>>(
      B, ldb, (int)K, (int)N, s, maxbits, sb, Bs);
  CUtensorMap ma, mb;
  if (!encode_i8(&ma, As, (uint64_t)K, (uint64_t)s * M, OZ_TM) || !encode_i8(&mb, Bs, (uint64_t)K, (uint64_t)s * N, OZ_TN))
    return cudaErrorInvalidValue;
  OzGemmParams p{};
  p.M = (int)M; p.N = (int)N; p.K = (int)K; p.s = s; p.triA = triA; p.triB = triB;
  p.sa = sa; p.sb = sb; p.C = C; p.ldc = ldc; p.alpha = alpha; p.beta = beta;
  p.tiles_n = (int)(N / OZ_TN);
  set_smem_once<oz_gemm_kernel>((int)OZ_SMEM);
  const unsigned tiles = (unsigned)((M / OZ_TM) * (N / OZ_TN));
  oz_gemm_kernel<<<tiles, OZ_THREADS, OZ_SMEM, st>>>(ma, mb, p);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

}  // namespace trinv
