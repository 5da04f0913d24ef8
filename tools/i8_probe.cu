// Feasibility probe for the "FP64 products on the INT8 tensor cores" direction
// (DESIGN.md §11): a plain tcgen05 kind::i8 GEMM, C (int32, M x N) = A (int8, M x K,
// K-major) * B^T (B int8, N x K, K-major), CTA tile 128 x 256, 128-byte K blocks staged
// by 2-D TMA with the 128-byte swizzle, accumulators in TMEM, one thread issuing MMA,
// four warps reading TMEM back.  Checked exactly against a simple int32 kernel; timed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/i8_probe tools/i8_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2307_07611_b200/csrc/ptx.cuh"
using namespace trinv;

constexpr int TM = 128, TN = 256, TK = 128, STAGES = 4;
constexpr int A_BYTES = TM * TK, B_BYTES = TN * TK, STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  // K-major, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B apart (SBO), LBO unused.
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;          // start address [0,14)
  d |= (uint64_t)1 << 16;             // leading byte offset (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // stride byte offset [32,46)
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // layout: SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  uint32_t d = 0;
  d |= 2u << 4;                 // C format S32
  d |= 1u << 7;                 // A signed 8-bit
  d |= 1u << 10;                // B signed 8-bit
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

__global__ void __launch_bounds__(128, 1)
    i8_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int32_t* C, int M,
            int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = blockIdx.x, tn = blockIdx.y;
  const int nk = K / TK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES, use = kt / STAGES;
      if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      tma_load_2d(sA + s * A_BYTES, &ma, kt * TK, tm * TM, &full[s]);
      tma_load_2d(sB + s * B_BYTES, &mb, kt * TK, tn * TN, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = idesc_i8(TM, TN);
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint64_t da = smem_desc_sw128(sA + s * A_BYTES), db = smem_desc_sw128(sB + s * B_BYTES);
#pragma unroll
      for (int k = 0; k < TK / 32; ++k) {  // UMMA_K = 32 int8: advance the start address by 32 B
        const uint32_t acc = (kt | k) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(done))
                 : "memory");
  }
  // epilogue: every warp reads its 32 TMEM lanes (= rows)
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = tm * TM + warp * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < TN; c += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    int32_t* dst = C + (int64_t)row * N + tn * TN + c;
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<int4*>(dst + j) = make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TN));
}

__global__ void ref_gemm(const int8_t* A, const int8_t* B, int32_t* C, int M, int N, int K) {
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  if (i >= M || j >= N) return;
  int32_t s = 0;
  for (int k = 0; k < K; ++k) s += (int32_t)A[(int64_t)i * K + k] * (int32_t)B[(int64_t)j * K + k];
  C[(int64_t)i * N + j] = s;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool enc(CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
  static EncFn fn = nullptr;
  if (!fn) {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = (EncFn)p;
  }
  cuuint64_t dims[2] = {cols, rows}, strides[1] = {cols};
  cuuint32_t box[2] = {bc, br}, es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 4096, N = argc > 2 ? atoi(argv[2]) : 4096, K = argc > 3 ? atoi(argv[3]) : 4096;
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
  uint64_t x = 88172645463325252ull;
  for (auto& v : hA) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int8_t)((x >> 24) % 255 - 127); }
  for (auto& v : hB) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int8_t)((x >> 24) % 255 - 127); }
  int8_t *A, *B; int32_t *C, *R;
  cudaMalloc(&A, hA.size()); cudaMalloc(&B, hB.size());
  cudaMalloc(&C, (size_t)M * N * 4); cudaMalloc(&R, (size_t)M * N * 4);
  cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  if (!enc(&ma, A, K, M, TK, TM) || !enc(&mb, B, K, N, TK, TN)) return 1;
  const size_t smem = STAGES * STAGE_BYTES + 1024 + 256;
  cudaFuncSetAttribute(i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(M / TM, N / TN);
  i8_gemm<<<grid, 128, smem>>>(ma, mb, C, M, N, K);
  cudaError_t e = cudaDeviceSynchronize();
  printf("i8_gemm: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  ref_gemm<<<dim3(N / 16, M / 16), dim3(16, 16)>>>(A, B, R, M, N, K);
  cudaDeviceSynchronize();
  std::vector<int32_t> hC((size_t)M * N), hR((size_t)M * N);
  cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hR.data(), R, hR.size() * 4, cudaMemcpyDeviceToHost);
  size_t bad = 0, first = (size_t)-1;
  for (size_t i = 0; i < hC.size(); ++i)
    if (hC[i] != hR[i]) { if (first == (size_t)-1) first = i; ++bad; }
  printf("mismatches: %zu of %zu", bad, hC.size());
  if (bad) printf(" (first at %zu: got %d want %d)", first, hC[first], hR[first]);
  printf("\n");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) i8_gemm<<<grid, 128, smem>>>(ma, mb, C, M, N, K);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) i8_gemm<<<grid, 128, smem>>>(ma, mb, C, M, N, K);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("M=N=%d K=%d: %.3f ms, %.1f TOPS\n", M, K, ms, 2.0 * M * N * K / ms / 1e9);
  return 0;
}
