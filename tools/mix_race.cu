// Standalone reproduction probe for the Strassen operand-sum pass under two concurrent streams:
// each stream runs (sum kernel -> check kernel) many times on its own buffers; the check counts
// entries that differ from the sum recomputed from the inputs.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda.h>

struct Mix {
  const double* in[7];
  int64_t ldin[7];
  double* out[5];
  int64_t ldout[5];
  double c[5][7];
  int nin, nout;
};
template <int NIN, int NOUT>
__global__ void __launch_bounds__(256) mix_kernel(int64_t rows, int64_t cols, double beta, const Mix m) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    for (int64_t j = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); j < cols;
         j += 2 * (int64_t)gridDim.x * blockDim.x) {
      double2 v[NIN];
#pragma unroll
      for (int q = 0; q < NIN; ++q) v[q] = __ldcg(reinterpret_cast<const double2*>(m.in[q] + i * m.ldin[q] + j));
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        double2* dst = reinterpret_cast<double2*>(m.out[o] + i * m.ldout[o] + j);
        double2 acc = make_double2(0.0, 0.0);
        if (beta != 0.0) { acc = __ldcg(dst); acc.x *= beta; acc.y *= beta; }
#pragma unroll
        for (int q = 0; q < NIN; ++q)
          if (m.c[o][q] != 0.0) { acc.x = fma(m.c[o][q], v[q].x, acc.x); acc.y = fma(m.c[o][q], v[q].y, acc.y); }
        *dst = acc;
      }
    }
  }
}
__global__ void check_kernel(int64_t q, const Mix m, unsigned long long* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q * q; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / q, j = e % q;
    for (int o = 0; o < m.nout; ++o) {
      double acc = 0.0;
      for (int k = 0; k < m.nin; ++k) if (m.c[o][k] != 0.0) acc = fma(m.c[o][k], m.in[k][i * m.ldin[k] + j], acc);
      if (m.out[o][i * m.ldout[o] + j] != acc) atomicAdd(bad, 1ull);
    }
  }
}
// TMA reader: each CTA loads [32 rows][4 cols] boxes of slot o via cp.async.bulk.tensor and compares
__global__ void tma_check_kernel(const __grid_constant__ CUtensorMap map, int64_t q, const Mix m, int o,
                                 unsigned long long* bad) {
  __shared__ __align__(128) double box[32 * 4];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sbox = (uint32_t)__cvta_generic_to_shared(box), sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int64_t t = blockIdx.x; t < (q / 32) * (q / 4); t += gridDim.x) {
    const int r0 = (int)(t / (q / 4)) * 32, c0 = (int)(t % (q / 4)) * 4;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(32 * 4 * 8) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sbox), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(r0), "r"(sbar) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(sbar), "r"(phase) : "memory");
    phase ^= 1;
    if (threadIdx.x < 128) {
      const int i = r0 + threadIdx.x / 4, j = c0 + threadIdx.x % 4;
      double acc = 0.0;
      for (int k = 0; k < m.nin; ++k) if (m.c[o][k] != 0.0) acc = fma(m.c[o][k], m.in[k][i * m.ldin[k] + j], acc);
      if (box[threadIdx.x] != acc) atomicAdd(bad, 1ull);
    }
    __syncthreads();
  }
}
__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}
__global__ void init_kernel(double* p, int64_t n, uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed + e) * 0x9E3779B97F4A7C15ull; z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    p[e] = (double)(z >> 11) * (1.0 / 9007199254740992.0);
  }
}

int main(int argc, char** argv) {
  const int64_t q = argc > 1 ? atoll(argv[1]) : 1024, n = 2 * q;
  const int reps = argc > 2 ? atoi(argv[2]) : 200;
  const int mode = argc > 3 ? atoi(argv[3]) : 1;  // 1 = two streams, 0 = one stream
  cudaStream_t st[2];
  cudaStreamCreateWithFlags(&st[0], cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&st[1], cudaStreamNonBlocking);
  double *A[2], *S[2];
  Mix m[2];
  unsigned long long* bad;
  cudaMalloc(&bad, 2 * sizeof(unsigned long long));
  cudaMemset(bad, 0, 2 * sizeof(unsigned long long));
  const double ac[5][4] = {{1, 0, 0, 1}, {0, 0, 1, 1}, {1, 1, 0, 0}, {-1, 0, 1, 0}, {0, 1, 0, -1}};
  for (int k = 0; k < 2; ++k) {
    cudaMalloc(&A[k], n * n * sizeof(double));
    cudaMalloc(&S[k], 5 * q * q * sizeof(double));
    init_kernel<<<1024, 256>>>(A[k], n * n, 1234567ull * (k + 1));
    m[k] = Mix{};
    m[k].nin = 4; m[k].nout = 5;
    const double* in[4] = {A[k], A[k] + q, A[k] + q * n, A[k] + q * n + q};
    for (int i = 0; i < 4; ++i) { m[k].in[i] = in[i]; m[k].ldin[i] = n; }
    for (int o = 0; o < 5; ++o) {
      m[k].out[o] = S[k] + o * q * q; m[k].ldout[o] = q;
      for (int i = 0; i < 4; ++i) m[k].c[o][i] = ac[o][i];
    }
  }
  CUtensorMap maps[2][5];
  for (int k = 0; k < 2; ++k)
    for (int o = 0; o < 5; ++o) {
      cuuint64_t dims[2] = {(cuuint64_t)q, (cuuint64_t)q}, strides[1] = {(cuuint64_t)q * 8};
      cuuint32_t box[2] = {4, 32}, es[2] = {1, 1};
      CUresult rc = cuTensorMapEncodeTiled(&maps[k][o], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, m[k].out[o], dims, strides,
                                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (rc != CUDA_SUCCESS) { printf("encode failed %d\n", (int)rc); return 1; }
    }
  cudaDeviceSynchronize();
  const int64_t bx = (q / 2 + 255) / 256;
  const dim3 grid((unsigned)(bx < 8 ? bx : 8), (unsigned)(q < 65535 ? q : 65535));
  for (int r = 0; r < reps; ++r)
    for (int k = 0; k < 2; ++k) {
      cudaStream_t s = (mode & 1) ? st[k] : st[0];
      fill_kernel<<<1024, 256, 0, s>>>(S[k], 5 * q * q, nan(""));
      mix_kernel<4, 5><<<grid, 256, 0, s>>>(q, q, 0.0, m[k]);
      if (mode & 2) {
        for (int o = 0; o < 5; ++o) tma_check_kernel<<<296, 128, 0, s>>>(maps[k][o], q, m[k], o, bad + k);
      } else {
        check_kernel<<<1024, 256, 0, s>>>(q, m[k], bad + k);
      }
    }
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
  printf("q=%lld reps=%d mode=%d: bad entries stream0 %llu stream1 %llu  (%s)\n", (long long)q, reps, mode, h[0], h[1],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
