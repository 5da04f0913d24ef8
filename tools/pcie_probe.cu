// PCIe probes for the host-buffer (e2e) path of config 1 (131072 x 32x32 fp64):
// copy engines vs SM zero-copy access to mapped pinned host memory, and host
// zero-fill of the upper 64-byte chunks by CPU threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pcie_probe tools/pcie_probe.cu -lcuda -lpthread
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include "../paper_2307_07611_b200/csrc/ptx.cuh"
using namespace trinv;

constexpr int64_t B = 131072;
constexpr size_t BYTES = (size_t)B * 32 * 32 * 8;

__global__ void read_plain(const double* __restrict__ A, double* out, int64_t batch) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * (int64_t)blockDim.x) >> 5;
  double s = 0;
  for (int64_t b = w; b < batch; b += W) {
    const double* m = A + b * 1024;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (lane < ((i >> 3) + 1) * 8) s += m[i * 32 + lane];  // lower triangle, 64-B granular
  }
  if (s == 12345.0) out[0] = s;
}

__global__ void write_plain(double* X, int64_t batch) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t b = w; b < batch; b += W) {
    double* m = X + b * 1024;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (lane < ((i >> 3) + 1) * 8) m[i * 32 + lane] = (double)(i - lane);
  }
}

// 4 TMA bands (8 rows x 8/16/24/32 cols) per matrix into a per-warp ring, sum, optional write-back.
template <bool WRITE>
__global__ void __launch_bounds__(256, 1) tma_rw(const __grid_constant__ CUtensorMap m8, const __grid_constant__ CUtensorMap m16,
                                                 const __grid_constant__ CUtensorMap m24, const __grid_constant__ CUtensorMap m32,
                                                 double* X, double* out, int64_t batch) {
  constexpr int NS = 4, SLOT = 640;  // 8*(8+16+24+32) doubles
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slots = reinterpret_cast<double*>(sm) + warp * NS * SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 8 * NS * SLOT * 8) + warp * NS;
  const int64_t gw = blockIdx.x * 8 + warp, TW = gridDim.x * 8;
  if (gw >= batch) return;
  const int64_t count = (batch - gw + TW - 1) / TW;
  if (lane == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1); fence_mbar_init(); }
  __syncwarp();
  auto issue = [&](int64_t t) {
    const int b = (int)(gw + t * TW);
    double* slot = slots + (t % NS) * SLOT;
    uint64_t* bar = &bars[t % NS];
    mbar_arrive_expect_tx(bar, SLOT * 8);
    tma_load_3d(slot, &m8, 0, 0, b, bar);
    tma_load_3d(slot + 64, &m16, 0, 8, b, bar);
    tma_load_3d(slot + 192, &m24, 0, 16, b, bar);
    tma_load_3d(slot + 384, &m32, 0, 24, b, bar);
  };
  if (lane == 0) for (int64_t t = 0; t < NS && t < count; ++t) issue(t);
  double s = 0;
  for (int64_t t = 0; t < count; ++t) {
    double* slot = slots + (t % NS) * SLOT;
    mbar_wait(&bars[t % NS], (uint32_t)((t / NS) & 1));
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int band = i >> 3, w = (band + 1) * 8, off = (band == 0 ? 0 : band == 1 ? 64 : band == 2 ? 192 : 384);
      v[i] = lane < w ? slot[off + (i & 7) * w + lane] : 0.0;
    }
    __syncwarp();
    if (t + NS < count && lane == 0) { fence_proxy_async_smem(); issue(t + NS); }
    if (WRITE) {
      double* m = X + (gw + t * TW) * 1024;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (lane < ((i >> 3) + 1) * 8) m[i * 32 + lane] = v[i] * 2.0;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) s += v[i];
    }
  }
  if (s == 12345.0) out[0] = s;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool enc(CUtensorMap* m, void* base, int cols) {
  static EncFn fn = nullptr;
  if (!fn) {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = (EncFn)p;
  }
  cuuint64_t dims[3] = {32, 32, (cuuint64_t)B}, strides[2] = {256, 8192};
  cuuint32_t box[3] = {(cuuint32_t)cols, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

static void zero_upper(double* X, int64_t b0, int64_t b1) {
  for (int64_t b = b0; b < b1; ++b) {
    double* m = X + b * 1024;
    for (int i = 0; i < 24; ++i) {
      const int c0 = ((i >> 3) + 1) * 8;
      memset(m + i * 32 + c0, 0, (32 - c0) * 8);
    }
  }
}

int main() {
  double *Ah, *Xh, *Ad, *Xd, *out;
  cudaHostAlloc(&Ah, BYTES, cudaHostAllocMapped);
  cudaHostAlloc(&Xh, BYTES, cudaHostAllocMapped);
  cudaMalloc(&Ad, BYTES); cudaMalloc(&Xd, BYTES); cudaMalloc(&out, 64);
  memset(Ah, 0, BYTES); memset(Xh, 0, BYTES);
  double *Ahd, *Xhd;
  cudaHostGetDevicePointer(&Ahd, Ah, 0); cudaHostGetDevicePointer(&Xhd, Xh, 0);
  printf("mapped device ptr == host ptr: %d\n", (int)(Ahd == Ah));
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0, s1); fn(); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %8.2f ms  %7.1f GB/s  (%s)\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("CE H2D 1 GiB", BYTES, [&] { cudaMemcpyAsync(Ad, Ah, BYTES, cudaMemcpyHostToDevice, s1); });
  timeit("CE D2H 1 GiB", BYTES, [&] { cudaMemcpyAsync(Xh, Xd, BYTES, cudaMemcpyDeviceToHost, s1); });
  timeit("CE H2D || D2H 1 GiB each (bytes one way)", BYTES, [&] {
    cudaEvent_t f; cudaEventCreate(&f); cudaEventRecord(f, s1); cudaStreamWaitEvent(s2, f, 0);
    cudaMemcpyAsync(Ad, Ah, BYTES, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(Xh, Xd, BYTES, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(f, s2); cudaStreamWaitEvent(s1, f, 0); cudaEventDestroy(f); });
  const double tri = (double)B * 8 * (64 + 128 + 192 + 256);
  timeit("SM plain read, 64B-granular triangle", tri, [&] { read_plain<<<148 * 8, 256, 0, s1>>>(Ahd, out, B); });
  timeit("SM plain write, 64B-granular triangle", tri, [&] { write_plain<<<148 * 8, 256, 0, s1>>>(Xhd, B); });
  CUtensorMap m8, m16, m24, m32;
  const size_t smem = 8 * 4 * 640 * 8 + 8 * 4 * 8;
  cudaFuncSetAttribute(tma_rw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(tma_rw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (enc(&m8, Ahd, 8) && enc(&m16, Ahd, 16) && enc(&m24, Ahd, 24) && enc(&m32, Ahd, 32)) {
    timeit("TMA read from host, 4 bands", tri, [&] { tma_rw<false><<<148, 256, smem, s1>>>(m8, m16, m24, m32, Xhd, out, B); });
    timeit("TMA read + SM write, host<->host (bytes one way)", tri,
           [&] { tma_rw<true><<<148, 256, smem, s1>>>(m8, m16, m24, m32, Xhd, out, B); });
  }
  for (int th : {1, 4, 8, 16}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (int k = 0; k < th; ++k) ts.emplace_back(zero_upper, Xh, B * k / th, B * (k + 1) / th);
    for (auto& t : ts) t.join();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    printf("CPU zero-fill of upper chunks, %2d threads          %8.2f ms  %7.1f GB/s\n", th, ms, B * 3072.0 / ms / 1e6);
  }
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  return 0;
}
