// Compressible-memory probe: does B200's generic memory compression cut the DRAM write
// traffic of the batched leaf's output (the full 32x32 inverse: lower triangle dense, the
// upper triangle +0.0 by contract)?  Writes 131072 such matrices (1 GiB) into (a) cudaMalloc
// memory and (b) a cuMemCreate allocation with CU_MEM_ALLOCATION_COMP_GENERIC, plus an
// all-nonzero and an all-zero pattern, and times each with CUDA events; ncu's
// dram__bytes_write.sum per launch gives the traffic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/comp_probe tools/comp_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

// pattern 0: leaf output (lower triangle nonzero, upper zero); 1: all nonzero; 2: all zero
__global__ void write_pattern(double2* __restrict__ dst, int batch, int pattern) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b = warp; b < batch; b += nwarps) {
    double2* m = dst + (size_t)b * 512;
    for (int r = 0; r < 32; ++r) {
      if (lane >= 16) continue;
      const int c0 = 2 * lane;
      double2 v;
      const double base = 1.0 + 1e-3 * (b & 1023) + 1e-6 * r;
      v.x = (pattern == 2 || (pattern == 0 && c0 > r)) ? 0.0 : base + 1e-9 * c0;
      v.y = (pattern == 2 || (pattern == 0 && c0 + 1 > r)) ? 0.0 : base + 1e-9 * (c0 + 1);
      m[r * 16 + lane] = v;
    }
  }
}

__global__ void read_sum(const double2* __restrict__ src, size_t n2, double* sink) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcg(src + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) sink[0] = acc;
}

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)

int main() {
  const int batch = 131072;
  const size_t bytes = (size_t)batch * 8192;
  cudaFree(0);
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int comp_ok = 0;
  CK(cuDeviceGetAttribute(&comp_ok, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev));
  printf("generic compression supported: %d\n", comp_ok);

  double2* plain;
  cudaMalloc(&plain, bytes);
  double* sink;
  cudaMalloc(&sink, 8);

  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.allocFlags.compressionType = CU_MEM_ALLOCATION_COMP_GENERIC;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, sz, &prop, 0));
  CUmemAllocationProp got = {};
  CK(cuMemGetAllocationPropertiesFromHandle(&got, h));
  printf("granularity %zu, compressionType after create: %d\n", gran, (int)got.allocFlags.compressionType);
  CUdeviceptr cptr;
  CK(cuMemAddressReserve(&cptr, sz, 0, 0, 0));
  CK(cuMemMap(cptr, sz, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(cptr, sz, &acc, 1));
  double2* comp = (double2*)cptr;

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"leaf-output", "all-nonzero", "all-zero"};
  for (int which = 0; which < 2; ++which) {
    double2* dst = which ? comp : plain;
    for (int p = 0; p < 3; ++p) {
      write_pattern<<<148 * 8, 256>>>(dst, batch, p);
      cudaEventRecord(e0);
      write_pattern<<<148 * 8, 256>>>(dst, batch, p);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      read_sum<<<148 * 8, 256>>>(dst, bytes / 16, sink);
      cudaEventRecord(e0);
      read_sum<<<148 * 8, 256>>>(dst, bytes / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float rms;
      cudaEventElapsedTime(&rms, e0, e1);
      printf("%-11s %-11s write %.3f ms (%.0f GB/s logical)  read %.3f ms (%.0f GB/s logical)\n",
             which ? "compressible" : "cudaMalloc", names[p], ms, bytes / ms / 1e6, rms, bytes / rms / 1e6);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
