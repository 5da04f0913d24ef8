// L2 fetch-granularity probe.  tools/sector_probe.cu showed that reading 32, 64 or 128 B of
// every 128-byte line moves whole lines from DRAM with the default settings.  This probe
// repeats that read under cudaLimitMaxL2FetchGranularity = default / 32 / 64 / 128 and adds
// the config-1 access pattern: the referenced lower triangle of 131072 row-major 32x32
// matrices read in 16-byte chunks (row i: ceil((i+1)/2) chunks), so that ncu's
// dram__bytes_read.sum per launch says what the 128-byte-line floor of the batched leaf is.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fetch_probe tools/fetch_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void lines(const double2* __restrict__ src, size_t nlines, int chunks_per_line, double* sink) {
  double acc = 0.0;
  for (size_t l = blockIdx.x * (size_t)blockDim.x + threadIdx.x; l < nlines * chunks_per_line;
       l += (size_t)gridDim.x * blockDim.x) {
    const size_t line = l / chunks_per_line, c = l % chunks_per_line;
    const double2 v = __ldcg(src + line * 8 + c);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) sink[0] = acc;
}

// chunk table: the 272 16-byte chunks of the referenced lower triangle (row, chunk-in-row)
__constant__ unsigned char c_row[272], c_col[272];

__global__ void triangle(const double2* __restrict__ src, int batch, double* sink) {
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b = warp; b < batch; b += nwarps) {
    const double2* m = src + (size_t)b * 512;  // 32 rows x 16 double2
    for (int c = lane; c < 272; c += 32) {
      const double2 v = __ldcg(m + c_row[c] * 16 + c_col[c]);
      acc += v.x + v.y;
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)2 << 30, nlines = bytes / 128;
  const int batch = 131072;
  unsigned char hr[272], hc[272];
  int k = 0;
  for (int i = 0; i < 32; ++i)
    for (int c = 0; c < (i + 2) / 2; ++c) { hr[k] = (unsigned char)i; hc[k] = (unsigned char)c; ++k; }
  if (k != 272) { printf("bad table %d\n", k); return 1; }
  cudaMemcpyToSymbol(c_row, hr, 272);
  cudaMemcpyToSymbol(c_col, hc, 272);
  double2* buf;
  double* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 0, bytes);
  size_t dflt = 0;
  cudaDeviceGetLimit(&dflt, cudaLimitMaxL2FetchGranularity);
  printf("default cudaLimitMaxL2FetchGranularity = %zu\n", dflt);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int g : {0, 32, 64, 128}) {
    if (g) {
      cudaError_t st = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
      size_t got = 0;
      cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
      printf("set %d -> %s, now %zu\n", g, cudaGetErrorString(st), got);
    }
    for (int cpl : {2, 4, 8}) {
      lines<<<148 * 8, 256>>>(buf, nlines, cpl, sink);
      cudaEventRecord(e0);
      lines<<<148 * 8, 256>>>(buf, nlines, cpl, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("gran %3d lines bytes/line %3d: %.3f ms, requested %.2f GB/s\n", g, cpl * 16, ms,
             nlines * cpl * 16.0 / ms / 1e6);
    }
    triangle<<<148 * 8, 256>>>(buf, batch, sink);
    cudaEventRecord(e0);
    triangle<<<148 * 8, 256>>>(buf, batch, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("gran %3d triangle (4352 B requested / matrix): %.3f ms, requested %.2f GB/s\n", g, ms,
           batch * 4352.0 / ms / 1e6);
  }
  cudaError_t st = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(st));
  return 0;
}
