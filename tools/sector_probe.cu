// DRAM read granularity probe: read `bytes_per_line` of every 128-byte line of a 2 GiB
// buffer (16-byte loads, L1 bypassed) and let ncu report dram__bytes_read.sum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sector_probe tools/sector_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(const double2* __restrict__ src, size_t lines, int chunks_per_line, double* sink) {
  double acc = 0.0;
  for (size_t l = blockIdx.x * (size_t)blockDim.x + threadIdx.x; l < lines * chunks_per_line;
       l += (size_t)gridDim.x * blockDim.x) {
    const size_t line = l / chunks_per_line, c = l % chunks_per_line;
    const double2 v = __ldcg(src + line * 8 + c);  // 8 x 16 B per 128-byte line
    acc += v.x + v.y;
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)2 << 30, lines = bytes / 128;
  double2* buf;
  double* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int cpl : {2, 4, 8}) {  // 32, 64, 128 bytes read per line
    probe<<<148 * 8, 256>>>(buf, lines, cpl, sink);
    cudaEventRecord(e0);
    probe<<<148 * 8, 256>>>(buf, lines, cpl, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bytes/line %3d: %.3f ms, requested %.2f GB/s\n", cpl * 16, ms, lines * cpl * 16.0 / ms / 1e6);
  }
  return 0;
}
