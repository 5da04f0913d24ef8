// FP64 peak microbenchmarks for B200 (sm_100a): register-only DMMA (mma.sync f64)
// and DFMA loops over all SMs. Output: one JSON object on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"device\": \"%s\", \"sms\": %d, \"smem_per_sm\": %zu, \"smem_optin_per_block\": %zu, \"l2_bytes\": %d, \"regs_per_sm\": %d",
         p.name, sms, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_rate_khz\": %d", clk);
  // DMMA: flops per mma.m8n8k4 = 2*8*8*4 = 512 per warp-instruction
  for (int warps : {4, 8, 16}) {
    int iters = 20000; int blocks = sms * 2;
    for (int rep = 0; rep < 2; ++rep) dmma_loop<8><<<blocks, warps * 32>>>(out, 200, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dmma_loop<8><<<blocks, warps * 32>>>(out, iters, 1.0); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 512.0 * 8 * iters * (double)blocks * warps;
    printf(", \"dmma_tflops_w%d\": %.3f", warps, flops / (best * 1e-3) / 1e12);
  }
  for (int warps : {4, 8, 16}) {
    int iters = 20000; int blocks = sms * 2;
    for (int rep = 0; rep < 2; ++rep) dfma_loop<8><<<blocks, warps * 32>>>(out, 200, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dfma_loop<8><<<blocks, warps * 32>>>(out, iters, 1.0); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)blocks * warps * 32;
    printf(", \"dfma_tflops_w%d\": %.3f", warps, flops / (best * 1e-3) / 1e12);
  }
  // sustained DMMA for ~4 s
  {
    int warps = 8, blocks = sms * 2, iters = 200000;
    cudaEventRecord(e0);
    int n = 0; float ms = 0;
    while (ms < 4000.0f) { dmma_loop<8><<<blocks, warps * 32>>>(out, iters, 1.0); ++n;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    double flops = 512.0 * 8 * iters * (double)blocks * warps * n;
    printf(", \"dmma_tflops_sustained\": %.3f", flops / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
