// probe.cu — live FP64 tensor-core peak for the roofline denominators (bench.py).
// A register-only loop of mma.sync m8n8k4 f64 (SASS DMMA.8x8x4, 512 flop per warp
// instruction) on every SM, timed with events on the caller's stream: the measured
// ceiling of the DMMA engine at the clocks of the run it is taken in.  Diagnostic only
// (it synchronises the stream); not on any product path.
#include <cuda_runtime.h>

#include "../../include/trinv.h"
#include "internal.h"
#include "ptx.cuh"

namespace trinv {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* sink, int iters, double seed) {
  const double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[threadIdx.x] = s;  // never true: keeps the loop live
}

}  // namespace trinv

extern "C" double trinv_probe_dmma_tflops(double ms_target, void* stream) {
  using namespace trinv;
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = device_sms();
  const int blocks = 2 * sms, threads = 256;
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1.0;
  double result = -1.0;
  int iters = 2000;
  for (int pass = 0; pass < 4; ++pass) {
    cudaEventRecord(e0, s);
    dmma_peak_kernel<<<blocks, threads, 0, s>>>(nullptr, iters, 1.0);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * 8.0 * iters * (double)blocks * (threads / 32);
    result = flops / (ms / 1e3) / 1e12;
    if (ms >= 0.5 * ms_target) break;
    iters = (int)(iters * (ms_target / (ms > 1e-3f ? ms : 1e-3f)));  // grow to the target duration
    if (iters > 1 << 26) iters = 1 << 26;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? result : -1.0;
}
