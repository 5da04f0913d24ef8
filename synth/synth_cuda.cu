// Device twin of synth.c (bit-identical; see synth.h). Not part of the method.
#include <cuda_runtime.h>
#include "synth.h"

__global__ void synth_fill_kernel(int64_t n, int64_t b0, int64_t count, uint64_t seed0, uint64_t tag,
                                  char uplo, int diag, double* out, int64_t ld, int64_t stride) {
  int64_t total = count * n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / (n * n), r = e - b * n * n, i = r / n, j = r - i * n;
    uint64_t key = synth_key(seed0 + (uint64_t)(b0 + b), tag);
    out[b * stride + i * ld + j] = synth_entry(key, n, i, j, uplo, diag);
  }
}

extern "C" int synth_fill_device(int64_t n, int64_t b0, int64_t count, uint64_t seed0, uint64_t tag,
                                 char uplo, int diag, double* out, int64_t ld, int64_t stride,
                                 void* stream) {
  if (n <= 0 || count <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  synth_fill_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(n, b0, count, seed0, tag, uplo, diag,
                                                               out, ld, stride);
  return (int)cudaGetLastError();
}
