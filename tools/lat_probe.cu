// Dependent-chain latency probes (cycles per op, one warp): DFMA, DMUL, DADD,
// FFMA, DMMA.8x8x4, LDS.64.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
__global__ void probe(double* out, long long* cyc, double a, double b, float fa) {
  __shared__ double sm[64];
  const int t = threadIdx.x;
  sm[t & 63] = (double)(t & 63) * 0 + (double)((t + 1) & 63);
  __syncthreads();
  double x = a, y = b;
  float f = fa;
  long long t0, t1;
  const int N = 1024;
  // DFMA chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = fma(x, a, b);
  t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) y = y * a;
  t1 = clock64();
  if (t == 0) cyc[1] = t1 - t0;
  double z = b;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) z = z + a;
  t1 = clock64();
  if (t == 0) cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) f = fmaf(f, fa, 1.0f);
  t1 = clock64();
  if (t == 0) cyc[3] = t1 - t0;
  double c0 = 0, c1 = 0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  t1 = clock64();
  if (t == 0) cyc[4] = (t1 - t0) * 4;
  int idx = t & 63;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) idx = (int)sm[idx];
  t1 = clock64();
  if (t == 0) cyc[5] = (t1 - t0) * 4;
  // throughput: 8 independent DFMA chains
  double v[8];
  for (int k = 0; k < 8; ++k) v[k] = a + k;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fma(v[k], a, b);
  t1 = clock64();
  if (t == 0) cyc[6] = t1 - t0;
  // MUFU.RCP64H chain (rcp.approx.ftz.f64)
  double r = a;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
  t1 = clock64();
  if (t == 0) cyc[7] = (t1 - t0) * 4;
  // SHFL chain
  int sh = t;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) sh = __shfl_sync(0xffffffffu, sh, (sh + 1) & 31);
  t1 = clock64();
  if (t == 0) cyc[8] = (t1 - t0) * 4;
  // __syncthreads loop
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) __syncthreads();
  t1 = clock64();
  if (t == 0) cyc[9] = (t1 - t0) * 4;
  // __drcp_rn chain
  double q = a;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) q = __drcp_rn(q) + 1e-300;
  t1 = clock64();
  if (t == 0) cyc[10] = (t1 - t0) * 16;
  double s = r + sh + q;
  for (int k = 0; k < 8; ++k) s += v[k];
  out[t] = x + y + z + f + c0 + c1 + idx + s;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 128);
  const char* names[] = {"DFMA", "DMUL", "DADD", "FFMA", "DMMA", "LDS", "DFMA x8 indep (per op-group of 1024)",
                         "MUFU.RCP64H", "SHFL.IDX", "BAR.SYNC", "__drcp_rn (+DADD)"};
  for (int w : {32, 128, 256}) {
    probe<<<1, w>>>(out, cyc, 1.0000001, 1e-9, 1.0000001f);
    cudaDeviceSynchronize();
    printf("threads=%d\n", w);
    for (int i = 0; i < 11; ++i) printf("  %-40s %.2f cyc/op\n", names[i], cyc[i] / 1024.0);
  }
  return 0;
}
