// Latency calibration on B200: dependent chains of FP64 ops, shuffles, smem and L2 loads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, const double* g, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x = out[threadIdx.x] + 1.0, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  t1 = clock64(); cyc[1] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  t1 = clock64(); cyc[2] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64(); cyc[3] = t1 - t0;
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64(); cyc[4] = t1 - t0;
  // smem dependent load chain
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v + i) & 1023; x += v; }
  t1 = clock64(); cyc[5] = t1 - t0;
  // L2 (ld.cg) dependent chain
  long gi = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = __ldcg(g + gi); gi = ((long)v + i * 4099) & ((1 << 20) - 1); x += v; }
  t1 = clock64(); cyc[6] = t1 - t0;
  // log1p chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = log1p(x * 1e-3);
  t1 = clock64(); cyc[7] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64(); cyc[8] = t1 - t0;
  // __syncthreads chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); cyc[9] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double *out, *g; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&g, (1 << 20) * 8 + 64); cudaMallocManaged(&cyc, 16 * 8);
  cudaMemset(out, 0, 1024 * 8); cudaMemset(g, 0, (1 << 20) * 8);
  const int n = 256;
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 256>>>(out, cyc, g, n); cudaDeviceSynchronize(); }
  const char* nm[] = {"dfma", "ddiv", "dsqrt", "drsqrt", "shfl", "lds", "ld.cg(L2)", "log1p", "dmul", "syncthreads(256)"};
  for (int i = 0; i < 10; ++i) printf("%-18s %7.1f cycles/op\n", nm[i], (double)cyc[i] / n);
  return 0;
}
