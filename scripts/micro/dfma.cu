// Dependent-chain latency of DFMA vs DMUL/DADD for several operand values (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* in, double* out, long long* cyc, int n) {
  double x = in[0], y = in[1], z = in[2];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) x = fma(x, y, z);
  long long t1 = clock64();
  double w = in[0];
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) w = w * y + z;  // contracted to DFMA too
  long long t3 = clock64();
  double u = in[0];
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) u = __dadd_rn(__dmul_rn(u, y), z);
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t5 - t4; }
  out[threadIdx.x] = x + w + u;
}
int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 64); cudaMallocManaged(&out, 4096); cudaMallocManaged(&cyc, 64);
  double cases[][3] = {{1.0, 0.999999, 1e-9}, {1.0, 1.0000001, 1e-9}, {0.5, 0.5, 0.25},
                       {3.0, 1.0, 0.0}, {1e-310, 1.0, 1e-312}};
  for (int th : {32, 256}) {
    for (auto& c : cases) {
      for (int rep = 0; rep < 2; ++rep) {
        in[0] = c[0]; in[1] = c[1]; in[2] = c[2];
        k<<<1, th>>>(in, out, cyc, 4000);
        cudaDeviceSynchronize();
      }
      printf("threads %3d x=%-6g y=%-10g z=%-6g: fma %.1f  mul+add-contracted %.1f  dmul_rn+dadd_rn %.1f cyc/iter\n",
             th, c[0], c[1], c[2], cyc[0] / 4000.0, cyc[1] / 4000.0, cyc[2] / 4000.0);
    }
  }
  return 0;
}
