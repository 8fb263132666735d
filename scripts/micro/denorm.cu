// FP64 latency with normal vs subnormal operands on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* io, long long* cyc, int n) {
  double x = io[0], y = io[1], z = io[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, z);
  long long t1 = clock64();
  cyc[0] = t1 - t0;
  double w = io[0];
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = w * y;
  t1 = clock64();
  cyc[1] = t1 - t0;
  double u = io[0];
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = u + z;
  t1 = clock64();
  cyc[2] = t1 - t0;
  io[3] = x + w + u;
}
int main() {
  double* io; long long* cyc;
  cudaMallocManaged(&io, 64); cudaMallocManaged(&cyc, 64);
  double cases[][3] = {{1.0, 0.999999, 1e-9}, {1e-310, 1.0, 1e-312}, {1e-300, 1.0, 1e-310}, {1e-310, 0.5, 0.0}};
  for (auto& c : cases) {
    for (int rep = 0; rep < 2; ++rep) {
      io[0] = c[0]; io[1] = c[1]; io[2] = c[2];
      k<<<1, 32>>>(io, cyc, 1000);
      cudaDeviceSynchronize();
    }
    printf("x=%g y=%g z=%g : dfma %.1f  dmul %.1f  dadd %.1f cycles/op\n", c[0], c[1], c[2],
           cyc[0] / 1000.0, cyc[1] / 1000.0, cyc[2] / 1000.0);
  }
  return 0;
}
