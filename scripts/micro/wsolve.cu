// Warp-0 triangular solve (shuffle column sweep) while 7 warps wait at a barrier.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int Q = 9;
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const double* Gin, double* out, long long* cyc, int reps) {
  __shared__ double Gm[Q * Q], dGi[Q];
  extern __shared__ double dyn[];
  if (MODE >= 1) { for (int e = threadIdx.x; e < 1000; e += blockDim.x) dyn[e] = e; }
  for (int e = threadIdx.x; e < Q * Q; e += blockDim.x) Gm[e] = Gin[e];
  if (threadIdx.x < Q) dGi[threadIdx.x] = 1.0 / Gin[threadIdx.x * Q + threadIdx.x];
  __syncthreads();
  double res = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < 32) {
      const int r = threadIdx.x;
      __syncwarp();
      double acc = (r < Q) ? 1.0 + r : 0.0, z = 0.0;
      const double gdi = (r < Q) ? dGi[r] : 0.0;
#pragma unroll 1
      for (int j = Q - 1; j >= 0; --j) {
        const double zj = __shfl_sync(0xffffffffu, acc * gdi, j);
        const double gji = (r < Q) ? Gm[j * Q + r] : 0.0;
        const double nacc = acc - gji * zj;
        z = (r == j) ? zj : z;
        acc = (r < j) ? nacc : acc;
      }
      res += z;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = res;
}
int main() {
  double *G, *out; long long* cyc;
  cudaMallocManaged(&G, Q * Q * 8); cudaMallocManaged(&out, 148 * 256 * 8); cudaMallocManaged(&cyc, 148 * 8);
  for (int i = 0; i < Q * Q; ++i) G[i] = (i % (Q + 1) == 0) ? 2.0 : 0.1;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int reps = 1000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      void* args[] = {&G, &out, &cyc, &reps};
      if (mode == 0) k<0><<<148, 256>>>(G, out, cyc, reps);
      else if (mode == 1) k<1><<<148, 256, 200 * 1024>>>(G, out, cyc, reps);
      else cudaLaunchCooperativeKernel((void*)k<2>, 148, 256, args, 200 * 1024, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) printf("err %s\n", cudaGetErrorString(e));
    }
    printf("mode %d: %.1f cycles per 9-step solve (%.1f per step)\n", mode, cyc[0] / 1000.0, cyc[0] / 9000.0);
  }
  return 0;
}
