#!/usr/bin/env python
"""Generate scripts/micro/bin/wsolve_icache.cu: the warp-0 triangular-solve instruction-cache
experiment ("Experiments that did not pay").  The kernel's BIG variant places a
6000-instruction straight-line FMA block in front of the solve so that the solve's code no
longer fits the instruction cache; that filler is generated here instead of being committed.

    python scripts/micro/gen_wsolve_icache.py && nvcc -gencode arch=compute_100a,code=sm_100a \
        -O3 -o scripts/micro/bin/wsolve_icache scripts/micro/bin/wsolve_icache.cu
"""
import os

HEAD = r"""// Warp-0 triangular solve (shuffle column sweep) while 7 warps wait at a barrier.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int Q = 9;
template <bool BIG>
__global__ void k(const double* Gin, double* out, long long* cyc, int reps) {
  __shared__ double Gm[Q * Q], dGi[Q];
  for (int e = threadIdx.x; e < Q * Q; e += blockDim.x) Gm[e] = Gin[e];
  if (threadIdx.x < Q) dGi[threadIdx.x] = 1.0 / Gin[threadIdx.x * Q + threadIdx.x];
  __syncthreads();
  double res = 0.0;
  long long t0 = clock64();
  double bx = Gin[0], by = Gin[1];
  long long tsolve = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (BIG) {"""
TAIL = r"""    }
    __syncthreads();
    const long long ts = clock64();
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
    tsolve += clock64() - ts;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = tsolve;
  (void)t1; (void)t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = res + bx + by;
}
int main() {
  double *G, *out; long long* cyc;
  cudaMallocManaged(&G, Q * Q * 8); cudaMallocManaged(&out, 148 * 256 * 8); cudaMallocManaged(&cyc, 148 * 8);
  for (int i = 0; i < Q * Q; ++i) G[i] = (i % (Q + 1) == 0) ? 2.0 : 0.1;
  for (int blocks : {1, 148}) for (int th : {32, 256}) {
    for (int rep = 0; rep < 2; ++rep) { k<false><<<blocks, th>>>(G, out, cyc, 100); cudaDeviceSynchronize(); }
    long long a = cyc[0];
    for (int rep = 0; rep < 2; ++rep) { k<true><<<blocks, th>>>(G, out, cyc, 100); cudaDeviceSynchronize(); }
    printf("blocks %3d threads %3d: solve-only %.0f cycles/rep, with 6000-FMA block %.0f cycles/rep\n", blocks, th,
           a / 100.0, cyc[0] / 100.0);
  }
  return 0;
}
"""


def main(n_fma: int = 6000) -> str:
    lines = []
    for i in range(1, n_fma + 1):
        a, b = ("bx", "by") if i % 2 else ("by", "bx")
        lines.append(f"    {a} = fma({a}, {b}, {i * 1e-9:.3e});")
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bin", "wsolve_icache.cu")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write(HEAD + "\n" + "\n".join(lines) + "\n" + TAIL)
    return out


if __name__ == "__main__":
    print(main())
