// FP64 tensor-core throughput by mma.sync shape and by the number of independent
// accumulator chains per warp (sm_100a): is m8n8k4 issue/latency-limited where m16n8k16 is not?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes dmma_shapes.cu && ./dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k884(double* out, int iters, double a0, double b0) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  double a = a0 + threadIdx.x, b = b0 - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k16816(double* out, int iters, double a0, double b0) {
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + threadIdx.x + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 - threadIdx.x - i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    const int thr = warps * 32;
#define RUN884(CH)                                                                          \
  {                                                                                         \
    double ms = timeit([&] { k884<CH><<<148, thr>>>(out, iters, 1.0, 2.0); });             \
    printf("m8n8k4   warps/SM %2d chains %d: %6.2f TFLOP/s\n", warps, CH,                    \
           2.0 * 256 * CH * (double)iters * warps * 148 / (ms * 1e-3) / 1e12);              \
  }
#define RUN16816(CH)                                                                        \
  {                                                                                         \
    double ms = timeit([&] { k16816<CH><<<148, thr>>>(out, iters / 8, 1.0, 2.0); });       \
    printf("m16n8k16 warps/SM %2d chains %d: %6.2f TFLOP/s\n", warps, CH,                    \
           2.0 * 2048 * CH * (double)(iters / 8) * warps * 148 / (ms * 1e-3) / 1e12);       \
  }
    RUN884(1) RUN884(2) RUN884(4) RUN884(8) RUN16816(1) RUN16816(2) RUN16816(4)
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
