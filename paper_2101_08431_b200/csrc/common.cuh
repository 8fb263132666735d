// Shared helpers for the nmf-b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define NMFB_MAX_K 16

// kernel launches issued by this library (reported by bench.py as gpu_launches)
extern unsigned long long g_nmfb_launches;

// Return codes of the C-ABI (0 = ok, negative = argument / launch error).
enum {
  NMFB_OK = 0,
  NMFB_EINVAL = -1,
  NMFB_ELAUNCH = -2,
  NMFB_ENOMEM = -3,
  NMFB_EUNSUPPORTED = -4,
};

// last CUDA error seen by NMFB_CHECK_LAUNCH (nmfb_last_cuda_error reports it)
extern int g_nmfb_last_cuda_error;

#define NMFB_CHECK_LAUNCH()                                   \
  do {                                                        \
    cudaError_t e__ = cudaGetLastError();                     \
    if (e__ != cudaSuccess) {                                 \
      g_nmfb_last_cuda_error = (int)e__;                      \
      return NMFB_ELAUNCH;                                    \
    }                                                         \
  } while (0)

// Dynamic shared memory opt-in.  The attribute is a per-function CAP, so a launch with
// more dynamic smem than an earlier, smaller setting fails; always raising it to the
// device's opt-in maximum keeps launches of one kernel at different sizes (problems of
// different k / m in one process) valid.  The launch's own size still sets occupancy.
static inline int nmfb_smem_optin_max() {
  static int v = [] {
    int d = 0, x = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return x;
  }();
  return v;
}
// per-kernel cap = opt-in maximum minus the kernel's static shared memory (a larger value
// is rejected), memoised by function address (the function TYPE is shared by kernels with
// the same signature)
static inline int nmfb_smem_cap(const void* f) {
  static const void* keys[256];
  static int caps[256];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == f) return caps[i];
  cudaFuncAttributes a;
  int c = nmfb_smem_optin_max();
  if (cudaFuncGetAttributes(&a, f) == cudaSuccess) c -= (int)a.sharedSizeBytes;
  if (n < 256) keys[n] = f, caps[n] = c, ++n;
  return c;
}
template <typename F>
static inline void nmfb_smem_attr(F* f, size_t bytes) {
  const int cap = nmfb_smem_cap((const void*)f);
  // a request above the cap is passed through: the launch itself reports the error
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (long)bytes > cap ? (int)bytes : cap);
}

static inline int nmfb_blocks(long n, int threads, int cap = 148 * 32) {
  long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic for a fixed
// blockDim).  `sh` needs blockDim.x/32 doubles.  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = -1.0 / 0.0;
  if (wid == 0) {
    r = lane < nw ? sh[lane] : -1.0 / 0.0;
    r = warp_max(r);
  }
  return r;
}
