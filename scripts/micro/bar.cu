// Grid-barrier latency on B200: per-CTA flags (release/relaxed poll), atomic counter,
// and cooperative_groups grid.sync, with 148 co-resident CTAs.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void bar_flags(unsigned* flags, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) st_release(flags + blockIdx.x, epoch);
  if (threadIdx.x < 32) {
    for (;;) {
      bool ok = true;
      for (int c = threadIdx.x; c < gridDim.x; c += 32) ok = ok && (ld_relaxed(flags + c) >= epoch);
      if (__all_sync(0xffffffffu, ok)) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__device__ void bar_flags_padded(unsigned* flags, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) st_release(flags + blockIdx.x * 32, epoch);
  if (threadIdx.x < 32) {
    for (;;) {
      bool ok = true;
      for (int c = threadIdx.x; c < gridDim.x; c += 32) ok = ok && (ld_relaxed(flags + c * 32) >= epoch);
      if (__all_sync(0xffffffffu, ok)) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__device__ void bar_atomic(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(bar, 1u);
    if (prev + 1u == epoch * gridDim.x) {
      st_release(bar + 32, epoch);
    } else {
      while (ld_acquire(bar + 32) < epoch) {}
    }
  }
  __syncthreads();
}
// one master CTA gathers, then broadcasts
__device__ void bar_master(unsigned* flags, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) st_release(flags + blockIdx.x, epoch);
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    for (;;) {
      bool ok = true;
      for (int c = threadIdx.x; c < gridDim.x; c += 32) ok = ok && (ld_relaxed(flags + c) >= epoch);
      if (__all_sync(0xffffffffu, ok)) break;
    }
    if (threadIdx.x == 0) st_release(flags + 1024, epoch);
  }
  if (threadIdx.x == 0) {
    while (ld_acquire(flags + 1024) < epoch) {}
  }
  __syncthreads();
}
__global__ void k(unsigned* w, long long* out, int n, int mode) {
  unsigned epoch = 0;
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < 4; ++i) {
    if (mode == 0) bar_flags(w, epoch);
    else if (mode == 1) bar_atomic(w, epoch);
    else if (mode == 2) grid.sync();
    else if (mode == 3) bar_flags_padded(w, epoch);
    else bar_master(w, epoch);
  }
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (mode == 0) bar_flags(w, epoch);
    else if (mode == 1) bar_atomic(w, epoch);
    else if (mode == 2) grid.sync();
    else if (mode == 3) bar_flags_padded(w, epoch);
    else bar_master(w, epoch);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* w; long long* out;
  cudaMalloc(&w, 1 << 20); cudaMallocManaged(&out, 1024 * 8);
  const char* nm[] = {"flags", "atomic", "cg.grid.sync", "flags padded", "master"};
  for (int G : {16, 32, 64, 148}) {
    for (int mode = 0; mode < 5; ++mode) {
      cudaMemset(w, 0, 1 << 20);
      int n = 1000;
      void* args[] = {&w, &out, &n, &mode};
      cudaLaunchCooperativeKernel((void*)k, G, 256, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      long long mx = 0;
      for (int i = 0; i < G; ++i) mx = out[i] > mx ? out[i] : mx;
      printf("G=%3d %-14s %7.1f cycles = %5.2f us per barrier (%s)\n", G, nm[mode], (double)mx / n,
             (double)mx / n / 1965.0, cudaGetErrorString(e));
    }
  }
  return 0;
}
