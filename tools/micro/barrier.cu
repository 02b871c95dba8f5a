// Microbenchmark: software grid barrier variants (tools only).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_empty() {}
template <int SLEEP>
__global__ void k_flat(int *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c, 1);
    while (*(volatile int *)c < (int)gridDim.x) __nanosleep(SLEEP);
    __threadfence();
  }
  __syncthreads();
}
// arrive on one counter; the last arriver releases 32 flags (one line each); CTAs poll their flag
__global__ void k_flags(int *c, int *flags) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(c, 1) == (int)gridDim.x - 1) {
      for (int g = 0; g < 32; g++) *(volatile int *)(flags + g * 32) = 1;
    } else {
      volatile int *f = flags + (blockIdx.x & 31) * 32;
      while (*f == 0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}
// arrive via ld.acquire polling with atom.add.release
__global__ void k_acq(int *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int v;
    asm volatile("atom.add.release.gpu.s32 %0, [%1], 1;" : "=r"(v) : "l"(c) : "memory");
    do {
      asm volatile("ld.acquire.gpu.s32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    } while (v < (int)gridDim.x);
  }
  __syncthreads();
}
__global__ void k_cg() { cg::this_grid().sync(); }
int main() {
  int *c, *f;
  cudaMalloc(&c, 1 << 20);
  cudaMalloc(&f, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, auto launch) {
    for (int w = 0; w < 3; w++) { cudaMemset(c, 0, 4096); cudaMemset(f, 0, 8192); launch(); }
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int it = 0; it < 30; it++) {
      cudaMemset(c, 0, 4096);
      cudaMemset(f, 0, 8192);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-36s %8.2f us  %s\n", name, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int n : {592, 1184, 1776, 2368}) {
    char nm[64];
    snprintf(nm, 64, "empty x%d", n); timeit(nm, [&] { k_empty<<<n, 64>>>(); });
    snprintf(nm, 64, "flat sleep32 x%d", n); timeit(nm, [&] { k_flat<32><<<n, 64>>>(c); });
    snprintf(nm, 64, "flat sleep256 x%d", n); timeit(nm, [&] { k_flat<256><<<n, 64>>>(c); });
    snprintf(nm, 64, "flat nosleep x%d", n); timeit(nm, [&] { k_flat<0><<<n, 64>>>(c); });
    snprintf(nm, 64, "release flags x%d", n); timeit(nm, [&] { k_flags<<<n, 64>>>(c, f); });
    snprintf(nm, 64, "acq/rel x%d", n); timeit(nm, [&] { k_acq<<<n, 64>>>(c); });
    snprintf(nm, 64, "cg grid.sync x%d", n);
    timeit(nm, [&] {
      void *args[] = {};
      cudaLaunchCooperativeKernel((void *)k_cg, dim3(n), dim3(64), args, 0, 0);
    });
  }
  return 0;
}
