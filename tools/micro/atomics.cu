// Microbenchmark: cost of same-address vs striped atomics from many CTAs, and
// of a software grid barrier (tools only; not part of the library).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_same(int *c, int reps) {
  if (threadIdx.x == 0)
    for (int r = 0; r < reps; r++) atomicAdd(c, 1);
}
__global__ void k_same_ret(int *c, int *out, int reps) {
  if (threadIdx.x == 0) {
    int s = 0;
    for (int r = 0; r < reps; r++) s += atomicAdd(c, 1);
    out[blockIdx.x] = s;
  }
}
__global__ void k_striped(int *c, int reps) {
  if (threadIdx.x == 0)
    for (int r = 0; r < reps; r++) atomicAdd(c + (blockIdx.x & 31) * 32, 1);
}
__global__ void k_warp_all(int *c) {   // every warp's lane 0
  if ((threadIdx.x & 31) == 0) atomicAdd(c, 1);
}
__global__ void k_load_same(const int *c, int *out) {   // every warp reads one word
  int v = __ldcg(c);
  if (v == 12345) out[0] = v;
}
__global__ void k_empty() {}
__global__ void k_barrier(int *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c, 1);
    while (*(volatile int *)c < (int)gridDim.x) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}
int main() {
  int *c, *out;
  cudaMalloc(&c, 1 << 20);
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, auto launch) {
    for (int w = 0; w < 3; w++) { cudaMemset(c, 0, 1 << 20); launch(); }
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int it = 0; it < 20; it++) {
      cudaMemset(c, 0, 1 << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %8.2f us\n", name, best * 1e3);
  };
  timeit("empty 1776x64", [&] { k_empty<<<1776, 64>>>(); });
  for (int n : {148, 592, 1184, 1776, 2368}) {
    char nm[64];
    snprintf(nm, 64, "same-addr RED x%d CTAs", n);
    timeit(nm, [&] { k_same<<<n, 64>>>(c, 1); });
    snprintf(nm, 64, "same-addr ATOM(ret) x%d CTAs", n);
    timeit(nm, [&] { k_same_ret<<<n, 64>>>(c, out, 1); });
    snprintf(nm, 64, "striped32 RED x%d CTAs", n);
    timeit(nm, [&] { k_striped<<<n, 64>>>(c, 1); });
  }
  timeit("same-addr RED 1184 CTAs x 8 reps", [&] { k_same<<<1184, 64>>>(c, 8); });
  timeit("warp-all RED 1184x128", [&] { k_warp_all<<<1184, 128>>>(c); });
  timeit("load same word 1184x128", [&] { k_load_same<<<1184, 128>>>(c, out); });
  timeit("grid barrier 1776x64", [&] { k_barrier<<<1776, 64>>>(c); });
  timeit("grid barrier 592x256", [&] { k_barrier<<<592, 256>>>(c); });
  return 0;
}
