// H2D copy time of one C2 f64 depth frame (2.46 MB) from pinned memory, one
// copy vs split over 2 / 4 streams, timed with events (no host overhead).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/micro/h2d tools/micro/h2d.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 640 * 480 * 8;
  char *h, *d;
  cudaMallocHost(&h, n * 4); cudaMalloc(&d, n * 4);
  cudaStream_t st[4]; for (auto &s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t bytes : {n, n / 4, n * 4}) {
    for (int parts : {1, 2, 4}) {
      float best = 1e9;
      for (int rep = 0; rep < 20; rep++) {
        cudaEventRecord(e0, st[0]);
        for (int p = 1; p < parts; p++) cudaStreamWaitEvent(st[p], e0, 0);
        for (int p = 0; p < parts; p++)
          cudaMemcpyAsync(d + p * bytes / parts, h + p * bytes / parts, bytes / parts, cudaMemcpyHostToDevice, st[p]);
        for (int p = 1; p < parts; p++) { cudaEvent_t ep; cudaEventCreate(&ep); cudaEventRecord(ep, st[p]); cudaStreamWaitEvent(st[0], ep, 0); cudaEventDestroy(ep); }
        cudaEventRecord(e1, st[0]);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%8zu B, %d stream(s): %7.1f us = %5.1f GB/s\n", bytes, parts, best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
