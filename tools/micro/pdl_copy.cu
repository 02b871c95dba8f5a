// Does an early programmatic trigger let a following (non-kernel) stream
// operation start before the triggering kernel completes?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/micro/pdl_copy tools/micro/pdl_copy.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void kA(int *flag, int spin_us, int trig, int pdl_launched) {
  if (trig) cudaTriggerProgrammaticLaunchCompletion();
  const unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)spin_us * 1000ull) {}
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) { __threadfence(); *(volatile int *)flag = 1; }
}
__global__ void kNop() {}
template <typename... KArgs, typename... Args>
static void launch(bool pdl, void (*k)(KArgs...), int grid, int block, cudaStream_t st, Args... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, a...);
}
int main() {
  int *flag, *hpin; cudaMalloc(&flag, 4); cudaMallocHost(&hpin, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char *names[] = {"A(pdl-launched, trig) -> memcpy D2H", "A(plain, trig) -> memcpy D2H",
                         "A(pdl-launched, no trig) -> memcpy D2H", "nop, A(pdl, trig) -> memcpy D2H",
                         "nop, A(pdl, trig) -> event record+sync, read via memcpy"};
  for (int c = 0; c < 5; c++) {
    int bad = 0;
    for (int rep = 0; rep < 20; rep++) {
      cudaMemsetAsync(flag, 0, 4, st); *hpin = -1;
      cudaStreamSynchronize(st);
      if (c >= 3) launch(false, kNop, 1, 32, st);
      launch(c != 1, kA, 148, 128, st, flag, 30, c != 2 ? 1 : 0, 1);
      if (c == 4) {
        cudaEvent_t ev; cudaEventCreate(&ev); cudaEventRecord(ev, st); cudaEventSynchronize(ev);
        cudaMemcpy(hpin, flag, 4, cudaMemcpyDeviceToHost); cudaEventDestroy(ev);
      } else {
        cudaMemcpyAsync(hpin, flag, 4, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
      }
      if (*hpin != 1) bad++;
    }
    printf("%-60s stale reads %d / 20  (%s)\n", names[c], bad, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
