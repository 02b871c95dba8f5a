// PDL semantics probe: A (spins, triggers early) -> B (PDL, no grid-dependency
// sync) -> C (PDL, cudaGridDependencySynchronize).  Does C wait for A?
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl tools/micro/pdl_chain.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void kA(int *flag, unsigned long long *out, int spin_us, int trig) {
  if (trig) cudaTriggerProgrammaticLaunchCompletion();
  const unsigned long long t0 = gt();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t0;
  while (gt() - t0 < (unsigned long long)spin_us * 1000ull) {}
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) { __threadfence(); atomicExch(flag, 1); out[1] = gt(); }
}
__global__ void kB(int *flag, unsigned long long *out, int spin_us) {
  const unsigned long long t0 = gt();
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[2] = t0; out[3] = *(volatile int *)flag; }
  while (gt() - t0 < (unsigned long long)spin_us * 1000ull) {}
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = gt();
}
__global__ void kC(int *flag, unsigned long long *out, int gds) {
  if (gds) cudaGridDependencySynchronize();
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[5] = gt(); out[6] = *(volatile int *)flag; }
}
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
  int *flag; unsigned long long *out, h[8];
  cudaMalloc(&flag, 4); cudaMalloc(&out, 64);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  struct Case { const char *name; int gridA, trig, pdlB, pdlC, gdsC, spinB; } cases[] = {
    {"A trig, B pdl short, C pdl+gds", 148, 1, 1, 1, 1, 2},
    {"A trig, B pdl short, C pdl no-gds", 148, 1, 1, 1, 0, 2},
    {"A trig, B pdl short, C plain", 148, 1, 1, 0, 0, 2},
    {"A no trig, B pdl, C pdl+gds", 148, 0, 1, 1, 1, 2},
    {"A trig (full SMs 8x148 CTAs), B pdl, C pdl+gds", 1184, 1, 1, 1, 1, 2},
  };
  for (auto &c : cases) {
    for (int rep = 0; rep < 3; rep++) {
      cudaMemsetAsync(flag, 0, 4, st); cudaMemsetAsync(out, 0, 64, st);
      cudaStreamSynchronize(st);
      launch(false, kA, c.gridA, 128, st, flag, out, 50, c.trig);
      launch(c.pdlB != 0, kB, 148, 128, st, flag, out, c.spinB);
      launch(c.pdlC != 0, kC, 148, 128, st, flag, out, c.gdsC);
      cudaStreamSynchronize(st);
      cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
      if (rep == 2)
        printf("%-50s A %.1f..%.1f  B start %.1f (flag %llu) end %.1f  C start %.1f flag %llu  err=%s\n", c.name, 0.0,
               (h[1] - h[0]) / 1e3, ((long long)h[2] - (long long)h[0]) / 1e3, h[3], ((long long)h[4] - (long long)h[0]) / 1e3,
               ((long long)h[5] - (long long)h[0]) / 1e3, h[6], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
