// Host cost of cudaLaunchKernelEx (PDL attribute) vs kernel parameter size.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/micro/launch_cost tools/micro/launch_cost.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct P { long long v[N / 8]; };
template <int N> __global__ void k(P<N> p) { if (p.v[0] == 12345 && threadIdx.x == 999) printf("x"); }
template <int N> double run(cudaStream_t st, int grid, bool pdl) {
  P<N> p{};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 100; i++) cudaLaunchKernelEx(&cfg, k<N>, p);
  cudaStreamSynchronize(st);
  auto t0 = std::chrono::steady_clock::now();
  const int n = 2000;
  for (int i = 0; i < n; i++) cudaLaunchKernelEx(&cfg, k<N>, p);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; pdl++) {
    printf("pdl=%d: 64B %.2f us, 512B %.2f us, 1024B %.2f us, 2048B %.2f us per launch (grid 740)\n", pdl,
           run<64>(st, 740, pdl), run<512>(st, 740, pdl), run<1024>(st, 740, pdl), run<2048>(st, 740, pdl));
  }
  return 0;
}
