// host cost of one cudaLaunchKernelEx (PDL attribute) against the kernel parameter size
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
struct P {
  char b[N];
};
template <int N>
__global__ void k_empty(const __grid_constant__ P<N> p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && p.b[0] == 42) printf("x");
}
template <int N>
double run(cudaStream_t s, bool pdl, int iters) {
  P<N> p = {};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k_empty<N>, p);
  cudaStreamSynchronize(s);
  auto t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, k_empty<N>, p);
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStreamSynchronize(s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, k_empty<N>, p);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("param %6d B pdl %d: host %.2f us/launch, device %.2f us/launch\n", N, (int)pdl,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / iters, ms * 1e3 / iters);
  return 0;
}
int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<64>(s, pdl, 2000);
    run<1024>(s, pdl, 2000);
    run<4096>(s, pdl, 2000);
    run<12288>(s, pdl, 2000);
    run<30000>(s, pdl, 2000);
  }
  return 0;
}
