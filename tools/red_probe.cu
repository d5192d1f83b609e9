// red_probe.cu -- does sharing a 32-B sector between the lanes of one RED instruction raise the
// L2 reduction rate?  (k_points issues 4 single-lane-per-sector REDs per cell
// group.)  Each warp instruction reduces into records of 4 x 8 B (one sector) spread pseudo-
// randomly over a region; `G` lanes of an instruction hit words 0..G-1 of the same record, and
// only `act` of the 32 lanes are active (k_points: ~7).  Reported: ops/s and records/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_probe tools/red_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool kF64>
__global__ void k_red(unsigned long long *buf, long long recs, int iters, int G, int act) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (lane >= act) return;
  const int grp = lane / G, word = lane % G;
  for (int it = 0; it < iters; ++it) {
    const unsigned long long key = (unsigned long long)((w * iters + it) * 32 + grp);
    const long long r = (long long)(((key * 2654435761ull) >> 7) & (unsigned long long)(recs - 1));  // recs: power of 2
    unsigned long long *p = buf + r * 4 + word;
    if (kF64)
      asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(1.0) : "memory");
    else
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory");
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long recs_l2 = 1 << 20;   // 32 MB of records (L2 resident, ~ the maps in flight)
  unsigned long long *buf;
  cudaMalloc(&buf, recs_l2 * 32);
  cudaMemset(buf, 0, recs_l2 * 32);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 3, threads = 256, iters = 512;
  const int Gs[] = {1, 2, 4};
  const int acts[] = {32, 8};
  for (int f64 = 0; f64 < 2; ++f64)
    for (int act : acts)
      for (int G : Gs) {
        auto run = [&] {
          if (f64) k_red<true><<<blocks, threads>>>(buf, recs_l2, iters, G, act);
          else k_red<false><<<blocks, threads>>>(buf, recs_l2, iters, G, act);
        };
        run();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
          cudaEventRecord(a);
          run();
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        const double ops = (double)blocks * (threads / 32) * act * iters;
        printf("%s act=%2d lanes/sector=%d: %8.1f us  %7.1f Gop/s  %7.1f Gsector/s\n", f64 ? "f64" : "u64", act, G,
               best * 1e3, ops / (best * 1e-3) / 1e9, ops / G / (best * 1e-3) / 1e9);
      }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
