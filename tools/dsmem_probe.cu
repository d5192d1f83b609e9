// dsmem_probe.cu -- reduction rates of the candidate accumulators for a cluster-privatised
// point pass: one map's per-cell sums held in the distributed shared memory of
// an 8-CTA cluster (8 x 192 KB) instead of an L2 scratch.  Each thread issues `iters`
// reductions to pseudo-random words of (a) its own CTA's shared memory, (b) any CTA of its
// cluster (`mapa` + red.shared::cluster), (c) a 32 MB global region (L2 REDs, the current
// design).  Reported: reductions per second over the whole GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kThreads = 512;
constexpr int kWords = 192 * 1024 / 8;  // f64 / u64 words per CTA

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

template <int kMode, int kT>  // kT: 0 u64, 1 f64, 2 u32, 3 f32
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(kThreads, 1)
    k_acc(unsigned long long *gbuf, int iters, unsigned long long *out) {
  extern __shared__ unsigned long long s[];
  for (int i = threadIdx.x; i < kWords; i += kThreads) s[i] = 0ull;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const unsigned seed = (blockIdx.x * kThreads + threadIdx.x) * 2654435761u;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(s);
  for (int it = 0; it < iters; ++it) {
    const unsigned h = hash(seed + it);
    const unsigned w = h % kWords;
    if (kMode == 0) {  // own CTA
      const unsigned addr = sbase + w * 8;
      if (kT == 1) asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(addr), "d"(1.0) : "memory");
      else if (kT == 0) asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(addr), "l"(1ull) : "memory");
      else if (kT == 2) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(1u) : "memory");
      else asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(addr), "f"(1.0f) : "memory");
    } else if (kMode == 1) {  // any CTA of the cluster
      unsigned remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(sbase + w * 8), "r"(h >> 29));
      if (kT == 1) asm volatile("red.shared::cluster.add.f64 [%0], %1;" ::"r"(remote), "d"(1.0) : "memory");
      else if (kT == 0) asm volatile("red.shared::cluster.add.u64 [%0], %1;" ::"r"(remote), "l"(1ull) : "memory");
      else if (kT == 2) asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(remote), "r"(1u) : "memory");
      else asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(remote), "f"(1.0f) : "memory");
    } else {  // global (L2)
      unsigned long long *p = gbuf + (h & ((1u << 22) - 1));
      if (kT == 1) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(1.0) : "memory");
      else asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory");
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

template <int kMode, int kF64>
static void run(const char *name, int grid, unsigned long long *gbuf, unsigned long long *out) {
  const int iters = 1024;
  const size_t smem = kWords * 8;
  cudaFuncSetAttribute(k_acc<kMode, kF64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_acc<kMode, kF64><<<grid, kThreads, smem>>>(gbuf, iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_acc<kMode, kF64><<<grid, kThreads, smem>>>(gbuf, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = (double)grid * kThreads * iters;
  printf("%-34s %8.1f us  %8.1f Gop/s\n", name, best * 1e3, ops / (best * 1e-3) / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms / 8 * 8;
  unsigned long long *gbuf, *out;
  cudaMalloc(&gbuf, 8ull << 22);
  cudaMemset(gbuf, 0, 8ull << 22);
  cudaMalloc(&out, 8 * grid);
  printf("grid %d CTAs (clusters of 8) x %d threads, 192 KB shared each\n", grid, kThreads);
  run<0, 0>("own-CTA shared red.u64", grid, gbuf, out);
  run<0, 1>("own-CTA shared red.f64", grid, gbuf, out);
  run<0, 2>("own-CTA shared red.u32", grid, gbuf, out);
  run<0, 3>("own-CTA shared red.f32", grid, gbuf, out);
  run<1, 0>("cluster DSMEM red.u64 (random CTA)", grid, gbuf, out);
  run<1, 1>("cluster DSMEM red.f64 (random CTA)", grid, gbuf, out);
  run<1, 2>("cluster DSMEM red.u32 (random CTA)", grid, gbuf, out);
  run<1, 3>("cluster DSMEM red.f32 (random CTA)", grid, gbuf, out);
  run<2, 0>("global L2 red.u64 (32 MB)", grid, gbuf, out);
  run<2, 1>("global L2 red.f64 (32 MB)", grid, gbuf, out);
  return 0;
}
