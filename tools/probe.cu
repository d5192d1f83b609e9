// probe.cu -- calibration microbenchmarks for the MEM kernels on B200 (not part of libmem).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe.cu && ./probe
// Prints one line per probe: name, time (us), rate.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void k_stream(const float4 *__restrict__ p, long long n, float *out) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p + i));
    acc += v.x + v.w;
  }
  if (acc == 12345.f) *out = acc;
}

template <int U>
__global__ void k_stream_unroll(const float4 *__restrict__ p, long long n, float *out) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + u * stride;
      v[u] = make_float4(0, 0, 0, 0);
      if (j < n)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                     : "l"(p + j));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
  }
  if (acc == 12345.f) *out = acc;
}

// RED throughput: each thread does `per` reductions to addresses idx(i) in a region of `cells`
// 8-byte words.  mode: 0 u64 add spread, 1 f64 add spread, 2 u64 add groups of 3 lanes same
// address, 3 f64 groups of 3, 4 u64 add fully random, 5 f64 random
__global__ void k_red(unsigned long long *buf, long long cells, long long total, int mode) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < total; i += nthreads) {
    long long a;
    if (mode <= 1)
      a = i % cells;
    else if (mode <= 3)
      a = (i / 3) % cells;
    else
      a = (long long)((unsigned long long)(i * 2654435761ull) % (unsigned long long)cells);
    if (mode & 1)
      asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(buf + a), "d"(1.0) : "memory");
    else
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(buf + a), "l"(1ull) : "memory");
  }
}

int main() {
  const long long n = 8388608;  // 134 MB of float4
  float4 *p;
  float *out;
  CK(cudaMalloc(&p, n * 16));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(p, 0, n * 16));
  float *flush;
  CK(cudaMalloc(&flush, 256 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char *name, double bytes, auto fn) {
    for (int r = 0; r < 3; ++r) fn();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaMemsetAsync(flush, r, 256 << 20));
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %9.1f us  %8.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  timeit("stream float4 grid=148x8x256", n * 16.0, [&] { k_stream<<<sms * 8, 256>>>(p, n, out); });
  timeit("stream float4 grid=148x16x128", n * 16.0, [&] { k_stream<<<sms * 16, 128>>>(p, n, out); });
  timeit("stream float4 unroll4 148x8x256", n * 16.0, [&] { k_stream_unroll<4><<<sms * 8, 256>>>(p, n, out); });
  timeit("stream float4 unroll8 148x4x256", n * 16.0, [&] { k_stream_unroll<8><<<sms * 4, 256>>>(p, n, out); });
  timeit("stream float4 unroll4 148x2x256", n * 16.0, [&] { k_stream_unroll<4><<<sms * 2, 256>>>(p, n, out); });

  unsigned long long *buf;
  const long long cells_small = 2560000;  // 20 MB region (L2 resident)
  CK(cudaMalloc(&buf, 8 * 64000000ll));
  CK(cudaMemset(buf, 0, 8 * 64000000ll));
  const long long total = 10000000;
  const char *names[] = {"red u64 spread (L2 20MB)", "red f64 spread (L2 20MB)", "red u64 3-lane same addr",
                         "red f64 3-lane same addr", "red u64 random (L2 20MB)", "red f64 random (L2 20MB)"};
  for (int mode = 0; mode < 6; ++mode) {
    char nm[96];
    snprintf(nm, sizeof nm, "%s 10M", names[mode]);
    cudaEventRecord(a);
    k_red<<<sms * 8, 256>>>(buf, cells_small, total, mode);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      k_red<<<sms * 8, 256>>>(buf, cells_small, total, mode);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %9.1f us  %8.1f Gop/s\n", nm, best * 1e3, total / (best * 1e-3) / 1e9);
  }
  // random over 512 MB (DRAM-resident lines)
  for (int mode = 4; mode < 6; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      k_red<<<sms * 8, 256>>>(buf, 64000000ll, total, mode);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %9.1f us  %8.1f Gop/s\n", mode == 4 ? "red u64 random (512 MB) 10M" : "red f64 random (512 MB) 10M",
           best * 1e3, total / (best * 1e-3) / 1e9);
  }
  return 0;
}
