// fp64 FMA throughput / latency on one SM (and fp32 for comparison)
#include <cstdio>
#include <cuda_runtime.h>
template <class T, int ILP>
__global__ void k_fma(T *out, int iters, long long *cyc) {
  T x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = (T)(threadIdx.x + i) * (T)1e-3;
  const T a = (T)0.999, b = (T)1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = x[i] * a + b;
  __syncthreads();
  long long t1 = clock64();
  T s = 0;
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <class T, int ILP>
void run(const char *name, int threads) {
  T *o;
  long long *c, h;
  cudaMalloc(&o, sizeof(T) * threads);
  cudaMalloc(&c, 8);
  const int iters = 4096;
  k_fma<T, ILP><<<1, threads>>>(o, iters, c);
  k_fma<T, ILP><<<1, threads>>>(o, iters, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)threads * iters * ILP;
  printf("%s threads %4d ILP %d: %.2f FMA/clk/SM, %.1f cycles per dependent FMA\n", name, threads, ILP, ops / h,
         (double)h / iters / ILP * (threads <= 32 ? ILP : 1));
  cudaFree(o);
  cudaFree(c);
}
int main() {
  run<double, 1>("f64", 32);
  run<double, 4>("f64", 32);
  run<double, 8>("f64", 512);
  run<double, 8>("f64", 1024);
  run<float, 1>("f32", 32);
  run<float, 8>("f32", 1024);
  return 0;
}
