// k_merge.cuh -- k_merge: typed fold of partial bands (sharded map, statistics exchange).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_merge (sharded map)
// own band scratch op= the other ranks' partials, typed per record word (f64 sums, u64 sums,
// u64 max), so the owner's k_cells sees the statistics of every rank's points.
__global__ void __launch_bounds__(kThreads) k_merge(const __grid_constant__ MergeArgs a) {
  const long long words = (long long)a.n * (1 + a.R);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < a.n) {  // counts: u64 n_in | n_out << 32
      unsigned long long v = a.cnt[a.lo + i];
      for (int p = 0; p < a.nsrc; ++p) v += a.src_cnt[(long long)p * a.n + i];
      a.cnt[a.lo + i] = v;
      continue;
    }
    const long long j = i - a.n;  // record word j of the band
    const int w = (int)(j % a.R);
    unsigned long long *dst = a.rec + (long long)a.lo * a.R + j;
    const int ty = a.wtype[w];
    if (ty == 0) {
      double v = __longlong_as_double((long long)*dst);
      for (int p = 0; p < a.nsrc; ++p) v += __longlong_as_double((long long)a.src_rec[(long long)p * a.n * a.R + j]);
      *dst = (unsigned long long)__double_as_longlong(v);
    } else if (ty == 1) {
      unsigned long long v = *dst;
      for (int p = 0; p < a.nsrc; ++p) v += a.src_rec[(long long)p * a.n * a.R + j];
      *dst = v;
    } else {
      unsigned long long v = *dst;
      for (int p = 0; p < a.nsrc; ++p) {
        const unsigned long long x = a.src_rec[(long long)p * a.n * a.R + j];
        v = x > v ? x : v;
      }
      *dst = v;
    }
  }
}
