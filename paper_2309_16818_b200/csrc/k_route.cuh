// k_route.cuh -- k_route: point routing of the sharded big map.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_route (sharded map, NEXT)
// a2-a5 for this rank's shard of a single map: dropped points are counted here, every
// in-window point is copied into the bucket of its cell's band owner (lanes with the same
// owner reserve their slots with one atomicAdd).  The owner then runs k_points + k_cells on
// what it received: the Mahalanobis test, accumulation and fusion all happen there.
__global__ void __launch_bounds__(kThreads) k_route(const __grid_constant__ PassArgs a, const RouteArgs r) {
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0)  // the other epoch is the next point input's (no memset per call)
    for (int i = threadIdx.x; i < kStatSlots * 8; i += kThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long packed = 0ull;
  unsigned npk = 0;
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31;
  const long long n = off_of(a, 1);
  const PointFrame f = frame_of(a, 0);
  const long long nthreads = (long long)gridDim.x * kThreads;
  for (long long i0 = (long long)blockIdx.x * kThreads; i0 < n; i0 += nthreads) {  // warp-uniform trip count
    const long long i = i0 + threadIdx.x;
    const bool in = i < n;
    const float *q = a.pts + (in ? i : 0) * (long long)a.stride;
    PointOut o;
    o.cell = -1;
    o.code = -1;
    if (in) o = bin_point(__ldg(q), __ldg(q + 1), __ldg(q + 2), f, g, a.np, 0);
    if (in && o.cell < 0) count_code(packed, npk, o.code, cnt);
    const int dest = o.cell >= 0 ? o.cell / r.band_n : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, dest);
    const int leader = __ffs(peers) - 1;
    unsigned base = 0u;
    if (dest >= 0 && lane == leader) base = atomicAdd(&r.cnt[dest], (unsigned)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (dest >= 0) {
      const long long pos = (long long)base + __popc(peers & lanemask_lt());
      float *d = r.buf + ((long long)dest * r.cap + pos) * a.stride;
      for (int k = 0; k < a.stride; ++k) d[k] = __ldg(q + k);
    }
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
