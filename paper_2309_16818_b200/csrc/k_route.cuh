// k_route.cuh -- point routing of the sharded big map: k_route_count,
// k_route_scan, k_route_scatter, k_code_return.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// a2-a5 of one tile of this rank's shard (one map, tiles of kTile points, the k_bin layout):
// the band owner of every in-window point (-1: dropped).  Dropped points are counted and their
// debug outputs written by the counting pass only.
template <bool kCount>
__device__ __forceinline__ void route_tile_bins(const PassArgs &a, const RouteArgs &r, long long wbeg, long long end,
                                                int (&dst)[kBinPerThread], unsigned (&cnt)[8]) {
  const int lane = threadIdx.x & 31;
  const PointFrame f = frame_of(a, 0);
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    const long long i = wbeg + u * 32 + lane;
    dst[u] = -1;
    if (i >= end) continue;
    const float *q = a.pts + i * (long long)a.stride;
    const PointOut o = bin_point(__ldg(q), __ldg(q + 1), __ldg(q + 2), f, a.geo, a.np, 0, a.r2lo, a.r2hi);
    if (o.cell >= 0) {
      dst[u] = o.cell / r.band_n;
    } else if (kCount) {
      cnt[1] += o.code == MEM_CODE_NONFINITE;
      cnt[2] += o.code == MEM_CODE_RANGE;
      cnt[3] += o.code == MEM_CODE_HEIGHT;
      cnt[4] += o.code == MEM_CODE_OOB;
      if (a.dbg_code) a.dbg_code[i] = (uint8_t)o.code;
    }
    if (kCount && a.dbg_cell) a.dbg_cell[i] = o.lcell;
  }
}

// pass 1: routed points per (tile, owner)
__global__ void __launch_bounds__(kBinThreads) k_route_count(const __grid_constant__ PassArgs a, const RouteArgs r) {
  __shared__ unsigned s_cnt[8];
  __shared__ unsigned s_own[64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 8) s_cnt[tid] = 0;
  if (tid < 64) s_own[tid] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0)  // the other epoch is the next point input's (no memset per call)
    for (int i = tid; i < kStatSlots * 8; i += kBinThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
  __syncthreads();
  const long long n = a.offi[1];
  const long long beg = (long long)blockIdx.x * kTile, end = beg + kTile < n ? beg + kTile : n;
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int dst[kBinPerThread];
  route_tile_bins<true>(a, r, beg + wid * 256, end, dst, cnt);
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    const unsigned peers = __match_any_sync(0xffffffffu, dst[u]);
    if (dst[u] >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_own[dst[u]], (unsigned)__popc(peers));
  }
  __syncthreads();
  if (tid < r.nranks) r.tcnt[(long long)blockIdx.x * r.nranks + tid] = s_own[tid];
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

// pass 2 (one CTA): per owner, the exclusive prefix of the tiles' counts (in place) and the total
__global__ void __launch_bounds__(kThreads) k_route_scan(const RouteArgs r) {
  __shared__ unsigned s_part[kThreads / 32];
  pdl_wait();
  pdl_trigger();
  for (int d = 0; d < r.nranks; ++d) {
    unsigned run = 0u;
    for (int tb = 0; tb < r.tiles; tb += kThreads) {
      const int t = tb + threadIdx.x;
      unsigned *p = r.tcnt + (long long)t * r.nranks + d;
      const unsigned v = t < r.tiles ? *p : 0u;
      unsigned tot;
      const unsigned pre = block_excl_scan<kThreads>(v, s_part, &tot);
      if (t < r.tiles) *p = run + pre;
      run += tot;
    }
    if (threadIdx.x == 0) r.cnt[d] = run;
  }
}

// pass 3: every routed point to its owner's bucket at (tile offset + stable rank in the tile):
// the buckets hold the shard's points in input order
__global__ void __launch_bounds__(kBinThreads) k_route_scatter(const __grid_constant__ PassArgs a, const RouteArgs r) {
  __shared__ uint16_t s_wcnt[kBinThreads / 32][64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < (kBinThreads / 32) * 64; i += kBinThreads) s_wcnt[i / 64][i % 64] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const long long n = a.offi[1];
  const long long beg = (long long)blockIdx.x * kTile, end = beg + kTile < n ? beg + kTile : n;
  const long long wbeg = beg + wid * 256;
  unsigned cnt[8];
  int dst[kBinPerThread];
  unsigned rk[kBinPerThread];
  route_tile_bins<false>(a, r, wbeg, end, dst, cnt);
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    const unsigned peers = __match_any_sync(0xffffffffu, dst[u]);
    unsigned base = 0u;
    if (dst[u] >= 0) base = s_wcnt[wid][dst[u]];
    __syncwarp();
    if (dst[u] >= 0) {
      rk[u] = base + (unsigned)__popc(peers & lanemask_lt());
      if (lane == __ffs(peers) - 1) s_wcnt[wid][dst[u]] = (uint16_t)(base + __popc(peers));
    }
    __syncwarp();
  }
  __syncthreads();
  for (int d = tid; d < r.nranks; d += kBinThreads) {  // warp bases (exclusive over warps)
    unsigned run = 0u;
#pragma unroll
    for (int w = 0; w < kBinThreads / 32; ++w) {
      const unsigned c = s_wcnt[w][d];
      s_wcnt[w][d] = (uint16_t)run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    if (dst[u] < 0) continue;
    const long long i = wbeg + u * 32 + lane;
    const long long pos = (long long)r.tcnt[(long long)blockIdx.x * r.nranks + dst[u]] + s_wcnt[wid][dst[u]] + rk[u];
    const float *q = a.pts + i * (long long)a.stride;
    float *o = r.buf + ((long long)dst[u] * r.cap + pos) * a.stride;
    for (int k = 0; k < a.stride; ++k) o[k] = __ldg(q + k);
    if (r.src) r.src[(long long)dst[u] * r.cap + pos] = (unsigned)i;
  }
}

// debug outputs of routed points: the owner's in/out codes back to the shard's point indices
__global__ void k_code_return(const uint8_t *codes, const unsigned *idx, long long n, uint8_t *dst) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    dst[idx[k]] = codes[k];
}
