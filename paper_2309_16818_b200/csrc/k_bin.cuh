// k_bin.cuh -- k_bin: a2-a6 for every point and the stable split of the in-window points by
// cell band.  Part of the single translation unit kernels.cu (included inside
// namespace memk, in order).
#pragma once

// per-map call parameters: inline (kernel parameter space) or staged
__device__ __forceinline__ const PointFrame &frame_of(const PassArgs &a, int m) {
  return a.frames ? a.frames[m] : a.fi[m];
}
__device__ __forceinline__ long long off_of(const PassArgs &a, int m) {
  return a.offsets ? __ldg(&a.offsets[m]) : a.offi[m];
}
__device__ __forceinline__ int ts_of(const PassArgs &a, int m) { return a.tstart ? __ldg(&a.tstart[m]) : a.tsi[m]; }

// the map of tile `tile` (tiles of map m are [tstart[m], tstart[m+1]))
__device__ __forceinline__ int map_of_tile(const PassArgs &a, int tile) {
  if (a.t_uniform > 0) {
    int rem;
    return divmod_fast(tile, a.t_uniform, a.inv_t_uniform, rem);
  }
  int lo = 0, hi = a.n_maps - 1;  // last m with tstart[m] <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts_of(a, mid) <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------- k_bin
// One CTA per tile of kTile consecutive points of one map (input order).  Warp w owns the tile's
// points [w * 256, (w + 1) * 256) -- 8 per lane, point w*256 + u*32 + lane in step u -- so the
// order (warp, step, lane) IS the input order.  Per point: a2-a6 (bin_point, the oracle's
// expressions).  Dropped points are counted (and their debug code written) here.  In-window
// points are split by cell band, stably: a lane's rank among the warp's earlier points of the
// same band comes from __match_any_sync plus a per-warp running count in shared memory; the
// tile then lays its records out band after band (tinfo[tile][band] = offset | count << 16),
// so every band's records sit in input order in each tile region and k_sort can gather them
// in input order without any global ordering pass.
//
// Record (16 B): x = cell within the band (bits 0-15) | usable-channel bit of bound group b
// (bit 16 + b, generic path), y = z (fp32), z = v (fp32), w = payload (fast paths: the point's
// channel word; generic: the point index).
template <bool kDebug, int kFast>
__global__ void __launch_bounds__(kBinThreads) k_bin(const __grid_constant__ PassArgs a) {
  __shared__ uint16_t s_wcnt[(kBinThreads / 32) * kMaxBands];  // [warp][band] (row stride NB): running count, then base
  __shared__ unsigned s_bofs[kMaxBands];                     // tile offset of each band's run
  __shared__ unsigned s_cnt[8];
  __shared__ unsigned s_part[kBinThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int m = map_of_tile(a, tile);
  const long long mbeg = off_of(a, m), mend = off_of(a, m + 1);
  const long long beg = mbeg + (long long)(tile - ts_of(a, m)) * kTile;
  const long long end = beg + kTile < mend ? beg + kTile : mend;
  const int NB = a.nbands;
  if (tid < 8) s_cnt[tid] = 0;
  for (int i = tid; i < (kBinThreads / 32) * NB; i += kBinThreads) s_wcnt[i] = 0;
  pdl_wait();  // the previous call's k_sort may still read the record buffers
  pdl_trigger();
  if (blockIdx.x == 0) {  // the other epoch is the next point input's (no memset per call)
    for (int i = tid; i < kStatSlots * 8; i += kBinThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
    if (tid == 0) a.ctl->n_rec = a.ctl->n_seg = a.ctl->n_lseg = a.ctl->n_mseg = 0u;
  }
  __syncthreads();
  const Geometry &g = a.geo;
  const PointFrame f = frame_of(a, m);
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int key[kBinPerThread];       // band of the point (-1: dropped)
  unsigned lc[kBinPerThread];   // cell within the band
  unsigned rk[kBinPerThread];   // rank within the warp's points of the same band
  float zz[kBinPerThread], vv[kBinPerThread];
  unsigned pay[kBinPerThread];
  const long long wbeg = beg + wid * 256;
  float4 q[kBinPerThread];
  if ((kFast == 1 || kFast == 2) || a.vec4) {  // all loads first (memory-level parallelism)
    const float4 *p4 = reinterpret_cast<const float4 *>(a.pts);
    const unsigned long long pol = evict_first_policy();
#pragma unroll
    for (int u = 0; u < kBinPerThread; ++u) {
      const long long i = wbeg + u * 32 + lane;
      q[u] = i < end ? ld_stream_f4(reinterpret_cast<const float *>(p4 + i), pol) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
#pragma unroll
    for (int u = 0; u < kBinPerThread; ++u) {
      const long long i = wbeg + u * 32 + lane;
      q[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < end) {
        const float *p = a.pts + i * (long long)a.stride;
        q[u].x = __ldg(p);
        q[u].y = __ldg(p + 1);
        q[u].z = __ldg(p + 2);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    const long long i = wbeg + u * 32 + lane;
    key[u] = -1;
    lc[u] = 0u;
    zz[u] = vv[u] = 0.0f;
    pay[u] = 0u;
    if (i < end) {
      const PointOut o = bin_point(q[u].x, q[u].y, q[u].z, f, g, a.np, 0, a.r2lo, a.r2hi);
      if (kDebug) a.dbg_cell[i] = o.lcell;
      if (o.cell >= a.cell_lo && o.cell < a.cell_hi) {
        int loc;
        key[u] = divmod_fast(o.cell - a.cell_lo, a.band_cells, a.inv_band, loc);
        lc[u] = (unsigned)loc;
        if (kFast == 0) {  // per bound group: are the point's channels usable (D31, D38)? bits 16..31
          for (int bi = 0; bi < a.nb; ++bi) lc[u] |= chan_ok(a, a.b[bi], (unsigned)i) ? (1u << (16 + bi)) : 0u;
        }
        zz[u] = o.z;
        vv[u] = o.v;
        pay[u] = kFast == 1 || kFast == 2 ? __float_as_uint(q[u].w) : (unsigned)i;
      } else {
        // o.cell >= 0 outside [cell_lo, cell_hi) cannot happen: a sharded owner receives only its
        // band's points (k_route); the unsharded pass covers every cell
        const int code = o.cell >= 0 ? MEM_CODE_OOB : o.code;
        cnt[1] += code == MEM_CODE_NONFINITE;  // mem_stats slots 1-4 (static indices: registers)
        cnt[2] += code == MEM_CODE_RANGE;
        cnt[3] += code == MEM_CODE_HEIGHT;
        cnt[4] += code == MEM_CODE_OOB;
        if (kDebug) a.dbg_code[i] = (uint8_t)code;
      }
    }
    // stable rank among the warp's points of the same band (steps are in input order)
    const unsigned peers = __match_any_sync(0xffffffffu, key[u]);
    unsigned base = 0u;
    if (key[u] >= 0) base = s_wcnt[wid * NB + key[u]];
    __syncwarp();
    if (key[u] >= 0) {
      rk[u] = base + (unsigned)__popc(peers & lanemask_lt());
      if (lane == __ffs(peers) - 1) s_wcnt[wid * NB + key[u]] = (uint16_t)(base + __popc(peers));
    }
    __syncwarp();
  }
  __syncthreads();
  // per band: warp bases (exclusive over warps) and the tile total
  for (int b = tid; b < NB; b += kBinThreads) {
    unsigned run = 0u;
#pragma unroll
    for (int w = 0; w < kBinThreads / 32; ++w) {
      const unsigned c = s_wcnt[w * NB + b];
      s_wcnt[w * NB + b] = (uint16_t)run;
      run += c;
    }
    s_bofs[b] = run;
  }
  __syncthreads();
  // exclusive scan of the band totals over the bands (thread t owns bands [t*k, (t+1)*k))
  {
    const int per = (NB + kBinThreads - 1) / kBinThreads;
    const int b0 = tid * per, b1 = b0 + per < NB ? b0 + per : NB;
    unsigned sum = 0u;
    for (int b = b0; b < b1; ++b) sum += s_bofs[b];
    unsigned tot;
    unsigned run = block_excl_scan<kBinThreads>(sum, s_part, &tot);
    unsigned *ti = a.tinfo + (long long)tile * NB;
    for (int b = b0; b < b1; ++b) {
      const unsigned v = s_bofs[b];
      s_bofs[b] = run;
      ti[b] = run | (v << 16);
      run += v;
    }
  }
  __syncthreads();
  uint4 *rt = a.recs + (long long)tile * kTile;
#pragma unroll
  for (int u = 0; u < kBinPerThread; ++u) {
    if (key[u] < 0) continue;
    const unsigned pos = s_bofs[key[u]] + s_wcnt[wid * NB + key[u]] + rk[u];
    __stcg(rt + pos, make_uint4(lc[u], __float_as_uint(zz[u]), __float_as_uint(vv[u]), pay[u]));
    if (kDebug) a.ridx[(long long)tile * kTile + pos] = (unsigned)(wbeg + u * 32 + lane);
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
