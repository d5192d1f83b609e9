// k_points.cuh -- k_points (a2-a8).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_points (a2-a8)
// Persistent grid-stride over the 128-point warp-items of one wave.  Per lane: its 4 points
// of the item, binning, one batched state gather (a7), then warp-aggregated REDs.  On the
// float4 path (stride 4, aligned) every lane prefetches its 4 points of the warp's NEXT item
// into shared memory with cp.async while it processes the current one (double buffer, each
// lane reads back only the slots it wrote itself, so no warp or CTA barrier is needed).

// per-map call parameters: inline (kernel parameter space) or staged
__device__ __forceinline__ const PointFrame &frame_of(const PassArgs &a, int m) {
  return a.frames ? a.frames[m] : a.fi[m];
}

__device__ __forceinline__ long long off_of(const PassArgs &a, int m) {
  return a.offsets ? __ldg(&a.offsets[m]) : a.offi[m];
}
__device__ __forceinline__ int ps_of(const PassArgs &a, int m) { return a.pstart ? __ldg(&a.pstart[m]) : a.psi[m]; }

// the map and point range of warp-item `it`
struct Item {
  int m;
  long long beg, end, base;
};
__device__ __forceinline__ Item item_of(const PassArgs &a, int it, int i0) {
  Item r;
  r.m = a.m0;
  if (a.p_uniform > 0) {
    int rem;
    r.m = a.m0 + divmod_fast(it - i0, a.p_uniform, a.inv_p_uniform, rem);
  } else if (a.m1 - a.m0 > 1) {  // last map m in [m0, m1) with pstart[m] <= it
    int lo = a.m0, hi = a.m1 - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ps_of(a, mid) <= it) lo = mid; else hi = mid - 1;
    }
    r.m = lo;
  }
  r.beg = off_of(a, r.m);
  r.end = off_of(a, r.m + 1);
  r.base = r.beg + (long long)(it - ps_of(a, r.m)) * kWarpPoints;
  return r;
}

// 16-byte async copy global -> shared (L1 bypass, L2 evict-first); src_size 0 zero-fills
__device__ __forceinline__ void cp_async_16(void *smem, const void *gmem, bool valid, unsigned long long pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool kDebug, int kFast, bool kFull = false>
__device__ __forceinline__ void process_item(const PassArgs &a, const Item &t, const float (&px)[kWarpPtsPerLane],
                                             const float (&py)[kWarpPtsPerLane], const float (&pz)[kWarpPtsPerLane],
                                             const float (&pw)[kWarpPtsPerLane],
                                             unsigned long long &packed, unsigned &npk, unsigned (&cnt)[8]) {
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31;
  const PointFrame f = frame_of(a, t.m);
  const int map_base = t.m * g.HW;
  const int sb = (int)scratch_base(a, t.m);
  // points of the item present: [0, nv) (32-bit indices within the item)
  const int nv = kFull ? kWarpPoints : t.end - t.base < kWarpPoints ? (int)(t.end - t.base) : kWarpPoints;
  PointOut o[kWarpPtsPerLane];
#pragma unroll
  for (int u = 0; u < kWarpPtsPerLane; ++u) {
    const bool in = u * 32 + lane < nv;
    if (in && !ABLATE(a, 8u)) {
      o[u] = bin_point(px[u], py[u], pz[u], f, g, a.np, map_base);
    } else {
      o[u].code = in ? MEM_CODE_NONFINITE : -1;
      o[u].cell = -1;
      o[u].test = false;
    }
  }
  if (!ABLATE(a, 4u)) mahalanobis(o, a.st, g, a.np.tau2);
#pragma unroll
  for (int u = 0; u < kWarpPtsPerLane; ++u) {
    const int k = u * 32 + lane;
    if (k < nv) {
      if (kDebug) {
        a.dbg_cell[t.base + k] = o[u].lcell;
        a.dbg_code[t.base + k] = (uint8_t)o[u].code;
      }
      if (o[u].code >= 0) packed += 1ull << (10 * o[u].code);  // flushed once per item, below
    }
    if (ABLATE(a, 2u)) continue;
    const float *pp = kFast != 0 ? nullptr : a.pts + (k < nv ? t.base + k : t.beg) * (long long)a.stride;
    accumulate_warp<kFast>(a, o[u], sb + (o[u].cell - map_base), pp, pw[u]);
  }
  npk += kWarpPtsPerLane;  // the 10-bit code fields are flushed before they can wrap
  if (npk > 1023u - kWarpPtsPerLane) {
#pragma unroll
    for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
    packed = 0ull;
    npk = 0;
  }
}

template <bool kDebug, int kFast>
__global__ void __launch_bounds__(kThreads, MEM_POINTS_MINB) k_points(const __grid_constant__ PassArgs a) {
  __shared__ unsigned s_cnt[8];
  __shared__ float4 s_pts[kThreads / 32][2][kWarpPoints];  // per warp: 2 stages x 128 points
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0)  // the other epoch is the next point input's (no memset per call)
    for (int i = threadIdx.x; i < kStatSlots * 8; i += kThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // by mem_stats slot
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (kThreads / 32);
  const int gw = blockIdx.x * (kThreads / 32) + wid;
  const int i0 = ps_of(a, a.m0);
  const int i1 = ps_of(a, a.m1);
  const unsigned long long pol = evict_first_policy();
  unsigned long long packed = 0ull;
  unsigned npk = 0;
  float px[kWarpPtsPerLane], py[kWarpPtsPerLane], pz[kWarpPtsPerLane], pw[kWarpPtsPerLane];
  if (kFast != 0 || a.vec4) {
    const float4 *pts4 = reinterpret_cast<const float4 *>(a.pts);
    auto issue = [&](const Item &t, int stage) {
      if (t.end - t.base >= kWarpPoints) {  // a full item (all but a map's last): no per-lane bounds
        const float4 *src = pts4 + t.base + lane;
#pragma unroll
        for (int u = 0; u < kWarpPtsPerLane; ++u) cp_async_16(&s_pts[wid][stage][u * 32 + lane], src + u * 32, true, pol);
      } else {
#pragma unroll
        for (int u = 0; u < kWarpPtsPerLane; ++u) {
          const long long i = t.base + u * 32 + lane;
          cp_async_16(&s_pts[wid][stage][u * 32 + lane], pts4 + (i < t.end ? i : t.beg), i < t.end, pol);
        }
      }
      cp_async_commit();
    };
    int it = i0 + gw, stage = 0;
    Item cur;
    // uniform maps: the (map, item-in-map) of the warp's next item follows from the current
    // one by an add and one carry (no division per item)
    int um = 0, ur = 0;
    const int ustep_m = a.p_uniform > 0 ? nwarps / a.p_uniform : 0;
    const int ustep_r = a.p_uniform > 0 ? nwarps - ustep_m * a.p_uniform : 0;
    if (it < i1) {
      cur = item_of(a, it, i0);
      if (a.p_uniform > 0) um = divmod_fast(it - i0, a.p_uniform, a.inv_p_uniform, ur);
      issue(cur, 0);
    }
    for (; it < i1; it += nwarps, stage ^= 1) {
      const int nx = it + nwarps;
      Item nxt;
      if (nx < i1) {
        if (a.p_uniform > 0) {
          um += ustep_m;
          ur += ustep_r;
          if (ur >= a.p_uniform) {
            ur -= a.p_uniform;
            ++um;
          }
          nxt.m = a.m0 + um;
          nxt.beg = off_of(a, nxt.m);
          nxt.end = off_of(a, nxt.m + 1);
          nxt.base = nxt.beg + (long long)ur * kWarpPoints;
        } else {
          nxt = item_of(a, nx, i0);
        }
        issue(nxt, stage ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
#pragma unroll
      for (int u = 0; u < kWarpPtsPerLane; ++u) {
        const float4 v = s_pts[wid][stage][u * 32 + lane];
        px[u] = v.x; py[u] = v.y; pz[u] = v.z; pw[u] = v.w;
      }
#if MEM_FULL_ITEMS
      if (cur.end - cur.base >= kWarpPoints)  // every lane holds 4 points: no bounds checks
        process_item<kDebug, kFast, true>(a, cur, px, py, pz, pw, packed, npk, cnt);
      else
#endif
        process_item<kDebug, kFast>(a, cur, px, py, pz, pw, packed, npk, cnt);
      cur = nxt;
    }
  } else {
    for (int it = i0 + gw; it < i1; it += nwarps) {
      const Item t = item_of(a, it, i0);
#pragma unroll
      for (int u = 0; u < kWarpPtsPerLane; ++u) {  // all loads first (memory-level parallelism)
        const long long i = t.base + u * 32 + lane;
        px[u] = py[u] = pz[u] = pw[u] = 0.0f;
        if (i < t.end) {
          const float *q = a.pts + i * (long long)a.stride;
          px[u] = __ldg(q); py[u] = __ldg(q + 1); pz[u] = __ldg(q + 2);
        }
      }
      process_item<kDebug, kFast>(a, t, px, py, pz, pw, packed, npk, cnt);
    }
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
