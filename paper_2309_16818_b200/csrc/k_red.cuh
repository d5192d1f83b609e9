// k_red.cuh -- k_points: a2-a8 with certified-exact fp64 reductions (reading
// D39).  Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

#ifndef MEM_SCRATCH_HINT
#define MEM_SCRATCH_HINT 2  // L2 priorities: 1 = k_cells zeroes the RED scratch evict-last (the next
                            // point pass REDs into it); 2 = also k_points' state gathers evict-first
                            // (C2x64 114.4 -> 112.6 us; REDs evict-last measured slower)
#endif

// ---------------------------------------------------------------- exactness certificates
// fp64 sums of fp32 terms are EXACT, in any order, when every partial sum is representable:
// with e_max / e_min the largest / smallest binary exponent among the (non-zero) terms and n
// terms, that holds when e_max - e_min + ceil(log2 n) <= 29 (every term is a multiple of
// 2^(e_min - 23), every partial sum below n 2^(e_max + 1) < 2^53 such quanta).
// An exact sum is the oracle's sequential sum bit for bit, so the atomic reductions below give
// the oracle's result whatever their order -- when a cell's certificate holds.  k_points keeps
// per cell the largest and (complemented) smallest |term| bit pattern of S = sum z/v (and of
// the average channel sum); k_cells checks them and hands any uncertified cell to k_refold,
// which recomputes it sequentially in input order.  P = sum 1/v is certified once per call on
// the host from the range of v.
//
// Storage: one 8-byte word per cell, four bf16 slots {e_max(S), 255 - e_min(S), e_max(X),
// 255 - e_min(X)} (exponent fields, subnormals counted as 1; integers <= 255 are exact in bf16,
// 0 = no non-zero term), reduced by ONE red.max.v2.bf16x2 per run of points (the four slots
// are independent maxima).
__device__ __forceinline__ unsigned bf16_int(unsigned v) { return __float_as_uint((float)v) >> 16; }
__device__ __forceinline__ unsigned int_bf16(unsigned h) { return (unsigned)__uint_as_float(h << 16); }
// {~min |t| bits, max |t| bits} (register form, 0 = no non-zero term) -> bf16x2 slots
__device__ __forceinline__ unsigned cert_slots(uint2 c) {
  if (c.y == 0u) return 0u;
  const unsigned emin = max((~c.x >> 23) & 255u, 1u), emax = max((c.y >> 23) & 255u, 1u);
  return bf16_int(emax) | bf16_int(255u - emin) << 16;
}
__device__ __forceinline__ void red_max_cert(unsigned *p, unsigned s, unsigned x) {  // p: 8-byte aligned
  asm volatile("red.relaxed.gpu.global.max.noftz.v2.bf16x2 [%0], {%1, %2};" ::"l"(p), "r"(s), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned cert_ceil_log2(unsigned n) { return n <= 1u ? 0u : 32u - __clz(n - 1u); }
// slots of one sum (bf16x2 word); n = number of terms
__device__ __forceinline__ bool cert_ok(unsigned w, unsigned n) {
  if (w == 0u) return true;  // every term zero
  const unsigned emax = int_bf16(w & 0xffffu), emin = 255u - int_bf16(w >> 16);
  return emax - emin + cert_ceil_log2(n) <= 29u;
}

// Block-certified sequential folding (k_refold, k_fuse): adding a block of fp32 terms to an fp64
// running sum V rounds nowhere when every value involved is a multiple of 2^q (q = the lowest
// set bit over V and the terms) and every partial sum is below 2^(q + 53); then V + (the block's
// exact sum, any order) is the sequential result bit for bit.
__device__ __forceinline__ int expo64(double x) { return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023; }
__device__ __forceinline__ int lsb64(double x) {  // x normal, non-zero
  const unsigned long long m = ((unsigned long long)__double_as_longlong(x) & 0xfffffffffffffull) | (1ull << 52);
  return expo64(x) - 52 + __ffsll((long long)m) - 1;
}
__device__ __forceinline__ int lsb32(float t) {  // t non-zero (normal or subnormal)
  const unsigned u = __float_as_uint(t) & 0x7fffffffu;
  const int fe = (int)(u >> 23);
  const unsigned m = (u & 0x7fffffu) | (fe ? 0x800000u : 0u);
  return (fe ? fe - 127 : -126) - 23 + __ffs((int)m) - 1;
}
// V + the block's terms, when the sequential fold provably rounds nowhere
__device__ __forceinline__ bool fold_exact(double V, double absum, int qb) {
  if (absum == 0.0) return true;  // only zero terms
  int q = qb;
  int e = expo64(absum);
  if (V != 0.0) {
    q = min(q, lsb64(V));
    e = max(e, expo64(V));
  }
  return e + 2 <= q + 53;  // |partial| <= |V| + absum < 2^(e + 2) <= 2^(q + 53)
}

// ---------------------------------------------------------------- a7, batched gathers
// a7 for a batch of points: issue every state gather first (one round trip), then decide.
// The valid flag is not read: an invalid cell always holds a NaN variance (reset_cell, and
// k_write keeps it so for state written through mem_set_layer), and a NaN h or s2 makes the
// comparison false -- exactly the oracle's "no test on an invalid cell" (D10).
template <int N>
__device__ __forceinline__ void mahalanobis(PointOut (&o)[N], const State &st, const Geometry &g, float tau2) {
  const float *elev = reinterpret_cast<const float *>(st.words) + (long long)kWordElev * g.BHW;
  const float *var = reinterpret_cast<const float *>(st.words) + (long long)kWordVar * g.BHW;
  float hv[N], sv[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    hv[u] = sv[u] = __int_as_float(0x7fc00000);
    if (o[u].test) {
#if MEM_SCRATCH_HINT >= 2
      const unsigned long long pf = evict_first_policy();
      hv[u] = ld_hint_f32(elev + o[u].cell, pf);
      sv[u] = ld_hint_f32(var + o[u].cell, pf);
#else
      hv[u] = __ldcg(elev + o[u].cell);
      sv[u] = __ldcg(var + o[u].cell);
#endif
    }
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    // outlier iff valid and (z - h)^2 > tau^2 (sigma^2 + v) (D10); NaN state compares false
    const float d = o[u].z - hv[u];
    if (d * d > tau2 * (sv[u] + o[u].v)) o[u].code = MEM_CODE_OUTLIER;
  }
}

// explicit fire-and-forget reductions (RED, never ATOM with a return)
__device__ __forceinline__ void red_add_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_f64(unsigned long long *p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Segmented reduction over runs of consecutive lanes holding the same cell (`heads`: the first
// lane of every run): after five shuffle-down steps the head lane of each run holds the run's
// total.  One pass reduces every statistic of the point (shared control flow).  A cell whose
// lanes are not contiguous gets one total per run (one RED set each): exact all the same.
__device__ __forceinline__ bool same_run_below(unsigned heads, int lane, int d) {
  // lanes (lane, lane + d] belong to lane's run (no head among them)
  return lane + d <= 31 && (heads & (((1u << d) - 1u) << (lane + 1))) == 0u;
}
template <int kFast>
__device__ __forceinline__ void reduce_runs(unsigned heads, double &w, double &zw, uint2 &cs, unsigned &rg,
                                            unsigned &bb, double &v, uint2 &cx) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const bool ok = same_run_below(heads, lane, d);
    const double tw = __shfl_down_sync(0xffffffffu, w, d), tz = __shfl_down_sync(0xffffffffu, zw, d);
    const unsigned c0 = __shfl_down_sync(0xffffffffu, cs.x, d), c1 = __shfl_down_sync(0xffffffffu, cs.y, d);
    unsigned r0 = 0u, r1 = 0u, x0 = 0u, x1 = 0u;
    double tv = 0.0;
    if (kFast == 1) {
      r0 = __shfl_down_sync(0xffffffffu, rg, d);
      r1 = __shfl_down_sync(0xffffffffu, bb, d);
    } else if (kFast == 2) {
      tv = __shfl_down_sync(0xffffffffu, v, d);
      x0 = __shfl_down_sync(0xffffffffu, cx.x, d);
      x1 = __shfl_down_sync(0xffffffffu, cx.y, d);
    }
    if (ok) {
      w += tw;
      zw += tz;
      cs.x = max(cs.x, c0);
      cs.y = max(cs.y, c1);
      if (kFast == 1) {
        rg += r0;
        bb += r1;
      } else if (kFast == 2) {
        v += tv;
        cx.x = max(cx.x, x0);
        cx.y = max(cx.y, x1);
      }
    }
  }
}

// |t| as the certificate pair {~bits, bits} (0, 0 for t = 0)
__device__ __forceinline__ uint2 cert_of(float t) {
  const unsigned b = __float_as_uint(t) & 0x7fffffffu;
  return b ? make_uint2(~b, b) : make_uint2(0u, 0u);
}

// a8: scatter-accumulate the sufficient statistics of the warp's current points (one per lane,
// `o.cell < 0` = dropped) into their scratch cells `sc`.  Lanes hitting the same cell are
// combined first (reduce_runs over runs of consecutive lanes) when >= 16 lanes repeat their
// neighbour's cell (dense clouds), so that one lane issues the REDs of each run.  All 32 lanes must call
// this.  kFast: 1 = one colour group, 2 = one 1-channel average group, 0 = no group (height).
// Scratch per cell: count word (colour: b | n << 32, else n_in | n_out << 32), record
// [P, S, colour: r | g << 32 / average: n_g, colour: n_out / average: X], certificates
// {~min, max} of |z/v| and of |channel|.
template <int kFast>
__device__ __forceinline__ void accumulate_warp(const PassArgs &a, const PointOut &o, int sc, float ch0) {
  unsigned long long *rec = a.rec + (long long)sc * 4;
  // the certificate word: record word 3 (colour, height only: the same 32-B sector as P and S),
  // the separate array for the average group (whose record holds n_g and X)
  unsigned *cert = kFast == 2 ? a.cert + (long long)sc * 2 : reinterpret_cast<unsigned *>(rec + 3);
  const bool act = o.cell >= 0;
  const unsigned act_b = __ballot_sync(0xffffffffu, act);
  if (act_b == 0u) return;
  const int lane = threadIdx.x & 31;
  const unsigned key = act ? (unsigned)sc : 0xffffffffu;
  const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned same = __ballot_sync(0xffffffffu, lane > 0 && prev == key);
  const unsigned dup = same & act_b;
  const bool agg = __popc(dup) >= 16;
  const bool single = !agg;
  // agg: runs of consecutive lanes of one cell are reduced to their head lane (reduce_runs)
  const unsigned heads = ~same;
  unsigned peers = 1u << lane;  // the lanes whose statistics this lane holds after the reduction
  if (agg) {
    const unsigned above = heads & ~((2u << lane) - 1u);  // heads after this lane (lane 31: none)
    const unsigned upto = above ? (above & (0u - above)) - 1u : 0xffffffffu;
    peers = upto & ~((1u << lane) - 1u);
  }
  const bool leader = act && (single || (heads >> lane & 1u));
  const bool inl = act && o.code == MEM_CODE_INLIER;
  const unsigned in_b = __ballot_sync(0xffffffffu, inl);
  // height statistics (inliers): sum 1/v, sum z/v, the certificate of z/v
  double w = 0.0, zw = 0.0;
  uint2 cs = make_uint2(0u, 0u);
  if (inl) {
    const float wf = 1.0f / o.v;
    const float t = o.z * wf;
    w = (double)wf;
    zw = (double)t;
    cs = cert_of(t);
  }
  // the group's statistics: colour words (kFast 1), the channel (kFast 2)
  unsigned rg = 0u, bb = 0u;
  double v = 0.0;
  uint2 cx = make_uint2(0u, 0u);
  bool fin = false;
  if (kFast == 1 && act) {
    const uint32_t bits = __float_as_uint(ch0);
    rg = ((bits >> 16) & 255u) | (((bits >> 8) & 255u) << 16);
    bb = bits & 255u;
  } else if (kFast == 2) {
    fin = act && isfinite(ch0);
    v = fin ? (double)ch0 : 0.0;
    cx = fin ? cert_of(ch0) : make_uint2(0u, 0u);
  }
  const unsigned fin_b = kFast == 2 ? __ballot_sync(0xffffffffu, fin) : 0u;
  if (!single) reduce_runs<kFast>(heads, w, zw, cs, rg, bb, v, cx);
  if constexpr (kFast == 1) {
    // colour: count word b | n << 25 | n_out << 43 (n = every filtered in-bounds point, D20;
    // n > 0 marks the cell touched), record [P, S, r | g << 32, certificate]
    unsigned n_in = (unsigned)__popc(peers & in_b), n_all = (unsigned)__popc(peers & act_b);
    bool lead = leader;
    if (single && __popc(dup) >= MEM_PAIR_MIN) {
      // a LiDAR scan line puts ~30% of its in-window points in the cell of the previous
      // lane: the head of each run absorbs its successor, so such a pair costs one RED set
      const bool fol = dup >> lane & 1u;
      const bool prev_fol = lane > 0 && (dup >> (lane - 1) & 1u);
      const bool absorbed = fol && !prev_fol;
      const bool absorbs = !fol && lane < 31 && (dup >> (lane + 1) & 1u);
      const double w2 = __shfl_down_sync(0xffffffffu, w, 1), zw2 = __shfl_down_sync(0xffffffffu, zw, 1);
      const unsigned rg2 = __shfl_down_sync(0xffffffffu, rg, 1), bb2 = __shfl_down_sync(0xffffffffu, bb, 1);
      const unsigned cx2 = __shfl_down_sync(0xffffffffu, cs.x, 1), cy2 = __shfl_down_sync(0xffffffffu, cs.y, 1);
      if (absorbs) {
        w += w2;
        zw += zw2;
        rg += rg2;
        bb += bb2;
        cs.x = max(cs.x, cx2);
        cs.y = max(cs.y, cy2);
        n_all = 2;
        n_in += in_b >> (lane + 1) & 1u;
      }
      lead = act && !absorbed;
    }
    if (lead) {  // count word b | n << 25 | n_out << 43 (kColourMaxPts: no field overflows)
      red_add_u64(&a.cnt[sc], (unsigned long long)bb | ((unsigned long long)n_all << 25) |
                                  ((unsigned long long)(n_all - n_in) << 43));
      if (n_in) {
        red_add_f64(rec + kRecP, w);
        red_add_f64(rec + kRecS, zw);
        if (cs.y) red_max_cert(cert, cert_slots(cs), 0u);
      }
      red_add_u64(rec + 2, (unsigned long long)(rg & 0xffffu) | ((unsigned long long)(rg >> 16) << 32));
    }
    return;
  }
  if (leader) {
    const unsigned n_in = (unsigned)__popc(peers & in_b), n_all = (unsigned)__popc(peers & act_b);
    red_add_u64(&a.cnt[sc], (unsigned long long)n_in | ((unsigned long long)(n_all - n_in) << 32));
    if (n_in) {
      red_add_f64(rec + kRecP, w);
      red_add_f64(rec + kRecS, zw);
    }
    if constexpr (kFast == 2) {  // Eq.(1) sums of one channel; non-finite values skip the group (D31)
      const unsigned ng = (unsigned)__popc(peers & fin_b);
      if (ng) {
        red_add_u64(rec + 2, (unsigned long long)ng);
        red_add_f64(rec + 3, v);
      }
      if ((n_in && cs.y) || (ng && cx.y)) red_max_cert(cert, n_in ? cert_slots(cs) : 0u, ng ? cert_slots(cx) : 0u);
    } else if (n_in && cs.y) {
      red_max_cert(cert, cert_slots(cs), 0u);
    }
  }
}

// ---------------------------------------------------------------- k_points (a2-a8, certified REDs)
// Persistent grid-stride over the 128-point warp-items of the call.  Per lane: its 4 points of
// the item, binning (bin_point), one batched state gather (a7), then warp-aggregated native
// 64-bit REDs of the per-cell statistics and the certificates (accumulate_warp).  On the float4
// path (stride 4, aligned) every lane prefetches its 4 points of the warp's NEXT item into
// shared memory with cp.async while it processes the current one.
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

template <bool kDebug, int kFast, bool kWave, bool kFull = false>
__device__ __forceinline__ void process_item(const PassArgs &a, const Item &t, const float (&px)[kWarpPtsPerLane],
                                             const float (&py)[kWarpPtsPerLane], const float (&pz)[kWarpPtsPerLane],
                                             const float (&pw)[kWarpPtsPerLane],
                                             unsigned long long &packed, unsigned &npk, unsigned (&cnt)[8]) {
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31;
  const PointFrame f = frame_of(a, t.m);
  const int map_base = t.m * g.HW;
  const int sb = (t.m - a.m0) * g.HW - a.sc_lo;  // the map's scratch cells (this wave's maps / cells)
  // points of the item present: [0, nv) (32-bit indices within the item)
  const int nv = kFull ? kWarpPoints : t.end - t.base < kWarpPoints ? (int)(t.end - t.base) : kWarpPoints;
  PointOut o[kWarpPtsPerLane];
#pragma unroll
  for (int u = 0; u < kWarpPtsPerLane; ++u) {
    const bool in = u * 32 + lane < nv;
    if (in) {
      o[u] = bin_point(px[u], py[u], pz[u], f, g, a.np, map_base, a.r2lo, a.r2hi);
      if (kWave) {  // cell waves: another wave's point is skipped, a dropped one counted once
        const int phys = o[u].cell - map_base;
        if (o[u].cell >= 0 ? phys < a.sc_lo || phys >= a.sc_hi : !a.wave_first) {
          o[u].code = -1;
          o[u].cell = -1;
          o[u].test = false;
        }
      }
    } else {
      o[u].code = in ? MEM_CODE_NONFINITE : -1;
      o[u].cell = -1;
      o[u].test = false;
    }
  }
  mahalanobis(o, a.st, g, a.np.tau2);
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
    accumulate_warp<kFast>(a, o[u], sb + (o[u].cell - map_base), pw[u]);
  }
  npk += kWarpPtsPerLane;  // the 10-bit code fields are flushed before they can wrap
  if (npk > 1023u - kWarpPtsPerLane) {
#pragma unroll
    for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
    packed = 0ull;
    npk = 0;
  }
}

#ifndef MEM_POINTS_MINB
#define MEM_POINTS_MINB 3  // k_points: CTAs per SM the registers are sized for
#endif
template <bool kDebug, int kFast, bool kWave>
__global__ void __launch_bounds__(kThreads, MEM_POINTS_MINB) k_points(const __grid_constant__ PassArgs a) {
  __shared__ unsigned s_cnt[8];
  __shared__ float4 s_pts[kThreads / 32][2][kWarpPoints];  // per warp: 2 stages x 128 points
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0) {  // the other epoch is the next point input's (no memset per call)
    for (int i = threadIdx.x; i < kStatSlots * 8; i += kThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
    if (threadIdx.x == 0) a.ctl->n_fb = a.ctl->n_fbpts = 0u;
  }
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
        process_item<kDebug, kFast, kWave, true>(a, cur, px, py, pz, pw, packed, npk, cnt);
      else
#endif
        process_item<kDebug, kFast, kWave>(a, cur, px, py, pz, pw, packed, npk, cnt);
      cur = nxt;
    }
  } else {
    float *s3 = reinterpret_cast<float *>(s_pts[wid][0]);  // the 3 x kWarpPoints floats of the warp's item (vec3)
    for (int it = i0 + gw; it < i1; it += nwarps) {
      const Item t = item_of(a, it, i0);
      if (a.vec3 && t.end - t.base >= kWarpPoints) {
        // stride 3, a full item: 96 coalesced float4 loads (3 per lane), the 128 points then
        // read back from shared memory (stride 3 words: conflict-free)
        const float4 *src = reinterpret_cast<const float4 *>(a.pts + t.base * 3);
        constexpr int kV3 = 3 * kWarpPoints / 4;  // float4 of the item
        float4 v[(kV3 + 31) / 32];
#pragma unroll
        for (int k = 0; k < (kV3 + 31) / 32; ++k)
          if (k * 32 + lane < kV3) v[k] = ld_stream_f4(reinterpret_cast<const float *>(src + k * 32 + lane), pol);
#pragma unroll
        for (int k = 0; k < (kV3 + 31) / 32; ++k)
          if (k * 32 + lane < kV3) reinterpret_cast<float4 *>(s3)[k * 32 + lane] = v[k];
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kWarpPtsPerLane; ++u) {
          const float *q = s3 + 3 * (u * 32 + lane);
          px[u] = q[0]; py[u] = q[1]; pz[u] = q[2]; pw[u] = 0.0f;
        }
        __syncwarp();  // the slice is rewritten by the warp's next item
        process_item<kDebug, kFast, kWave, MEM_FULL_ITEMS != 0>(a, t, px, py, pz, pw, packed, npk, cnt);
        continue;
      }
#pragma unroll
      for (int u = 0; u < kWarpPtsPerLane; ++u) {  // all loads first (memory-level parallelism)
        const long long i = t.base + u * 32 + lane;
        px[u] = py[u] = pz[u] = pw[u] = 0.0f;
        if (i < t.end) {
          const float *q = a.pts + i * (long long)a.stride;
          px[u] = __ldg(q); py[u] = __ldg(q + 1); pz[u] = __ldg(q + 2);
        }
      }
      process_item<kDebug, kFast, kWave>(a, t, px, py, pz, pw, packed, npk, cnt);
    }
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
