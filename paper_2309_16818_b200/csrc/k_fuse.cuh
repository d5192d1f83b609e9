// k_fuse.cuh -- k_fuse: a7-a10 for every touched cell of a point input, in input order
// (DESIGN.md §4.2).  Part of the single translation unit kernels.cu (included inside namespace
// memk, in order).
#pragma once

#ifndef MEM_FUSE_MINB0
#define MEM_FUSE_MINB0 4  // k_fuse short cells, generic groups: CTAs per SM the registers are sized for
                           // (8: spills; 4: paper sweep 3-5% faster)
#endif

// ---------------------------------------------------------------- k_fuse
// Persistent grid-stride over the call's segments (one touched cell each: its records are
// contiguous in the sorted array, in input order, k_sort).  One thread per cell runs the
// oracle's per-point loop: the Mahalanobis test against the pre-frame state (a7), then the
// sufficient statistics summed sequentially in input order -- P += (double)(1/v),
// S += (double)(z/v), channel sums in fp64, colour in integers (a8) -- then the Kalman height
// update and the group rules (a9, a10) with the oracle's expressions.  The results are the
// oracle's, operation for operation, whatever the thread schedule or launch configuration
// (reading D39).  kFast: 1 one colour group, 2 one 1-channel average group (the channel word
// rides in the record), 3 no group, 0 generic (channels read from the points by index).
// the state of one cell after its frame statistics: a9 (Kalman height, D7/D11) and, for the fast
// groups, a10 (Eq.(1)+(2)); the generic groups follow in fuse_generic
template <int kFast>
__device__ __forceinline__ void fuse_state(const PassArgs &a, long long gc, float h, float s2, uint8_t vd0,
                                           const float *th, uint8_t ob, unsigned nin, unsigned nout, double P,
                                           double S, unsigned cr, unsigned cg, unsigned cb, unsigned na, double X) {
  constexpr int NCH = kFast == 1 ? 3 : kFast == 2 ? 1 : 0;
  const long long BHW = a.geo.BHW;
  float *vals = reinterpret_cast<float *>(a.st.words);
  uint8_t vd = vd0;
  kalman_height(h, s2, vd, (double)nin, (double)nout, P, S, a.np.v_out);
  if (vd) {
    vals[(long long)kWordElev * BHW + gc] = h;
    vals[(long long)kWordVar * BHW + gc] = s2;
    if (!vd0) a.st.flags[(long long)kFlagValid * BHW + gc] = 1;
  }
  if (NCH > 0 && na != 0u) {
    const GroupDesc &gd = a.b[0].g;
    const unsigned sums[3] = {cr, cg, cb};
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      vals[(long long)(gd.word0 + k) * BHW + gc] =
          rule_average(th[k], ob != 0, kFast == 1 ? (double)sums[k] : X, (double)na, gd.w);
    if (!ob) a.st.flags[(long long)gd.flag * BHW + gc] = 1;
  }
}

// a10 for the generic groups of one cell: per group, per channel, in input order (channels
// read from the points by index, usable-channel bits in the records)
__device__ __forceinline__ void fuse_generic(const PassArgs &a, long long gc, const uint4 *rec, int n) {
  const long long BHW = a.geo.BHW;
  float *vals = reinterpret_cast<float *>(a.st.words);
  // a10, generic groups: per group, per channel, in input order (channels read by point index)
  for (int bi = 0; bi < a.nb; ++bi) {
    const BindDesc &b = a.b[bi];
    const GroupDesc &gd = b.g;
    if (gd.rule == MEM_COLOR) {  // D20: packed 0x00RRGGBB, never skipped
      unsigned r_ = 0u, g_ = 0u, b_ = 0u;
      for (int r = 0; r < n; ++r) {
        const uint32_t bits = __float_as_uint(chan_value(a, b, __ldcg(&rec[r].w), 0));
        r_ += (bits >> 16) & 255u;
        g_ += (bits >> 8) & 255u;
        b_ += bits & 255u;
      }
      uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
      const bool obb = *obs != 0;
      const unsigned sums[3] = {r_, g_, b_};
      for (int k = 0; k < 3; ++k) {
        float *t = vals + (long long)(gd.word0 + k) * BHW + gc;
        *t = rule_average(*t, obb, (double)sums[k], (double)n, gd.w);
      }
      *obs = 1;
      continue;
    }
    if (gd.rule == MEM_CLASS_MAX) {  // D19: the frame's winner, an order-free maximum
      unsigned long long key = 0ull;
      for (int r = 0; r < n; ++r) {
        const uint4 q = __ldcg(rec + r);
        if (q.x >> (16 + bi) & 1u) {
          const unsigned long long k = chan_key(a, b, q.w);
          key = k > key ? k : key;
        }
      }
      if (key != 0ull) {
        reinterpret_cast<int *>(a.st.words)[(long long)gd.label * BHW + gc] =
            gd.nch - 1 - (int)(uint32_t)(key & 0xffffffffull);
        vals[(long long)gd.word0 * BHW + gc] = f32_of_ord((uint32_t)(key >> 32));
      }
      continue;
    }
    // the points whose channels are usable (D31, D38): bit 16 + bi of the record (k_bin); a
    // short cell (n <= kShortSeg): its point indices in registers, then per channel every
    // point's value in flight together, summed in input order
    unsigned ng = 0u, okm = 0u, pidx[kShortSeg];
#pragma unroll
    for (int r = 0; r < kShortSeg; ++r) {
      pidx[r] = 0u;
      if (r < n) {
        const uint4 q = __ldcg(rec + r);
        pidx[r] = q.w;
        if (q.x >> (16 + bi) & 1u) okm |= 1u << r;
      }
    }
    ng = __popc(okm);
    if (ng == 0u) continue;  // no finite point: the group is not updated (D31)
    uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
    const bool obb = *obs != 0;
    for (int k = 0; k < gd.nch; ++k) {
      float cv[kShortSeg];
#pragma unroll
      for (int r = 0; r < kShortSeg; ++r) cv[r] = (okm >> r & 1u) ? chan_value(a, b, pidx[r], k) : 0.0f;
      double sum = 0.0;
#pragma unroll
      for (int r = 0; r < kShortSeg; ++r)
        if (okm >> r & 1u) sum += (double)cv[r];
      float *t = vals + (long long)(gd.word0 + k) * BHW + gc;
      switch (gd.rule) {
        case MEM_AVERAGE:
        case MEM_CLASS_AVERAGE: *t = rule_average(*t, obb, sum, (double)ng, gd.w); break;
        case MEM_GAUSSIAN: {
          float *vr = vals + (long long)(gd.word0 + gd.nch + k) * BHW + gc;
          float mu = *t, vv = *vr;
          rule_gaussian(mu, vv, obb, sum, (double)ng, gd);
          *t = mu;
          *vr = vv;
          break;
        }
        case MEM_CLASS_BAYESIAN: *t = rule_dirichlet(*t, obb, sum, gd.a0); break;
        default: break;
      }
    }
    *obs = 1;
  }
}

// the loads of one short cell (its pre-frame state and its first kCellB records), issued
// together so that a thread can have the next cell's loads in flight while it fuses this one
constexpr int kCellB = 4;
template <int kFast>
struct CellIn {
  uint4 seg;
  float h, s2, th[kFast == 1 ? 3 : 1];
  uint8_t vd, ob;
  uint4 q[kCellB];
};

template <int kFast>
__device__ __forceinline__ void load_cell(const PassArgs &a, const uint4 seg, CellIn<kFast> &c) {
  constexpr int NCH = kFast == 1 ? 3 : kFast == 2 ? 1 : 0;
  const long long BHW = a.geo.BHW;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  c.seg = seg;
  const long long gc = c.seg.x;
  c.h = __ldcg(vals + (long long)kWordElev * BHW + gc);
  c.s2 = __ldcg(vals + (long long)kWordVar * BHW + gc);
  c.vd = __ldcg(a.st.flags + (long long)kFlagValid * BHW + gc);
  c.ob = 0;
  if (NCH > 0) {
    const GroupDesc &gd = a.b[0].g;
#pragma unroll
    for (int k = 0; k < NCH; ++k) c.th[k] = __ldcg(vals + (long long)(gd.word0 + k) * BHW + gc);
    c.ob = __ldcg(a.st.flags + (long long)gd.flag * BHW + gc);
  }
  const uint4 *rec = a.srec + c.seg.y;
#pragma unroll
  for (int u = 0; u < kCellB; ++u)
    if (u < (int)c.seg.z) c.q[u] = __ldcg(rec + u);
}

// a7 + a8 for the short cell's points in input order, then a9 + a10 (one thread)
template <bool kDebug, int kFast>
__device__ __forceinline__ void fuse_cell(const PassArgs &a, const CellIn<kFast> &c, unsigned (&cnt)[8]) {
  const long long gc = c.seg.x;  // m * HW + physical cell
  const uint4 *rec = a.srec + c.seg.y;
  const int n = (int)c.seg.z;
  const float h = c.h, s2 = c.s2;
  const float tau2 = a.np.tau2;
  double P = 0.0, S = 0.0;
  unsigned nin = 0u, nout = 0u;
  unsigned cr = 0u, cg = 0u, cb = 0u, na = 0u;  // colour sums and count / average count
  double X = 0.0;                               // 1-channel average sum
  auto point = [&](const uint4 q, int r) {
    const float z = __uint_as_float(q.y), v = __uint_as_float(q.z);
    const float d = z - h;  // a7 (D10): NaN state (invalid cell) compares false
    const bool outl = d * d > tau2 * (s2 + v);
    if (outl) {
      ++nout;
    } else {
      ++nin;
      const float w = 1.0f / v;  // a8: the oracle's fp32 terms, summed in fp64 in input order
      P += (double)w;
      S += (double)(z * w);
    }
    if (kFast == 1) {  // D20: packed 0x00RRGGBB, exact integer sums
      cr += (q.w >> 16) & 255u;
      cg += (q.w >> 8) & 255u;
      cb += q.w & 255u;
      ++na;
    } else if (kFast == 2) {  // D31: a non-finite channel skips the group
      const float ch = __uint_as_float(q.w);
      if (isfinite(ch)) {
        ++na;
        X += (double)ch;
      }
    }
    if (kDebug) a.dbg_code[__ldcg(a.sridx + c.seg.y + r)] = (uint8_t)(outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER);
  };
#pragma unroll
  for (int u = 0; u < kCellB; ++u)
    if (u < n) point(c.q[u], u);
  for (int r = kCellB; r < n; r += kCellB) {  // the rest of a longer cell, kCellB in flight
    uint4 qb[kCellB];
#pragma unroll
    for (int u = 0; u < kCellB; ++u)
      if (r + u < n) qb[u] = __ldcg(rec + r + u);
#pragma unroll
    for (int u = 0; u < kCellB; ++u)
      if (r + u < n) point(qb[u], r + u);
  }
  cnt[5] += nin;
  cnt[6] += nout;
  ++cnt[7];
  fuse_state<kFast>(a, gc, h, s2, c.vd, c.th, c.ob, nin, nout, P, S, cr, cg, cb, na, X);
  if constexpr (kFast == 0) fuse_generic(a, gc, rec, n);
}

// One long cell (more than kShortSeg points) on one warp: lane l takes record b0 + l of each
// batch of 32 (coalesced loads, the per-point fp32 terms in parallel), then every lane folds
// the batch's terms in lane order -- i.e. input order -- with shuffles, so the fp64 sums are the
// oracle's sequential ones; integer sums and counts are order-free warp reductions.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o > v ? o : v;
  }
  return v;
}

// One cell on a group of G lanes (G = 8: mid-size cells, 4 per warp; G = 32: long cells): lane
// li of the group takes record b0 + li of each batch of G, and every lane of the group folds the
// batch's terms in lane order -- input order -- with shuffles.
template <int G>
__device__ __forceinline__ unsigned group_sum(unsigned v) {
  if constexpr (G == 32) {
    return __reduce_add_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
  }
}

template <bool kDebug, int kFast, int G>
__device__ __forceinline__ void fuse_cell_group(const PassArgs &a, const uint4 seg, unsigned (&cnt)[8]) {
  constexpr int NCH = kFast == 1 ? 3 : kFast == 2 ? 1 : 0;
  const int lane = threadIdx.x & 31, li = lane & (G - 1);
  const unsigned gsh = (unsigned)(lane & ~(G - 1));  // the group's first lane
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  const long long gc = seg.x;
  const uint4 *rec = a.srec + seg.y;
  const int n = (int)seg.z;  // 0: this group has no cell (uniform control flow is kept)
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  float h = 0.0f, s2 = 0.0f;
  uint8_t vd0 = 0;
  float th[NCH > 0 ? NCH : 1] = {};
  uint8_t ob = 0;
  if (n > 0) {
    h = __ldcg(vals + (long long)kWordElev * BHW + gc);
    s2 = __ldcg(vals + (long long)kWordVar * BHW + gc);
    vd0 = __ldcg(a.st.flags + (long long)kFlagValid * BHW + gc);
    if (NCH > 0) {
      const GroupDesc &gd = a.b[0].g;
#pragma unroll
      for (int k = 0; k < NCH; ++k) th[k] = __ldcg(vals + (long long)(gd.word0 + k) * BHW + gc);
      ob = __ldcg(a.st.flags + (long long)gd.flag * BHW + gc);
    }
  }
  const float tau2 = a.np.tau2;
  double P = 0.0, S = 0.0, X = 0.0;
  unsigned nin = 0u, nout = 0u, cr = 0u, cg = 0u, cb = 0u, na = 0u;
  // the longest cell of the warp's groups bounds the batch loop (every lane runs it)
  int nmax = n;
#pragma unroll
  for (int d = 16; d >= G; d >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, d));
  constexpr unsigned gmask = (unsigned)((1ull << G) - 1ull);
  // pass 1: a7, the counts and colour sums, and the fp64 sums as group trees with the
  // exactness certificate of the cell's terms (k_red.cuh): when it holds the trees are the
  // oracle's sequential sums bit for bit; pass 2 (only groups whose certificate fails) folds
  // sequentially in input order
  unsigned ewx = 0u, ewn = 255u, ezx = 0u, ezn = 255u, ecx = 0u, ecn = 255u;
  uint4 q = make_uint4(0u, 0u, 0u, 0u);
  if (li < n) q = __ldcg(rec + li);
  for (int b0 = 0; b0 < nmax; b0 += G) {
    const int m_ = n - b0 < G ? (n - b0 > 0 ? n - b0 : 0) : G;
    const bool act = li < m_;
    uint4 nq = make_uint4(0u, 0u, 0u, 0u);  // the next batch in flight
    if (b0 + G + li < n) nq = __ldcg(rec + b0 + G + li);
    const float z = __uint_as_float(q.y), v = __uint_as_float(q.z);
    const float d = z - h;  // a7 (D10)
    const bool outl = act && d * d > tau2 * (s2 + v);
    const bool inl = act && !outl;
    float w = 0.0f, zw = 0.0f;
    if (inl) {
      w = 1.0f / v;  // a8: the oracle's fp32 terms
      zw = z * w;
      const unsigned e1 = max((__float_as_uint(w) >> 23) & 255u, 1u);
      ewx = max(ewx, e1);
      ewn = min(ewn, e1);
      if (zw != 0.0f) {
        const unsigned e2 = max((__float_as_uint(zw) >> 23) & 255u, 1u);
        ezx = max(ezx, e2);
        ezn = min(ezn, e2);
      }
    }
    nin += __popc((__ballot_sync(0xffffffffu, inl) >> gsh) & gmask);
    nout += __popc((__ballot_sync(0xffffffffu, outl) >> gsh) & gmask);
    float c = 0.0f;
    if (kFast == 1) {  // D20: exact integer sums, order-free
      cr += group_sum<G>(act ? (q.w >> 16) & 255u : 0u);
      cg += group_sum<G>(act ? (q.w >> 8) & 255u : 0u);
      cb += group_sum<G>(act ? q.w & 255u : 0u);
      na += m_;
    } else if (kFast == 2) {  // D31
      const float cc = __uint_as_float(q.w);
      const bool fin = act && isfinite(cc);
      na += __popc((__ballot_sync(0xffffffffu, fin) >> gsh) & gmask);
      if (fin) {
        c = cc;
        if (cc != 0.0f) {
          const unsigned e3 = max((__float_as_uint(cc) >> 23) & 255u, 1u);
          ecx = max(ecx, e3);
          ecn = min(ecn, e3);
        }
      }
    }
    double tw = (double)w, tz = (double)zw, tc = (double)c;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      tw += __shfl_xor_sync(0xffffffffu, tw, o);
      tz += __shfl_xor_sync(0xffffffffu, tz, o);
      if (kFast == 2) tc += __shfl_xor_sync(0xffffffffu, tc, o);
    }
    P += tw;
    S += tz;
    if (kFast == 2) X += tc;
    if (kDebug && act) a.dbg_code[__ldcg(a.sridx + seg.y + b0 + li)] = (uint8_t)(outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER);
    q = nq;
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    ewx = max(ewx, __shfl_xor_sync(0xffffffffu, ewx, o));
    ewn = min(ewn, __shfl_xor_sync(0xffffffffu, ewn, o));
    ezx = max(ezx, __shfl_xor_sync(0xffffffffu, ezx, o));
    ezn = min(ezn, __shfl_xor_sync(0xffffffffu, ezn, o));
    if (kFast == 2) {
      ecx = max(ecx, __shfl_xor_sync(0xffffffffu, ecx, o));
      ecn = min(ecn, __shfl_xor_sync(0xffffffffu, ecn, o));
    }
  }
  const unsigned lg = cert_ceil_log2(nin);
  const bool exact = (nin == 0u || ewx - ewn + lg <= 29u) && (ezx < ezn || ezx - ezn + lg <= 29u) &&
                     (kFast != 2 || ecx < ecn || ecx - ecn + cert_ceil_log2(na) <= 29u);
  if (__any_sync(0xffffffffu, !exact)) {  // pass 2: every lane runs it (full-warp shuffles)
    double P2 = 0.0, S2 = 0.0, X2 = 0.0;
    if (li < n) q = __ldcg(rec + li);
    for (int b0 = 0; b0 < nmax; b0 += G) {
      const int m_ = n - b0 < G ? (n - b0 > 0 ? n - b0 : 0) : G;
      const bool act = li < m_;
      uint4 nq = make_uint4(0u, 0u, 0u, 0u);
      if (b0 + G + li < n) nq = __ldcg(rec + b0 + G + li);
      const float z = __uint_as_float(q.y), v = __uint_as_float(q.z);
      const float d = z - h;
      const bool inl = act && !(d * d > tau2 * (s2 + v));
      float w = 0.0f, zw = 0.0f, c = 0.0f;
      if (inl) {
        w = 1.0f / v;
        zw = z * w;
      }
      const unsigned im = (__ballot_sync(0xffffffffu, inl) >> gsh) & gmask;
      unsigned fm = 0u;
      if (kFast == 2) {
        c = __uint_as_float(q.w);
        fm = (__ballot_sync(0xffffffffu, act && isfinite(c)) >> gsh) & gmask;
        if (!(fm >> li & 1u)) c = 0.0f;
      }
      // block-certified: the batch's exact sum when adding it to the running sum provably
      // rounds nowhere (fold_exact), else term by term in input order
      double bs[3] = {(double)w, (double)zw, (double)c}, ba[3] = {(double)w, fabs((double)zw), fabs((double)c)};
      int bq[3] = {w != 0.0f ? lsb32(w) : 0x7fffffff, zw != 0.0f ? lsb32(zw) : 0x7fffffff,
                   c != 0.0f ? lsb32(c) : 0x7fffffff};
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if (k == 2 && kFast != 2) continue;
          bs[k] += __shfl_xor_sync(0xffffffffu, bs[k], o);
          ba[k] += __shfl_xor_sync(0xffffffffu, ba[k], o);
          bq[k] = min(bq[k], __shfl_xor_sync(0xffffffffu, bq[k], o));
        }
      }
      const bool okP = fold_exact(P2, ba[0], bq[0]), okS = fold_exact(S2, ba[1], bq[1]);
      const bool okX = kFast != 2 || fold_exact(X2, ba[2], bq[2]);
      if (okP) P2 += bs[0];
      if (okS) S2 += bs[1];
      if (kFast == 2 && okX) X2 += bs[2];
      if (__any_sync(0xffffffffu, !(okP && okS && okX))) {
        for (int j0 = 0; j0 < G; j0 += 8) {  // input order; 8 lanes' terms fetched ahead of the adds
          float wj[8], zj[8], cj[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            wj[u] = __shfl_sync(0xffffffffu, w, j0 + u, G);
            zj[u] = __shfl_sync(0xffffffffu, zw, j0 + u, G);
            if (kFast == 2) cj[u] = __shfl_sync(0xffffffffu, c, j0 + u, G);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (im >> (j0 + u) & 1u) {
              if (!okP) P2 += (double)wj[u];
              if (!okS) S2 += (double)zj[u];
            }
            if (kFast == 2 && !okX && (fm >> (j0 + u) & 1u)) X2 += (double)cj[u];
          }
        }
      }
      q = nq;
    }
    if (!exact) {
      P = P2;
      S = S2;
      X = X2;
    }
  }
  if (li == 0 && n > 0) {
    cnt[5] += nin;
    cnt[6] += nout;
    ++cnt[7];
    fuse_state<kFast>(a, gc, h, s2, vd0, th, ob, nin, nout, P, S, cr, cg, cb, na, X);
  }
}

template <bool kDebug, int kFast>
__device__ __forceinline__ void fuse_cell_warp(const PassArgs &a, const uint4 seg, unsigned (&cnt)[8]) {
  constexpr int NCH = kFast == 1 ? 3 : kFast == 2 ? 1 : 0;
  const int lane = threadIdx.x & 31;
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  const long long gc = seg.x;
  const uint4 *rec = a.srec + seg.y;
  const int n = (int)seg.z;
  if constexpr (kFast != 0) {  // a 16-lane group (the upper half-warp idles; ptxas rejects the
                               // 32-lane colour variant: C7600)
    fuse_cell_group<kDebug, kFast, 16>(a, lane < 16 ? seg : make_uint4(0u, 0u, 0u, 0u), cnt);
    return;
  }
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const float h = __ldcg(vals + (long long)kWordElev * BHW + gc), s2 = __ldcg(vals + (long long)kWordVar * BHW + gc);
  const uint8_t vd0 = __ldcg(a.st.flags + (long long)kFlagValid * BHW + gc);
  float th[NCH > 0 ? NCH : 1];
  uint8_t ob = 0;
  const float tau2 = a.np.tau2;
  double P = 0.0, S = 0.0, X = 0.0;
  unsigned nin = 0u, nout = 0u, cr = 0u, cg = 0u, cb = 0u, na = 0u;
  // pass 1: the a7 decisions, the counts, and the fp64 sums as warp trees together with the
  // exactness certificate of the cell's terms (k_red.cuh): when it holds, every partial sum is
  // exact and the trees equal the oracle's sequential sums bit for bit
  uint4 q = make_uint4(0u, 0u, 0u, 0u);
  if (lane < n) q = __ldcg(rec + lane);
  unsigned ewmax = 0u, ewmin = 255u, ezmax = 0u, ezmin = 255u;
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int m_ = n - b0 < 32 ? n - b0 : 32;
    const bool act = lane < m_;
    uint4 nq = make_uint4(0u, 0u, 0u, 0u);
    if (b0 + 32 + lane < n) nq = __ldcg(rec + b0 + 32 + lane);
    const float z = __uint_as_float(q.y), v = __uint_as_float(q.z);
    const float d = z - h;  // a7 (D10)
    const bool outl = act && d * d > tau2 * (s2 + v);
    const bool inl = act && !outl;
    float w = 0.0f, zw = 0.0f;
    if (inl) {
      w = 1.0f / v;
      zw = z * w;
      const unsigned ew = max((__float_as_uint(w) >> 23) & 255u, 1u);
      ewmax = max(ewmax, ew);
      ewmin = min(ewmin, ew);
      if (zw != 0.0f) {
        const unsigned ez = max((__float_as_uint(zw) >> 23) & 255u, 1u);
        ezmax = max(ezmax, ez);
        ezmin = min(ezmin, ez);
      }
    }
    nin += __popc(__ballot_sync(0xffffffffu, inl));
    nout += __popc(__ballot_sync(0xffffffffu, outl));
    double tw = (double)w, tz = (double)zw;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tw += __shfl_xor_sync(0xffffffffu, tw, o);
      tz += __shfl_xor_sync(0xffffffffu, tz, o);
    }
    P += tw;
    S += tz;
    if (kDebug && act) a.dbg_code[__ldcg(a.sridx + seg.y + b0 + lane)] = (uint8_t)(outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER);
    q = nq;
  }
  ewmax = __reduce_max_sync(0xffffffffu, ewmax);
  ewmin = __reduce_min_sync(0xffffffffu, ewmin);
  ezmax = __reduce_max_sync(0xffffffffu, ezmax);
  ezmin = __reduce_min_sync(0xffffffffu, ezmin);
  const unsigned lg = cert_ceil_log2(nin);
  const bool exact = (nin == 0u || ewmax - ewmin + lg <= 29u) && (ezmax < ezmin || ezmax - ezmin + lg <= 29u);
  if (!exact) {  // pass 2: the oracle's sequential fold
    P = S = 0.0;
    if (lane < n) q = __ldcg(rec + lane);
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int m_ = n - b0 < 32 ? n - b0 : 32;
      const bool act = lane < m_;
      uint4 nq = make_uint4(0u, 0u, 0u, 0u);
      if (b0 + 32 + lane < n) nq = __ldcg(rec + b0 + 32 + lane);
      const float z = __uint_as_float(q.y), v = __uint_as_float(q.z);
      const float d = z - h;  // a7 (D10)
      const bool inl = act && !(d * d > tau2 * (s2 + v));
      float w = 0.0f, zw = 0.0f;
      if (inl) {
        w = 1.0f / v;
        zw = z * w;
      }
      const unsigned im = __ballot_sync(0xffffffffu, inl);
      for (int j = 0; j < m_; ++j) {  // input order
        const float wj = __shfl_sync(0xffffffffu, w, j), zj = __shfl_sync(0xffffffffu, zw, j);
        if (im >> j & 1u) {
          P += (double)wj;
          S += (double)zj;
        }
      }
      q = nq;
    }
  }
  if (lane == 0) {
    cnt[5] += nin;
    cnt[6] += nout;
    ++cnt[7];
    fuse_state<kFast>(a, gc, h, s2, vd0, th, ob, nin, nout, P, S, cr, cg, cb, na, X);
  }
  if constexpr (kFast == 0) {  // generic groups, warp-parallel over the points of each batch
    float *wv = reinterpret_cast<float *>(a.st.words);
    for (int bi = 0; bi < a.nb; ++bi) {
      const BindDesc &b = a.b[bi];
      const GroupDesc &gd = b.g;
      if (gd.rule == MEM_COLOR) {
        unsigned r_ = 0u, g_ = 0u, b_ = 0u;
        for (int b0 = 0; b0 < n; b0 += 32) {
          unsigned bits = 0u;
          if (b0 + lane < n) bits = __float_as_uint(chan_value(a, b, __ldcg(&rec[b0 + lane].w), 0));
          r_ += __reduce_add_sync(0xffffffffu, (bits >> 16) & 255u);
          g_ += __reduce_add_sync(0xffffffffu, (bits >> 8) & 255u);
          b_ += __reduce_add_sync(0xffffffffu, bits & 255u);
        }
        if (lane == 0) {
          uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
          const bool obb = *obs != 0;
          const unsigned sums[3] = {r_, g_, b_};
          for (int k = 0; k < 3; ++k) {
            float *t = wv + (long long)(gd.word0 + k) * BHW + gc;
            *t = rule_average(*t, obb, (double)sums[k], (double)n, gd.w);
          }
          *obs = 1;
        }
        continue;
      }
      if (gd.rule == MEM_CLASS_MAX) {  // D19: order-free maximum
        unsigned long long key = 0ull;
        for (int b0 = 0; b0 < n; b0 += 32) {
          unsigned long long k = 0ull;
          if (b0 + lane < n) {
            const uint4 r = __ldcg(rec + b0 + lane);
            if (r.x >> (16 + bi) & 1u) k = chan_key(a, b, r.w);
          }
          k = warp_max_u64(k);
          key = k > key ? k : key;
        }
        if (lane == 0 && key != 0ull) {
          reinterpret_cast<int *>(a.st.words)[(long long)gd.label * BHW + gc] =
              gd.nch - 1 - (int)(uint32_t)(key & 0xffffffffull);
          wv[(long long)gd.word0 * BHW + gc] = f32_of_ord((uint32_t)(key >> 32));
        }
        continue;
      }
      unsigned ng = 0u;
      for (int b0 = 0; b0 < n; b0 += 32)
        ng += __popc(__ballot_sync(0xffffffffu, b0 + lane < n && (__ldcg(&rec[b0 + lane].x) >> (16 + bi) & 1u)));
      if (ng == 0u) continue;  // D31
      uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
      const bool obb = *obs != 0;
      // lane = point: each channel's values of a batch of 32 points are gathered by one warp
      // load and summed by a warp tree; lane kk of block k0 keeps channel k0 + kk's sum and the
      // exactness certificate of its terms (k_red.cuh: exponent range + ceil(log2 ng) <= 29 makes
      // every partial sum exact, so the tree sums equal the oracle's sequential ones); a channel
      // whose certificate fails is re-summed by its lane sequentially in input order
      for (int k0 = 0; k0 < gd.nch; k0 += 32) {
        const int nk = gd.nch - k0 < 32 ? gd.nch - k0 : 32;
        double acc = 0.0;
        unsigned emx = 0u, emn = 255u;
        for (int b0 = 0; b0 < n; b0 += 32) {
          unsigned pid = 0u;
          bool ok = false;
          if (b0 + lane < n) {
            const uint4 r = __ldcg(rec + b0 + lane);
            ok = r.x >> (16 + bi) & 1u;
            pid = r.w;
          }
          for (int kk0 = 0; kk0 < nk; kk0 += 4) {
            float cv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) cv[u] = ok && kk0 + u < nk ? chan_value(a, b, pid, k0 + kk0 + u) : 0.0f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const unsigned e = cv[u] != 0.0f ? max((__float_as_uint(cv[u]) >> 23) & 255u, 1u) : 0u;
              const unsigned ex = __reduce_max_sync(0xffffffffu, e);
              const unsigned en = __reduce_min_sync(0xffffffffu, e ? e : 255u);
              double t = (double)cv[u];
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
              if (lane == kk0 + u) {
                acc += t;
                emx = max(emx, ex);
                emn = min(emn, en);
              }
            }
          }
        }
        const int k = k0 + lane;
        if (lane < nk && !(emx < emn || emx - emn + cert_ceil_log2(ng) <= 29u)) {
          acc = 0.0;  // uncertified: the oracle's sequential sum of this channel
          for (int r = 0; r < n; ++r) {
            const uint4 q = __ldcg(rec + r);
            if (q.x >> (16 + bi) & 1u) acc += (double)chan_value(a, b, q.w, k);
          }
        }
        const double sum = acc;
        if (lane < nk) {
          float *t = wv + (long long)(gd.word0 + k) * BHW + gc;
          switch (gd.rule) {
            case MEM_AVERAGE:
            case MEM_CLASS_AVERAGE: *t = rule_average(*t, obb, sum, (double)ng, gd.w); break;
            case MEM_GAUSSIAN: {
              float *vr = wv + (long long)(gd.word0 + gd.nch + k) * BHW + gc;
              float mu = *t, vv = *vr;
              rule_gaussian(mu, vv, obb, sum, (double)ng, gd);
              *t = mu;
              *vr = vv;
              break;
            }
            case MEM_CLASS_BAYESIAN: *t = rule_dirichlet(*t, obb, sum, gd.a0); break;
            default: break;
          }
        }
      }
      __syncwarp();  // every lane has read `obb`
      if (lane == 0) *obs = 1;
    }
  }
}

// kPart 0: the short cells (a thread each); kPart 1: long cells (16 lanes each), then mid-size
// ones (8 lanes each).  Two kernels, so that the common short-cell kernel keeps few registers.
template <bool kDebug, int kFast, int kPart>
__global__ void __launch_bounds__(kFuseThreads, kPart == 0 ? (kFast == 0 ? MEM_FUSE_MINB0 : 8) : 4) k_fuse(const __grid_constant__ PassArgs a) {
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if constexpr (kPart == 1) {
    const unsigned nlong = *(volatile unsigned *)&a.ctl->n_lseg, nmid = *(volatile unsigned *)&a.ctl->n_mseg;
    const unsigned gw = (blockIdx.x * kFuseThreads + threadIdx.x) >> 5, nw = gridDim.x * (kFuseThreads / 32);
    for (unsigned s = gw; s < nlong; s += nw) fuse_cell_warp<kDebug, kFast>(a, __ldcg(a.segs + (a.seg_cap - 1 - s)), cnt);
    if constexpr (kFast != 0) {
      const unsigned grp = (blockIdx.x * kFuseThreads + threadIdx.x) >> 3, ngrp = gridDim.x * (kFuseThreads / 8);
      for (unsigned s0 = grp & ~3u; s0 < nmid; s0 += ngrp) {  // warp-uniform trip count
        const unsigned s = s0 + (grp & 3u);
        const uint4 sg = s < nmid ? __ldcg(a.segs + a.seg_cap + s) : make_uint4(0u, 0u, 0u, 0u);
        fuse_cell_group<kDebug, kFast, 8>(a, sg, cnt);
      }
    }
  } else {
    const unsigned nseg = *(volatile unsigned *)&a.ctl->n_seg;
    for (unsigned s = blockIdx.x * kFuseThreads + threadIdx.x; s < nseg; s += gridDim.x * kFuseThreads) {
      CellIn<kFast> c;
      load_cell<kFast>(a, __ldcg(a.segs + s), c);
      fuse_cell<kDebug, kFast>(a, c, cnt);
    }
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
