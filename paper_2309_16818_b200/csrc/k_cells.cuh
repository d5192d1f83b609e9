// k_cells.cuh -- k_cells (a9-a10 + lazy a13 after k_points) and k_refold (the sequential
// recomputation of uncertified cells).  Part of the single translation unit kernels.cu
// (included inside namespace memk, in order).
#pragma once

// One lane fuses up to N touched cells (phys[u] >= 0) of map m from the RED statistics.  Every
// load of a cell (scratch record, certificates, h, s2, valid, observed, theta_k) is issued in one
// round before any math or store.  A cell whose certificate fails (cert_ok) is not fused: it is
// appended to the fallback list for k_refold, which recomputes it in input order.
// kFast: 1 colour, 2 one 1-channel average group, 0 height only.
template <int N, int kFast>
__device__ __forceinline__ void fuse_cells_red(const PassArgs &a, int m, const int (&phys)[N],
                                               const unsigned long long (&cnt)[N], unsigned (&stc)[8]) {
  constexpr int NCH = kFast == 1 ? 3 : kFast == 2 ? 1 : 0;
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  double P[N], S[N];
  unsigned long long w0[N], w1[N];
  uint2 ce[N];
  float h[N], s2[N], th[N][NCH > 0 ? NCH : 1];
  uint8_t vd[N], ob[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {  // one round of loads
    if (phys[u] < 0) continue;
    const int c = m * g.HW + phys[u];                // state
    const int q = (m - a.m0) * g.HW + phys[u] - a.sc_lo;  // scratch (this wave's maps / cells)
    const ulonglong2 *r = reinterpret_cast<const ulonglong2 *>(a.rec + (long long)q * 4);
    const ulonglong2 ps = __ldcg(r), ww = __ldcg(r + 1);
    P[u] = __longlong_as_double((long long)ps.x);
    S[u] = __longlong_as_double((long long)ps.y);
    w0[u] = ww.x;
    w1[u] = ww.y;
    if (kFast == 2) ce[u] = __ldcg(reinterpret_cast<const uint2 *>(a.cert) + q);
    h[u] = elev[c];
    s2[u] = var[c];
    vd[u] = validp[c];
    ob[u] = 0;
    if (NCH > 0) {
      const GroupDesc &gd = a.b[0].g;
      ob[u] = a.st.flags[(long long)gd.flag * BHW + c];
#pragma unroll
      for (int k = 0; k < NCH; ++k) th[u][k] = vals[(long long)(gd.word0 + k) * BHW + c];
    }
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (phys[u] < 0) continue;
    const int c = m * g.HW + phys[u];
    // counts: colour count word b | n << 25 | n_out << 43, else n_in | n_out << 32; colour and
    // height only keep the certificate in record word 3
    if (kFast != 2) ce[u] = make_uint2((unsigned)w1[u], (unsigned)(w1[u] >> 32));
    const unsigned n_out = kFast == 1 ? (unsigned)(cnt[u] >> 43) : (unsigned)(cnt[u] >> 32);
    const unsigned n_in = kFast == 1 ? (unsigned)((cnt[u] >> 25) & 0x3ffffull) - n_out : (unsigned)(cnt[u] & 0xffffffffull);
    const unsigned ng = kFast == 1 ? (unsigned)((cnt[u] >> 25) & 0x3ffffull) : kFast == 2 ? (unsigned)w0[u] : 0u;
    const bool ok = cert_ok(ce[u].x, n_in) && (kFast != 2 || cert_ok(ce[u].y, ng));
    if (ok) {
      ++stc[7];
      // a9: Kalman height fusion (D7, D11)
      float hh = h[u], ss = s2[u];
      uint8_t vv = vd[u];
      kalman_height(hh, ss, vv, (double)n_in, (double)n_out, P[u], S[u], a.np.v_out);
      if (vv) {
        elev[c] = hh;
        var[c] = ss;
        if (!vd[u]) validp[c] = 1;
      }
      // a10: Eq.(1)+(2) per channel
      if (NCH > 0 && ng != 0u) {
        const GroupDesc &gd = a.b[0].g;
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          double sk;
          if (kFast == 1) {
            const uint32_t v = k == 0 ? (uint32_t)(w0[u] & 0xffffffffull)
                                      : k == 1 ? (uint32_t)(w0[u] >> 32) : (uint32_t)(cnt[u] & 0x1ffffffull);
            sk = (double)v;  // exact integer colour sums (D20)
          } else {
            sk = __longlong_as_double((long long)w1[u]);
          }
          vals[(long long)(gd.word0 + k) * BHW + c] = rule_average(th[u][k], ob[u] != 0, sk, (double)ng, gd.w);
        }
        if (!ob[u]) a.st.flags[(long long)gd.flag * BHW + c] = 1;
      }
    } else {  // uncertified: its points listed and recomputed in input order by k_refold
      const unsigned k = atomicAdd(&a.ctl->n_fb, 1u);
      const unsigned n = n_in + n_out;  // the cell's in-window points
      const unsigned off = atomicAdd(&a.ctl->n_fbpts, n);
      a.fb[2 * k] = (unsigned long long)c;
      a.fb[2 * k + 1] = (unsigned long long)off | (unsigned long long)n << 32;
      a.fbmark[c] = (int)k;
      a.fbmap[m] = 1u;
    }
    // re-zero the scratch for the next wave / point input
    const int q = (m - a.m0) * g.HW + phys[u] - a.sc_lo;
    unsigned long long *r = a.rec + (long long)q * 4;
#if MEM_SCRATCH_HINT
    {  // evict-last: the zeroed lines should still be in L2 when the next point pass REDs into them
      const unsigned long long pol = evict_last_policy();
      st_hint_u64(a.cnt + q, 0ull, pol);
      st_hint_u64x2(r, 0ull, 0ull, pol);
      st_hint_u64x2(r + 2, 0ull, 0ull, pol);
    }
#else
    __stcg(a.cnt + q, 0ull);
    __stcg(reinterpret_cast<ulonglong2 *>(r), make_ulonglong2(0ull, 0ull));
    __stcg(reinterpret_cast<ulonglong2 *>(r) + 1, make_ulonglong2(0ull, 0ull));
#endif
    if (kFast == 2) __stcg(reinterpret_cast<uint2 *>(a.cert) + q, make_uint2(0u, 0u));
  }
}

// ---------------------------------------------------------------- k_cells (a9-a10, lazy a13)
constexpr int kChunkPerLane = 4;                 // cells per lane per chunk
constexpr int kChunk = 32 * kChunkPerLane;        // 128-cell chunk per warp

// Warp-persistent grid-stride over 128-cell chunks of the call's maps (newest map first: its
// scratch was touched last by k_points and is still in L2).  Each warp, independently of the
// others (no CTA barrier): 4 count loads per lane in flight, the pending shift strips reset,
// its touched cells compacted in its own shared-memory slice, then fused 2 per lane per round.
#ifndef MEM_CELLS_MINB
#define MEM_CELLS_MINB 3  // k_cells: CTAs per SM the registers are sized for
#endif
// kCPL: cells per lane per chunk -- 4 (128-cell chunks) when the call has chunks for every
// resident warp, else 1 (32-cell chunks: a small map spreads over more SMs, shorter chains)
template <int kFast, int kCPL>
__global__ void __launch_bounds__(kThreads, MEM_CELLS_MINB) k_cells(const __grid_constant__ PassArgs a) {
  constexpr int kCh = 32 * kCPL;
  __shared__ int s_phys[kThreads / 32][kCh];
  __shared__ unsigned long long s_cntv[kThreads / 32][kCh];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (kThreads / 32);
  const int gw = blockIdx.x * (kThreads / 32) + wid;
  const int cpm = (a.cell_hi - a.cell_lo + kCh - 1) / kCh;  // chunks per map (band)
  const int total = (a.m1 - a.m0) * cpm;  // this wave's maps
  int *sp = s_phys[wid];
  unsigned long long *sc = s_cntv[wid];
  for (int rt = gw; rt < total; rt += nwarps) {
    const int chunk = total - 1 - rt;
    const int mi = chunk / cpm;
    const int m = a.m0 + mi;
    const int t0 = a.cell_lo + (chunk - mi * cpm) * kCh;
    const int sb = mi * g.HW - a.sc_lo;  // scratch
    unsigned long long cv[kCPL];
#pragma unroll
    for (int u = 0; u < kCPL; ++u) {  // counts first (memory-level parallelism)
      const int phys = t0 + u * 32 + lane;
      cv[u] = phys < a.cell_hi ? __ldcg(a.cnt + sb + phys) : 0ull;
    }
    const PointFrame f = frame_of(a, m);
    if (t0 == a.cell_lo && lane == 0) a.ring[m] = make_int2(f.r0, f.c0);
    int n = 0;
#pragma unroll
    for (int u = 0; u < kCPL; ++u) {
      const int phys = t0 + u * 32 + lane;
      if (phys < a.cell_hi && (f.sr != 0 || f.sc != 0)) {  // lazy ring shift: reset the scrolled-in cells (a13)
        int pcol;
        const int prow = divmod_fast(phys, g.W, g.inv_W, pcol);
        int row = prow - f.r0, col = pcol - f.c0;
        row += row < 0 ? g.H : 0;
        col += col < 0 ? g.W : 0;
        if (in_strip(row, col, f, g)) reset_cell(a.st, g.BHW, (long long)m * g.HW + phys, a.reset);
      }
      const bool t = cv[u] != 0ull;  // untouched cells stay bit-identical
      const unsigned b = __ballot_sync(0xffffffffu, t);
      if (t) {
        const int k = n + __popc(b & lanemask_lt());
        sp[k] = phys;
        sc[k] = cv[u];
      }
      n += __popc(b);
    }
    __syncwarp();
    for (int k0 = 0; k0 < n; k0 += 64) {
      int ph[2];
      unsigned long long cc[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u * 32 + lane;
        ph[u] = k < n ? sp[k] : -1;
        cc[u] = k < n ? sc[k] : 0ull;
      }
      fuse_cells_red<2, kFast>(a, m, ph, cc, cnt);
    }
    __syncwarp();  // this warp's slice is rewritten by its next chunk
  }
  __syncthreads();
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

// ---------------------------------------------------------------- k_refold
// The cells k_cells could not certify (their fp64 sums might depend on the order of the REDs)
// are recomputed from their points in input order, exactly as the oracle folds them.
//
// k_refold is a cooperative launch (all CTAs resident) and returns at once when no cell is
// listed.  Phase 1 (collect_points): a grid-stride pass over the warp-items of the maps that
// have a listed cell: a2-a6 for each point (bin_point); a point whose cell is listed appends its
// index (relative to the map's first point) to the cell's slice of fblist (an atomic slot: any
// order).  A grid barrier, then phase 2 below.
__device__ __forceinline__ void collect_points(const PassArgs &a) {
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x / 32);
  const int gw = blockIdx.x * (blockDim.x / 32) + wid;
  const int i0 = ps_of(a, a.m0), i1 = ps_of(a, a.m1);
  for (int it = i0 + gw; it < i1; it += nwarps) {
    const Item t = item_of(a, it, i0);
    if (__ldcg(a.fbmap + t.m) == 0u) continue;  // warp-uniform
    const PointFrame f = frame_of(a, t.m);
    const int map_base = t.m * g.HW;
#pragma unroll
    for (int u = 0; u < kWarpPtsPerLane; ++u) {
      const long long i = t.base + u * 32 + lane;
      if (i >= t.end) continue;
      const float *p = a.pts + i * (long long)a.stride;
      const PointOut o = bin_point(__ldg(p), __ldg(p + 1), __ldg(p + 2), f, g, a.np, map_base, a.r2lo, a.r2hi);
      if (o.cell < 0) continue;
      const int k = __ldcg(a.fbmark + o.cell);
      if (k < 0) continue;
      const unsigned off = (unsigned)__ldcg(a.fb + 2 * k + 1);
      const unsigned slot = atomicAdd(a.fbfill + k, 1u);
      a.fblist[off + slot] = (unsigned)(i - t.beg);
    }
  }
}

// k_refold: one CTA per listed cell.  Its point indices are sorted into input order (a block
// radix sort in shared memory; cells of more than kRefoldCap points walk the whole map instead).
// Then, 512 points at a time, warps 1-15 evaluate the next chunk's per-point
// terms -- a2-a7 (bin_point, the Mahalanobis test against the pre-frame state, which k_cells
// left untouched), the oracle's fp32 terms 1/v and z*(1/v) of the inliers, the channel -- while
// one thread of warp 0 folds the current chunk into the fp64 sums P, S (, X) in input order,
// operation for operation the oracle's loop (a term of +0.0 stands for a skipped point: the
// sums start at +0.0 and never become -0.0, so adding +0.0 leaves them bit-identical).  The
// integer statistics are order-free (shared-memory atomics).  Then a9 + a10 (fuse_state).
#ifndef MEM_REFOLD_THREADS
#define MEM_REFOLD_THREADS 512
#endif
constexpr int kRefoldThreads = MEM_REFOLD_THREADS;
constexpr int kRefoldItems = 32;
constexpr int kRefoldCap = kRefoldThreads * kRefoldItems;  // points of a cell sorted in shared memory
constexpr int kRefoldChunk = 512;                          // terms folded per step

struct RefoldTerms {
  unsigned nin, nout, cr, cg, cb, na;
};

// the terms of point i (absolute index) of map m for a cell `cell` (global index); returns
// false if the point does not reach the cell (the scan path)
template <int kFast>
__device__ __forceinline__ bool refold_term(const PassArgs &a, const PointFrame &f, int map_base, long long i,
                                            long long cell, float h, float s2, float &w, float &zw, float &c,
                                            RefoldTerms &t) {
  const float *p = a.pts + i * (long long)a.stride;
  const PointOut o = bin_point(__ldg(p), __ldg(p + 1), __ldg(p + 2), f, a.geo, a.np, map_base, a.r2lo, a.r2hi);
  w = zw = c = 0.0f;
  if ((long long)o.cell != cell) return false;
  const float z = o.z, v = o.v;
  const float d = z - h;  // a7 (D10)
  if (d * d > a.np.tau2 * (s2 + v)) {
    ++t.nout;
  } else {
    ++t.nin;
    w = 1.0f / v;  // a8: the oracle's fp32 terms
    zw = z * w;
  }
  if (kFast == 1) {  // D20: exact integer sums
    const uint32_t bits = __float_as_uint(__ldg(p + 3));
    t.cr += (bits >> 16) & 255u;
    t.cg += (bits >> 8) & 255u;
    t.cb += bits & 255u;
    ++t.na;
  } else if (kFast == 2) {  // D31: finite channels only
    const float ch = __ldg(p + 3);
    if (isfinite(ch)) {
      ++t.na;
      c = ch;
    }
  }
  return true;
}

// the oracle's sequential fold of n terms (inputs in order; loads issued 4 ahead of the adds)
template <int kFast>
__device__ __forceinline__ void refold_fold(const float *w, const float *zw, const float *c, int n, double &P,
                                            double &S, double &X) {
  int j = 0;
  for (; j + 4 <= n; j += 4) {
    float wj[4], zj[4], cj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      wj[u] = w[j + u];
      zj[u] = zw[j + u];
      cj[u] = kFast == 2 ? c[j + u] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      P += (double)wj[u];
      S += (double)zj[u];
      if (kFast == 2) X += (double)cj[u];
    }
  }
  for (; j < n; ++j) {
    P += (double)w[j];
    S += (double)zw[j];
    if (kFast == 2) X += (double)c[j];
  }
}

// Block-certified sequential folding.  Within a block of 32 consecutive terms the oracle's
// sequential fp64 sum V <- V + t_1 <- ... rounds nowhere when every value involved is a multiple
// of 2^q (q = the lowest set bit over V and the block's terms) and every partial sum is below
// 2^(q + 53); then V + (the block's exact sum, any order) is the sequential result bit for bit.
// The block sums and their lowest-bit / magnitude summaries are computed in parallel; only the
// chain over blocks (and the rare block that fails the test) is sequential.
struct FoldBlock {
  double t[3], a[3];  // block sums (P, S, X) and sums of magnitudes
  int q[3];           // lowest set bit over the block's non-zero terms (INT_MAX: none)
};
// the block's summary from lane l's terms (all 32 lanes of a warp)
template <int kFast>
__device__ __forceinline__ FoldBlock fold_block(float w, float zw, float c) {
  FoldBlock fb;
  const float v[3] = {w, zw, c};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k == 2 && kFast != 2) {
      fb.t[k] = fb.a[k] = 0.0;
      fb.q[k] = 0x7fffffff;
      continue;
    }
    double t = (double)v[k], aa = fabs((double)v[k]);
    int q = v[k] != 0.0f ? lsb32(v[k]) : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      aa += __shfl_xor_sync(0xffffffffu, aa, o);
      q = min(q, __shfl_xor_sync(0xffffffffu, q, o));
    }
    fb.t[k] = t;
    fb.a[k] = aa;
    fb.q[k] = q;
  }
  return fb;
}

template <int kFast>
struct RefoldSmem {
  using Sort = cub::BlockRadixSort<unsigned, kRefoldThreads, kRefoldItems>;
  static constexpr int NC = kFast == 2 ? kRefoldChunk : 1;
  struct Bufs {
    float w[2][kRefoldChunk], zw[2][kRefoldChunk], c[2][NC];
  };
  union {
    typename Sort::TempStorage sort;
    Bufs b;
  } u;
  unsigned idx[kRefoldCap];
  FoldBlock blk[2][kRefoldChunk / 32];
};
template <int kFast>
size_t refold_smem_bytes() { return sizeof(RefoldSmem<kFast>); }

template <int kFast>
__global__ void __launch_bounds__(kRefoldThreads) k_refold(const __grid_constant__ PassArgs a) {
  using Sort = typename RefoldSmem<kFast>::Sort;
  extern __shared__ __align__(16) unsigned char s_raw[];
  RefoldSmem<kFast> &sm = *reinterpret_cast<RefoldSmem<kFast> *>(s_raw);
  auto &s_u = sm.u;
  unsigned *s_idx = sm.idx;
  __shared__ unsigned s_t[6];
  __shared__ unsigned s_part[kRefoldThreads / 32];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Geometry &g = a.geo;
  const unsigned nfb = *(volatile unsigned *)&a.ctl->n_fb;
  if (nfb == 0u) return;  // uniform over the grid
  collect_points(a);
  cooperative_groups::this_grid().sync();
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  for (unsigned k = blockIdx.x; k < nfb; k += gridDim.x) {
    const long long gc = (long long)__ldcg(a.fb + 2 * k);
    const unsigned long long e = __ldcg(a.fb + 2 * k + 1);
    const unsigned off = (unsigned)e, n = (unsigned)(e >> 32);
    const int m = (int)(gc / g.HW);
    const int map_base = m * g.HW;
    const PointFrame f = frame_of(a, m);
    const long long beg = off_of(a, m), end = off_of(a, m + 1);
    const float h = __ldcg(vals + (long long)kWordElev * g.BHW + gc), s2 = __ldcg(vals + (long long)kWordVar * g.BHW + gc);
    if (threadIdx.x < 6) s_t[threadIdx.x] = 0u;
    RefoldTerms t = {0u, 0u, 0u, 0u, 0u, 0u};
    double P = 0.0, S = 0.0, X = 0.0;
    if (n <= (unsigned)kRefoldCap) {
      // the cell's point indices into input order
      const unsigned span = (unsigned)(end - beg);
      const int end_bit = span <= 1u ? 1 : 32 - __clz(span - 1u);
      unsigned keys[kRefoldItems];
#pragma unroll
      for (int q = 0; q < kRefoldItems; ++q) {  // any arrangement: coalesced loads
        const unsigned j = q * kRefoldThreads + threadIdx.x;
        keys[q] = j < n ? __ldcg(a.fblist + off + j) : 0xffffffffu;
      }
      Sort(s_u.sort).Sort(keys, 0, end_bit);
#pragma unroll
      for (int q = 0; q < kRefoldItems; ++q) {  // the sorted keys: blocked arrangement
        const unsigned j = threadIdx.x * kRefoldItems + q;
        if (j < n) s_idx[j] = keys[q];
      }
      __syncthreads();  // s_idx complete; the sort's storage (aliasing the term buffers) is free
      // chunk ch's 16 blocks of 32 positions: block bk is produced by warp bk % W for the first
      // chunk (W warps), by warp 1 + bk % (W - 1) for the others (warp 0 folds meanwhile); a producing
      // warp writes the terms (for a block that must fold sequentially) and the block summary
      constexpr int kBlocks = kRefoldChunk / 32;
      const int nch = (int)((n + kRefoldChunk - 1) / kRefoldChunk);
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      auto produce = [&](int ch, int bk) {
        const int bb = ch & 1, j = bk * 32 + lane, pos = ch * kRefoldChunk + j;
        float w = 0.0f, zw = 0.0f, c = 0.0f;
        if (pos < (int)n) refold_term<kFast>(a, f, map_base, beg + s_idx[pos], gc, h, s2, w, zw, c, t);
        s_u.b.w[bb][j] = w;
        s_u.b.zw[bb][j] = zw;
        if (kFast == 2) s_u.b.c[bb][j] = c;
        const FoldBlock fb = fold_block<kFast>(w, zw, c);
        if (lane == 0) sm.blk[bb][bk] = fb;
      };
      for (int bk = wid; bk < kBlocks; bk += kRefoldThreads / 32) produce(0, bk);
      __syncthreads();
      for (int ch = 0; ch < nch; ++ch) {
        const int bb = ch & 1;
        if (wid == 0) {  // warp 0: the chain over chunk ch's blocks
          if (lane == 0) {
            const int len = (int)n - ch * kRefoldChunk < kRefoldChunk ? (int)n - ch * kRefoldChunk : kRefoldChunk;
            for (int bk = 0; bk * 32 < len; ++bk) {
              const FoldBlock &fb = sm.blk[bb][bk];
              const int bl = len - bk * 32 < 32 ? len - bk * 32 : 32;
              double *acc[3] = {&P, &S, &X};
              const float *src[3] = {s_u.b.w[bb] + bk * 32, s_u.b.zw[bb] + bk * 32, s_u.b.c[bb] + bk * 32};
#pragma unroll
              for (int k = 0; k < (kFast == 2 ? 3 : 2); ++k) {
                if (fold_exact(*acc[k], fb.a[k], fb.q[k])) {
                  *acc[k] += fb.t[k];
                } else {  // the oracle's sequential fold of this block
                  double v = *acc[k];
                  for (int i = 0; i < bl; ++i) v += (double)src[k][i];
                  *acc[k] = v;
                }
              }
            }
          }
        } else if (ch + 1 < nch) {  // warps 1-15: chunk ch + 1
          for (int bk = wid - 1; bk < kBlocks; bk += (kRefoldThreads / 32) - 1) produce(ch + 1, bk);
        }
        __syncthreads();
      }
    } else {
      // more points than the sort holds: walk the map's points in input order, 512 at a time,
      // and compact the cell's terms in order (block scan)
      for (long long b0 = beg; b0 < end; b0 += kRefoldThreads) {
        const long long i = b0 + threadIdx.x;
        float w = 0.0f, zw = 0.0f, c = 0.0f;
        const bool in = i < end && refold_term<kFast>(a, f, map_base, i, gc, h, s2, w, zw, c, t);
        unsigned tot;
        const unsigned pos = block_excl_scan<kRefoldThreads>(in ? 1u : 0u, s_part, &tot);
        if (in) {
          s_u.b.w[0][pos] = w;
          s_u.b.zw[0][pos] = zw;
          if (kFast == 2) s_u.b.c[0][pos] = c;
        }
        __syncthreads();
        if (threadIdx.x == 0) refold_fold<kFast>(s_u.b.w[0], s_u.b.zw[0], s_u.b.c[0], (int)tot, P, S, X);
        __syncthreads();
      }
    }
    // the integer statistics (order-free)
    if (t.nin) atomicAdd(&s_t[0], t.nin);
    if (t.nout) atomicAdd(&s_t[1], t.nout);
    if (kFast == 1 && t.na) {
      atomicAdd(&s_t[2], t.cr);
      atomicAdd(&s_t[3], t.cg);
      atomicAdd(&s_t[4], t.cb);
    }
    if (t.na) atomicAdd(&s_t[5], t.na);
    __syncthreads();
    if (threadIdx.x == 0) {
      ++cnt[7];
      float th[3] = {0.0f, 0.0f, 0.0f};
      uint8_t ob = 0;
      if (kFast != 0) {
        const GroupDesc &gd = a.b[0].g;
        for (int c = 0; c < (kFast == 1 ? 3 : 1); ++c) th[c] = __ldcg(vals + (long long)(gd.word0 + c) * g.BHW + gc);
        ob = __ldcg(a.st.flags + (long long)gd.flag * g.BHW + gc);
      }
      fuse_state<kFast == 0 ? 3 : kFast>(a, gc, h, s2, __ldcg(a.st.flags + (long long)kFlagValid * g.BHW + gc), th, ob,
                                         s_t[0], s_t[1], P, S, s_t[2], s_t[3], s_t[4], s_t[5], X);
      a.fbmark[gc] = -1;  // the lists are empty again for the next point input
      a.fbfill[k] = 0u;
      a.fbmap[m] = 0u;
    }
    __syncthreads();
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
