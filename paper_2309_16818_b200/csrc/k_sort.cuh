// k_sort.cuh -- k_sort: the in-window points of one cell band, sorted by cell STABLY (input
// order within each cell), plus the lazy ring-shift reset of the band (a13).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_sort
// One CTA per (map, band of band_cells physical cells).  k_bin left the band's in-window points
// as per-tile runs (input order within each run, runs in tile order), so walking the runs in
// tile order visits the band's points in input order (band position p).  The CTA
//   1. resets the band's cells in the strips that scrolled in with the pending shift (a13);
//   2. prefix-sums the runs' counts (tinfo) over the map's tiles;
//   3. counts the records per cell (shared-memory atomics: order-free integers);
//   4. turns the counts into cell starts (exclusive scan over the cells); every touched cell
//      becomes a segment {cell, first sorted record, count} of the call's list (k_fuse; cells
//      of more than kShortSeg points at the back);
//   5. ranks every record among the earlier records of its cell -- warp w walks the positions
//      [w*S, (w+1)*S) in input order, 32 at a time (__match_any_sync rank + the warp's running
//      count per cell), then each cell's per-warp counts are prefix-summed over the warps --
//      and scatters the record to (cell start + rank): a stable counting sort, each cell's
//      records in the input order the oracle sums them in.
// Bands of more than kSortCap records run step 5 window by window.
struct SortSmem {  // dynamic shared memory layout of k_sort (host and device)
  size_t bar, rec, tcnt, tpre, cst, wc, rank, total;
  __host__ __device__ SortSmem(int tmax, int band_cells) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
      const size_t at = o;
      o = (o + bytes + 15) & ~(size_t)15;
      return at;
    };
    bar = take(16);                                                           // mbarrier (bulk copies)
    rec = take(sizeof(uint4) * kSortCap);                                     // the window's records
    tcnt = take(sizeof(unsigned) * (size_t)tmax);
    tpre = take(sizeof(unsigned) * (size_t)(tmax + 1));
    cst = take(sizeof(unsigned) * (size_t)band_cells);                       // count -> start
    wc = take(sizeof(uint16_t) * (kSortThreads / 32) * (size_t)band_cells);   // [warp][cell]
    rank = take(sizeof(uint16_t) * kSortCap);
    total = o;
  }
};

template <bool kDebug>
__global__ void __launch_bounds__(kSortThreads) k_sort(const __grid_constant__ PassArgs a) {
  constexpr int kW = kSortThreads / 32;
  __shared__ unsigned s_part[kW];
  __shared__ unsigned s_base[4];  // this band's first record / short / long / mid-size segment
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const Geometry &g = a.geo;
  int bb;
  const int m = divmod_fast(blockIdx.x, a.nbands, a.inv_nbands, bb);
  const int c0 = a.cell_lo + bb * a.band_cells;
  const int c1 = c0 + a.band_cells < a.cell_hi ? c0 + a.band_cells : a.cell_hi;
  const int ncell = c1 - c0;
  const int t0 = ts_of(a, m), T = ts_of(a, m + 1) - t0;
  const SortSmem L(a.tmax, a.band_cells);
  const unsigned bar = smem_addr(s_dyn + L.bar);
  uint4 *rec_s = reinterpret_cast<uint4 *>(s_dyn + L.rec);
  unsigned *tcnt_s = reinterpret_cast<unsigned *>(s_dyn + L.tcnt);
  unsigned *tpre_s = reinterpret_cast<unsigned *>(s_dyn + L.tpre);
  unsigned *cst_s = reinterpret_cast<unsigned *>(s_dyn + L.cst);
  uint16_t *wc_s = reinterpret_cast<uint16_t *>(s_dyn + L.wc);
  uint16_t *rank_s = reinterpret_cast<uint16_t *>(s_dyn + L.rank);
  const long long gb = (long long)m * g.HW + c0;  // global index of the band's first cell
  for (int i = tid; i < ncell; i += kSortThreads) cst_s[i] = 0u;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  pdl_wait();
  pdl_trigger();
  const PointFrame f = frame_of(a, m);
  if (bb == 0 && tid == 0) a.ring[m] = make_int2(f.r0, f.c0);
  // 1. a13: the band's cells in the strips that scrolled in are reset (before k_fuse reads them)
  if (f.sr != 0 || f.sc != 0) {
    for (int i = tid; i < ncell; i += kSortThreads) {
      int pcol;
      const int prow = divmod_fast(c0 + i, g.W, g.inv_W, pcol);
      int row = prow - f.r0, col = pcol - f.c0;
      row += row < 0 ? g.H : 0;
      col += col < 0 ? g.W : 0;
      if (in_strip(row, col, f, g)) reset_cell(a.st, g.BHW, gb + i, a.reset);
    }
  }
  // 2. the runs of this band in the map's tiles, and their prefix (input order): all the
  // (strided) tinfo loads in flight first, then the scan over shared memory
  for (int tb = 0; tb < T; tb += 4 * kSortThreads) {
    unsigned v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = tb + u * kSortThreads + tid;
      v[u] = t < T ? __ldcg(a.tinfo + (long long)(t0 + t) * a.nbands + bb) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = tb + u * kSortThreads + tid;
      if (t < T) tcnt_s[t] = v[u];
    }
  }
  __syncthreads();
  unsigned K = 0u;
  for (int tb = 0; tb < T; tb += kSortThreads) {
    const int t = tb + tid;
    const unsigned v = t < T ? tcnt_s[t] : 0u;
    unsigned tot;
    const unsigned pre = block_excl_scan<kSortThreads>(v >> 16, s_part, &tot);
    if (t < T) tpre_s[t] = K + pre;
    K += tot;
  }
  if (tid == 0) tpre_s[T] = K;
  __syncthreads();
  const int nwin = (int)((K + kSortCap - 1) / kSortCap);
  // runs of a few records in a map of many tiles (a sparse band: C5b's uniform cloud) are gathered
  // by every thread with plain loads; otherwise every run by one bulk copy (warp 0)
  const bool short_runs = T > kSortThreads && 4ull * K < (unsigned long long)T * kSortBulkRun4;
  unsigned phase = 0u;
  // the window [p0, p0 + n) of band positions into rec_s, all the copies in flight together;
  // every thread waits for the lot
  auto load_window = [&](unsigned p0, unsigned n) {
    if (short_runs) {
      for (int tb = 0; tb < T; tb += 4 * kSortThreads) {  // 4 tiles per thread in flight
        unsigned lo[4], hi[4];
        const uint4 *src[4];
        uint4 r0[4], r1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = tb + u * kSortThreads + tid;
          lo[u] = hi[u] = 0u;
          src[u] = a.recs;
          if (t < T) {
            lo[u] = tpre_s[t] > p0 ? tpre_s[t] : p0;
            hi[u] = tpre_s[t + 1] < p0 + n ? tpre_s[t + 1] : p0 + n;
            src[u] = a.recs + (long long)(t0 + t) * kTile + (tcnt_s[t] & 0xffffu) - tpre_s[t];
          }
          if (hi[u] > lo[u]) r0[u] = __ldcg(src[u] + lo[u]);
          if (hi[u] > lo[u] + 1) r1[u] = __ldcg(src[u] + lo[u] + 1);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (hi[u] > lo[u]) rec_s[lo[u] - p0] = r0[u];
          if (hi[u] > lo[u] + 1) rec_s[lo[u] + 1 - p0] = r1[u];
          for (unsigned r = lo[u] + 2; r < hi[u]; ++r) rec_s[r - p0] = __ldcg(src[u] + r);
        }
      }
      __syncthreads();
      return;
    }
    if (wid == 0) {
      if (lane == 0) mbar_arrive_expect_tx(bar, 16u * n);
      __syncwarp();
      for (int t = lane; t < T; t += 32) {
        const unsigned lo = tpre_s[t] > p0 ? tpre_s[t] : p0, hi = tpre_s[t + 1] < p0 + n ? tpre_s[t + 1] : p0 + n;
        if (hi > lo)
          bulk_load(smem_addr(rec_s + (lo - p0)),
                    a.recs + (long long)(t0 + t) * kTile + (tcnt_s[t] & 0xffffu) + (lo - tpre_s[t]), 16u * (hi - lo),
                    bar);
      }
    }
    mbar_wait(bar, phase & 1u);
    ++phase;
  };
  // 3. records per cell (order-free); a band of one window keeps its records for step 5
  for (int w = 0; w < nwin; ++w) {
    const unsigned p0 = (unsigned)w * kSortCap, n = K - p0 < (unsigned)kSortCap ? K - p0 : (unsigned)kSortCap;
    if (w > 0) __syncthreads();  // rec_s is refilled
    load_window(p0, n);
    for (unsigned j = tid; j < n; j += kSortThreads) atomicAdd(&cst_s[rec_s[j].x & 0xffffu], 1u);
  }
  __syncthreads();
  // 4. cell starts (exclusive over the cells) and the touched cells' segments; thread t owns
  // the cells [t*cpt, (t+1)*cpt)
  {
    const int cpt = (ncell + kSortThreads - 1) / kSortThreads;
    const int cb = tid * cpt, ce = cb + cpt < ncell ? cb + cpt : ncell;
    // fast paths: short cells (<= kShortSeg points) a thread each, mid-size cells (<= kMidSeg)
    // 8 lanes each, long cells 16 lanes each; generic groups: a thread (<= kShortSeg) or a warp
    const unsigned smax = (unsigned)kShortSeg, mmax = a.fast ? (unsigned)kMidSeg : (unsigned)kShortSeg;
    unsigned tot = 0u, ns = 0u, nm = 0u, nl = 0u;
    for (int cc = cb; cc < ce; ++cc) {
      const unsigned x = cst_s[cc];
      tot += x;
      ns += x != 0u && x <= smax;
      nm += x > smax && x <= mmax;
      nl += x > mmax;
    }
    unsigned K2, nsm, nlong;
    unsigned st = block_excl_scan<kSortThreads>(tot, s_part, &K2);
    const unsigned psm = block_excl_scan<kSortThreads>(ns | (nm << 16), s_part, &nsm);
    unsigned sl = block_excl_scan<kSortThreads>(nl, s_part, &nlong);
    const unsigned nshort = nsm & 0xffffu, nmid = nsm >> 16;
    if (tid == 0) {
      s_base[0] = K ? atomicAdd(&a.ctl->n_rec, K) : 0u;
      s_base[1] = nshort ? atomicAdd(&a.ctl->n_seg, nshort) : 0u;
      s_base[2] = nlong ? atomicAdd(&a.ctl->n_lseg, nlong) : 0u;
      s_base[3] = nmid ? atomicAdd(&a.ctl->n_mseg, nmid) : 0u;
    }
    __syncthreads();
    const unsigned rbase = s_base[0], lbase = s_base[2];
    unsigned ss = s_base[1] + (psm & 0xffffu), sm = a.seg_cap + s_base[3] + (psm >> 16);
    // short segments from the front of the list, long ones from its back, mid-size ones in
    // its second half
    for (int cc = cb; cc < ce; ++cc) {
      const unsigned x = cst_s[cc];
      cst_s[cc] = rbase + st;
      if (x) {
        const uint4 sgm = make_uint4((unsigned)(gb + cc), rbase + st, x, 0u);
        if (x <= smax) a.segs[ss++] = sgm;
        else if (x <= mmax) a.segs[sm++] = sgm;
        else a.segs[a.seg_cap - 1 - (lbase + sl++)] = sgm;
      }
      st += x;
    }
  }
  // 5. stable scatter, window by window
  for (int w = 0; w < nwin; ++w) {
    const unsigned p0 = (unsigned)w * kSortCap, n = K - p0 < (unsigned)kSortCap ? K - p0 : (unsigned)kSortCap;
    const unsigned S = ((n + kW - 1) / kW + 31) / 32 * 32;  // window positions per warp
    for (int i = tid; i < kW * ncell; i += kSortThreads) wc_s[i] = 0;
    __syncthreads();
    if (nwin > 1) load_window(p0, n);
    // warp wid ranks the positions [wid*S, (wid+1)*S) in input order
    for (unsigned b0 = wid * S; b0 < (wid + 1) * S && b0 < n; b0 += 32) {
      const unsigned j = b0 + lane;
      const int key = j < n ? (int)(rec_s[j].x & 0xffffu) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      unsigned base = 0u;
      if (key >= 0) base = wc_s[wid * ncell + key];
      __syncwarp();
      if (key >= 0) {
        rank_s[j] = (uint16_t)(base + __popc(peers & lanemask_lt()));
        if (lane == __ffs(peers) - 1) wc_s[wid * ncell + key] = (uint16_t)(base + __popc(peers));
      }
      __syncwarp();
    }
    __syncthreads();
    for (int cc = tid; cc < ncell; cc += kSortThreads) {  // warp bases: exclusive over the warps
      unsigned run = 0u;
#pragma unroll
      for (int ww = 0; ww < kW; ++ww) {
        const unsigned x = wc_s[ww * ncell + cc];
        wc_s[ww * ncell + cc] = (uint16_t)run;
        run += x;
      }
    }
    __syncthreads();
    for (unsigned j = tid; j < n; j += kSortThreads) {
      const uint4 r = rec_s[j];
      const unsigned key = r.x & 0xffffu;
      const unsigned pos = cst_s[key] + wc_s[(j / S) * ncell + key] + rank_s[j];
      __stcg(a.srec + pos, r);
      if (kDebug) {  // the point index of the record (debug outputs only)
        const unsigned p = p0 + j;
        int lo = 0, hi = T - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (tpre_s[mid] <= p) lo = mid; else hi = mid - 1;
        }
        a.sridx[pos] = __ldcg(a.ridx + (long long)(t0 + lo) * kTile + (tcnt_s[lo] & 0xffffu) + (p - tpre_s[lo]));
      }
    }
    __syncthreads();
    if (w + 1 < nwin) {  // the cells' starts move past this window's records
      for (unsigned j = tid; j < n; j += kSortThreads) atomicAdd(&cst_s[rec_s[j].x & 0xffffu], 1u);
      __syncthreads();
    }
  }
}
