// k_accum.cuh -- k_accum: the opt-in bucketed fast path.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_accum (a8 end, a9-a10, lazy a13)
// Bucketed fast path.  Grid-stride over the (map, band) units of the wave (band = 1024 cells,
// 4 per thread).  Per unit: each thread issues the loads of its 4 cells' state (one round trip,
// kept in registers); the band's records (<= kSortCap, the bucket capacity) are counting-sorted
// by cell in shared memory (one native shared atomic per record for the histogram, one for the
// scatter); then each thread sums its cells' records in registers (fp64, no atomics), merges the
// scratch of a spilled band, resets its cells in a scrolled-in strip, fuses its touched cells
// and stores the cells it changed.  The band's state is contiguous: loads and stores coalesce.
constexpr int kAccumPerThread = 4;
constexpr int kBand = kThreads * kAccumPerThread;  // 1024 cells
constexpr int kSortCap = 4096;                     // records sorted per unit (= max bucket capacity)

size_t accum_smem_bytes(int) { return (size_t)kSortCap * sizeof(uint4); }
int accum_sort_cap() { return kSortCap; }

// exclusive prefix sum of cnt[0, kBand) in place (256 threads, 4 consecutive cells each);
// beg[c] receives the same offsets; returns the total
__device__ __forceinline__ unsigned band_scan(unsigned *cnt, unsigned *beg, unsigned *wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c0 = threadIdx.x * kAccumPerThread;
  unsigned v[kAccumPerThread], t = 0;
#pragma unroll
  for (int j = 0; j < kAccumPerThread; ++j) {
    v[j] = t;
    t += cnt[c0 + j];
  }
  unsigned x = t;  // inclusive warp scan of the thread totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  unsigned wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const unsigned ws = wsum[w];
    wbase += w < wid ? ws : 0u;
    total += ws;
  }
  const unsigned base = wbase + x - t;
#pragma unroll
  for (int j = 0; j < kAccumPerThread; ++j) {
    cnt[c0 + j] = base + v[j];
    beg[c0 + j] = base + v[j];
  }
  return total;
}

template <int kFast>
__global__ void __launch_bounds__(kThreads, 2) k_accum(const __grid_constant__ PassArgs a) {
  constexpr int NCH = kFast == 1 ? 3 : 1;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  uint4 *s_rec = reinterpret_cast<uint4 *>(s_dyn);  // [kSortCap] records sorted by cell
  __shared__ unsigned s_cur[kBand];                  // counts -> scatter cursors
  __shared__ unsigned s_beg[kBand + 1];              // first sorted record of each cell
  __shared__ unsigned s_wsum[kThreads / 32];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  const GroupDesc &gd = a.b[0].g;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  uint8_t *obsp = a.st.flags + (long long)gd.flag * BHW;
  const int units = ABLATE(a, 1u) ? 0 : (a.m1 - a.m0) * a.nbands;
  auto key_of = [&](int un) {
    const int mi = un / a.nbands;
    return (a.slot0 + mi) * a.nbands + (un - mi * a.nbands);
  };
  unsigned ntot_next = blockIdx.x < units ? __ldcg(a.bcnt + key_of(blockIdx.x)) : 0u;
  for (int un = blockIdx.x; un < units; un += gridDim.x) {
    const int mi = un / a.nbands, band = un - mi * a.nbands;
    const int m = a.m0 + mi;
    const int key = (a.slot0 + mi) * a.nbands + band;
    const int lo = band * kBand;
    const int ncell = min(kBand, g.HW - lo);
    const long long cbase = (long long)m * g.HW + lo;
    const unsigned ntot = ntot_next;
    const unsigned nrec = min(ntot, a.bcap);  // bcap <= kSortCap (host)
    const uint4 *rp = a.recs + (long long)key * a.bcap;
    // (1) the frame, the next unit's record count; clear the histogram
#pragma unroll
    for (int u = 0; u < kAccumPerThread; ++u) s_cur[u * kThreads + threadIdx.x] = 0u;
    const PointFrame f = frame_of(a, m);
    ntot_next = un + (int)gridDim.x < units ? __ldcg(a.bcnt + key_of(un + gridDim.x)) : 0u;
    __syncthreads();
    // (2) histogram of the records' cells
    for (unsigned r0 = threadIdx.x; r0 < nrec; r0 += 4 * kThreads) {
      unsigned kx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned r = r0 + u * kThreads;
        kx[u] = r < nrec ? __ldcg(reinterpret_cast<const unsigned *>(rp + r)) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (kx[u] != 0xffffffffu) atomicAdd(&s_cur[kx[u] & 0x7fffffffu], 1u);
    }
    __syncthreads();
    // (3) offsets, then the scatter into cell order
    band_scan(s_cur, s_beg, s_wsum);
    if (threadIdx.x == 0) s_beg[kBand] = nrec;
    __syncthreads();
    for (unsigned r0 = threadIdx.x; r0 < nrec; r0 += 4 * kThreads) {
      uint4 rr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned r = r0 + u * kThreads;
        if (r < nrec) rr[u] = __ldcg(rp + r);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r0 + u * kThreads < nrec) s_rec[atomicAdd(&s_cur[rr[u].x & 0x7fffffffu], 1u)] = rr[u];
    }
    if (threadIdx.x == 0) {
      a.bcnt[key] = 0u;  // ready for the next frame
      if (band == 0) a.ring[m] = make_int2(f.r0, f.c0);
    }
    __syncthreads();
    // (4) per cell: sum the sorted records (+ the scratch of a spilled band); then, two cells
    // at a time, one round of state loads for the cells that change (touched or scrolled in),
    // strip reset, fusion, stores
    const bool shift = f.sr != 0 || f.sc != 0;
    const bool spilled = ntot > a.bcap;
    const int sb = spilled ? (int)scratch_base(a, m) : 0;
#pragma unroll
    for (int u0 = 0; u0 < kAccumPerThread; u0 += 2) {
      unsigned nin[2], nout[2], c0[2], c1[2], c2[2];
      double P[2], S[2], X[2];
      bool strip[2], dirty[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int c = (u0 + v) * kThreads + threadIdx.x;
        nin[v] = nout[v] = c0[v] = c1[v] = c2[v] = 0u;
        P[v] = S[v] = X[v] = 0.0;
        strip[v] = dirty[v] = false;
        if (c >= ncell) continue;
        const unsigned e = s_beg[c + 1];
        for (unsigned r = s_beg[c]; r < e; ++r) {
          const uint4 q = s_rec[r];
          if (q.x >> 31) {
            ++nout[v];
          } else {
            ++nin[v];
            P[v] += (double)__uint_as_float(q.y);
            S[v] += (double)__uint_as_float(q.z);
          }
          if (kFast == 1) {  // D20: 0x00RRGGBB, exact integer sums
            c0[v] += (q.w >> 16) & 255u;
            c1[v] += (q.w >> 8) & 255u;
            c2[v] += q.w & 255u;
          } else {  // D31: a non-finite channel skips the group
            const float x = __uint_as_float(q.w);
            if (isfinite(x)) {
              ++c0[v];
              X[v] += (double)x;
            }
          }
        }
        if (spilled) {  // merge (and re-zero) the scratch of this cell
          const unsigned long long cv = __ldcg(a.cnt + sb + lo + c);
          if (cv != 0ull) {
            ulonglong2 *rq = reinterpret_cast<ulonglong2 *>(a.rec + (long long)(sb + lo + c) * 4);
            const ulonglong2 ps = __ldcg(rq), ww = __ldcg(rq + 1);
            P[v] += __longlong_as_double((long long)ps.x);
            S[v] += __longlong_as_double((long long)ps.y);
            if (kFast == 1) {  // colour layout: b | n << 32, [P, S, r | g << 32, n_out]
              nout[v] += (unsigned)ww.y;
              nin[v] += (unsigned)(cv >> 32) - (unsigned)ww.y;
              c0[v] += (unsigned)(ww.x & 0xffffffffull);
              c1[v] += (unsigned)(ww.x >> 32);
              c2[v] += (unsigned)(cv & 0xffffffffull);
            } else {
              nin[v] += (unsigned)(cv & 0xffffffffull);
              nout[v] += (unsigned)(cv >> 32);
              c0[v] += (unsigned)ww.x;
              X[v] += __longlong_as_double((long long)ww.y);
            }
            __stcg(a.cnt + sb + lo + c, 0ull);
            __stcg(rq, make_ulonglong2(0ull, 0ull));
            __stcg(rq + 1, make_ulonglong2(0ull, 0ull));
          }
        }
        if (shift) {  // lazy ring shift: the scrolled-in cells start from the reset state (a13)
          int pcol;
          const int prow = divmod_fast(lo + c, g.W, g.inv_W, pcol);
          int row = prow - f.r0, col = pcol - f.c0;
          row += row < 0 ? g.H : 0;
          col += col < 0 ? g.W : 0;
          strip[v] = in_strip(row, col, f, g);
        }
        // untouched cells outside the strips stay bit-identical
        dirty[v] = strip[v] || (nin[v] + nout[v] != 0u && !ABLATE(a, 512u));
      }
      float h[2], s2[2], th[2][NCH];
      uint8_t vd[2], ob[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {  // one round of loads
        const long long cc = cbase + (u0 + v) * kThreads + threadIdx.x;
        if (!dirty[v] || strip[v]) continue;
        h[v] = elev[cc];
        s2[v] = var[cc];
#pragma unroll
        for (int k = 0; k < NCH; ++k) th[v][k] = vals[(long long)(gd.word0 + k) * BHW + cc];
        vd[v] = validp[cc];
        ob[v] = obsp[cc];
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        if (!dirty[v]) continue;
        const long long cc = cbase + (u0 + v) * kThreads + threadIdx.x;
        if (strip[v]) {
          h[v] = s2[v] = __int_as_float(0x7fc00000);
#pragma unroll
          for (int k = 0; k < NCH; ++k) th[v][k] = 0.0f;
          vd[v] = ob[v] = 0;
        }
        if (nin[v] + nout[v] != 0u && !ABLATE(a, 512u)) {
          ++cnt[7];
          // a9: Kalman height fusion (D7), outliers inflate first (D11); reciprocals (D29b)
          if (vd[v]) {
            const double sp = (double)s2[v] + (double)nout[v] * (double)a.np.v_out;
            if (nin[v] > 0u) {
              const double rden = 1.0 / (1.0 + P[v] * sp);
              h[v] = __double2float_rn(((double)h[v] + S[v] * sp) * rden);
              s2[v] = __double2float_rn(sp * rden);
            } else {
              s2[v] = __double2float_rn(sp);
            }
          } else if (nin[v] > 0u) {
            const double rP = 1.0 / P[v];
            h[v] = __double2float_rn(S[v] * rP);
            s2[v] = __double2float_rn(rP);
            vd[v] = 1;
          }
          // a10: Eq.(1)+(2); colour n = every filtered in-bounds point (D20), average n = finite (D31)
          const unsigned nn = kFast == 1 ? nin[v] + nout[v] : c0[v];
          if (nn != 0u) {
            const double rn = 1.0 / (double)nn;
            if (kFast == 1) {
              th[v][0] = rule_average_r(th[v][0], ob[v] != 0, (double)c0[v], rn, gd.w);
              th[v][1 % NCH] = rule_average_r(th[v][1 % NCH], ob[v] != 0, (double)c1[v], rn, gd.w);
              th[v][2 % NCH] = rule_average_r(th[v][2 % NCH], ob[v] != 0, (double)c2[v], rn, gd.w);
            } else {
              th[v][0] = rule_average_r(th[v][0], ob[v] != 0, X[v], rn, gd.w);
            }
            ob[v] = 1;
          }
        }
        elev[cc] = h[v];
        var[cc] = s2[v];
#pragma unroll
        for (int k = 0; k < NCH; ++k) vals[(long long)(gd.word0 + k) * BHW + cc] = th[v][k];
        validp[cc] = vd[v];
        obsp[cc] = ob[v];
      }
    }
    __syncthreads();  // s_cur / s_beg / s_rec are rewritten by the next unit
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
