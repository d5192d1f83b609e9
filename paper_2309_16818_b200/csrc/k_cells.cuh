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
  uint4 ce[N];
  float h[N], s2[N], th[N][NCH > 0 ? NCH : 1];
  uint8_t vd[N], ob[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {  // one round of loads
    if (phys[u] < 0) continue;
    const int c = m * g.HW + phys[u];
    const ulonglong2 *r = reinterpret_cast<const ulonglong2 *>(a.rec + (long long)c * 4);
    const ulonglong2 ps = __ldcg(r), ww = __ldcg(r + 1);
    P[u] = __longlong_as_double((long long)ps.x);
    S[u] = __longlong_as_double((long long)ps.y);
    w0[u] = ww.x;
    w1[u] = ww.y;
    ce[u] = __ldcg(reinterpret_cast<const uint4 *>(a.cert) + c);
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
    // counts: colour count word b | n << 32 with n_out in the record, else n_in | n_out << 32
    const unsigned n_out = kFast == 1 ? (unsigned)w1[u] : (unsigned)(cnt[u] >> 32);
    const unsigned n_in = kFast == 1 ? (unsigned)(cnt[u] >> 32) - n_out : (unsigned)(cnt[u] & 0xffffffffull);
    const unsigned ng = kFast == 1 ? (unsigned)(cnt[u] >> 32) : kFast == 2 ? (unsigned)w0[u] : 0u;
    const bool ok = cert_ok(make_uint2(ce[u].x, ce[u].y), n_in) && (kFast != 2 || cert_ok(make_uint2(ce[u].z, ce[u].w), ng));
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
                                      : k == 1 ? (uint32_t)(w0[u] >> 32) : (uint32_t)(cnt[u] & 0xffffffffull);
            sk = (double)v;  // exact integer colour sums (D20)
          } else {
            sk = __longlong_as_double((long long)w1[u]);
          }
          vals[(long long)(gd.word0 + k) * BHW + c] = rule_average(th[u][k], ob[u] != 0, sk, (double)ng, gd.w);
        }
        if (!ob[u]) a.st.flags[(long long)gd.flag * BHW + c] = 1;
      }
    } else {  // uncertified: recomputed in input order by k_refold
      const unsigned k = atomicAdd(&a.ctl->n_fb, 1u);
      a.fb[k] = (long long)c;
    }
    // re-zero the scratch for the next point input
    unsigned long long *r = a.rec + (long long)c * 4;
    __stcg(a.cnt + c, 0ull);
    __stcg(reinterpret_cast<ulonglong2 *>(r), make_ulonglong2(0ull, 0ull));
    __stcg(reinterpret_cast<ulonglong2 *>(r) + 1, make_ulonglong2(0ull, 0ull));
    __stcg(reinterpret_cast<uint4 *>(a.cert) + c, make_uint4(0u, 0u, 0u, 0u));
  }
}

// ---------------------------------------------------------------- k_cells (a9-a10, lazy a13)
constexpr int kChunkPerLane = 4;                 // cells per lane per chunk
constexpr int kChunk = 32 * kChunkPerLane;        // 128-cell chunk per warp

// Warp-persistent grid-stride over 128-cell chunks of the call's maps (newest map first: its
// scratch was touched last by k_points and is still in L2).  Each warp, independently of the
// others (no CTA barrier): 4 count loads per lane in flight, the pending shift strips reset,
// its touched cells compacted in its own shared-memory slice, then fused 2 per lane per round.
template <int kFast>
__global__ void __launch_bounds__(kThreads, 3) k_cells(const __grid_constant__ PassArgs a) {
  __shared__ int s_phys[kThreads / 32][kChunk];
  __shared__ unsigned long long s_cntv[kThreads / 32][kChunk];
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
  const int cpm = (a.cell_hi - a.cell_lo + kChunk - 1) / kChunk;  // chunks per map (band)
  const int total = a.n_maps * cpm;
  int *sp = s_phys[wid];
  unsigned long long *sc = s_cntv[wid];
  for (int rt = gw; rt < total; rt += nwarps) {
    const int chunk = total - 1 - rt;
    const int m = chunk / cpm;
    const int t0 = a.cell_lo + (chunk - m * cpm) * kChunk;
    const int sb = m * g.HW;
    unsigned long long cv[kChunkPerLane];
#pragma unroll
    for (int u = 0; u < kChunkPerLane; ++u) {  // counts first (memory-level parallelism)
      const int phys = t0 + u * 32 + lane;
      cv[u] = phys < a.cell_hi ? __ldcg(a.cnt + sb + phys) : 0ull;
    }
    const PointFrame f = frame_of(a, m);
    if (t0 == a.cell_lo && lane == 0) a.ring[m] = make_int2(f.r0, f.c0);
    int n = 0;
#pragma unroll
    for (int u = 0; u < kChunkPerLane; ++u) {
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
// The cells k_cells could not certify (their fp64 sums might depend on the order of the REDs):
// one CTA per listed cell walks its map's points in input order, 256 at a time -- a2-a7 for each
// (bin_point, the Mahalanobis test against the pre-frame state, which k_cells left untouched)
// -- compacts the points of the cell in order (ballots and a block scan) and folds their terms
// sequentially in fp64, exactly as the oracle does; then a9 + a10 (fuse_state).  A rare path:
// the certificate fails only when a cell's terms span more than ~29 binades minus log2(n).
template <int kFast>
__global__ void __launch_bounds__(kThreads) k_refold(const __grid_constant__ PassArgs a) {
  __shared__ float s_z[kThreads], s_v[kThreads], s_c[kThreads];
  __shared__ unsigned s_part[kThreads / 32];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Geometry &g = a.geo;
  const unsigned nfb = *(volatile unsigned *)&a.ctl->n_fb;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  for (unsigned k = blockIdx.x; k < nfb; k += gridDim.x) {
    const long long gc = __ldcg(a.fb + k);
    const int m = (int)(gc / g.HW), phys = (int)(gc - (long long)m * g.HW);
    const PointFrame f = frame_of(a, m);
    const long long beg = off_of(a, m), end = off_of(a, m + 1);
    const float h = __ldcg(vals + (long long)kWordElev * g.BHW + gc), s2 = __ldcg(vals + (long long)kWordVar * g.BHW + gc);
    double P = 0.0, S = 0.0, X = 0.0;
    unsigned nin = 0u, nout = 0u, cr = 0u, cg = 0u, cb = 0u, na = 0u;
    for (long long b0 = beg; b0 < end; b0 += kThreads) {
      const long long i = b0 + threadIdx.x;
      bool in = false;
      float z = 0.0f, v = 0.0f, ch = 0.0f;
      if (i < end) {
        const float *p = a.pts + i * (long long)a.stride;
        const PointOut o = bin_point(__ldg(p), __ldg(p + 1), __ldg(p + 2), f, g, a.np, 0, a.r2lo, a.r2hi);
        if (o.cell == phys) {
          in = true;
          z = o.z;
          v = o.v;
          if (kFast != 0) ch = __ldg(p + 3);
        }
      }
      unsigned tot;
      const unsigned pos = block_excl_scan<kThreads>(in ? 1u : 0u, s_part, &tot);
      if (in) {
        s_z[pos] = z;
        s_v[pos] = v;
        s_c[pos] = ch;
      }
      __syncthreads();
      if (threadIdx.x == 0) {  // the oracle's per-point loop, in input order
        for (unsigned j = 0; j < tot; ++j) {
          const float zj = s_z[j], vj = s_v[j];
          const float d = zj - h;  // a7 (D10)
          if (d * d > a.np.tau2 * (s2 + vj)) {
            ++nout;
          } else {
            ++nin;
            const float w = 1.0f / vj;
            P += (double)w;
            S += (double)(zj * w);
          }
          if (kFast == 1) {
            const uint32_t bits = __float_as_uint(s_c[j]);
            cr += (bits >> 16) & 255u;
            cg += (bits >> 8) & 255u;
            cb += bits & 255u;
            ++na;
          } else if (kFast == 2 && isfinite(s_c[j])) {
            ++na;
            X += (double)s_c[j];
          }
        }
      }
      __syncthreads();
    }
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
                                         nin, nout, P, S, cr, cg, cb, na, X);
    }
    __syncthreads();
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
