// cell_pass.cuh -- a9-a10 device functions: batched per-cell fusion (generic and fast).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- a9-a10, batched
// One lane fuses up to N touched cells (phys[u] >= 0) of map m.  Every phase issues all of its
// loads for the N cells before any math or store (the compiler cannot hoist loads over stores
// to possibly aliasing layers), so a lane keeps N independent round trips in flight.
template <int N>
__device__ __forceinline__ void fuse_cells(const PassArgs &a, int m, int sb, const int (&phys)[N],
                                           const unsigned long long (&cnt)[N]) {
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  int c[N], sc[N];
  unsigned hit = 0;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    c[u] = m * g.HW + phys[u];
    sc[u] = sb + phys[u];
    hit |= phys[u] >= 0 ? (1u << u) : 0u;
  }
  // ---- a9: Kalman height fusion (D7, kalman_height)
  {
    double P[N], S[N];
    float h[N], s2[N];
    uint8_t vd[N];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (!(hit >> u & 1u)) continue;
      const unsigned long long *r = a.rec + (long long)sc[u] * a.R;
      P[u] = __longlong_as_double((long long)__ldcg(r + kRecP));
      S[u] = __longlong_as_double((long long)__ldcg(r + kRecS));
      h[u] = elev[c[u]];
      s2[u] = var[c[u]];
      vd[u] = validp[c[u]];
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (!(hit >> u & 1u)) continue;
      const double n_in = (double)(uint32_t)(cnt[u] & 0xffffffffull);
      const double n_out = (double)(uint32_t)(cnt[u] >> 32);
      {
        float hh = h[u], ss = s2[u];
        uint8_t vv = vd[u];
        kalman_height(hh, ss, vv, n_in, n_out, P[u], S[u], a.np.v_out);
        if (vv) {
          elev[c[u]] = hh;
          var[c[u]] = ss;
          if (!vd[u]) validp[c[u]] = 1;
        }
      }
      unsigned long long *r = a.rec + (long long)sc[u] * a.R;  // re-zero for the slot's next map
      __stcg(a.cnt + sc[u], 0ull);
      __stcg(r + kRecP, 0ull);
      __stcg(r + kRecS, 0ull);
    }
  }
  // ---- a10: each bound group by its rule, batched over the N cells
  for (int bi = 0; bi < a.nb; ++bi) {
    const GroupDesc &gd = a.b[bi].g;
    unsigned long long *ga[N];
#pragma unroll
    for (int u = 0; u < N; ++u) ga[u] = a.rec + (long long)sc[u] * a.R + gd.acc0;
    if (gd.rule == MEM_CLASS_MAX) {  // D19: the frame's winner overwrites (label, conf)
      unsigned long long key[N];
#pragma unroll
      for (int u = 0; u < N; ++u) key[u] = (hit >> u & 1u) ? __ldcg(ga[u]) : 0ull;
#pragma unroll
      for (int u = 0; u < N; ++u) {
        if (key[u] == 0ull) continue;
        reinterpret_cast<int *>(a.st.words)[(long long)gd.label * BHW + c[u]] =
            gd.nch - 1 - (int)(uint32_t)(key[u] & 0xffffffffull);
        vals[(long long)gd.word0 * BHW + c[u]] = f32_of_ord((uint32_t)(key[u] >> 32));
        __stcg(ga[u], 0ull);
      }
      continue;
    }
    uint8_t *obsp = a.st.flags + (long long)gd.flag * BHW;
    unsigned long long w0[N], w1[N];  // count (or color r|g<<32) and color b|n<<32
    unsigned obs = 0, any = 0;
#pragma unroll
    for (int u = 0; u < N; ++u) {
      w0[u] = w1[u] = 0ull;
      if (!(hit >> u & 1u)) continue;
      w0[u] = __ldcg(ga[u]);
      if (gd.rule == MEM_COLOR) w1[u] = __ldcg(ga[u] + 1);
      obs |= obsp[c[u]] ? (1u << u) : 0u;
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const unsigned long long nn = gd.rule == MEM_COLOR ? (w1[u] >> 32) : w0[u];
      any |= nn != 0ull ? (1u << u) : 0u;
    }
    for (int k = 0; k < gd.nch; ++k) {
      double sum[N];
      float th[N], th2[N];
#pragma unroll
      for (int u = 0; u < N; ++u) {  // loads for channel k of every cell first
        if (!(any >> u & 1u)) continue;
        if (gd.rule == MEM_COLOR) {
          const uint32_t v = k == 0 ? (uint32_t)(w0[u] & 0xffffffffull) : k == 1 ? (uint32_t)(w0[u] >> 32)
                                                                          : (uint32_t)(w1[u] & 0xffffffffull);
          sum[u] = (double)v;  // exact integer colour sums (D20)
        } else {
          sum[u] = __longlong_as_double((long long)__ldcg(ga[u] + 1 + k));
        }
        th[u] = vals[(long long)(gd.word0 + k) * BHW + c[u]];
        if (gd.rule == MEM_GAUSSIAN) th2[u] = vals[(long long)(gd.word0 + gd.nch + k) * BHW + c[u]];
      }
#pragma unroll
      for (int u = 0; u < N; ++u) {
        if (!(any >> u & 1u)) continue;
        const double n = (double)(gd.rule == MEM_COLOR ? (w1[u] >> 32) : w0[u]);
        const bool ob = obs >> u & 1u;
        float *dst = vals + (long long)(gd.word0 + k) * BHW + c[u];
        switch (gd.rule) {
          case MEM_AVERAGE:
          case MEM_CLASS_AVERAGE:
          case MEM_COLOR: *dst = rule_average(th[u], ob, sum[u], n, gd.w); break;
          case MEM_GAUSSIAN: {
            float mu = th[u], vv = th2[u];
            rule_gaussian(mu, vv, ob, sum[u], n, gd);
            *dst = mu;
            vals[(long long)(gd.word0 + gd.nch + k) * BHW + c[u]] = vv;
            break;
          }
          case MEM_CLASS_BAYESIAN: *dst = rule_dirichlet(th[u], ob, sum[u], gd.a0); break;
          default: break;
        }
        if (gd.rule != MEM_COLOR) __stcg(ga[u] + 1 + k, 0ull);
      }
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (!(any >> u & 1u)) continue;
      obsp[c[u]] = 1;
      __stcg(ga[u], 0ull);
      if (gd.rule == MEM_COLOR) __stcg(ga[u] + 1, 0ull);
    }
  }
}

// Fast path of fuse_cells for the common configuration "one average or colour group with
// nch <= 3 channels bound" (C1, C2, C5a): every load of a cell (scratch record, h, s2, valid,
// observed, theta_k) is issued in ONE round for both cells before any math or store.
template <int N, int NCH, bool kColor>
__device__ __forceinline__ void fuse_cells_avg(const PassArgs &a, int m, int sb, const int (&phys)[N],
                                               const unsigned long long (&cnt)[N]) {
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  const GroupDesc &gd = a.b[0].g;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  uint8_t *obsp = a.st.flags + (long long)gd.flag * BHW;
  double P[N], S[N], sum[N][NCH];
  unsigned long long w0[N], w1[N];
  float h[N], s2[N], th[N][NCH];
  uint8_t vd[N], ob[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {  // one round of loads
    if (phys[u] < 0) continue;
    const int c = m * g.HW + phys[u];
    // the record is [P, S, w0, w1] (colour: r|g<<32, b|n<<32; average: count, sum): 2 x 16 B
    const ulonglong2 *r = reinterpret_cast<const ulonglong2 *>(a.rec + (long long)(sb + phys[u]) * 4);
    const ulonglong2 ps = __ldcg(r), ww = __ldcg(r + 1);
    P[u] = __longlong_as_double((long long)ps.x);
    S[u] = __longlong_as_double((long long)ps.y);
    w0[u] = ww.x;
    w1[u] = ww.y;
    if (!kColor) sum[u][0] = __longlong_as_double((long long)ww.y);
    h[u] = elev[c];
    s2[u] = var[c];
    vd[u] = validp[c];
    ob[u] = obsp[c];
#pragma unroll
    for (int k = 0; k < NCH; ++k) th[u][k] = vals[(long long)(gd.word0 + k) * BHW + c];
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (phys[u] < 0) continue;
    const int c = m * g.HW + phys[u];
    unsigned long long *r = a.rec + (long long)(sb + phys[u]) * 4;
    // a9: Kalman height fusion (D7), outliers inflate first (D11).  Colour layout: count word
    // b | n << 32, record [P, S, r | g << 32, n_out] (n_in > 0 iff P > 0)
    const double n_in = kColor ? (P[u] > 0.0 ? 1.0 : 0.0) : (double)(uint32_t)(cnt[u] & 0xffffffffull);
    const double n_out = kColor ? (double)w1[u] : (double)(uint32_t)(cnt[u] >> 32);
    {
      float hh = h[u], ss = s2[u];
      uint8_t vv = vd[u];
      kalman_height(hh, ss, vv, n_in, n_out, P[u], S[u], a.np.v_out);
      if (vv) {
        elev[c] = hh;
        var[c] = ss;
        if (!vd[u]) validp[c] = 1;
      }
    }
    // a10: Eq.(1)+(2) per channel
    const unsigned long long nn = kColor ? (cnt[u] >> 32) : w0[u];
    if (nn != 0ull) {
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        double sk;
        if (kColor) {
          const uint32_t v = k == 0 ? (uint32_t)(w0[u] & 0xffffffffull)
                                    : k == 1 ? (uint32_t)(w0[u] >> 32) : (uint32_t)(cnt[u] & 0xffffffffull);
          sk = (double)v;  // exact integer colour sums (D20)
        } else {
          sk = sum[u][k];
        }
        vals[(long long)(gd.word0 + k) * BHW + c] = rule_average(th[u][k], ob[u] != 0, sk, (double)nn, gd.w);
      }
      obsp[c] = 1;
    }
    // re-zero the scratch for the slot's next map (fast-path records are 4 words, 32 B)
    __stcg(a.cnt + sb + phys[u], 0ull);
    __stcg(reinterpret_cast<ulonglong2 *>(r), make_ulonglong2(0ull, 0ull));
    __stcg(reinterpret_cast<ulonglong2 *>(r) + 1, make_ulonglong2(0ull, 0ull));
  }
}

// scratch cell base of map m of this wave: its map-slot in the wave's half of the pool
__device__ __forceinline__ long long scratch_base(const PassArgs &a, int m) {
  return (long long)(a.slot0 + m - a.m0) * a.geo.HW;
}

// per-lane code counters packed in one u64: 10 bits per code, flushed before they can wrap
__device__ __forceinline__ void count_code(unsigned long long &packed, unsigned &n, int code, unsigned (&cnt)[8]) {
  if (code >= 0) packed += 1ull << (10 * code);
  if (++n == 1000u) {
#pragma unroll
    for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
    packed = 0ull;
    n = 0;
  }
}

// per-CTA counters: warp reduce, one smem add per warp, one global add per counter
__device__ __forceinline__ void flush_stats(unsigned *s_cnt, const unsigned (&cnt)[8], unsigned long long *out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const unsigned v = __reduce_add_sync(0xffffffffu, cnt[c]);
    if (lane == 0 && v) atomicAdd(&s_cnt[c], v);
  }
  __syncthreads();
  if (threadIdx.x < 8 && s_cnt[threadIdx.x])
    atomicAdd(&out[(blockIdx.x % kStatSlots) * 8 + threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}
