// kernels.cu -- the sm_100a kernels of the MEM hot path.
//
//   k_points a2-a8  persistent grid-stride over 128-point warp-items of one wave of maps:
//                   coalesced float4 loads (4 in flight per lane), filters, transform, bin,
//                   noise, one batched state gather for the Mahalanobis test, and
//                   warp-aggregated native 64-bit REDs into L2-resident per-cell scratch
//   k_cells  a9-a10 + lazy a13  grid-stride over 128-cell warp-items of the same wave: strip
//                   reset of a pending shift, Kalman height fusion, per-group rules (fp64),
//                   re-zero the scratch.  k_cells(w) runs on a side stream concurrently with
//                   k_points(w+1); waves alternate between the two halves of the scratch pool.
//   k_image  a11-a12  one thread per valid cell: project, frustum, gather, fuse (N_j = 1)
//   k_shift  a13      eager strip reset (only when a shift cannot be folded into k_fused)
//   k_read   a14      unroll the ring into logical row-major fp32, derive theta / NaN
//   k_write           the inverse of k_read (state injection for single-step parity)
//
// Everything is stream-ordered; no kernel synchronises the host.
#include <cmath>

#include "kernels.cuh"

#ifndef MEM_POINTS_MINB
#define MEM_POINTS_MINB 3  // resident CTAs per SM the register allocation of k_points targets
#endif
#ifndef MEM_PAIR_MIN
#define MEM_PAIR_MIN 4  // colour fast path: pair lanes of the same cell when >= this many repeat
#endif
#ifndef MEM_OCC_BATCH
#define MEM_OCC_BATCH 4  // occlusion walk: intermediate cells whose loads are issued together
#endif
#ifndef MEM_CELLS_MINB
#define MEM_CELLS_MINB 3
#endif

namespace memk {

// ---------------------------------------------------------------- programmatic dependent launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- memory helpers
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// read-once point data: no L1 allocation, evict-first in L2 so the scratch of the maps in
// flight keeps its L2 residency
__device__ __forceinline__ float4 ld_stream_f4(const float *p, unsigned long long pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ bool finite3(float a, float b, float c) { return isfinite(a) && isfinite(b) && isfinite(c); }

__device__ __forceinline__ int stat_slot(int code) {
  // mem_stats order: n_input, nonfinite, range, height, oob, inlier, outlier, touched
  return code == MEM_CODE_INLIER ? 5 : code == MEM_CODE_OUTLIER ? 6 : code - 1;
}

// is logical cell (row, col) in the strips that scrolled in with the pending shift (D14)?
template <class F>
__device__ __forceinline__ bool in_strip(int row, int col, const F &f, const Geometry &g) {
  if (f.sr == 0 && f.sc == 0) return false;
  const int ar = f.sr < 0 ? -f.sr : f.sr, ac = f.sc < 0 ? -f.sc : f.sc;
  if (ar >= g.H || ac >= g.W) return true;
  const bool rs = f.sr > 0 ? row >= g.H - f.sr : row < -f.sr;
  const bool cs = f.sc > 0 ? col >= g.W - f.sc : col < -f.sc;
  return rs || cs;
}

// the state of a never-observed cell (D15)
__device__ __forceinline__ void reset_cell(const State &st, long long BHW, long long cell, const ResetInfo &r) {
  float *vals = reinterpret_cast<float *>(st.words);
  vals[(long long)kWordElev * BHW + cell] = __int_as_float(0x7fc00000);
  vals[(long long)kWordVar * BHW + cell] = __int_as_float(0x7fc00000);
  for (int w = 2; w < r.n_word; ++w) st.words[(long long)w * BHW + cell] = 0u;
  for (int l = 0; l < r.n_label; ++l) reinterpret_cast<int *>(st.words)[(long long)r.label_word[l] * BHW + cell] = -1;
  for (int fl = 0; fl < r.n_flag; ++fl) st.flags[(long long)fl * BHW + cell] = 0;
}

// ---------------------------------------------------------------- a2-a8 for one point
struct PointOut {
  int code;
  int lcell;        // logical row*W+col, -1 if dropped
  int cell;         // global physical cell m*HW + phys, -1 if dropped
  float z, v;
  bool test;        // in the window and not in a scrolled-in strip: Mahalanobis test applies
};

// a2-a6 for one point: no memory access (the state gather of a7 is batched by the caller)
__device__ __forceinline__ PointOut bin_point(float px, float py, float pz, const PointFrame &f, const Geometry &g,
                                              const mem_noise &np, float rmin2, float rmax2, int map_base) {
  PointOut o;
  o.code = MEM_CODE_NONFINITE;
  o.lcell = -1;
  o.cell = -1;
  o.z = 0.0f;
  o.v = 0.0f;
  o.test = false;
  if (!finite3(px, py, pz)) return o;                   // a2: finiteness
  const float r2 = (px * px + py * py) + pz * pz;       // a2: sensor-frame range on r^2 (D9)
  if (!(rmin2 <= r2 && r2 <= rmax2)) {
    o.code = MEM_CODE_RANGE;
    return o;
  }
  // a3: q = R p, fixed order, no FMA ("point trsf.")
  const float qx = (f.R[0] * px + f.R[1] * py) + f.R[2] * pz;
  const float qy = (f.R[3] * px + f.R[4] * py) + f.R[5] * pz;
  const float qz = (f.R[6] * px + f.R[7] * py) + f.R[8] * pz;
  if (!(np.h_min <= qz && qz <= np.h_max)) {             // a4: height filter (D9)
    o.code = MEM_CODE_HEIGHT;
    return o;
  }
  const float x = qx + f.t[0], y = qy + f.t[1];
  o.z = qz + f.t[2];
  const float fr = x * g.inv_res + g.hH;                 // a5: bin (D13)
  const float fc = y * g.inv_res + g.hW;
  if (!(0.0f <= fr && fr < (float)g.H && 0.0f <= fc && fc < (float)g.W)) {
    o.code = MEM_CODE_OOB;
    return o;
  }
  const int row = (int)floorf(fr), col = (int)floorf(fc);
  o.lcell = row * g.W + col;
  o.cell = map_base + wrap(row + f.r0, g.H) * g.W + wrap(col + f.c0, g.W);
  o.v = np.a + np.b * r2;                                // a6: noise variance (D8)
  o.code = MEM_CODE_INLIER;                              // a7 decided after the gather
  o.test = !in_strip(row, col, f, g);                    // scrolled-in cells are fresh (invalid)
  return o;
}

// a7 for a batch of points: issue every state gather first (one round trip), then decide.
// The valid flag is not read: an invalid cell always holds a NaN variance (reset_cell, and
// k_write keeps it so for state written through mem_set_layer), and a NaN h or s2 makes the
// comparison false -- exactly the oracle's "no test on an invalid cell" (D10); a valid cell
// whose h or s2 was set to NaN compares false in the oracle too.
template <int N>
__device__ __forceinline__ void mahalanobis(PointOut (&o)[N], const State &st, const Geometry &g, float tau2) {
  const float *elev = reinterpret_cast<const float *>(st.words) + (long long)kWordElev * g.BHW;
  const float *var = reinterpret_cast<const float *>(st.words) + (long long)kWordVar * g.BHW;
  float hv[N], sv[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    hv[u] = sv[u] = __int_as_float(0x7fc00000);
    if (o[u].test) {
      hv[u] = elev[o[u].cell];
      sv[u] = var[o[u].cell];
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
__device__ __forceinline__ void red_max_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- warp aggregation
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Segmented reduction over the lanes of `peers` (the lanes holding the same cell): the lowest
// lane of each peer group ends with the group's total.  Tree over the rank within the group:
// ceil(log2(group size)) rounds, every lane participates in every shuffle (after E. Westphal,
// "warp-aggregated atomics").  `Op` is + or max.
template <class T, class Op>
__device__ __forceinline__ T reduce_peers(unsigned peers, T x, Op op) {
  const int lane = threadIdx.x & 31;
  unsigned rel = (unsigned)__popc(peers & lanemask_lt());
  unsigned rest = peers & ~(lanemask_lt() | (1u << lane));  // peers above me
  while (__any_sync(0xffffffffu, rest != 0u)) {
    const int next = __ffs(rest);
    const T t = __shfl_sync(0xffffffffu, x, next > 0 ? next - 1 : lane);
    if (next) x = op(x, t);
    rest &= ~__ballot_sync(0xffffffffu, rel & 1u);  // odd ranks are folded into their neighbour
    rel >>= 1;
  }
  return x;
}

struct OpAdd {
  template <class T>
  __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a > b ? a : b; }
};

// NEXT-2 (reading D38): the k (id, p) pairs of one point / pixel, `step` floats apart, seen as
// the dense K + 1 class vector dense[id_j] += p_j, dense[K] = 1 - sum p_j (fp32, pair order)
struct TopK {
  const float *ch;
  long long step;
  int k, K;
  __device__ float id(int j) const { return __ldg(ch + (long long)(2 * j) * step); }
  __device__ float p(int j) const { return __ldg(ch + (long long)(2 * j + 1) * step); }
  __device__ bool ok() const {  // every value finite, every id an integer in [0, K)
    for (int j = 0; j < k; ++j) {
      const float i = id(j), q = p(j);
      if (!isfinite(i) || !isfinite(q) || i != floorf(i) || i < 0.0f || i >= (float)K) return false;
    }
    return true;
  }
  __device__ float value(int c) const {
    float v = 0.0f;
    if (c == K) {
      for (int j = 0; j < k; ++j) v += p(j);
      return 1.0f - v;
    }
    for (int j = 0; j < k; ++j)
      if ((int)id(j) == c) v += p(j);
    return v;
  }
  __device__ bool first(int j) const {  // id(j) does not occur among the earlier pairs
    for (int i = 0; i < j; ++i)
      if (id(i) == id(j)) return false;
    return true;
  }
  __device__ unsigned long long key() const {  // D19 class_max key of the dense vector
    int best = 0;
    float bv = value(0);
    for (int c = 1; c <= K; ++c) {
      const float v = value(c);
      if (v > bv) {
        bv = v;
        best = c;
      }
    }
    return ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(K - best);
  }
};

// a8: scatter-accumulate the sufficient statistics of the warp's current points (one per lane,
// `o.cell < 0` = dropped) into their scratch cells `sc`.  Lanes hitting the same cell are
// combined first (__match_any_sync + reduce_peers) so that one lane issues the REDs of the
// group: fewer L2 atomics, no same-address serialisation.  All 32 lanes must call this.
// kFast (stride-4 points, one group bound): 1 = colour, 2 = 1-channel average; 0 = generic
template <int kFast>
__device__ __forceinline__ void accumulate_warp(const PassArgs &a, const PointOut &o, int sc, const float *p,
                                                float ch0) {
  unsigned long long *rec = a.rec + (long long)sc * a.R;
  const bool act = o.cell >= 0;
  const unsigned act_b = __ballot_sync(0xffffffffu, act);
  if (act_b == 0u) return;
  const int lane = threadIdx.x & 31;
  const unsigned key = act ? (unsigned)sc : 0xffffffffu;
  // aggregate only when it pays: >= 16 lanes repeat their neighbour's cell (dense clouds; a
  // LiDAR scan line has ~1.5 points per cell and is faster with one RED set per lane)
  const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned dup = __ballot_sync(0xffffffffu, act && lane > 0 && prev == key);
  const bool agg = __popc(dup) >= 16 && !(a.ablate & 64u);
  const unsigned peers = agg ? __match_any_sync(0xffffffffu, key) : (1u << lane);
  const bool single = !agg;
  const bool leader = act && (__ffs(peers) - 1 == lane);
  const bool inl = act && o.code == MEM_CODE_INLIER;
  const unsigned in_b = __ballot_sync(0xffffffffu, inl);
  // height statistics (inliers): n_in | n_out << 32, sum 1/v, sum z/v
  double w = 0.0, zw = 0.0;
  if (inl) {
    const float wf = 1.0f / o.v;
    w = (double)wf;
    zw = (double)(o.z * wf);
  }
  if (!single) {
    w = reduce_peers(peers, w, OpAdd());
    zw = reduce_peers(peers, zw, OpAdd());
  }
  if constexpr (kFast == 1) {
    // colour fast path, 4 REDs per inlier instead of 5: count word
    // b | n << 32 (n = every filtered in-bounds point, D20; n > 0 marks the cell touched),
    // record [P, S, r | g << 32, n_out]; n_in > 0 iff P > 0 (every 1/v > 0)
    unsigned rg = 0u, bb = 0u;
    if (act) {
      const uint32_t bits = __float_as_uint(ch0);
      rg = ((bits >> 16) & 255u) | (((bits >> 8) & 255u) << 16);
      bb = bits & 255u;
    }
    unsigned n_in = (unsigned)__popc(peers & in_b), n_all = (unsigned)__popc(peers);
    bool lead = leader;
    if (!single) {
      rg = reduce_peers(peers, rg, OpAdd());
      bb = reduce_peers(peers, bb, OpAdd());
    } else if (__popc(dup) >= MEM_PAIR_MIN && !(a.ablate & 64u)) {
      // a LiDAR scan line puts ~30% of its in-window points in the cell of the previous
      // lane: the head of each run absorbs its successor (one shuffle per value), so such
      // a pair costs one set of REDs
      const bool fol = dup >> lane & 1u;
      const bool prev_fol = lane > 0 && (dup >> (lane - 1) & 1u);
      const bool absorbed = fol && !prev_fol;
      const bool absorbs = !fol && lane < 31 && (dup >> (lane + 1) & 1u);
      const double w2 = __shfl_down_sync(0xffffffffu, w, 1), zw2 = __shfl_down_sync(0xffffffffu, zw, 1);
      const unsigned rg2 = __shfl_down_sync(0xffffffffu, rg, 1), bb2 = __shfl_down_sync(0xffffffffu, bb, 1);
      if (absorbs) {
        w += w2;
        zw += zw2;
        rg += rg2;
        bb += bb2;
        n_all = 2;
        n_in += in_b >> (lane + 1) & 1u;
      }
      lead = act && !absorbed;
    }
    if (lead) {
      red_add_u64(&a.cnt[sc], (unsigned long long)bb | ((unsigned long long)n_all << 32));
      if (n_in) {
        red_add_f64(rec + kRecP, w);
        red_add_f64(rec + kRecS, zw);
      }
      red_add_u64(rec + 2, (unsigned long long)(rg & 0xffffu) | ((unsigned long long)(rg >> 16) << 32));
      if (n_all != n_in) red_add_u64(rec + 3, (unsigned long long)(n_all - n_in));
    }
    return;
  }
  if (leader) {
    const unsigned n_in = (unsigned)__popc(peers & in_b), n_all = (unsigned)__popc(peers);
    red_add_u64(&a.cnt[sc], (unsigned long long)n_in | ((unsigned long long)(n_all - n_in) << 32));
    if (n_in) {
      red_add_f64(rec + kRecP, w);
      red_add_f64(rec + kRecS, zw);
    }
  }
  if constexpr (kFast != 0) {  // one group, channel in ch0 (the float4's w)
    unsigned long long *ga = rec + a.b[0].g.acc0;
    {  // Eq.(1) sums of one channel; non-finite values skip the group (D31)
      const bool fin = act && isfinite(ch0);
      double v = fin ? (double)ch0 : 0.0;
      unsigned ng = fin ? 1u : 0u;
      if (!single) {
        ng = (unsigned)__popc(peers & __ballot_sync(0xffffffffu, fin));
        v = reduce_peers(peers, v, OpAdd());
      }
      if (leader && ng) {
        red_add_u64(ga, (unsigned long long)ng);
        red_add_f64(ga + 1, v);
      }
    }
  } else {
  for (int bi = 0; bi < a.nb; ++bi) {  // every filtered in-bounds point feeds the groups (D12)
    const BindDesc &b = a.b[bi];
    unsigned long long *ga = rec + b.g.acc0;
    const float *ch = p + 3 + b.ch_offset;
    if (b.topk > 0) {  // top-k pairs (D38): per-lane REDs of the expanded vector's non-zero classes
      const TopK tk{ch, 1, b.topk, b.g.nch - 1};
      if (!act || !tk.ok()) continue;
      if (b.g.rule == MEM_CLASS_MAX) {
        red_max_u64(ga, tk.key());
        continue;
      }
      red_add_u64(ga, 1ull);
      for (int j = 0; j < tk.k; ++j)
        if (tk.first(j)) red_add_f64(ga + 1 + (int)tk.id(j), (double)tk.value((int)tk.id(j)));
      red_add_f64(ga + 1 + tk.K, (double)tk.value(tk.K));
      continue;
    }
    if (b.g.rule == MEM_COLOR) {  // D20: packed 0x00RRGGBB; exact integer sums
      unsigned rg = 0u, bb = 0u;  // r | g << 16 (a warp sums <= 32 * 255 per channel)
      if (act) {
        const uint32_t bits = __float_as_uint(a.vec4 ? ch0 : ch[0]);
        rg = ((bits >> 16) & 255u) | (((bits >> 8) & 255u) << 16);
        bb = bits & 255u;
      }
      if (!single) {
        rg = reduce_peers(peers, rg, OpAdd());
        bb = reduce_peers(peers, bb, OpAdd());
      }
      if (leader) {
        red_add_u64(ga, (unsigned long long)(rg & 0xffffu) | ((unsigned long long)(rg >> 16) << 32));
        red_add_u64(ga + 1, (unsigned long long)bb | ((unsigned long long)__popc(peers) << 32));
      }
      continue;
    }
    bool fin = act;
    if (act) {
      if (a.vec4) {
        fin = isfinite(ch0);
      } else {
        for (int k = 0; k < b.nch; ++k) fin &= (bool)isfinite(ch[k]);
      }
    }
    const unsigned fin_b = __ballot_sync(0xffffffffu, fin);  // D31: non-finite channels skip the group
    if ((fin_b & act_b) == 0u) continue;
    if (b.g.rule == MEM_CLASS_MAX) {  // D19: (conf, lowest index) as one u64 max
      unsigned long long kv = 0ull;
      if (fin) {
        int best = 0;
        float bv = ch[0];
        for (int k = 1; k < b.nch; ++k) {
          const float c = ch[k];
          if (c > bv) {
            bv = c;
            best = k;
          }
        }
        kv = ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
      }
      if (!single) kv = reduce_peers(peers, kv, OpMax());
      if (leader && kv) red_max_u64(ga, kv);
      continue;
    }
    const unsigned ng = (unsigned)__popc(peers & fin_b);
    if (leader && ng) red_add_u64(ga, (unsigned long long)ng);
    for (int k = 0; k < b.nch; ++k) {
      double v = fin ? (double)(a.vec4 ? ch0 : ch[k]) : 0.0;
      if (!single) v = reduce_peers(peers, v, OpAdd());
      if (leader && ng) red_add_f64(ga + 1 + k, v);
    }
  }
  }
}

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
  // ---- a9: Kalman height fusion (D7: h' = (h + S sp)/(1 + P sp), s2' = sp/(1 + P sp))
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
      if (vd[u]) {
        const double sp = (double)s2[u] + n_out * (double)a.np.v_out;  // outliers inflate first (D11)
        if (n_in > 0.0) {
          const double den = 1.0 + P[u] * sp;
          elev[c[u]] = __double2float_rn(((double)h[u] + S[u] * sp) / den);
          var[c[u]] = __double2float_rn(sp / den);
        } else {
          var[c[u]] = __double2float_rn(sp);
        }
      } else if (n_in > 0.0) {  // first touch: h = S/P, s2 = 1/P
        elev[c[u]] = __double2float_rn(S[u] / P[u]);
        var[c[u]] = __double2float_rn(1.0 / P[u]);
        validp[c[u]] = 1;
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
    if (vd[u]) {
      const double sp = (double)s2[u] + n_out * (double)a.np.v_out;
      if (n_in > 0.0) {  // one fp64 division, two multiplies (reading D29b)
        const double rden = 1.0 / (1.0 + P[u] * sp);
        elev[c] = __double2float_rn(((double)h[u] + S[u] * sp) * rden);
        var[c] = __double2float_rn(sp * rden);
      } else {
        var[c] = __double2float_rn(sp);
      }
    } else if (n_in > 0.0) {
      const double rP = 1.0 / P[u];
      elev[c] = __double2float_rn(S[u] * rP);
      var[c] = __double2float_rn(rP);
      validp[c] = 1;
    }
    // a10: Eq.(1)+(2) per channel
    const unsigned long long nn = kColor ? (cnt[u] >> 32) : w0[u];
    if (nn != 0ull) {
      const double rn = 1.0 / (double)nn;
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
        vals[(long long)(gd.word0 + k) * BHW + c] = rule_average_r(th[u][k], ob[u] != 0, sk, rn, gd.w);
      }
      obsp[c] = 1;
    }
    // re-zero the scratch for the slot's next map (fast-path records are 4 words, 32 B)
    __stcg(a.cnt + sb + phys[u], 0ull);
    __stcg(reinterpret_cast<ulonglong2 *>(r), make_ulonglong2(0ull, 0ull));
    __stcg(reinterpret_cast<ulonglong2 *>(r) + 1, make_ulonglong2(0ull, 0ull));
  }
}

// a8, bucketed fast path: one 16-B record per in-window point, appended to the bucket of its
// (map-slot, band): {local cell | outlier << 31, 1/v (fp32, 0 for outliers), z * (1/v) (fp32),
// the channel word}.  These are exactly the fp32 terms the oracle sums in fp64,
// so k_accum's sums equal the RED path's.  Lanes of the same bucket reserve their slots with one
// atomicAdd (match_any).  A bucket that is full sends the point to the scratch with REDs instead
// (accumulate_warp); k_accum merges the scratch of such a band.  All 32 lanes must call this.
template <int kFast>
__device__ __forceinline__ void bucket_warp(const PassArgs &a, const PointOut &o, int phys, int slot, int sc,
                                            const float *p, float ch0) {
  const bool act = o.cell >= 0;
  if (!__any_sync(0xffffffffu, act)) return;
  const int lane = threadIdx.x & 31;
  int band = 0, local = 0;
  if (act) band = divmod_fast(phys, a.band_cells, a.inv_band, local);
  const int key = act ? slot * a.nbands + band : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int leader = __ffs(peers) - 1;
  unsigned base = 0u;
  if (act && lane == leader) base = atomicAdd(&a.bcnt[key], (unsigned)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  const unsigned pos = base + (unsigned)__popc(peers & lanemask_lt());
  const bool spill = act && pos >= a.bcap;
  if (act && !spill) {
    const bool inl = o.code == MEM_CODE_INLIER;
    float wf = 0.0f, zw = 0.0f;
    if (inl) {
      wf = 1.0f / o.v;
      zw = o.z * wf;
    }
    uint4 r;
    r.x = (unsigned)local | (inl ? 0u : 0x80000000u);
    r.y = __float_as_uint(wf);
    r.z = __float_as_uint(zw);
    r.w = __float_as_uint(ch0);
    __stcg(a.recs + (long long)key * a.bcap + pos, r);
  }
  if (__any_sync(0xffffffffu, spill)) {
    PointOut q = o;
    if (!spill) q.cell = -1;
    accumulate_warp<kFast>(a, q, sc, p, ch0);
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

template <bool kDebug, int kFast, bool kBucket>
__device__ __forceinline__ void process_item(const PassArgs &a, const Item &t, const float (&px)[kWarpPtsPerLane],
                                             const float (&py)[kWarpPtsPerLane], const float (&pz)[kWarpPtsPerLane],
                                             const float (&pw)[kWarpPtsPerLane], float rmin2, float rmax2,
                                             unsigned long long &packed, unsigned &npk, unsigned (&cnt)[8]) {
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31;
  const PointFrame f = frame_of(a, t.m);
  const int map_base = t.m * g.HW;
  const int sb = (int)scratch_base(a, t.m);
  // points of the item present: [0, nv) (32-bit indices within the item)
  const int nv = t.end - t.base < kWarpPoints ? (int)(t.end - t.base) : kWarpPoints;
  PointOut o[kWarpPtsPerLane];
#pragma unroll
  for (int u = 0; u < kWarpPtsPerLane; ++u) {
    const bool in = u * 32 + lane < nv;
    if (in && !(a.ablate & 8u)) {
      o[u] = bin_point(px[u], py[u], pz[u], f, g, a.np, rmin2, rmax2, map_base);
    } else {
      o[u].code = in ? MEM_CODE_NONFINITE : -1;
      o[u].cell = -1;
      o[u].test = false;
    }
  }
  if (!(a.ablate & 4u)) mahalanobis(o, a.st, g, a.np.tau2);
#pragma unroll
  for (int u = 0; u < kWarpPtsPerLane; ++u) {
    const int k = u * 32 + lane;
    if (k < nv) {
      if (kDebug) {
        a.dbg_cell[t.base + k] = o[u].lcell;
        a.dbg_code[t.base + k] = (uint8_t)o[u].code;
      }
      count_code(packed, npk, o[u].code, cnt);
    }
    if (a.ablate & 2u) continue;
    const float *pp = kFast != 0 ? nullptr : a.pts + (k < nv ? t.base + k : t.beg) * (long long)a.stride;
    if constexpr (kBucket)
      bucket_warp<kFast>(a, o[u], o[u].cell - map_base, a.slot0 + t.m - a.m0, sb + (o[u].cell - map_base), pp,
                         pw[u]);
    else
      accumulate_warp<kFast>(a, o[u], sb + (o[u].cell - map_base), pp, pw[u]);
  }
}

template <bool kDebug, int kFast, bool kBucket>
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
  const float rmin2 = a.np.r_min * a.np.r_min, rmax2 = a.np.r_max * a.np.r_max;  // D9
  unsigned long long packed = 0ull;
  unsigned npk = 0;
  float px[kWarpPtsPerLane], py[kWarpPtsPerLane], pz[kWarpPtsPerLane], pw[kWarpPtsPerLane];
  if (kFast != 0 || a.vec4) {
    const float4 *pts4 = reinterpret_cast<const float4 *>(a.pts);
    auto issue = [&](const Item &t, int stage) {
#pragma unroll
      for (int u = 0; u < kWarpPtsPerLane; ++u) {
        const long long i = t.base + u * 32 + lane;
        cp_async_16(&s_pts[wid][stage][u * 32 + lane], pts4 + (i < t.end ? i : t.beg), i < t.end, pol);
      }
      cp_async_commit();
    };
    int it = i0 + gw, stage = 0;
    Item cur;
    if (it < i1) {
      cur = item_of(a, it, i0);
      issue(cur, 0);
    }
    for (; it < i1; it += nwarps, stage ^= 1) {
      const int nx = it + nwarps;
      Item nxt;
      if (nx < i1) {
        nxt = item_of(a, nx, i0);
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
      process_item<kDebug, kFast, kBucket>(a, cur, px, py, pz, pw, rmin2, rmax2, packed, npk, cnt);
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
      process_item<kDebug, kFast, kBucket>(a, t, px, py, pz, pw, rmin2, rmax2, packed, npk, cnt);
    }
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

// ---------------------------------------------------------------- k_cells (a9-a10, lazy a13)
// Persistent grid-stride over 1024-cell tiles of one wave.  Phase 1 reads every cell's count
// (coalesced), applies the pending strip reset and compacts the touched cells into shared
// memory; phase 2 fuses the touched cells densely (2 per lane in flight), so no lane idles on
// untouched cells.
constexpr int kChunkPerLane = 4;                 // cells per lane per chunk
constexpr int kChunk = 32 * kChunkPerLane;        // 128-cell chunk per warp

// Warp-persistent grid-stride over 128-cell chunks of the wave's maps (newest map first: its
// scratch was touched last by k_points and is still in L2).  Each warp, independently of the
// others (no CTA barrier): 4 count loads per lane in flight, the pending shift strips reset,
// its touched cells compacted in its own shared-memory slice, then fused 2 per lane per round.
template <int kFast>
__global__ void __launch_bounds__(kThreads, MEM_CELLS_MINB) k_cells(const __grid_constant__ PassArgs a) {
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
  const int total = (a.ablate & 1u) ? 0 : (a.m1 - a.m0) * cpm;
  int *sp = s_phys[wid];
  unsigned long long *sc = s_cntv[wid];
  for (int rt = gw; rt < total; rt += nwarps) {
    const int chunk = (a.ablate & 32u) ? rt : total - 1 - rt;
    const int mi = chunk / cpm;
    const int m = a.m0 + mi;
    const int t0 = a.cell_lo + (chunk - mi * cpm) * kChunk;
    const int sb = (int)scratch_base(a, m);
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
    cnt[7] += lane == 0 ? (unsigned)n : 0u;
    for (int k0 = 0; k0 < ((a.ablate & 512u) ? 0 : n); k0 += 64) {
      int ph[2];
      unsigned long long cc[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u * 32 + lane;
        ph[u] = k < n ? sp[k] : -1;
        cc[u] = k < n ? sc[k] : 0ull;
      }
      if (kFast == 1)
        fuse_cells_avg<2, 3, true>(a, m, sb, ph, cc);
      else if (kFast == 2)
        fuse_cells_avg<2, 1, false>(a, m, sb, ph, cc);
      else
        fuse_cells<2>(a, m, sb, ph, cc);
    }
    __syncwarp();  // this warp's slice is rewritten by its next chunk
  }
  __syncthreads();
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

// ---------------------------------------------------------------- k_smap (small maps, sort by cell)
// One CTA per map (grid-stride over the wave's maps) for the fast rules on small maps
// (H*W <= kSmapCells, <= kSmapPoints points per map): no scratch, no atomics outside shared
// memory.  P1 bins every point (streamed once from HBM) into a shared-memory histogram of its
// cell; P2 turns it into offsets; P3 re-bins (the map's points are L2-resident) and scatters
// the point indices by cell; P4 gives every cell to one thread, which sorts the cell's indices
// (input order, like the oracle), re-reads and re-bins those points, tests them against the
// cell's pre-frame state (a7), sums in fp64 in input order and fuses the cell with the
// oracle's exact formulas -- so this path is deterministic and reproduces the oracle's sums
// operation for operation.  (The north_star's "sort-by-cell segmented reduction".)
#ifndef MEM_SMAP_THREADS
#define MEM_SMAP_THREADS 1024  // P4 walks the cells one per thread: more threads, shorter chains
#endif
#ifndef MEM_SMAP_MINB
#define MEM_SMAP_MINB 1
#endif
constexpr int kSmapThreads = MEM_SMAP_THREADS;
constexpr int kSmapCells = 16384;
constexpr int kSmapPoints = 65535;
constexpr int kSmapSortMax = 256;  // cells with more points keep the scatter order (still exact sums, any order)

// shared memory: the per-cell counts / offsets as packed u16 pairs (a map has < 65536 points)
// and the u16 point indices
constexpr int kSmapChunk = 64;  // P4: points per warp step
__host__ __device__ inline size_t smap_tmp_offset(int HW, long long max_pts) {
  return (sizeof(unsigned) * (size_t)((HW + 1) / 2) + sizeof(uint16_t) * (size_t)max_pts + 15) & ~(size_t)15;
}
size_t smap_smem_bytes(int HW, long long max_pts) {
  return smap_tmp_offset(HW, max_pts) + sizeof(float4) * (size_t)kSmapChunk * (kSmapThreads / 32);
}
bool smap_eligible(int HW, long long max_pts) {
  return HW <= kSmapCells && max_pts <= kSmapPoints && smap_smem_bytes(HW, max_pts) <= 220 * 1024;
}

template <bool kDebug, int kFast>
__global__ void __launch_bounds__(kSmapThreads, MEM_SMAP_MINB) k_smap(const __grid_constant__ PassArgs a) {
  constexpr int NCH = kFast == 1 ? 3 : 1;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const Geometry &g = a.geo;
  unsigned *hist = reinterpret_cast<unsigned *>(s_dyn);  // cell c: 16-bit half (c & 1) of word c >> 1
  uint16_t *idx = reinterpret_cast<uint16_t *>(hist + (g.HW + 1) / 2);
  auto h16 = [&](int c) { return (hist[c >> 1] >> (16 * (c & 1))) & 0xffffu; };
  float4 *s_tmp = reinterpret_cast<float4 *>(s_dyn + smap_tmp_offset(g.HW, a.smap_maxpts));  // P4 slices
  __shared__ unsigned s_part[kSmapThreads];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0)  // the other epoch is the next point input's (no memset per call)
    for (int i = threadIdx.x; i < kStatSlots * 8; i += kSmapThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long packed = 0ull;
  unsigned npk = 0;
  const unsigned long long pol = evict_first_policy();
  const float rmin2 = a.np.r_min * a.np.r_min, rmax2 = a.np.r_max * a.np.r_max;  // D9
  const long long BHW = g.BHW;
  const GroupDesc &gd = a.b[0].g;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  uint8_t *obsp = a.st.flags + (long long)gd.flag * BHW;
  const float4 *pts4 = reinterpret_cast<const float4 *>(a.pts);
  for (int m = a.m0 + blockIdx.x; m < a.m1; m += gridDim.x) {
    const long long beg = off_of(a, m);
    const int np = (int)(off_of(a, m + 1) - beg);
    const PointFrame f = frame_of(a, m);
    const int map_base = m * g.HW;
    for (int c = threadIdx.x; c < (g.HW + 1) / 2; c += kSmapThreads) hist[c] = 0u;
    if (threadIdx.x == 0) a.ring[m] = make_int2(f.r0, f.c0);
    __syncthreads();
    // P1: bin every point (a2-a6), histogram of the in-window points' cells
    for (int i0 = threadIdx.x; i0 < np; i0 += 4 * kSmapThreads) {
      float4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i < np) q[u] = ld_stream_f4(reinterpret_cast<const float *>(pts4 + beg + i), pol);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i >= np) continue;
        const PointOut o = bin_point(q[u].x, q[u].y, q[u].z, f, g, a.np, rmin2, rmax2, map_base);
        if (o.cell >= 0) {
          const int c = o.cell - map_base;
          atomicAdd(&hist[c >> 1], 1u << (16 * (c & 1)));
        } else {
          count_code(packed, npk, o.code, cnt);
          if (kDebug) {
            a.dbg_cell[beg + i] = -1;
            a.dbg_code[beg + i] = (uint8_t)o.code;
          }
        }
      }
    }
    __syncthreads();
    // P2: exclusive scan of the counts: each warp scans a contiguous run of words (2 cells each,
    // lanes on consecutive words), then the warps' totals are offset
    {
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      constexpr int kWarps = kSmapThreads / 32;
      const int nw = (g.HW + 1) / 2;
      const int seg = ((nw + kWarps - 1) / kWarps + 31) & ~31;
      const int w0 = wid * seg, w1 = min(w0 + seg, nw);
      unsigned run = 0;
      for (int w = w0; w < w1; w += 32) {
        const unsigned word = w + lane < w1 ? hist[w + lane] : 0u;
        const unsigned lo = word & 0xffffu, pair = lo + (word >> 16);
        unsigned x = pair;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const unsigned off = run + x - pair;
        if (w + lane < w1) hist[w + lane] = off | ((off + lo) << 16);
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) s_part[wid] = run;
      __syncthreads();
      unsigned off = 0;
      for (int w = 0; w < wid; ++w) off += s_part[w];
      for (int w = w0 + lane; w < w1; w += 32) hist[w] += off | (off << 16);
    }
    __syncthreads();
    // P3: scatter the in-window points' indices by cell (the map's points are now in L2)
    for (int i0 = threadIdx.x; i0 < np; i0 += 4 * kSmapThreads) {
      float4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i < np) q[u] = __ldg(pts4 + beg + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i >= np) continue;
        const PointOut o = bin_point(q[u].x, q[u].y, q[u].z, f, g, a.np, rmin2, rmax2, map_base);
        if (o.cell >= 0) {
          const int c = o.cell - map_base;
          idx[(atomicAdd(&hist[c >> 1], 1u << (16 * (c & 1))) >> (16 * (c & 1))) & 0xffffu] = (uint16_t)i;
        }
      }
    }
    __syncthreads();
    // P4: warps take groups of 32 consecutive cells (lane = cell).  Each lane sorts its cell's
    // point indices into input order and loads its cell's pre-frame state; the warp then walks
    // the group's points (contiguous in idx) 64 at a time, lane-parallel: re-read, re-bin,
    // outlier test against the owner lane's state (shuffle), contributions staged in the
    // warp's shared slice; each lane then adds its own cell's contributions in input order --
    // the oracle's sequential fp64 sums -- and finally fuses and stores its cell.
    const bool shift = f.sr != 0 || f.sc != 0;
    {
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      float4 *tmp = s_tmp + wid * kSmapChunk;
      for (int gbase = wid * 32; gbase < g.HW; gbase += kSmapThreads) {
        const int c = gbase + lane;
        const bool inmap = c < g.HW;
        unsigned s0 = 0u, s1 = 0u;
        bool strip = false;
        if (inmap) {
          s0 = c == 0 ? 0u : h16(c - 1);
          s1 = h16(c);  // the count of c is now its end
          if (shift) {
            int pcol;
            const int prow = divmod_fast(c, g.W, g.inv_W, pcol);
            int row = prow - f.r0, col = pcol - f.c0;
            row += row < 0 ? g.H : 0;
            col += col < 0 ? g.W : 0;
            strip = in_strip(row, col, f, g);
          }
          if (s1 - s0 > 1u && s1 - s0 <= (unsigned)kSmapSortMax) {  // input order (insertion sort)
            for (unsigned r = s0 + 1; r < s1; ++r) {
              const uint16_t key = idx[r];
              unsigned q = r;
              while (q > s0 && idx[q - 1] > key) {
                idx[q] = idx[q - 1];
                --q;
              }
              idx[q] = key;
            }
          }
        }
        const bool live = inmap && (s1 != s0 || strip);  // untouched cells stay bit-identical
        const long long cc = (long long)map_base + (inmap ? c : 0);
        float h = __int_as_float(0x7fc00000), s2 = h, th[NCH];
        uint8_t vd = 0, ob = 0;
#pragma unroll
        for (int k = 0; k < NCH; ++k) th[k] = 0.0f;
        if (live && !strip) {  // a scrolled-in cell starts from the reset state (a13)
          h = elev[cc];
          s2 = var[cc];
          vd = validp[cc];
          ob = obsp[cc];
#pragma unroll
          for (int k = 0; k < NCH; ++k) th[k] = vals[(long long)(gd.word0 + k) * BHW + cc];
        }
        const unsigned last = __reduce_max_sync(0xffffffffu, inmap ? (unsigned)lane : 0u);
        const unsigned R0 = __shfl_sync(0xffffffffu, s0, 0), R1 = __shfl_sync(0xffffffffu, s1, last);
        __syncwarp();  // every lane's sorted segment is visible
        unsigned nin = 0, nout = 0, ng = 0, cr = 0, cg = 0, cbl = 0;
        double P = 0.0, S = 0.0, X = 0.0;
        for (unsigned cb0 = R0; cb0 < R1; cb0 += kSmapChunk) {
          const unsigned ce = min(cb0 + (unsigned)kSmapChunk, R1);
#pragma unroll
          for (int k = 0; k < kSmapChunk / 32; ++k) {
            const unsigned r = cb0 + k * 32 + lane;
            const bool act = r < ce;
            const int i = act ? idx[r] : 0;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (act) q = __ldg(pts4 + beg + i);
            PointOut o;
            o.cell = -1;
            o.test = false;
            o.z = o.v = 0.0f;
            o.lcell = -1;
            if (act) o = bin_point(q.x, q.y, q.z, f, g, a.np, rmin2, rmax2, map_base);
            const int owner = act ? o.cell - map_base - gbase : lane;  // the lane holding its cell
            const float ho = __shfl_sync(0xffffffffu, h, owner), so = __shfl_sync(0xffffffffu, s2, owner);
            const int vo = __shfl_sync(0xffffffffu, (int)vd, owner);
            if (act) {
              bool outl = false;
              if (o.test && vo) {  // (z - h)^2 > tau^2 (sigma^2 + v) against the pre-frame state (D10)
                const float d = o.z - ho;
                outl = d * d > a.np.tau2 * (so + o.v);
              }
              const int code = outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER;
              count_code(packed, npk, code, cnt);
              if (kDebug) {
                a.dbg_cell[beg + i] = o.lcell;
                a.dbg_code[beg + i] = (uint8_t)code;
              }
              float wf = 0.0f, zw = 0.0f;
              if (!outl) {
                wf = 1.0f / o.v;
                zw = o.z * wf;
              }
              tmp[k * 32 + lane] = make_float4(wf, zw, q.w, outl ? 1.0f : 0.0f);
            }
          }
          __syncwarp();
          const unsigned lo = max(s0, cb0), hi = min(s1, ce);
          for (unsigned r = lo; r < hi; ++r) {  // this cell's points of the chunk, in input order
            const float4 t4 = tmp[r - cb0];
            if (t4.w != 0.0f) {
              ++nout;
            } else {
              ++nin;
              P += (double)t4.x;
              S += (double)t4.y;
            }
            if (kFast == 1) {  // D20: 0x00RRGGBB, exact integer sums
              const uint32_t bits = __float_as_uint(t4.z);
              cr += (bits >> 16) & 255u;
              cg += (bits >> 8) & 255u;
              cbl += bits & 255u;
            } else if (isfinite(t4.z)) {  // D31
              ++ng;
              X += (double)t4.z;
            }
          }
          __syncwarp();  // the slice is refilled by the next chunk
        }
        if (!live) continue;
        if (s1 > s0 && !(a.ablate & 512u)) {
          ++cnt[7];
          // a9 (D7, D11) in the oracle's exact form
          if (vd) {
            const double sp = (double)s2 + (double)nout * (double)a.np.v_out;
            if (nin > 0u) {
              const double den = 1.0 + P * sp;
              h = __double2float_rn(((double)h + S * sp) / den);
              s2 = __double2float_rn(sp / den);
            } else {
              s2 = __double2float_rn(sp);
            }
          } else if (nin > 0u) {
            h = __double2float_rn(S / P);
            s2 = __double2float_rn(1.0 / P);
            vd = 1;
          }
          // a10: Eq.(1)+(2)
          const unsigned nn = kFast == 1 ? nin + nout : ng;
          if (nn != 0u) {
            if (kFast == 1) {
              th[0] = rule_average(th[0], ob != 0, (double)cr, (double)nn, gd.w);
              th[1 % NCH] = rule_average(th[1 % NCH], ob != 0, (double)cg, (double)nn, gd.w);
              th[2 % NCH] = rule_average(th[2 % NCH], ob != 0, (double)cbl, (double)nn, gd.w);
            } else {
              th[0] = rule_average(th[0], ob != 0, X, (double)nn, gd.w);
            }
            ob = 1;
          }
        }
        elev[cc] = h;
        var[cc] = s2;
#pragma unroll
        for (int k = 0; k < NCH; ++k) vals[(long long)(gd.word0 + k) * BHW + cc] = th[k];
        validp[cc] = vd;
        obsp[cc] = ob;
      }
    }
    __syncthreads();  // hist / idx are reused by the next map
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

// ---------------------------------------------------------------- k_route (sharded map, NEXT)
// a2-a5 for this rank's shard of a single map: dropped points are counted here, every
// in-window point is copied into the bucket of its cell's band owner (lanes with the same
// owner reserve their slots with one atomicAdd).  The owner then runs k_points + k_cells on
// what it received: the Mahalanobis test, accumulation and fusion all happen there.
__global__ void __launch_bounds__(kThreads) k_route(const __grid_constant__ PassArgs a, const RouteArgs r) {
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0)  // the other epoch is the next point input's (no memset per call)
    for (int i = threadIdx.x; i < kStatSlots * 8; i += kThreads) (&a.ctl->stats[a.epoch ^ 1][0][0])[i] = 0ull;
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long packed = 0ull;
  unsigned npk = 0;
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31;
  const long long n = off_of(a, 1);
  const PointFrame f = frame_of(a, 0);
  const float rmin2 = a.np.r_min * a.np.r_min, rmax2 = a.np.r_max * a.np.r_max;  // D9
  const long long nthreads = (long long)gridDim.x * kThreads;
  for (long long i0 = (long long)blockIdx.x * kThreads; i0 < n; i0 += nthreads) {  // warp-uniform trip count
    const long long i = i0 + threadIdx.x;
    const bool in = i < n;
    const float *q = a.pts + (in ? i : 0) * (long long)a.stride;
    PointOut o;
    o.cell = -1;
    o.code = -1;
    if (in) o = bin_point(__ldg(q), __ldg(q + 1), __ldg(q + 2), f, g, a.np, rmin2, rmax2, 0);
    if (in && o.cell < 0) count_code(packed, npk, o.code, cnt);
    const int dest = o.cell >= 0 ? o.cell / r.band_n : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, dest);
    const int leader = __ffs(peers) - 1;
    unsigned base = 0u;
    if (dest >= 0 && lane == leader) base = atomicAdd(&r.cnt[dest], (unsigned)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (dest >= 0) {
      const long long pos = (long long)base + __popc(peers & lanemask_lt());
      float *d = r.buf + ((long long)dest * r.cap + pos) * a.stride;
      for (int k = 0; k < a.stride; ++k) d[k] = __ldg(q + k);
    }
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}

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
  const int units = (a.ablate & 1u) ? 0 : (a.m1 - a.m0) * a.nbands;
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
        dirty[v] = strip[v] || (nin[v] + nout[v] != 0u && !(a.ablate & 512u));
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
        if (nin[v] + nout[v] != 0u && !(a.ablate & 512u)) {
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

// ---------------------------------------------------------------- plugins (NEXT-3)
// The oracle's definitions (om_plugin_*, readings D35-D37) with the same fp32 operations in
// the same order; neighbours are logical cells (no wrap), mapped through the ring.
struct PostCtx {
  const PostArgs &a;
  int m;
  int2 ring;
  __device__ long long phys(int i, int j) const {
    const Geometry &g = a.geo;
    return (long long)m * g.HW + (long long)wrap(i + ring.x, g.H) * g.W + wrap(j + ring.y, g.W);
  }
  __device__ bool valid(int i, int j) const {
    const Geometry &g = a.geo;
    return i >= 0 && i < g.H && j >= 0 && j < g.W && a.st.flags[(long long)kFlagValid * g.BHW + phys(i, j)];
  }
  __device__ float h(int i, int j) const {
    return reinterpret_cast<const float *>(a.st.words)[(long long)kWordElev * a.geo.BHW + phys(i, j)];
  }
  __device__ bool grad(int i, int j, int di, int dj, float &gr) const {
    const bool vp = valid(i + di, j + dj), vm = valid(i - di, j - dj);
    const float res = a.geo.res;
    if (vp && vm) gr = (h(i + di, j + dj) - h(i - di, j - dj)) / (2.0f * res);
    else if (vp) gr = (h(i + di, j + dj) - h(i, j)) / res;
    else if (vm) gr = (h(i, j) - h(i - di, j - dj)) / res;
    else return false;
    return true;
  }
  __device__ bool normal(int i, int j, float (&n)[3]) const {
    float gx, gy;
    if (!valid(i, j) || !grad(i, j, 1, 0, gx) || !grad(i, j, 0, 1, gy)) return false;
    const float norm = sqrtf((gx * gx + gy * gy) + 1.0f);
    n[0] = -gx / norm;
    n[1] = -gy / norm;
    n[2] = 1.0f / norm;
    return true;
  }
};

__global__ void __launch_bounds__(kThreads) k_post(const __grid_constant__ PostArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int i = t / g.W, j = t - (t / g.W) * g.W;
  const PostCtx c{a, m, a.ring[m]};
  const long long o = (long long)m * g.HW + t, L = g.BHW;  // output layer stride = n_maps * HW
  const float nan = __int_as_float(0x7fc00000);
  if (a.op == 0) {  // normals
    float n[3];
    if (!c.normal(i, j, n)) n[0] = n[1] = n[2] = nan;
    a.out[o] = n[0];
    a.out[L + o] = n[1];
    a.out[2 * L + o] = n[2];
  } else if (a.op == 1) {  // traversability (D36)
    float n[3];
    if (!c.normal(i, j, n)) {
      a.out[o] = nan;
      return;
    }
    const float slope = (n[2] - a.cos_max) / (1.0f - a.cos_max);
    const float hc = c.h(i, j);
    float mx = 0.0f;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        if ((di == 0 && dj == 0) || !c.valid(i + di, j + dj)) continue;
        const float d = fabsf(c.h(i + di, j + dj) - hc);
        if (d > mx) mx = d;
      }
    const float step = 1.0f - mx / a.step_max;
    float sc = slope < step ? slope : step;
    sc = sc < 0.0f ? 0.0f : sc;
    a.out[o] = sc > 1.0f ? 1.0f : sc;
  } else {  // semantic argmax (D37)
    const long long p = c.phys(i, j);
    const float *vals = reinterpret_cast<const float *>(a.st.words);
    float id = -1.0f, conf = 0.0f;
    if (a.rule == MEM_CLASS_MAX) {
      const int lab = reinterpret_cast<const int *>(a.st.words)[(long long)a.label * g.BHW + p];
      if (lab >= 0) {
        id = (float)lab;
        conf = vals[(long long)a.first * g.BHW + p];
      }
    } else if (a.st.flags[(long long)a.flag * g.BHW + p]) {
      double tot = 0.0;
      if (a.rule == MEM_CLASS_BAYESIAN)
        for (int k = 0; k < a.K; ++k) tot += (double)vals[(long long)(a.first + k) * g.BHW + p];
      for (int k = 0; k < a.K; ++k) {
        const float v = vals[(long long)(a.first + k) * g.BHW + p];
        const float th = a.rule == MEM_CLASS_BAYESIAN ? __double2float_rn((double)v / tot) : v;
        if (k == 0 || th > conf) {
          conf = th;
          id = (float)k;
        }
      }
    }
    a.out[o] = id;
    a.out[L + o] = conf;
  }
}

// ---------------------------------------------------------------- occlusion (NEXT-1)
// Is logical cell (row, col) of map m seen from the camera at (tx, ty, tz) (map-centred, fp32)?
// every intermediate cell of the Bresenham line from the camera's footprint
// cell to the target must lie below the ray; readings D32-D34: the line is walked
// from the lexicographically smaller endpoint (all-octant integer form), cells outside the map
// and unknown cells do not occlude, the ray height is linear in the 2D distance between the
// camera height and the target elevation, tolerance eps_occ.  fp32 in the oracle's order.
__device__ __forceinline__ bool cell_visible(const ImageArgs &a, int m, int row, int col, float tx, float ty,
                                             float tz, float hb, int2 ring) {
  const Geometry &g = a.geo;
  const float *elev = reinterpret_cast<const float *>(a.st.words) + (long long)kWordElev * g.BHW;
  const uint8_t *validp = a.st.flags + (long long)kFlagValid * g.BHW;
  const int rc = (int)floorf(tx * g.inv_res + g.hH), cc = (int)floorf(ty * g.inv_res + g.hW);
  const float xb = ((float)row + 0.5f - g.hH) * g.res, yb = ((float)col + 0.5f - g.hW) * g.res;
  const float dxb = xb - tx, dyb = yb - ty;
  const float db = sqrtf(dxb * dxb + dyb * dyb);
  int r0 = rc, c0 = cc, r1 = row, c1 = col;
  if (r1 < r0 || (r1 == r0 && c1 < c0)) {
    r0 = row; c0 = col; r1 = rc; c1 = cc;
  }
  const int dx = abs(r1 - r0), dy = -abs(c1 - c0);
  const int sx = r0 < r1 ? 1 : -1, sy = c0 < c1 ? 1 : -1;
  int err = dx + dy, x = r0, y = c0;
  const long long mbase = (long long)m * g.HW;
  // the line has max(dx, -dy) - 1 intermediate cells; they are generated kOccBatch at a time
  // and all their (valid, h) loads issued before any test (one round trip per batch)
  constexpr int kOccBatch = MEM_OCC_BATCH;
  int left = max(dx, -dy) - 1;
  while (left > 0) {
    int bx[kOccBatch], by[kOccBatch];
    long long bj[kOccBatch];
    uint8_t bv[kOccBatch];
    float bh[kOccBatch];
#pragma unroll
    for (int k = 0; k < kOccBatch; ++k) {
      bj[k] = -1;
      if (k < left) {
        const int e2 = 2 * err;
        if (e2 >= dy) { err += dy; x += sx; }
        if (e2 <= dx) { err += dx; y += sy; }
        bx[k] = x;
        by[k] = y;
        if (x >= 0 && x < g.H && y >= 0 && y < g.W)  // outside the map: no occluder
          bj[k] = mbase + (long long)wrap(x + ring.x, g.H) * g.W + wrap(y + ring.y, g.W);
      }
    }
#pragma unroll
    for (int k = 0; k < kOccBatch; ++k) {
      bv[k] = 0;
      if (bj[k] >= 0) {
        bv[k] = validp[bj[k]];
        bh[k] = elev[bj[k]];
      }
    }
#pragma unroll
    for (int k = 0; k < kOccBatch; ++k) {
      if (!bv[k]) continue;  // unknown terrain does not occlude
      const float xi = ((float)bx[k] + 0.5f - g.hH) * g.res, yi = ((float)by[k] + 0.5f - g.hW) * g.res;
      const float dxi = xi - tx, dyi = yi - ty;
      const float di = sqrtf(dxi * dxi + dyi * dyi);
      const float ray = tz + (di / db) * (hb - tz);
      if (bh[k] > ray + a.eps_occ) return false;
    }
    left -= kOccBatch;
  }
  return true;
}

// ---------------------------------------------------------------- k_image (a11-a12)
__global__ void __launch_bounds__(kThreads) k_image(const __grid_constant__ ImageArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;  // logical cell
  const int2 ring = a.ring[m];
  const int prow = wrap(row + ring.x, g.H);
  if (prow < a.row_lo || prow >= a.row_hi) return;  // another rank's band (sharded map)
  const long long cell = (long long)m * g.HW + (long long)prow * g.W + wrap(col + ring.y, g.W);
  if (!a.st.flags[(long long)kFlagValid * g.BHW + cell]) return;
  const MapFrame &f = a.frames ? a.frames[m] : a.f0;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  // a11: cell centre at its elevation, relative to the map centre (D13), into the camera (D17)
  const float xc = ((float)row + 0.5f - g.hH) * g.res;
  const float yc = ((float)col + 0.5f - g.hW) * g.res;
  const float dx = xc - f.t[0], dy = yc - f.t[1];
  const float hcell = vals[(long long)kWordElev * g.BHW + cell];
  const float dz = hcell - f.t[2];
  const float pcx = (f.R[0] * dx + f.R[3] * dy) + f.R[6] * dz;
  const float pcy = (f.R[1] * dx + f.R[4] * dy) + f.R[7] * dz;
  const float pcz = (f.R[2] * dx + f.R[5] * dy) + f.R[8] * dz;
  if (!(pcz > 1e-6f)) return;
  const float ux = pcx / pcz, uy = pcy / pcz;
  const float u = (f.K[0] * ux + f.K[1] * uy) + f.K[2];  // pinhole
  const float v = f.K[3] * uy + f.K[4];
  const float fu = floorf(u + 0.5f), fv = floorf(v + 0.5f);  // nearest pixel (D16)
  if (!(0.0f <= fu && fu < (float)a.IW && 0.0f <= fv && fv < (float)a.IH)) return;  // frustum
  if (a.occlusion && !cell_visible(a, m, row, col, f.t[0], f.t[1], f.t[2], hcell, ring)) return;
  const long long plane = (long long)a.IH * a.IW;
  const float *pix = a.img + (long long)m * a.map_stride + (long long)(int)fv * a.IW + (int)fu;
  // a12: sample and fuse with N_j = 1
  for (int bi = 0; bi < a.nb; ++bi) {
    const BindDesc &b = a.b[bi];
    const float *ch = pix + (long long)b.ch_offset * plane;
    if (b.topk > 0) {  // top-k pairs (D38)
      const TopK tk{ch, plane, b.topk, b.g.nch - 1};
      if (!tk.ok()) continue;
      const unsigned long long key = b.g.rule == MEM_CLASS_MAX ? tk.key() : 0ull;
      apply_group(a.st, g.BHW, cell, b.g, 1.0, [&](int k) { return (double)tk.value(k); }, key);
      continue;
    }
    bool fin = true;
    for (int k = 0; k < b.nch; ++k) fin &= (bool)isfinite(__ldg(ch + k * plane));
    if (!fin) continue;  // D21
    unsigned long long key = 0ull;
    if (b.g.rule == MEM_CLASS_MAX) {
      int best = 0;
      float bv = __ldg(ch);
      for (int k = 1; k < b.nch; ++k) {
        const float c = __ldg(ch + k * plane);
        if (c > bv) {
          bv = c;
          best = k;
        }
      }
      key = ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
    }
    apply_group(a.st, g.BHW, cell, b.g, 1.0, [&](int k) { return (double)__ldg(ch + k * plane); }, key);
  }
}

// ---------------------------------------------------------------- k_shift (eager a13)
__global__ void __launch_bounds__(kThreads) k_shift(const __grid_constant__ ShiftArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const ShiftRec r = a.recs ? a.recs[m] : a.rec0;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) a.ring[m] = make_int2(r.r0, r.c0);
  const int ar = r.sr < 0 ? -r.sr : r.sr, ac = r.sc < 0 ? -r.sc : r.sc;
  int row, col;  // logical cell of the NEW window that scrolled in
  if (ar >= g.H || ac >= g.W) {
    if (t >= g.HW) return;
    row = t / g.W;
    col = t - row * g.W;
  } else if (t < ar * g.W) {
    const int k = t / g.W;
    row = r.sr > 0 ? g.H - r.sr + k : k;
    col = t - k * g.W;
  } else if (t < ar * g.W + ac * g.H) {
    const int t2 = t - ar * g.W;
    const int k = t2 / g.H;
    col = r.sc > 0 ? g.W - r.sc + k : k;
    row = t2 - k * g.H;
  } else {
    return;
  }
  const long long cell = (long long)m * g.HW + (long long)wrap(row + r.r0, g.H) * g.W + wrap(col + r.c0, g.W);
  reset_cell(a.st, g.BHW, cell, a.reset);
}

// ---------------------------------------------------------------- k_read / k_write (a14)
__global__ void __launch_bounds__(kThreads) k_read(const __grid_constant__ ReadArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;
  const int2 ring = a.ring[m];
  const long long cell = (long long)m * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  float out = 0.0f;
  switch (a.kind) {
    case RK_ELEV:
    case RK_VAR:
      out = a.st.flags[(long long)kFlagValid * g.BHW + cell] ? vals[(long long)a.idx * g.BHW + cell]
                                                              : __int_as_float(0x7fc00000);
      break;
    case RK_WORD: out = vals[(long long)a.idx * g.BHW + cell]; break;
    case RK_LABEL: out = (float)reinterpret_cast<const int *>(a.st.words)[(long long)a.idx * g.BHW + cell]; break;
    case RK_FLAG: out = (float)a.st.flags[(long long)a.idx * g.BHW + cell]; break;
    case RK_THETA: {  // Eq.(11) posterior mean, derived at readout (D5)
      if (!a.st.flags[(long long)a.flag * g.BHW + cell]) break;  // unobserved -> 0 (D15)
      double tot = 0.0;
      for (int k = 0; k < a.K; ++k) tot += (double)vals[(long long)(a.first + k) * g.BHW + cell];
      out = __double2float_rn((double)vals[(long long)a.idx * g.BHW + cell] / tot);
      break;
    }
  }
  a.out[(long long)m * g.HW + t] = out;
}

__global__ void __launch_bounds__(kThreads) k_write(const __grid_constant__ ReadArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;
  const int2 ring = a.ring[m];
  const long long cell = (long long)m * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
  float v = a.src[(long long)m * g.HW + t];
  float *var = reinterpret_cast<float *>(a.st.words) + (long long)kWordVar * g.BHW;
  const uint8_t *validp = a.st.flags + (long long)kFlagValid * g.BHW;
  switch (a.kind) {
    case RK_VAR:  // invariant: an invalid cell holds a NaN variance (see mahalanobis)
      if (!validp[cell]) v = __int_as_float(0x7fc00000);
      var[cell] = v;
      break;
    case RK_ELEV:
    case RK_WORD: reinterpret_cast<float *>(a.st.words)[(long long)a.idx * g.BHW + cell] = v; break;
    case RK_LABEL: reinterpret_cast<int *>(a.st.words)[(long long)a.idx * g.BHW + cell] = (int)v; break;
    case RK_FLAG:
      a.st.flags[(long long)a.idx * g.BHW + cell] = v != 0.0f;
      if (a.idx == kFlagValid && v == 0.0f) var[cell] = __int_as_float(0x7fc00000);
      break;
    default: break;
  }
}

// ---------------------------------------------------------------- PCA readout (a14, C4)
// Moments over the observed cells of one map: sum x and the upper triangle of sum x x^T in
// fp64 (a tile of cells staged in shared memory, one thread per (a, b) pair, native fp64 REDs).
constexpr int kPcaTileBytes = 32768;
__global__ void __launch_bounds__(kThreads) k_pca_moments(const __grid_constant__ PcaArgs a) {
  extern __shared__ float s_x[];  // [d][tile]
  __shared__ int s_n;
  const Geometry &g = a.geo;
  const int d = a.d;
  const int tile = kPcaTileBytes / (4 * d);
  const int c0 = blockIdx.x * tile;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const long long mb = (long long)a.map * g.HW;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < tile; t += blockDim.x) {  // physical cells: order is irrelevant
    const int phys = c0 + t;
    const bool obs = phys < g.HW && a.st.flags[(long long)a.flag * g.BHW + mb + phys];
    for (int k = 0; k < d; ++k) s_x[k * tile + t] = obs ? vals[(long long)(a.word0 + k) * g.BHW + mb + phys] : 0.0f;
    if (obs) atomicAdd(&s_n, 1);
  }
  __syncthreads();
  const int pairs = d * (d + 1) / 2;
  for (int p = threadIdx.x; p < d + pairs; p += blockDim.x) {
    double acc = 0.0;
    if (p < d) {
      for (int t = 0; t < tile; ++t) acc += (double)s_x[p * tile + t];
    } else {
      int q = p - d, ra = 0;  // q -> (ra, rb), ra <= rb, row-major upper triangle
      while (q >= d - ra) {
        q -= d - ra;
        ++ra;
      }
      const int rb = ra + q;
      for (int t = 0; t < tile; ++t) acc += (double)s_x[ra * tile + t] * (double)s_x[rb * tile + t];
    }
    if (acc != 0.0) atomicAdd(&a.sums[p], acc);
  }
  if (threadIdx.x == 0 && s_n) atomicAdd(&a.sums[d + pairs], (double)s_n);
}

__device__ __forceinline__ unsigned long long ord_f64(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double f64_of_ord(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}

// pass 0: projections p_c = (x - mu) . e_c in fp64 (sequential over d), min/max per component;
// pass 1: min-max scaling to [0, 1] (0 when max == min); unobserved cells 0.
__global__ void __launch_bounds__(kThreads) k_pca_project(const __grid_constant__ PcaArgs a, int pass) {
  const Geometry &g = a.geo;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;
  const int2 ring = a.ring[a.map];
  const long long cell = (long long)a.map * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
  const bool obs = a.st.flags[(long long)a.flag * g.BHW + cell] != 0;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  for (int c = 0; c < a.k; ++c) {
    float *o = a.out + (long long)c * g.HW + t;
    if (!obs) {
      if (pass == 1) *o = 0.0f;
      continue;
    }
    double p = 0.0;
    for (int k = 0; k < a.d; ++k)
      p += ((double)vals[(long long)(a.word0 + k) * g.BHW + cell] - a.mean[k]) * a.comp[c * a.d + k];
    if (pass == 0) {
      atomicMin(&a.minmax[2 * c], ord_f64(p));
      atomicMax(&a.minmax[2 * c + 1], ord_f64(p));
    } else {
      const double lo = f64_of_ord(a.minmax[2 * c]), hi = f64_of_ord(a.minmax[2 * c + 1]);
      *o = hi > lo ? __double2float_rn((p - lo) / (hi - lo)) : 0.0f;
    }
  }
}

// ---------------------------------------------------------------- k_merge (sharded map)
// own band scratch op= the other ranks' partials, typed per record word (f64 sums, u64 sums,
// u64 max), so the owner's k_cells sees the statistics of every rank's points.
__global__ void __launch_bounds__(kThreads) k_merge(const __grid_constant__ MergeArgs a) {
  const long long words = (long long)a.n * (1 + a.R);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < a.n) {  // counts: u64 n_in | n_out << 32
      unsigned long long v = a.cnt[a.lo + i];
      for (int p = 0; p < a.nsrc; ++p) v += a.src_cnt[(long long)p * a.n + i];
      a.cnt[a.lo + i] = v;
      continue;
    }
    const long long j = i - a.n;  // record word j of the band
    const int w = (int)(j % a.R);
    unsigned long long *dst = a.rec + (long long)a.lo * a.R + j;
    const int ty = a.wtype[w];
    if (ty == 0) {
      double v = __longlong_as_double((long long)*dst);
      for (int p = 0; p < a.nsrc; ++p) v += __longlong_as_double((long long)a.src_rec[(long long)p * a.n * a.R + j]);
      *dst = (unsigned long long)__double_as_longlong(v);
    } else if (ty == 1) {
      unsigned long long v = *dst;
      for (int p = 0; p < a.nsrc; ++p) v += a.src_rec[(long long)p * a.n * a.R + j];
      *dst = v;
    } else {
      unsigned long long v = *dst;
      for (int p = 0; p < a.nsrc; ++p) {
        const unsigned long long x = a.src_rec[(long long)p * a.n * a.R + j];
        v = x > v ? x : v;
      }
      *dst = v;
    }
  }
}

// ---------------------------------------------------------------- launchers
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

int points_blocks_per_sm(bool debug) {
  int n = 0;
  if (debug)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_points<true, 0, false>, kThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_points<false, 0, false>, kThreads, 0);
  return n > 0 ? n : 1;
}

int cells_blocks_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_cells<0>, kThreads, 0);
  return n > 0 ? n : 1;
}

// Programmatic dependent launch: k_points, k_cells and k_accum may be scheduled while the
// kernel before them on the stream drains (its CTAs retire); each waits on griddepcontrol.wait
// before it reads anything the previous kernel wrote, and lets its own dependent launch early.
template <class K>
static cudaError_t launch_pdl(K kernel, int grid, size_t smem, cudaStream_t s, const PassArgs &a) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

cudaError_t launch_points(const PassArgs &a, int grid, cudaStream_t s) {
  // the fast variants need the channel in the float4's w (vec4) and exactly one group bound
  const int f = a.vec4 ? a.fast : 0;
  if (a.dbg_cell) {
    if (f == 1 && a.bucketed) return launch_pdl(k_points<true, 1, true>, grid, 0, s, a);
    else if (f == 2 && a.bucketed) return launch_pdl(k_points<true, 2, true>, grid, 0, s, a);
    else if (f == 1) return launch_pdl(k_points<true, 1, false>, grid, 0, s, a);
    else if (f == 2) return launch_pdl(k_points<true, 2, false>, grid, 0, s, a);
    else return launch_pdl(k_points<true, 0, false>, grid, 0, s, a);
  } else {
    if (f == 1 && a.bucketed) return launch_pdl(k_points<false, 1, true>, grid, 0, s, a);
    else if (f == 2 && a.bucketed) return launch_pdl(k_points<false, 2, true>, grid, 0, s, a);
    else if (f == 1) return launch_pdl(k_points<false, 1, false>, grid, 0, s, a);
    else if (f == 2) return launch_pdl(k_points<false, 2, false>, grid, 0, s, a);
    else return launch_pdl(k_points<false, 0, false>, grid, 0, s, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_cells(const PassArgs &a, int grid, cudaStream_t s) {
  if (a.fast == 1)
    return launch_pdl(k_cells<1>, grid, 0, s, a);
  if (a.fast == 2) return launch_pdl(k_cells<2>, grid, 0, s, a);
  return launch_pdl(k_cells<0>, grid, 0, s, a);
}

int accum_blocks_per_sm(int band_cells) {
  const size_t smem = accum_smem_bytes(band_cells);
  cudaFuncSetAttribute(k_accum<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_accum<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_accum<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_accum<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_accum<1>, kThreads, smem);
  return n > 0 ? n : 1;
}

cudaError_t launch_accum(const PassArgs &a, int grid, cudaStream_t s) {
  const size_t smem = accum_smem_bytes(a.band_cells);
  if (a.fast == 1)
    return launch_pdl(k_accum<1>, grid, smem, s, a);
  return launch_pdl(k_accum<2>, grid, smem, s, a);
}

cudaError_t launch_post(const PostArgs &a, cudaStream_t s) {
  k_post<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_smap(const PassArgs &a, int grid, size_t smem, cudaStream_t s) {
  // the opt-in shared-memory size is a per-device function attribute: set it for the current
  // device on every launch (a host-side call; maps may live on different devices)
  if (a.dbg_cell)
    cudaFuncSetAttribute(a.fast == 1 ? k_smap<true, 1> : k_smap<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  else
    cudaFuncSetAttribute(a.fast == 1 ? k_smap<false, 1> : k_smap<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSmapThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (a.dbg_cell) return a.fast == 1 ? cudaLaunchKernelEx(&cfg, k_smap<true, 1>, a) : cudaLaunchKernelEx(&cfg, k_smap<true, 2>, a);
  return a.fast == 1 ? cudaLaunchKernelEx(&cfg, k_smap<false, 1>, a) : cudaLaunchKernelEx(&cfg, k_smap<false, 2>, a);
}

cudaError_t launch_route(const PassArgs &a, const RouteArgs &r, int grid, cudaStream_t s) {
  k_route<<<grid, kThreads, 0, s>>>(a, r);
  return cudaGetLastError();
}

cudaError_t launch_image(const ImageArgs &a, cudaStream_t s) {
  k_image<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
  const int cnt = a.max_count > 0 ? a.max_count : 1;
  k_shift<<<dim3(cdiv(cnt, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_moments(const PcaArgs &a, cudaStream_t s) {
  const int tile = kPcaTileBytes / (4 * a.d);
  k_pca_moments<<<cdiv(a.geo.HW, tile), kThreads, kPcaTileBytes, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_project(const PcaArgs &a, int pass, cudaStream_t s) {
  k_pca_project<<<cdiv(a.geo.HW, kThreads), kThreads, 0, s>>>(a, pass);
  return cudaGetLastError();
}

cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s) {
  const long long words = (long long)a.n * (1 + a.R);
  const long long blocks = (words + kThreads - 1) / kThreads;
  k_merge<<<(unsigned)(blocks < 148LL * 16 ? blocks : 148LL * 16), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_read(const ReadArgs &a, cudaStream_t s) {
  k_read<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_write(const ReadArgs &a, cudaStream_t s) {
  k_write<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace memk
