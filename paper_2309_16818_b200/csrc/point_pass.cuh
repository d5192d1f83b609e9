// point_pass.cuh -- a2-a8 device functions: binning, the Mahalanobis gate, REDs, warp aggregation, top-k, accumulate_warp.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

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
                                              const mem_noise &np, int map_base) {
  PointOut o;
  o.code = MEM_CODE_NONFINITE;
  o.lcell = -1;
  o.cell = -1;
  o.z = 0.0f;
  o.v = 0.0f;
  o.test = false;
  if (!finite3(px, py, pz)) return o;                   // a2: finiteness
  const float r2 = (px * px + py * py) + pz * pz;       // a2: sensor-frame range (D9)
  const float r = __fsqrt_rn(r2);                       // IEEE sqrt, as the oracle's sqrtf
  if (!(np.r_min <= r && r <= np.r_max)) {
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
  const float fr = __fdiv_rn(x, g.res) + g.hH;           // a5: bin (D13), IEEE division
  const float fc = __fdiv_rn(y, g.res) + g.hW;
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
#ifndef MEM_STATE_LD
#define MEM_STATE_LD 2  // state gathers: 0 plain LDG, 1 __ldg (.nc), 2 __ldcg (L2 only)
#endif
template <int N>
__device__ __forceinline__ void mahalanobis(PointOut (&o)[N], const State &st, const Geometry &g, float tau2) {
  const float *elev = reinterpret_cast<const float *>(st.words) + (long long)kWordElev * g.BHW;
  const float *var = reinterpret_cast<const float *>(st.words) + (long long)kWordVar * g.BHW;
  float hv[N], sv[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    hv[u] = sv[u] = __int_as_float(0x7fc00000);
    if (o[u].test) {
#if MEM_STATE_LD == 1
      hv[u] = __ldg(elev + o[u].cell);
      sv[u] = __ldg(var + o[u].cell);
#elif MEM_STATE_LD == 2
      hv[u] = __ldcg(elev + o[u].cell);
      sv[u] = __ldcg(var + o[u].cell);
#else
      hv[u] = elev[o[u].cell];
      sv[u] = var[o[u].cell];
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
  // the fast paths' records are 4 words (mem_api selects them only then)
  unsigned long long *rec = a.rec + (long long)sc * (kFast != 0 ? 4 : a.R);
  const bool act = o.cell >= 0;
  const unsigned act_b = __ballot_sync(0xffffffffu, act);
  if (act_b == 0u) return;
  const int lane = threadIdx.x & 31;
  const unsigned key = act ? (unsigned)sc : 0xffffffffu;
  // aggregate only when it pays: >= 16 lanes repeat their neighbour's cell (dense clouds; a
  // LiDAR scan line has ~1.5 points per cell and is faster with one RED set per lane)
  const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned dup = __ballot_sync(0xffffffffu, act && lane > 0 && prev == key);
  const bool agg = __popc(dup) >= 16 && !ABLATE(a, 64u);
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
    } else if (__popc(dup) >= MEM_PAIR_MIN && !ABLATE(a, 64u)) {
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
