// point_pass.cuh -- a2-a6 for one point (bin_point) and the top-k class input decoder (NEXT-2).
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
                                              const mem_noise &np, int map_base, float r2lo, float r2hi) {
  PointOut o;
  o.code = MEM_CODE_NONFINITE;
  o.lcell = -1;
  o.cell = -1;
  o.z = 0.0f;
  o.v = 0.0f;
  o.test = false;
  if (!finite3(px, py, pz)) return o;                   // a2: finiteness
  const float r2 = (px * px + py * py) + pz * pz;       // a2: sensor-frame range (D9)
  // r_min <= sqrtf(r2) <= r_max, decided on r2 against the exact equivalent bounds the host
  // derived from the correctly rounded sqrt (PassArgs::r2lo / r2hi): the oracle's decision
  if (!(r2 >= r2lo && r2 <= r2hi)) {
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

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

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


// the channel value k of a bound group for the point at index pi (dense or top-k, D38)
__device__ __forceinline__ float chan_value(const PassArgs &a, const BindDesc &b, unsigned pi, int k) {
  const float *ch = a.pts + (long long)pi * a.stride + 3 + b.ch_offset;
  if (b.topk > 0) return TopK{ch, 1, b.topk, b.g.nch - 1}.value(k);
  return __ldg(ch + k);
}

// D31 / D38: the group takes the point iff its channels are finite (top-k: valid pairs);
// colour never skips (D20)
__device__ __forceinline__ bool chan_ok(const PassArgs &a, const BindDesc &b, unsigned pi) {
  if (b.g.rule == MEM_COLOR) return true;
  const float *ch = a.pts + (long long)pi * a.stride + 3 + b.ch_offset;
  if (b.topk > 0) return TopK{ch, 1, b.topk, b.g.nch - 1}.ok();
  for (int k = 0; k < b.nch; ++k)
    if (!isfinite(__ldg(ch + k))) return false;
  return true;
}

// D19: (conf, lowest class) of the point as one u64 key
__device__ __forceinline__ unsigned long long chan_key(const PassArgs &a, const BindDesc &b, unsigned pi) {
  const float *ch = a.pts + (long long)pi * a.stride + 3 + b.ch_offset;
  if (b.topk > 0) return TopK{ch, 1, b.topk, b.g.nch - 1}.key();
  int best = 0;
  float bv = __ldg(ch);
  for (int k = 1; k < b.nch; ++k) {
    const float c = __ldg(ch + k);
    if (c > bv) {
      bv = c;
      best = k;
    }
  }
  return ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
}

