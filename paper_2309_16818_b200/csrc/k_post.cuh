// k_post.cuh -- k_post: post-processing plugins (NEXT-3).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

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
