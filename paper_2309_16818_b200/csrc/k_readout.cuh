// k_readout.cuh -- k_shift (eager a13), k_read / k_write (a14), PCA readout (C4).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

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
