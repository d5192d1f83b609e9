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
// fp64.  Persistent CTAs walk tiles of kPcaTile cells staged in shared memory (row stride
// kPcaTile + 1: conflict-free), every thread owning up to kPcaSlots of the moments in
// registers; each CTA writes its partial sums to its own row (no atomics), k_pca_eigen adds
// the rows in a fixed order.
constexpr int kPcaTile = 128;
constexpr int kPcaSlots = 9;  // ceil((64 + 64 * 65 / 2 + 1) / 256)
__global__ void __launch_bounds__(kThreads) k_pca_moments(const __grid_constant__ PcaArgs a) {
  extern __shared__ float s_x[];  // [d][kPcaTile + 1]
  __shared__ int s_n;
  const Geometry &g = a.geo;
  const int d = a.d, ld = kPcaTile + 1;
  const int pairs = d * (d + 1) / 2, nv = d + pairs + 1;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const long long mb = (long long)a.map * g.HW;
  int ra[kPcaSlots], rb[kPcaSlots];
  double acc[kPcaSlots];
#pragma unroll
  for (int j = 0; j < kPcaSlots; ++j) {  // slot v: sum x_v (v < d), pair (ra, rb), or the count
    const int v = threadIdx.x + j * kThreads;
    acc[j] = 0.0;
    ra[j] = rb[j] = -1;
    if (v < d) {
      ra[j] = v;
    } else if (v < d + pairs) {
      int q = v - d, r = 0;  // q -> (r, r + q'), row-major upper triangle
      while (q >= d - r) {
        q -= d - r;
        ++r;
      }
      ra[j] = r;
      rb[j] = r + q;
    }
  }
  long long nobs = 0;
  for (int c0 = blockIdx.x * kPcaTile; c0 < g.HW; c0 += gridDim.x * kPcaTile) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < kPcaTile; t += kThreads) {  // physical cells: order is irrelevant
      const int phys = c0 + t;
      const bool obs = phys < g.HW && a.st.flags[(long long)a.flag * g.BHW + mb + phys];
      for (int k = 0; k < d; ++k) s_x[k * ld + t] = obs ? vals[(long long)(a.word0 + k) * g.BHW + mb + phys] : 0.0f;
      if (obs) atomicAdd(&s_n, 1);
    }
    __syncthreads();
    nobs += s_n;
#pragma unroll
    for (int j = 0; j < kPcaSlots; ++j) {
      if (ra[j] < 0) continue;
      const float *xa = s_x + ra[j] * ld;
      double s = 0.0;
      if (rb[j] < 0) {
        for (int t = 0; t < kPcaTile; ++t) s += (double)xa[t];
      } else {
        const float *xb = s_x + rb[j] * ld;
        for (int t = 0; t < kPcaTile; ++t) s += (double)xa[t] * (double)xb[t];
      }
      acc[j] += s;
    }
    __syncthreads();
  }
  double *row = a.part + (long long)blockIdx.x * nv;
#pragma unroll
  for (int j = 0; j < kPcaSlots; ++j) {
    const int v = threadIdx.x + j * kThreads;
    if (v < d + pairs) row[v] = acc[j];
    else if (v == d + pairs) row[v] = (double)nobs;
  }
}

__device__ __forceinline__ unsigned long long ord_f64(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double f64_of_ord(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}

// pass 0: projections p_c = (x - mu) . e_c in fp64 (sequential over d) kept in a.proj, their
// min / max per component (a block reduction, then one atomic per CTA); pass 1: min-max
// scaling to [0, 1] (0 when max == min); unobserved cells 0.
__global__ void __launch_bounds__(kThreads) k_pca_project(const __grid_constant__ PcaArgs a, int pass) {
  __shared__ unsigned long long s_mm[2][kThreads / 32];
  const Geometry &g = a.geo;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool obs = false;
  long long cell = 0;
  if (t < g.HW) {
    const int row = t / g.W, col = t - (t / g.W) * g.W;
    const int2 ring = a.ring[a.map];
    cell = (long long)a.map * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
    obs = a.st.flags[(long long)a.flag * g.BHW + cell] != 0;
  }
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  for (int c = 0; c < a.k; ++c) {
    if (pass == 1) {
      if (t < g.HW) {
        const double lo = f64_of_ord(a.minmax[2 * c]), hi = f64_of_ord(a.minmax[2 * c + 1]);
        a.out[(long long)c * g.HW + t] =
            obs && hi > lo ? __double2float_rn((a.proj[(long long)c * g.HW + t] - lo) / (hi - lo)) : 0.0f;
      }
      continue;
    }
    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (obs) {
      double p = 0.0;
      for (int k = 0; k < a.d; ++k)
        p += ((double)vals[(long long)(a.word0 + k) * g.BHW + cell] - a.mean[k]) * a.comp[c * a.d + k];
      a.proj[(long long)c * g.HW + t] = p;
      kmin = kmax = ord_f64(p);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, kmin, o), y = __shfl_xor_sync(0xffffffffu, kmax, o);
      kmin = x < kmin ? x : kmin;
      kmax = y > kmax ? y : kmax;
    }
    if (lane == 0) {
      s_mm[0][wid] = kmin;
      s_mm[1][wid] = kmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // one atomic pair per CTA and component
      for (int w = 1; w < kThreads / 32; ++w) {
        kmin = s_mm[0][w] < kmin ? s_mm[0][w] : kmin;
        kmax = s_mm[1][w] > kmax ? s_mm[1][w] : kmax;
      }
      if (kmax) {
        atomicMin(&a.minmax[2 * c], kmin);
        atomicMax(&a.minmax[2 * c + 1], kmax);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- PCA eigen-solve on the device
// One CTA: the d x d covariance (fp64, from the moments of k_pca_moments) diagonalised by the
// parallel cyclic Jacobi method (round-robin ordering: every round rotates d/2 disjoint (p, q)
// pairs at once -- columns of A and V, then rows of A), sweeps until the off-diagonal mass is
// below 1e-26 of the total (at most 30 sweeps); then the top-k eigenvectors in
// decreasing eigenvalue order, each signed so that its largest-|.| coefficient is positive
// (reading D25), a component left 0 once the rank is exhausted (lambda <= 1e-12 lambda_max),
// the mean, and the min / max keys of the projection reset -- all on the stream, no host trip.
#ifndef MEM_PCA_TOL
#define MEM_PCA_TOL 1e-26  // Jacobi convergence: off-diagonal mass / total
#endif
constexpr int kPcaEigThreads = 512;
__global__ void __launch_bounds__(kPcaEigThreads) k_pca_eigen(const __grid_constant__ PcaArgs a) {
  extern __shared__ double s_m[];  // A [dp][dp], V [dp][dp] (dp = d rounded up to even)
  __shared__ int s_pair[2][32 * 4];
  __shared__ double s_cs[2][32 * 4];
  __shared__ double s_red[2][kPcaEigThreads / 32];
  __shared__ int s_done;
  const int d = a.d, dp = (d + 1) & ~1, ld = dp + 1, tid = threadIdx.x;  // ld: odd row stride (no bank conflicts)
  double *A = s_m, *V = s_m + dp * ld;
  const int pairs = d * (d + 1) / 2, nv = d + pairs + 1;
  for (int v = tid; v < nv; v += kPcaEigThreads) {  // the CTAs' partial moments, in a fixed order
    double s = 0.0;
    for (int b = 0; b < a.nparts; ++b) s += a.part[(long long)b * nv + v];
    a.sums[v] = s;
  }
  __syncthreads();
  const double n = a.sums[d + pairs];
  // covariance from the moments: c_ij = sum x_i x_j / n - mean_i mean_j (the host's formula);
  // a padding row/column (odd d) is zero and never rotates into the others
  for (int e = tid; e < dp * dp; e += kPcaEigThreads) {
    const int i = e / dp, j = e - i * dp;
    double c = 0.0;
    if (i < d && j < d && n > 0.0) {
      const int ra = i < j ? i : j, rb = i < j ? j : i;
      const int p = d + ra * d - ra * (ra - 1) / 2 + (rb - ra);
      c = a.sums[p] / n - (a.sums[i] / n) * (a.sums[j] / n);
    }
    A[i * ld + j] = c;
    V[i * ld + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;  // convergence: off-diagonal mass <= 1e-26 of the total
    for (int e = tid; e < dp * dp; e += kPcaEigThreads) {
      const int i = e / dp, j = e - i * dp;
      const double x = A[i * ld + j] * A[i * ld + j];
      tot += x;
      if (i != j) off += x;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((tid & 31) == 0) {
      s_red[0][tid >> 5] = off;
      s_red[1][tid >> 5] = tot;
    }
    __syncthreads();
    if (tid == 0) {
      double o2 = 0.0, t2 = 0.0;
      for (int w = 0; w < kPcaEigThreads / 32; ++w) {
        o2 += s_red[0][w];
        t2 += s_red[1][w];
      }
      s_done = (o2 <= MEM_PCA_TOL * t2 || o2 == 0.0) ? 1 : 0;
    }
    __syncthreads();
    if (s_done) break;
    for (int round = 0; round < dp - 1; ++round) {
      // round-robin pairing of dp indices: index 0 fixed, the others rotate
      const int h = dp / 2;
      if (tid < h) {
        int p, q;
        if (tid == 0) {
          p = 0;
          q = 1 + (round % (dp - 1));
        } else {
          p = 1 + ((round + tid) % (dp - 1));
          q = 1 + ((round + dp - 1 - tid) % (dp - 1));
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        const double apq = A[p * ld + q];
        double c = 1.0, sn = 0.0;
        if (apq != 0.0) {
          const double theta = (A[q * ld + q] - A[p * ld + p]) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          sn = t * c;
        }
        s_pair[0][tid] = p;
        s_pair[1][tid] = q;
        s_cs[0][tid] = c;
        s_cs[1][tid] = sn;
      }
      __syncthreads();
      for (int e = tid; e < h * dp; e += kPcaEigThreads) {  // A <- A J, V <- V J (columns)
        const int pi = e / dp, k = e - pi * dp;
        const int p = s_pair[0][pi], q = s_pair[1][pi];
        const double c = s_cs[0][pi], sn = s_cs[1][pi];
        const double akp = A[k * ld + p], akq = A[k * ld + q];
        A[k * ld + p] = c * akp - sn * akq;
        A[k * ld + q] = sn * akp + c * akq;
        const double vkp = V[k * ld + p], vkq = V[k * ld + q];
        V[k * ld + p] = c * vkp - sn * vkq;
        V[k * ld + q] = sn * vkp + c * vkq;
      }
      __syncthreads();
      for (int e = tid; e < h * dp; e += kPcaEigThreads) {  // A <- J^T A (rows)
        const int pi = e / dp, k = e - pi * dp;
        const int p = s_pair[0][pi], q = s_pair[1][pi];
        const double c = s_cs[0][pi], sn = s_cs[1][pi];
        const double apk = A[p * ld + k], aqk = A[q * ld + k];
        A[p * ld + k] = c * apk - sn * aqk;
        A[q * ld + k] = sn * apk + c * aqk;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {  // top-k by eigenvalue (stable: the lower index first on ties), signs (D25)
    double *mean = const_cast<double *>(a.mean), *comp = const_cast<double *>(a.comp);
    for (int i = 0; i < d; ++i) mean[i] = n > 0.0 ? a.sums[i] / n : 0.0;
    for (int e = 0; e < a.k * d; ++e) comp[e] = 0.0;
    if (n > 0.0) {
      unsigned long long used[4] = {0ull, 0ull, 0ull, 0ull};  // d <= kMaxCh = 256
      double lmax = 0.0;
      for (int c = 0; c < a.k; ++c) {
        int best = -1;
        for (int i = 0; i < d; ++i) {
          if (used[i >> 6] >> (i & 63) & 1ull) continue;
          if (best < 0 || A[i * ld + i] > A[best * ld + best]) best = i;
        }
        used[best >> 6] |= 1ull << (best & 63);
        const double w = A[best * ld + best];
        if (c == 0) lmax = w;
        if (!(w > 0.0) || w <= 1e-12 * lmax) break;  // rank exhausted: the component stays 0
        int big = 0;
        for (int i = 1; i < d; ++i)
          if (fabs(V[i * ld + best]) > fabs(V[big * ld + best])) big = i;
        const double sg = V[big * ld + best] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < d; ++i) comp[c * d + i] = sg * V[i * ld + best];
      }
    }
    for (int c = 0; c < a.k; ++c) {  // min keys start at all-ones, max keys at zero
      a.minmax[2 * c] = ~0ull;
      a.minmax[2 * c + 1] = 0ull;
    }
  }
}
