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
// fp64 (products of fp32 values are exact in fp64).  Persistent CTAs walk tiles of kPcaTile
// cells staged in shared memory in fp64 by all threads ([channel][cell], channels padded to a
// multiple of 4 with zeros, the observed flags staged first); thread b < nb (nb + 1) / 2 owns
// the 4 x 4 block (bi, bj), bi <= bj, of the Gram matrix in 16 fp64 registers and the
// diagonal-block threads the sums of their 4 channels; each CTA writes its partial moments to
// its own row (no atomics), k_pca_eigen adds the rows in a fixed order.
constexpr int kPcaTile = 128;
__host__ __device__ inline int pca_ldc(int d) { return ((d + 3) & ~3) * (kPcaTile + 1); }  // doubles of the staged tile
__global__ void __launch_bounds__(kThreads) k_pca_moments(const __grid_constant__ PcaArgs a) {
  extern __shared__ double s_xd[];  // [d4][kPcaTile + 1]: the tile's values in fp64, converted once
  __shared__ unsigned char s_obs[kPcaTile];
  __shared__ int s_n;
  const Geometry &g = a.geo;
  const int d = a.d, d4 = (d + 3) & ~3, nb = d4 / 4, ld = kPcaTile + 1;
  const int pairs = d * (d + 1) / 2, nv = d + pairs + 1;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const long long mb = (long long)a.map * g.HW;
  const int nblk = nb * (nb + 1) / 2;
  // d <= 64 (mem_pca_readout): at most 136 blocks, one per thread
  const int b = threadIdx.x;
  int bi = 0, bj = 0;
  if (b < nblk) {  // b -> (bi, bj), row-major upper triangle of blocks
    int q = b;
    while (q >= nb - bi) {
      q -= nb - bi;
      ++bi;
    }
    bj = bi + q;
  }
  double acc[4][4], sum[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    sum[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  }
  long long nobs = 0;
  double *row = a.part + (long long)blockIdx.x * nv;
  for (int c0 = blockIdx.x * kPcaTile; c0 < g.HW; c0 += gridDim.x * kPcaTile) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    if (threadIdx.x < kPcaTile) {  // physical cells: order is irrelevant
      const int phys = c0 + threadIdx.x;
      const bool obs = phys < g.HW && a.st.flags[(long long)a.flag * g.BHW + mb + phys];
      s_obs[threadIdx.x] = obs;
      if (obs) atomicAdd(&s_n, 1);
    }
    __syncthreads();
    // every thread stages: channel k of cell t at [k][t] (coalesced loads, conflict-free stores)
    for (int e = threadIdx.x; e < kPcaTile * d4; e += kThreads) {
      const int k = e / kPcaTile, t = e - k * kPcaTile;
      const int phys = c0 + t;
      s_xd[k * ld + t] = k < d && s_obs[t] ? (double)vals[(long long)(a.word0 + k) * g.BHW + mb + phys] : 0.0;
    }
    __syncthreads();
    nobs += s_n;
    if (b < nblk) {
      const double *xa = s_xd + 4 * bi * ld, *xb = s_xd + 4 * bj * ld;
#pragma unroll 2
      for (int t = 0; t < kPcaTile; ++t) {
        double va[4], vb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          va[i] = xa[i * ld + t];
          vb[i] = xb[i * ld + t];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sum[i] += va[i];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] += va[i] * vb[j];  // exact products of fp32 values
        }
      }
    }
    __syncthreads();
  }
  if (b < nblk) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ra = 4 * bi + i;
      if (ra >= d) continue;
      if (bi == bj) row[ra] = sum[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rb = 4 * bj + j;
        if (rb < ra || rb >= d) continue;
        row[d + ra * d - ra * (ra - 1) / 2 + (rb - ra)] = acc[i][j];
      }
    }
  }
  if (threadIdx.x == 0) row[d + pairs] = (double)nobs;
}

__device__ __forceinline__ unsigned long long ord_f64(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double f64_of_ord(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}

// pass 0: projections p_c = (x - mu) . e_c in fp64 (sequential over d; 4 components per read
// of the cell's values) kept in a.proj, their
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
  if (pass == 1) {
    for (int c = 0; c < a.k; ++c)
      if (t < g.HW) {
        const double lo = f64_of_ord(a.minmax[2 * c]), hi = f64_of_ord(a.minmax[2 * c + 1]);
        a.out[(long long)c * g.HW + t] =
            obs && hi > lo ? __double2float_rn((a.proj[(long long)c * g.HW + t] - lo) / (hi - lo)) : 0.0f;
      }
    return;
  }
  for (int c0 = 0; c0 < a.k; c0 += 4) {  // 4 components per pass over the cell's values
    const int nc = a.k - c0 < 4 ? a.k - c0 : 4;
    double p[4] = {0.0, 0.0, 0.0, 0.0};
    if (obs)
      for (int k = 0; k < a.d; ++k) {
        const double x = (double)vals[(long long)(a.word0 + k) * g.BHW + cell] - a.mean[k];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nc) p[j] += x * a.comp[(c0 + j) * a.d + k];
      }
    for (int j = 0; j < nc; ++j) {
      const int c = c0 + j;
      unsigned long long kmin = ~0ull, kmax = 0ull;
      if (obs) {
        a.proj[(long long)c * g.HW + t] = p[j];
        kmin = kmax = ord_f64(p[j]);
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
}

// ---------------------------------------------------------------- PCA eigen-solve on the device
// One CTA, fp64, d <= 64 (mem_pca_readout):
//   1. the covariance C = sum x x^T / n - mu mu^T from the moments of k_pca_moments (the CTAs'
//      partial rows added in a fixed order);
//   2. Householder tridiagonalisation Q^T C Q = T (d - 2 reflections: the norm and the
//      reflector by warp 0, p = beta A v with 8 lanes per row, A -= v w^T + w v^T with
//      w = p - (beta/2)(v^T p) v -- three barriers per reflection; v kept in place below the
//      sub-diagonal);
//   3. the top-k eigenvalues of T by Sturm-count multisection (one warp per eigenvalue, 32
//      points per step, to relative width ~4 eps);
//   4. their eigenvectors by inverse iteration on T - lambda I (tridiagonal LU with partial
//      pivoting, 3 solves, one lane each), orthogonalised within clusters of close eigenvalues
//      (Gram-Schmidt in eigenvalue order), mapped back through the reflectors (one warp each);
//   5. each signed so that its largest-|.| coefficient is positive (reading D25); components
//      with lambda <= 1e-12 lambda_max (or <= 0) are left 0 (rank exhausted); the
//      mean and the min / max keys of the projection reset -- all on the stream, no host trip.
// (The oracle uses power iteration with deflation; both converge to the eigenvectors of the
// same fp64 covariance, compared at 1e-4 on the scaled outputs, reading D28.)
constexpr int kPcaEigThreads = 512;
constexpr int kPcaMaxD = 64;
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// 1 / a to a few ulp: the MUFU approximation and three Newton steps (|a| >= DBL_MIN here)
__device__ __forceinline__ double rcp64(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  r = r + r * (1.0 - a * r);  // unfused (no FMA anywhere in the library, tests/test_abi.py)
  r = r + r * (1.0 - a * r);
  return r + r * (1.0 - a * r);
}
// number of eigenvalues of T (diagonal dg, squared off-diagonal e2) below x (Sturm count)
__device__ __forceinline__ int sturm_count(const double *dg, const double *e2, int n, double x, double pivmin) {
  double q = dg[0] - x;
  int c = q < 0.0;
  for (int i = 1; i < n; ++i) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = (dg[i] - x) - e2[i - 1] * rcp64(q);
    c += q < 0.0;
  }
  return c;
}
// LU factors (partial pivoting) of T - lam I: U's diagonals u0 (stored inverted), u1, u2, the
// multipliers and the row swaps (n <= 64)
__device__ void tri_lu(const double *dg, const double *ev, int n, double lam, double pivmin, double *u0, double *u1,
                       double *u2, double *mlt, unsigned long long &sw) {
  sw = 0ull;
  double ai = dg[0] - lam, bi = n > 1 ? ev[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    const double ci = ev[i], an = dg[i + 1] - lam, bn = i + 1 < n - 1 ? ev[i + 1] : 0.0;
    if (fabs(ai) >= fabs(ci)) {
      if (fabs(ai) < pivmin) ai = ai < 0.0 ? -pivmin : pivmin;
      const double ri = rcp64(ai), m = ci * ri;
      u0[i] = ri;
      u1[i] = bi;
      u2[i] = 0.0;
      mlt[i] = m;
      ai = an - m * bi;
      bi = bn;
    } else {
      const double ri = rcp64(ci), m = ai * ri;
      u0[i] = ri;
      u1[i] = an;
      u2[i] = bn;
      mlt[i] = m;
      sw |= 1ull << i;
      ai = bi - m * an;
      bi = -m * bn;
    }
  }
  if (fabs(ai) < pivmin) ai = ai < 0.0 ? -pivmin : pivmin;
  u0[n - 1] = rcp64(ai);
}
__device__ void tri_solve(int n, const double *u0, const double *u1, const double *u2, const double *mlt,
                          unsigned long long sw, double *y, bool apply_l) {
  if (apply_l)
    for (int i = 0; i < n - 1; ++i) {
      if (sw >> i & 1ull) {
        const double t = y[i];
        y[i] = y[i + 1];
        y[i + 1] = t - mlt[i] * y[i];
      } else {
        y[i + 1] -= mlt[i] * y[i];
      }
    }
  for (int i = n - 1; i >= 0; --i) {
    double t = y[i];
    if (i + 1 < n) t -= u1[i] * y[i + 1];
    if (i + 2 < n) t -= u2[i] * y[i + 2];
    y[i] = t * u0[i];
  }
}

// the CTAs' partial moment rows summed in a fixed order (deterministic): CTA b owns 32 sums,
// warp w adds the rows [w P / 8, (w + 1) P / 8) (coalesced over the lanes), warp 0 the 8 parts
__global__ void __launch_bounds__(kThreads) k_pca_sum(const __grid_constant__ PcaArgs a) {
  __shared__ double s_part[kThreads / 32][32];
  const int d = a.d, nv = d + d * (d + 1) / 2 + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + lane;
  constexpr int W = kThreads / 32;
  const int b0 = (int)((long long)a.nparts * wid / W), b1 = (int)((long long)a.nparts * (wid + 1) / W);
  double s = 0.0;
  if (v < nv) {
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(a.part + (long long)(b + u) * nv + v);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += x[u];
    }
    for (; b < b1; ++b) s += __ldcg(a.part + (long long)b * nv + v);
  }
  s_part[wid][lane] = s;
  __syncthreads();
  if (wid == 0 && v < nv) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) t += s_part[w][lane];
    a.sums[v] = t;
  }
}

__global__ void __launch_bounds__(kPcaEigThreads) k_pca_eigen(const __grid_constant__ PcaArgs a) {
  extern __shared__ double s_m[];  // A [d][d + 1]; X [k][d] (eigenvectors); LU scratch [4][k][d]
  __shared__ double s_dg[kPcaMaxD], s_ev[kPcaMaxD], s_e2[kPcaMaxD], s_beta[kPcaMaxD], s_p[kPcaMaxD], s_v[kPcaMaxD];
  __shared__ double s_lam[kPcaMaxD];
  __shared__ double s_bounds[3];
  __shared__ int s_fa[kPcaEigThreads / 32];
  const int d = a.d, ld = d + 1, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#if MEM_PCA_CLOCKS
  long long ck[9];
  const long long ck_start = clock64();
#endif
  const int K = a.k;
  double *A = s_m, *X = s_m + d * ld, *LU = X + K * d;
  const int pairs = d * (d + 1) / 2;
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[0] = clock64();
#endif
  const double n = a.sums[d + pairs];
  // 1. covariance from the moments: c_ij = sum x_i x_j / n - mean_i mean_j
  for (int e = tid; e < d * d; e += kPcaEigThreads) {
    const int i = e / d, j = e - i * d;
    double c = 0.0;
    if (n > 0.0) {
      const int ra = i < j ? i : j, rb = i < j ? j : i;
      const int p = d + ra * d - ra * (ra - 1) / 2 + (rb - ra);
      c = a.sums[p] / n - (a.sums[i] / n) * (a.sums[j] / n);
    }
    A[i * ld + j] = c;
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[1] = clock64();
#endif
  // 2. Householder tridiagonalisation: reflection k zeroes A[k+2..d-1][k]
  for (int k = 0; k + 2 < d; ++k) {
    const int m = d - k - 1;  // x = A[k+1..d-1][k]
    double *col = A + (k + 1) * ld + k;  // col[i * ld] = x_i
    if (wid == 0) {
      double s = 0.0;
      for (int i = 1 + lane; i < m; i += 32) s += col[i * ld] * col[i * ld];
      s = warp_sum_d(s);
      const double x0 = col[0];
      const double nrm = sqrt(x0 * x0 + s), alpha = x0 <= 0.0 ? nrm : -nrm;
      for (int i = lane; i < m; i += 32) s_v[i] = i == 0 ? x0 - alpha : col[i * ld];  // v = x - alpha e1
      if (lane == 0) {
        if (s == 0.0) {  // already reduced: no reflection
          s_beta[k] = 0.0;
          s_ev[k] = x0;
        } else {
          col[0] = x0 - alpha;                         // kept in place for the back-transformation
          s_beta[k] = 1.0 / (nrm * nrm - x0 * alpha);  // 2 / (v^T v)
          s_ev[k] = alpha;
        }
      }
    }
    __syncthreads();
    const double beta = s_beta[k];
    if (beta == 0.0) continue;  // uniform
    {  // p = beta A22 v, 8 lanes per row
      const int i = tid >> 3, part = tid & 7;
      double s = 0.0;
      if (i < m) {
        const double *row = A + (k + 1 + i) * ld + (k + 1);
        for (int j = part; j < m; j += 8) s += row[j] * s_v[j];
      }
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      if (i < m && part == 0) s_p[i] = beta * s;
    }
    __syncthreads();

    {  // K = (beta / 2) v^T p (every warp, redundantly), w = p - K v, A22 -= v w^T + w v^T;
       // thread: column j = tid % 64, rows tid / 64 + 8 r
      double s = 0.0;
      for (int i = lane; i < m; i += 32) s += s_v[i] * s_p[i];
      const double Kc = 0.5 * beta * warp_sum_d(s);
      const int j = tid & 63;
      if (j < m) {
        const double vj = s_v[j], wj = s_p[j] - Kc * vj;
        double *aj = A + (k + 1) * ld + (k + 1) + j;
        for (int i = tid >> 6; i < m; i += kPcaEigThreads / 64) {
          const double vi = s_v[i], wi = s_p[i] - Kc * vi;
          aj[i * ld] -= vi * wj + wi * vj;
        }
      }
    }
    __syncthreads();
  }

#if MEM_PCA_CLOCKS
  if (tid == 0) ck[2] = clock64();
#endif
  // T: diagonal s_dg, off-diagonal s_ev (the last one was never reflected)
  if (tid < d) s_dg[tid] = A[tid * ld + tid];
  if (tid == 0 && d >= 2) s_ev[d - 2] = A[(d - 1) * ld + (d - 2)];
  __syncthreads();
  if (tid < d) s_e2[tid] = tid < d - 1 ? s_ev[tid] * s_ev[tid] : 0.0;
  if (tid == 0) {  // Gershgorin interval and the pivot floor
    double lo = 0.0, hi = 0.0, tn = 0.0, emax2 = 0.0;
    for (int i = 0; i < d; ++i) {
      const double r = (i > 0 ? fabs(s_ev[i - 1]) : 0.0) + (i < d - 1 ? fabs(s_ev[i]) : 0.0);
      lo = i == 0 ? s_dg[i] - r : fmin(lo, s_dg[i] - r);
      hi = i == 0 ? s_dg[i] + r : fmax(hi, s_dg[i] + r);
      if (i < d - 1) emax2 = fmax(emax2, s_ev[i] * s_ev[i]);
    }
    tn = fmax(fabs(lo), fabs(hi));
    s_bounds[0] = lo - 4.0 * DBL_EPSILON * tn - DBL_MIN;
    s_bounds[1] = hi + 4.0 * DBL_EPSILON * tn + DBL_MIN;
    s_bounds[2] = fmax(DBL_MIN, DBL_MIN / DBL_EPSILON * emax2);  // LAPACK's pivmin
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[3] = clock64();
#endif
  const double pivmin = s_bounds[2];
  // 3. the j-th largest eigenvalue (index d - 1 - j ascending): G = 16 / K warps per eigenvalue
  //    (at least one), 32 G points per step; every warp of a group takes the same decisions
  {
    constexpr int NW = kPcaEigThreads / 32;
    const int G = K >= NW ? 1 : NW / K, slots = NW / G;
    const int slot = wid / G, gw = wid - slot * G;
    for (int j0 = 0; j0 < K; j0 += slots) {
      const int j = j0 + slot;
      const bool mine = slot < slots && j < K;
      const int r = d - 1 - (mine ? j : 0);
      double lo = s_bounds[0], hi = s_bounds[1];
      for (int it = 0; it < 64; ++it) {
        const double w = hi - lo;
        const bool conv = !mine || !(w > 4.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin);
        if (__syncthreads_and(conv)) break;
        const double x = lo + w * (double)(gw * 32 + lane + 1) / (double)(32 * G + 1);
        const bool below = mine && !conv && sturm_count(s_dg, s_e2, d, x, pivmin) <= r;  // lambda_r >= x
        const unsigned bm = __ballot_sync(0xffffffffu, below);
        if (lane == 0) s_fa[wid] = bm == 0xffffffffu ? 32 : __ffs(~bm) - 1;
        __syncthreads();
        if (mine && !conv) {  // the first transition over the group's points (increasing in gw, lane)
          int q = G * 32;
          for (int u = 0; u < G; ++u)
            if (s_fa[slot * G + u] < 32) {
              q = u * 32 + s_fa[slot * G + u];
              break;
            }
          const double nlo = q > 0 ? lo + w * (double)q / (double)(32 * G + 1) : lo;
          const double nhi = q < 32 * G ? lo + w * (double)(q + 1) / (double)(32 * G + 1) : hi;
          lo = nlo;
          hi = nhi;
        }
      }
      if (mine && gw == 0 && lane == 0) s_lam[j] = 0.5 * (lo + hi);
    }
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[4] = clock64();
#endif
  // 4. inverse iteration, one lane per eigenvalue (tridiagonal space), then clusters
  //    orthogonalised in order and the vectors mapped back through the reflectors
  const double tnorm = fmax(fabs(s_bounds[0]), fabs(s_bounds[1]));
  for (int j = tid; j < K; j += kPcaEigThreads) {
    double *x = X + j * d, *u0 = LU + (0 * K + j) * d, *u1 = LU + (1 * K + j) * d, *u2 = LU + (2 * K + j) * d,
           *ml = LU + (3 * K + j) * d;
    unsigned long long sw;
    tri_lu(s_dg, s_ev, d, s_lam[j], fmax(pivmin, DBL_EPSILON * tnorm), u0, u1, u2, ml, sw);
    for (int i = 0; i < d; ++i) x[i] = 1.0 + 1e-3 * (double)((i * 7 + j * 3) % 11);  // not orthogonal to any eigenvector in practice
    for (int it = 0; it < 3; ++it) {
      tri_solve(d, u0, u1, u2, ml, sw, x, it > 0);
      double nr = 0.0;
      for (int i = 0; i < d; ++i) nr += x[i] * x[i];
      nr = 1.0 / sqrt(nr);
      for (int i = 0; i < d; ++i) x[i] *= nr;
    }
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[5] = clock64();
#endif
  if (wid == 0) {  // Gram-Schmidt within clusters (|lambda_i - lambda_j| <= 1e-3 |T|), eigenvalue order
    for (int j = 1; j < K; ++j)
      for (int i = 0; i < j; ++i) {
        if (!(fabs(s_lam[i] - s_lam[j]) <= 1e-3 * tnorm)) continue;
        double s = 0.0;
        for (int q = lane; q < d; q += 32) s += X[i * d + q] * X[j * d + q];
        s = warp_sum_d(s);
        double nr = 0.0;
        for (int q = lane; q < d; q += 32) {
          X[j * d + q] -= s * X[i * d + q];
          nr += X[j * d + q] * X[j * d + q];
        }
        nr = 1.0 / sqrt(warp_sum_d(nr));
        for (int q = lane; q < d; q += 32) X[j * d + q] *= nr;
        __syncwarp();
      }
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[6] = clock64();
#endif
  for (int j = wid; j < K; j += kPcaEigThreads / 32) {  // x <- H_0 H_1 ... H_{d-3} x
    double *x = X + j * d;
    for (int k = d - 3; k >= 0; --k) {
      const double beta = s_beta[k];
      if (beta == 0.0) continue;
      const int m = d - k - 1;
      const double *col = A + (k + 1) * ld + k;
      double s = 0.0;
      for (int i = lane; i < m; i += 32) s += col[i * ld] * x[k + 1 + i];
      s = beta * warp_sum_d(s);
      for (int i = lane; i < m; i += 32) x[k + 1 + i] -= s * col[i * ld];
      __syncwarp();
    }
  }
  __syncthreads();
#if MEM_PCA_CLOCKS
  if (tid == 0) ck[7] = clock64();
#endif
  if (tid == 0) {  // 5. order, rank, signs (D25); mean; projection keys reset
    double *mean = const_cast<double *>(a.mean), *comp = const_cast<double *>(a.comp);
    for (int i = 0; i < d; ++i) mean[i] = n > 0.0 ? a.sums[i] / n : 0.0;
    for (int e = 0; e < K * d; ++e) comp[e] = 0.0;
    if (n > 0.0) {
      const double lmax = s_lam[0];
      for (int c = 0; c < K; ++c) {
        const double w = s_lam[c];
        if (!(w > 0.0) || w <= 1e-12 * lmax) break;  // rank exhausted: the component stays 0
        const double *x = X + c * d;
        int big = 0;
        for (int i = 1; i < d; ++i)
          if (fabs(x[i]) > fabs(x[big])) big = i;
        const double sg = x[big] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < d; ++i) comp[c * d + i] = sg * x[i];
      }
    }
    for (int c = 0; c < K; ++c) {  // min keys start at all-ones, max keys at zero
      a.minmax[2 * c] = ~0ull;
      a.minmax[2 * c + 1] = 0ull;
    }
#if MEM_PCA_CLOCKS
    printf("pca eigen cycles: sums %lld cov %lld tridiag %lld bounds %lld eigvals %lld inviter %lld gs %lld backtr %lld\n",
           ck[0] - ck_start, ck[1] - ck[0], ck[2] - ck[1], ck[3] - ck[2], ck[4] - ck[3], ck[5] - ck[4], ck[6] - ck[5], ck[7] - ck[6]);
#endif
  }
}
