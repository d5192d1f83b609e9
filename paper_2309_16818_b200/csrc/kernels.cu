// kernels.cu -- the sm_100a kernels of the MEM hot path.
//
//   k_point  a2-a8   one thread per point: load, finiteness/range/height filters, transform,
//                    bin, noise variance, Mahalanobis test against the pre-frame state,
//                    scatter-accumulate the sufficient statistics (native 64-bit REDs)
//   k_cell   a9-a10  one thread per touched cell: Kalman height fusion, per-group rules,
//                    re-zero the statistics it consumed
//   k_image  a11-a12 one thread per valid cell: project, frustum, gather, fuse (N_j = 1)
//   k_shift  a13     reset the scrolled-in strips of the ring buffer, advance ring offsets
//   k_read   a14     unroll the ring into logical row-major fp32, derive theta / NaN
//
// Everything is stream-ordered; no kernel synchronises the host.
#include <cmath>

#include "kernels.cuh"

namespace memk {

// ---------------------------------------------------------------- loads
__device__ __forceinline__ float4 ld_stream_f4(const float *p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ bool finite3(float a, float b, float c) {
  return isfinite(a) && isfinite(b) && isfinite(c);
}

__device__ __forceinline__ int stat_slot(int code) {
  // mem_stats order: n_input, nonfinite, range, height, oob, inlier, outlier, touched
  return code == MEM_CODE_INLIER ? 5 : code == MEM_CODE_OUTLIER ? 6 : code - 1;
}

// ---------------------------------------------------------------- k_point (a2-a8)
template <bool kDebug>
__global__ void __launch_bounds__(kPointThreads) k_point(const __grid_constant__ PointArgs a) {
  const int m = blockIdx.y;
  long long beg = 0, end = a.n_single;
  if (a.offsets) {
    beg = a.offsets[m];
    end = a.offsets[m + 1];
  }
  const long long base = beg + (long long)blockIdx.x * kPointsPerBlock;
  if (base >= end) return;  // block-uniform

  __shared__ unsigned s_cnt[6];
  if (threadIdx.x < 6) s_cnt[threadIdx.x] = 0;
  __syncthreads();

  const MapFrame &f = a.frames ? a.frames[m] : a.f0;
  const int2 ring = a.ring[m];
  const Geometry &g = a.geo;
  const mem_noise &np = a.np;
  const long long map_base = (long long)m * g.HW;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const uint8_t *valid = a.st.flags + (long long)kFlagValid * g.BHW;
  unsigned long long *acc = a.st.acc;
  const int lane = threadIdx.x & 31;

#pragma unroll
  for (int u = 0; u < kPointsPerThread; ++u) {
    const long long i = base + (long long)u * kPointThreads + threadIdx.x;
    const bool live = i < end;
    int code = MEM_CODE_NONFINITE;
    int lcell = -1;
    long long cell = -1;
    float z = 0.0f, v = 0.0f;
    float ch0 = 0.0f;  // stride-4 points: the one channel arrives with the float4
    const float *p = a.pts + i * (long long)a.stride;
    if (live) {
      float px, py, pz;
      if (a.vec4) {
        const float4 q = ld_stream_f4(p);
        px = q.x; py = q.y; pz = q.z; ch0 = q.w;
      } else {
        px = __ldg(p); py = __ldg(p + 1); pz = __ldg(p + 2);
      }
      if (finite3(px, py, pz)) {                          // a2: finiteness
        const float r2 = (px * px + py * py) + pz * pz;    // a2: range in the sensor frame (D9)
        const float r = sqrtf(r2);
        if (!(np.r_min <= r && r <= np.r_max)) {
          code = MEM_CODE_RANGE;
        } else {
          // a3: q = R p, fixed order, no FMA ("point trsf.")
          const float qx = (f.R[0] * px + f.R[1] * py) + f.R[2] * pz;
          const float qy = (f.R[3] * px + f.R[4] * py) + f.R[5] * pz;
          const float qz = (f.R[6] * px + f.R[7] * py) + f.R[8] * pz;
          if (!(np.h_min <= qz && qz <= np.h_max)) {       // a4: height filter (D9)
            code = MEM_CODE_HEIGHT;
          } else {
            const float x = qx + f.t[0], y = qy + f.t[1];
            z = qz + f.t[2];
            const float fr = x / g.res + g.hH;              // a5: bin (D13)
            const float fc = y / g.res + g.hW;
            if (!(0.0f <= fr && fr < (float)g.H && 0.0f <= fc && fc < (float)g.W)) {
              code = MEM_CODE_OOB;
            } else {
              const int row = (int)floorf(fr), col = (int)floorf(fc);
              lcell = row * g.W + col;
              cell = map_base + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
              v = np.a + np.b * r2;                         // a6: noise variance (D8)
              bool outlier = false;                         // a7: Mahalanobis test (D10)
              if (valid[cell]) {
                const float d = z - vals[(long long)kWordElev * g.BHW + cell];
                outlier = d * d > np.tau2 * (vals[(long long)kWordVar * g.BHW + cell] + v);
              }
              code = outlier ? MEM_CODE_OUTLIER : MEM_CODE_INLIER;
            }
          }
        }
      }
      if (kDebug) {
        a.dbg_cell[i] = lcell;
        a.dbg_code[i] = (uint8_t)code;
      }
    }
    // per-code counters: one ballot per code per warp, one smem add per code per warp
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const unsigned bal = __ballot_sync(0xffffffffu, live && code == c);
      if (lane == 0 && bal) atomicAdd(&s_cnt[c], (unsigned)__popc(bal));
    }
    if (cell < 0) continue;

    // a8: scatter-accumulate (hard part #7: native 64-bit global REDs)
    if (code == MEM_CODE_OUTLIER) {
      atomicAdd(&acc[(long long)kAccCnt * g.BHW + cell], 1ull << 32);
    } else {
      const float w = 1.0f / v;
      atomicAdd(&acc[(long long)kAccCnt * g.BHW + cell], 1ull);
      atomicAdd(reinterpret_cast<double *>(&acc[(long long)kAccP * g.BHW + cell]), (double)w);
      atomicAdd(reinterpret_cast<double *>(&acc[(long long)kAccS * g.BHW + cell]), (double)(z * w));
    }
    for (int bi = 0; bi < a.nb; ++bi) {  // every filtered in-bounds point feeds the groups (D12)
      const BindDesc &b = a.b[bi];
      const float *ch = p + 3 + b.ch_offset;
      unsigned long long *ga = acc + (long long)b.g.acc0 * g.BHW + cell;
      if (a.vec4) {  // stride 4: the single channel is ch0 (bindings were validated against stride)
        if (b.g.rule == MEM_COLOR) {
          const uint32_t bits = __float_as_uint(ch0);
          const unsigned long long rr = (bits >> 16) & 255u, gg = (bits >> 8) & 255u, bb = bits & 255u;
          atomicAdd(ga, rr | (gg << 32));
          atomicAdd(ga + g.BHW, bb | (1ull << 32));
        } else if (isfinite(ch0)) {  // nch == 1 (class rules need >= 2 channels)
          atomicAdd(ga, 1ull);
          atomicAdd(reinterpret_cast<double *>(ga + g.BHW), (double)ch0);
        }
        continue;
      }
      if (b.g.rule == MEM_COLOR) {  // D20: packed 0x00RRGGBB; exact integer sums packed in u64
        const uint32_t bits = __float_as_uint(__ldg(ch));
        const unsigned long long rr = (bits >> 16) & 255u, gg = (bits >> 8) & 255u, bb = bits & 255u;
        atomicAdd(ga, rr | (gg << 32));
        atomicAdd(ga + g.BHW, bb | (1ull << 32));
        continue;
      }
      bool fin = true;
      for (int k = 0; k < b.nch; ++k) fin &= (bool)isfinite(__ldg(ch + k));
      if (!fin) continue;  // D31
      if (b.g.rule == MEM_CLASS_MAX) {  // D19
        int best = 0;
        float bv = __ldg(ch);
        for (int k = 1; k < b.nch; ++k) {
          const float c = __ldg(ch + k);
          if (c > bv) { bv = c; best = k; }
        }
        const unsigned long long key = ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
        atomicMax(ga, key);
        continue;
      }
      atomicAdd(ga, 1ull);
      for (int k = 0; k < b.nch; ++k)
        atomicAdd(reinterpret_cast<double *>(ga + (long long)(1 + k) * g.BHW), (double)__ldg(ch + k));
    }
  }
  __syncthreads();
  if (threadIdx.x < 6 && s_cnt[threadIdx.x]) atomicAdd(&a.stats[stat_slot(threadIdx.x)], (unsigned long long)s_cnt[threadIdx.x]);
}

// ---------------------------------------------------------------- k_cell (a9-a10)
__global__ void __launch_bounds__(256) k_cell(const __grid_constant__ CellArgs a) {
  const Geometry &g = a.geo;
  unsigned long long *acc = a.st.acc;
  float *vals = reinterpret_cast<float *>(a.st.words);
  uint8_t *valid = a.st.flags + (long long)kFlagValid * g.BHW;
  unsigned touched = 0;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < g.BHW;
       c += (long long)gridDim.x * blockDim.x) {
    const unsigned long long cnt = __ldcg(&acc[(long long)kAccCnt * g.BHW + c]);
    if (cnt == 0) continue;  // untouched cells stay bit-identical
    ++touched;
    const double n_in = (double)(uint32_t)(cnt & 0xffffffffull);
    const double n_out = (double)(uint32_t)(cnt >> 32);
    const double P = __longlong_as_double((long long)__ldcg(&acc[(long long)kAccP * g.BHW + c]));
    const double S = __longlong_as_double((long long)__ldcg(&acc[(long long)kAccS * g.BHW + c]));
    float *h = vals + (long long)kWordElev * g.BHW + c;
    float *s2 = vals + (long long)kWordVar * g.BHW + c;
    // a9: Kalman height fusion, information form (D7), outliers inflate first (D11)
    if (valid[c]) {
      const double sp = (double)*s2 + n_out * (double)a.v_out;
      if (n_in > 0.0) {
        const double den = 1.0 / sp + P;
        const double hn = ((double)*h / sp + S) / den;
        *h = __double2float_rn(hn);
        *s2 = __double2float_rn(1.0 / den);
      } else {
        *s2 = __double2float_rn(sp);
      }
    } else if (n_in > 0.0) {  // first touch
      *h = __double2float_rn(S / P);
      *s2 = __double2float_rn(1.0 / P);
      valid[c] = 1;
    }
    acc[(long long)kAccCnt * g.BHW + c] = 0ull;
    acc[(long long)kAccP * g.BHW + c] = 0ull;
    acc[(long long)kAccS * g.BHW + c] = 0ull;
    // a10: each bound group by its rule
    for (int bi = 0; bi < a.nb; ++bi) {
      const GroupDesc &gd = a.b[bi].g;
      unsigned long long *ga = acc + (long long)gd.acc0 * g.BHW + c;
      if (gd.rule == MEM_CLASS_MAX) {
        const unsigned long long key = __ldcg(ga);
        if (key == 0ull) continue;
        apply_group(a.st, g.BHW, c, gd, 1.0, [](int) { return 0.0; }, key);
        *ga = 0ull;
      } else if (gd.rule == MEM_COLOR) {
        const unsigned long long rg = __ldcg(ga), bn = __ldcg(ga + g.BHW);
        const uint32_t n = (uint32_t)(bn >> 32);
        if (n == 0) continue;
        const double sr = (double)(uint32_t)(rg & 0xffffffffull), sg = (double)(uint32_t)(rg >> 32),
                     sb = (double)(uint32_t)(bn & 0xffffffffull);
        apply_group(a.st, g.BHW, c, gd, (double)n,
                    [&](int k) { return k == 0 ? sr : k == 1 ? sg : sb; }, 0ull);
        ga[0] = 0ull;
        ga[g.BHW] = 0ull;
      } else {
        const unsigned long long n = __ldcg(ga);
        if (n == 0ull) continue;
        apply_group(a.st, g.BHW, c, gd, (double)n,
                    [&](int k) { return __longlong_as_double((long long)__ldcg(ga + (long long)(1 + k) * g.BHW)); },
                    0ull);
        ga[0] = 0ull;
        for (int k = 0; k < gd.nch; ++k) ga[(long long)(1 + k) * g.BHW] = 0ull;
      }
    }
  }
  // n_cells_touched: warp reduce, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) touched += __shfl_xor_sync(0xffffffffu, touched, o);
  if ((threadIdx.x & 31) == 0 && touched) atomicAdd(&a.stats[7], (unsigned long long)touched);
}

// ---------------------------------------------------------------- k_image (a11-a12)
__global__ void __launch_bounds__(256) k_image(const __grid_constant__ ImageArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;  // logical cell
  const int2 ring = a.ring[m];
  const long long cell = (long long)m * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
  if (!a.st.flags[(long long)kFlagValid * g.BHW + cell]) return;
  const MapFrame &f = a.frames ? a.frames[m] : a.f0;
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  // a11: cell centre at its elevation, relative to the map centre (D13), into the camera (D17)
  const float xc = ((float)row + 0.5f - g.hH) * g.res;
  const float yc = ((float)col + 0.5f - g.hW) * g.res;
  const float dx = xc - f.t[0], dy = yc - f.t[1];
  const float dz = vals[(long long)kWordElev * g.BHW + cell] - f.t[2];
  const float pcx = (f.R[0] * dx + f.R[3] * dy) + f.R[6] * dz;
  const float pcy = (f.R[1] * dx + f.R[4] * dy) + f.R[7] * dz;
  const float pcz = (f.R[2] * dx + f.R[5] * dy) + f.R[8] * dz;
  if (!(pcz > 1e-6f)) return;
  const float ux = pcx / pcz, uy = pcy / pcz;
  const float u = (f.K[0] * ux + f.K[1] * uy) + f.K[2];  // pinhole
  const float v = f.K[3] * uy + f.K[4];
  const float fu = floorf(u + 0.5f), fv = floorf(v + 0.5f);  // nearest pixel (D16)
  if (!(0.0f <= fu && fu < (float)a.IW && 0.0f <= fv && fv < (float)a.IH)) return;  // frustum
  const long long plane = (long long)a.IH * a.IW;
  const float *pix = a.img + (long long)m * a.map_stride + (long long)(int)fv * a.IW + (int)fu;
  // a12: sample and fuse with N_j = 1
  for (int bi = 0; bi < a.nb; ++bi) {
    const BindDesc &b = a.b[bi];
    const float *ch = pix + (long long)b.ch_offset * plane;
    bool fin = true;
    for (int k = 0; k < b.nch; ++k) fin &= (bool)isfinite(__ldg(ch + k * plane));
    if (!fin) continue;  // D21
    unsigned long long key = 0ull;
    if (b.g.rule == MEM_CLASS_MAX) {
      int best = 0;
      float bv = __ldg(ch);
      for (int k = 1; k < b.nch; ++k) {
        const float c = __ldg(ch + k * plane);
        if (c > bv) { bv = c; best = k; }
      }
      key = ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
    }
    apply_group(a.st, g.BHW, cell, b.g, 1.0, [&](int k) { return (double)__ldg(ch + k * plane); }, key);
  }
}

// ---------------------------------------------------------------- reset of a cell
__device__ __forceinline__ void reset_cell(const State &st, long long BHW, long long cell, int n_word, int n_flag,
                                           const int *label_word, int n_label) {
  float *vals = reinterpret_cast<float *>(st.words);
  vals[(long long)kWordElev * BHW + cell] = __int_as_float(0x7fc00000);
  vals[(long long)kWordVar * BHW + cell] = __int_as_float(0x7fc00000);
  for (int w = 2; w < n_word; ++w) st.words[(long long)w * BHW + cell] = 0u;
  for (int l = 0; l < n_label; ++l) reinterpret_cast<int *>(st.words)[(long long)label_word[l] * BHW + cell] = -1;
  for (int fl = 0; fl < n_flag; ++fl) st.flags[(long long)fl * BHW + cell] = 0;
}

// ---------------------------------------------------------------- k_shift (a13)
__global__ void __launch_bounds__(256) k_shift(const __grid_constant__ ShiftArgs a) {
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
  reset_cell(a.st, g.BHW, cell, a.n_word, a.n_flag, a.label_word, a.n_label);
}

// ---------------------------------------------------------------- k_read / k_write (a14)
__global__ void __launch_bounds__(256) k_read(const __grid_constant__ ReadArgs a) {
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
    case RK_THETA: {  // Eq.(11) posterior mean, derived at readout (D5); idx = alpha layer of class k
      if (!a.st.flags[(long long)a.flag * g.BHW + cell]) break;  // unobserved -> 0 (D15)
      double tot = 0.0;
      for (int k = 0; k < a.K; ++k) tot += (double)vals[(long long)(a.first + k) * g.BHW + cell];
      out = __double2float_rn((double)vals[(long long)a.idx * g.BHW + cell] / tot);
      break;
    }
  }
  a.out[(long long)m * g.HW + t] = out;
}

__global__ void __launch_bounds__(256) k_write(const __grid_constant__ ReadArgs a) {
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;
  const int2 ring = a.ring[m];
  const long long cell = (long long)m * g.HW + (long long)wrap(row + ring.x, g.H) * g.W + wrap(col + ring.y, g.W);
  const float v = a.src[(long long)m * g.HW + t];
  switch (a.kind) {
    case RK_ELEV:
    case RK_VAR:
    case RK_WORD: reinterpret_cast<float *>(a.st.words)[(long long)a.idx * g.BHW + cell] = v; break;
    case RK_LABEL: reinterpret_cast<int *>(a.st.words)[(long long)a.idx * g.BHW + cell] = (int)v; break;
    case RK_FLAG: a.st.flags[(long long)a.idx * g.BHW + cell] = v != 0.0f; break;
    default: break;
  }
}

// ---------------------------------------------------------------- launchers
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

cudaError_t launch_point(const PointArgs &a, cudaStream_t s) {
  const unsigned bx = cdiv(a.max_n > 0 ? a.max_n : 1, kPointsPerBlock);
  const dim3 grid(bx, a.geo.n_maps);
  if (a.dbg_cell)
    k_point<true><<<grid, kPointThreads, 0, s>>>(a);
  else
    k_point<false><<<grid, kPointThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_cell(const CellArgs &a, cudaStream_t s) {
  const long long blocks = (a.geo.BHW + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 148LL * 16 ? blocks : 148LL * 16);
  k_cell<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_image(const ImageArgs &a, cudaStream_t s) {
  k_image<<<dim3(cdiv(a.geo.HW, 256), a.geo.n_maps), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
  const int cnt = a.max_count > 0 ? a.max_count : 1;
  k_shift<<<dim3(cdiv(cnt, 256), a.geo.n_maps), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_read(const ReadArgs &a, cudaStream_t s) {
  k_read<<<dim3(cdiv(a.geo.HW, 256), a.geo.n_maps), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_write(const ReadArgs &a, cudaStream_t s) {
  k_write<<<dim3(cdiv(a.geo.HW, 256), a.geo.n_maps), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace memk
