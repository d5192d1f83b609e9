// k_image.cuh -- occlusion walk (NEXT-1) and k_image (a11-a12).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

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
  const int rc = (int)floorf(__fdiv_rn(tx, g.res) + g.hH), cc = (int)floorf(__fdiv_rn(ty, g.res) + g.hW);
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
// kImgLanes lanes per logical cell (consecutive lanes of one warp: a "group"); every lane of a
// group computes the cell's projection (a11, identical operands and order), the occlusion walk
// runs on the group's first lane.  The channels of a binding are split over the lanes --
// channel k on lane k % L -- so each lane's pixel and state loads (at most kImgBatch channels
// per batch) are all in flight together; the D21 finiteness test is an AND over the group and
// the class_max argmax a (value, lowest channel) reduction over the group.  Every channel is
// fused by exactly the rule calls of apply_group (same operands, same order per channel), so
// results are identical to the one-thread-per-cell form.
#ifndef MEM_IMG_BATCH
#define MEM_IMG_BATCH 16
#endif
#ifndef MEM_IMG_LANES
#define MEM_IMG_LANES 4
#endif
constexpr int kImgBatch = MEM_IMG_BATCH;
constexpr int kImgLanes = MEM_IMG_LANES;
// the group's channels k = sub, sub + L, ... of one binding fused with N_j = 1
template <bool kSimple, int kB>
__device__ __forceinline__ void image_fuse_words(const State &st, long long BHW, long long cell, const GroupDesc &g,
                                                 const float *ch, long long plane, int sub, unsigned gmask) {
  float *vals = reinterpret_cast<float *>(st.words);
  uint8_t *obs = st.flags + (long long)g.flag * BHW + cell;
  const bool observed = *obs != 0;
  const bool dir = g.rule == MEM_CLASS_BAYESIAN;
  constexpr int L = kImgLanes;
  if (!kSimple && g.rule == MEM_GAUSSIAN) {  // two words per channel: mean at word0 + k, variance at word0 + nch + k
    for (int k0 = 0; k0 < g.nch; k0 += kB * L) {
      float p[kB], mu[kB], var[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + u * L + sub;
        if (k < g.nch) {
          p[u] = __ldg(ch + (long long)k * plane);
          mu[u] = vals[(long long)(g.word0 + k) * BHW + cell];
          var[u] = vals[(long long)(g.word0 + g.nch + k) * BHW + cell];
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + u * L + sub;
        if (k < g.nch) {
          rule_gaussian(mu[u], var[u], observed, (double)p[u], 1.0, g);
          vals[(long long)(g.word0 + k) * BHW + cell] = mu[u];
          vals[(long long)(g.word0 + g.nch + k) * BHW + cell] = var[u];
        }
      }
    }
  } else {
    for (int k0 = 0; k0 < g.nch; k0 += kB * L) {
      float p[kB], th[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + u * L + sub;
        if (k < g.nch) {
          p[u] = __ldg(ch + (long long)k * plane);
          th[u] = vals[(long long)(g.word0 + k) * BHW + cell];
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k = k0 + u * L + sub;
        if (k < g.nch)
          vals[(long long)(g.word0 + k) * BHW + cell] =
              dir ? rule_dirichlet(th[u], observed, (double)p[u], g.a0) : rule_average(th[u], observed, (double)p[u], 1.0, g.w);
      }
    }
  }
  __syncwarp(gmask);  // every lane has read `observed`
  if (sub == 0) *obs = 1;
}

#ifndef MEM_IMG_THREADS
#define MEM_IMG_THREADS 256
#endif
constexpr int kImgThreads = MEM_IMG_THREADS;
constexpr int kImgCells = kImgThreads / kImgLanes;  // cells per CTA
// kSimple: no top-k binding, no gaussian group, no occlusion walk (C3, C4): a leaner kernel
// kB: channels per lane per batch of loads in flight (kImgBatch; 8 for bindings of <= 32 channels)
template <bool kSimple, int kB>
__global__ void __launch_bounds__(kImgThreads) k_image(const __grid_constant__ ImageArgs a) {
  constexpr int L = kImgLanes;
  const Geometry &g = a.geo;
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31, sub = lane & (L - 1);
  const unsigned gmask = (unsigned)((1ull << L) - 1ull) << (lane & ~(L - 1));
  const int t = blockIdx.x * kImgCells + (int)(threadIdx.x / L);
  // every exit below depends on the cell only: uniform over the group
  if (t >= g.HW) return;
  const int row = t / g.W, col = t - (t / g.W) * g.W;  // logical cell
  const int2 ring = a.ring[m];
  const int prow = wrap(row + ring.x, g.H);
  if (prow < a.row_lo || prow >= a.row_hi) return;  // another rank's band (sharded map)
  const long long cell = (long long)m * g.HW + (long long)prow * g.W + wrap(col + ring.y, g.W);
  const float *vals = reinterpret_cast<const float *>(a.st.words);
  const uint8_t valid = a.st.flags[(long long)kFlagValid * g.BHW + cell];
  const float hcell = vals[(long long)kWordElev * g.BHW + cell];  // loaded with the flag (one round trip)
  if (!valid) return;
  const MapFrame &f = a.frames ? a.frames[m] : a.f0;
  // a11: cell centre at its elevation, relative to the map centre (D13), into the camera (D17)
  const float xc = ((float)row + 0.5f - g.hH) * g.res;
  const float yc = ((float)col + 0.5f - g.hW) * g.res;
  const float dx = xc - f.t[0], dy = yc - f.t[1];
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
  if (!kSimple && a.occlusion) {  // the walk on the group's first lane
    bool vis = false;
    if (sub == 0) vis = cell_visible(a, m, row, col, f.t[0], f.t[1], f.t[2], hcell, ring);
    if (!__shfl_sync(gmask, vis, 0, L)) return;
  }
  const long long plane = (long long)a.IH * a.IW;
  const float *pix = a.img + (long long)m * a.map_stride + (long long)(int)fv * a.IW + (int)fu;
  // a12: sample and fuse with N_j = 1
  for (int bi = 0; bi < a.nb; ++bi) {
    const BindDesc &b = a.b[bi];
    const float *ch = pix + (long long)b.ch_offset * plane;
    if (!kSimple && b.topk > 0) {  // top-k pairs (D38): the group's first lane
      if (sub == 0) {
        const TopK tk{ch, plane, b.topk, b.g.nch - 1};
        if (tk.ok()) {
          const unsigned long long key = b.g.rule == MEM_CLASS_MAX ? tk.key() : 0ull;
          apply_group(a.st, g.BHW, cell, b.g, 1.0, [&](int k) { return (double)tk.value(k); }, key);
        }
      }
      __syncwarp(gmask);
      continue;
    }
    // D21 finiteness over all channels, and class_max's first maximum in channel order
    bool fin = true;
    float bv = -INFINITY;
    int best = -1;
    for (int k0 = 0; k0 < b.nch; k0 += kB * L) {  // loads of a batch in flight together
      float c[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int k = k0 + q * L + sub;
        c[q] = k < b.nch ? __ldg(ch + (long long)k * plane) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int k = k0 + q * L + sub;
        if (k < b.nch) {
          fin &= (bool)isfinite(c[q]);
          if (best < 0 || c[q] > bv) {  // this lane's channels in increasing order
            bv = c[q];
            best = k;
          }
        }
      }
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) {
      fin &= (bool)__shfl_xor_sync(gmask, (int)fin, o, L);
      const float ov = __shfl_xor_sync(gmask, bv, o, L);
      const int ob = __shfl_xor_sync(gmask, best, o, L);
      if (ob >= 0 && (best < 0 || ov > bv || (ov == bv && ob < best))) {  // larger, or equal and earlier
        bv = ov;
        best = ob;
      }
    }
    if (!fin) continue;  // D21 (uniform over the group)
    if (b.g.rule == MEM_CLASS_MAX) {
      if (sub == 0) {
        const unsigned long long key = ((unsigned long long)ord_f32(bv) << 32) | (unsigned)(b.nch - 1 - best);
        apply_group(a.st, g.BHW, cell, b.g, 1.0, [&](int k) { return (double)__ldg(ch + k * plane); }, key);
      }
      __syncwarp(gmask);
      continue;
    }
    image_fuse_words<kSimple, kB>(a.st, g.BHW, cell, b.g, ch, plane, sub, gmask);
  }
}
