// k_smap.cuh -- k_smap: small maps sorted by cell (deterministic, oracle order).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_smap (small maps, sort by cell)
// One CTA per map (grid-stride over the wave's maps) for the fast rules on small maps
// (H*W <= kSmapCells, <= kSmapPoints points per map): no scratch, no atomics outside shared
// memory.  P1 bins every point (streamed once from HBM) into a shared-memory histogram of its
// cell (and records the cell of every point when shared memory allows); P2 turns it into
// offsets; P3 scatters the point indices by cell (from the recorded cells, else re-binned
// from L2); P4 gives every cell to one lane, which sorts the cell's indices (input order,
// like the oracle); the warp re-reads those points, recomputes z and v and tests them
// against the cell's pre-frame state (a7); the lane sums in fp64 in input order and fuses the cell with the
// oracle's exact formulas -- so this path is deterministic and reproduces the oracle's sums
// operation for operation.  (The north_star's "sort-by-cell segmented reduction".)
#ifndef MEM_SMAP_THREADS
#define MEM_SMAP_THREADS 1024  // P4 walks the cells one per thread: more threads, shorter chains
#endif
#ifndef MEM_SMAP_MINB
#define MEM_SMAP_MINB 1
#endif
constexpr int kSmapThreads = MEM_SMAP_THREADS;
#ifndef MEM_SMAP_P1
#define MEM_SMAP_P1 2  // P1: points per thread in flight (C5a: 4 -> 2: 3.18 -> 3.13 ms)
#endif
constexpr int kSmapP1 = MEM_SMAP_P1;
constexpr int kSmapCells = 16384;
constexpr int kSmapPoints = 65535;

// shared memory: the per-cell counts / offsets as packed u16 pairs (a map has < 65536 points)
// and the u16 point indices
constexpr int kSmapChunk = 64;  // P4: points per warp step
// The P4 slices share their space with the u16 cell of every point that P1 records for P3
// (P3 then scatters from shared memory instead of re-reading and re-binning the points).
#ifndef MEM_SMAP_CACHE
#define MEM_SMAP_CACHE 1
#endif
__host__ __device__ inline size_t smap_tmp_offset(int HW, long long max_pts) {
  return (sizeof(unsigned) * (size_t)((HW + 1) / 2) + sizeof(uint16_t) * (size_t)max_pts + 15) & ~(size_t)15;
}
constexpr size_t kSmapTmpBytes = sizeof(float4) * (size_t)kSmapChunk * (kSmapThreads / 32);
constexpr size_t kSmapMaxSmem = 220 * 1024;
__host__ __device__ inline bool smap_cached(int HW, long long max_pts) {
  const size_t pc = sizeof(uint16_t) * (size_t)max_pts;
  return MEM_SMAP_CACHE && smap_tmp_offset(HW, max_pts) + (pc > kSmapTmpBytes ? pc : kSmapTmpBytes) <= kSmapMaxSmem;
}
size_t smap_smem_bytes(int HW, long long max_pts) {
  const size_t pc = smap_cached(HW, max_pts) ? sizeof(uint16_t) * (size_t)max_pts : 0;
  return smap_tmp_offset(HW, max_pts) + (pc > kSmapTmpBytes ? pc : kSmapTmpBytes);
}
bool smap_eligible(int HW, long long max_pts) {
  return HW <= kSmapCells && max_pts <= kSmapPoints && smap_smem_bytes(HW, max_pts) <= kSmapMaxSmem;
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
  uint16_t *pcell = reinterpret_cast<uint16_t *>(s_tmp);  // P1 -> P3: cell of every point (0xffff: dropped)
  const bool cached = smap_cached(g.HW, a.smap_maxpts);
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
    for (int i0 = threadIdx.x; i0 < np; i0 += kSmapP1 * kSmapThreads) {
      float4 q[kSmapP1];
#pragma unroll
      for (int u = 0; u < kSmapP1; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i < np) q[u] = ld_stream_f4(reinterpret_cast<const float *>(pts4 + beg + i), pol);
      }
#pragma unroll
      for (int u = 0; u < kSmapP1; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i >= np) continue;
        const PointOut o = bin_point(q[u].x, q[u].y, q[u].z, f, g, a.np, map_base, a.r2lo, a.r2hi);
        if (cached) pcell[i] = o.cell >= 0 ? (uint16_t)(o.cell - map_base) : (uint16_t)0xffffu;
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
    // P3: scatter the in-window points' indices by cell
    if (cached) {
      for (int i = threadIdx.x; i < np; i += kSmapThreads) {
        const unsigned c = pcell[i];
        if (c != 0xffffu) idx[(atomicAdd(&hist[c >> 1], 1u << (16 * (c & 1))) >> (16 * (c & 1))) & 0xffffu] = (uint16_t)i;
      }
    }
    for (int i0 = threadIdx.x; i0 < (cached ? 0 : np); i0 += kSmapP1 * kSmapThreads) {  // re-binned (points in L2)
      float4 q[kSmapP1];
#pragma unroll
      for (int u = 0; u < kSmapP1; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i < np) q[u] = __ldg(pts4 + beg + i);
      }
#pragma unroll
      for (int u = 0; u < kSmapP1; ++u) {
        const int i = i0 + u * kSmapThreads;
        if (i >= np) continue;
        const PointOut o = bin_point(q[u].x, q[u].y, q[u].z, f, g, a.np, map_base, a.r2lo, a.r2hi);
        if (o.cell >= 0) {
          const int c = o.cell - map_base;
          idx[(atomicAdd(&hist[c >> 1], 1u << (16 * (c & 1))) >> (16 * (c & 1))) & 0xffffu] = (uint16_t)i;
        }
      }
    }
    __syncthreads();
    // P4: warps take groups of 32 consecutive cells (lane = cell).  Each lane sorts its cell's
    // point indices into input order and loads its cell's pre-frame state; the warp then walks
    // the group's points (contiguous in idx) 64 at a time, lane-parallel: re-read, recompute
    // z and v, find the owner lane (the segment holding the position), outlier test against
    // the owner lane's state (shuffle), contributions staged in the
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
          if (s1 - s0 > 1u) {  // input order (insertion sort; every cell)
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
        const unsigned e = inmap ? s1 : 0xffffffffu;  // segment ends, non-decreasing over the lanes
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
            int owner = lane;  // the lane holding the point's cell
            if (kDebug) {
              if (act) o = bin_point(q.x, q.y, q.z, f, g, a.np, map_base, a.r2lo, a.r2hi);
              if (act) owner = o.cell - map_base - gbase;
            } else {
              // the point is known to be in the window: only z and v are recomputed (bin_point's
              // expressions, same rounding), and its cell is the segment that holds position r
              // (binary search over the lanes' segment ends).  A scrolled-in strip cell has
              // vd = 0 (reset state), so the test flag of bin_point is not needed.
              if (act) {
                const float r2 = (q.x * q.x + q.y * q.y) + q.z * q.z;
                const float qz = (f.R[6] * q.x + f.R[7] * q.y) + f.R[8] * q.z;
                o.z = qz + f.t[2];
                o.v = a.np.a + a.np.b * r2;
                o.test = true;
              }
              int lo = 0;
#pragma unroll
              for (int st = 16; st > 0; st >>= 1) {
                const unsigned eo = __shfl_sync(0xffffffffu, e, lo + st - 1);
                lo += eo <= r ? st : 0;
              }
              if (act) owner = lo;
            }
            const float ho = __shfl_sync(0xffffffffu, h, owner), so = __shfl_sync(0xffffffffu, s2, owner);
            const int vo = __shfl_sync(0xffffffffu, (int)vd, owner);
            if (act) {
              bool outl = false;
              if (o.test && vo) {  // (z - h)^2 > tau^2 (sigma^2 + v) against the pre-frame state (D10)
                const float d = o.z - ho;
                outl = d * d > a.np.tau2 * (so + o.v);
              }
              const int code = outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER;
              cnt[5] += outl ? 0u : 1u;  // stat_slot(INLIER), stat_slot(OUTLIER)
              cnt[6] += outl ? 1u : 0u;
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
        if (s1 > s0) {
          ++cnt[7];
          // a9 (D7, D11) in the oracle's exact form
          kalman_height(h, s2, vd, (double)nin, (double)nout, P, S, a.np.v_out);
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
