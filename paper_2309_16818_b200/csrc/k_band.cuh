// k_band.cuh -- k_band: a7-a10 (+ lazy a13) for one cell band of one map, in input order
// (DESIGN.md §4.2).  Part of the single translation unit kernels.cu (included inside namespace
// memk, in order).
#pragma once

// ---------------------------------------------------------------- k_band
// One CTA per (map, band of band_cells physical cells).  The band's in-window points were
// split out by k_bin into per-tile runs (input order within each run, runs in tile order), so
// walking the runs in tile order visits the band's points in input order.  The CTA:
//   1. resets the band's cells in the strips that scrolled in with the pending shift (a13);
//   2. prefix-sums the runs' counts (tinfo) over the map's tiles;
//   3. per chunk of kChunkRecs records (in input order): gathers them into shared memory,
//      sorts (cell, position) with a stable block radix sort on the cell (the positions are
//      the input order, so ties keep it), finds the per-cell segments, and gives every
//      segment to one thread, which runs the oracle's per-point loop for its cell: the
//      Mahalanobis test against the pre-frame state (a7), then the sufficient statistics
//      summed sequentially in input order -- P += (double)(1/v), S += (double)(z/v), channel
//      sums in fp64, colour in integers (a8) -- and, at the cell's last chunk, the Kalman
//      height update and the group rules (a9, a10) with the oracle's expressions.
// The sums are thus the oracle's, operation for operation, whatever the thread schedule or
// launch configuration (reading D39): results are bit-identical to the oracle and run to run.
// A band with more records than one chunk keeps each cell's partial sums in the per-cell
// scratch between chunks (a cell's last chunk is known from a pre-pass over the records).
constexpr int kBandChunk = kChunkRecs;

struct BandSmem {  // dynamic shared memory layout of k_band (host and device)
  size_t rec, key, idx, seg, fin, ridx, tcnt, tpre, last, seen, total;
  __host__ __device__ BandSmem(int tmax, int band_cells) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
      const size_t at = o;
      o = (o + bytes + 15) & ~(size_t)15;
      return at;
    };
    rec = take(sizeof(uint3) * kBandChunk);
    key = take(sizeof(uint16_t) * kBandChunk);
    idx = take(sizeof(uint16_t) * kBandChunk);
    seg = take(sizeof(uint16_t) * (kBandChunk + 1));
    fin = take(sizeof(uint16_t) * kBandChunk);
    ridx = take(sizeof(unsigned) * kBandChunk);
    tcnt = take(sizeof(unsigned) * (size_t)tmax);
    tpre = take(sizeof(unsigned) * (size_t)(tmax + 1));
    last = take(sizeof(uint16_t) * (size_t)band_cells);
    seen = take(sizeof(unsigned) * (size_t)((band_cells + 31) / 32));
    total = o;
  }
};

// block-wide exclusive scan of one value per thread; returns the prefix, *total the sum
template <int kT>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned *s_part, unsigned *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  __syncthreads();  // s_part may still be read by a previous scan
  if (lane == 31) s_part[wid] = incl;
  __syncthreads();
  unsigned wpre = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    const unsigned p = s_part[w];
    wpre += w < wid ? p : 0u;
    tot += p;
  }
  *total = tot;
  return wpre + incl - v;
}

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

// One cell's points [s0, s1) of the sorted chunk: a7 + a8 in input order, then (at the cell's
// last chunk) a9 + a10.  `first`: no earlier chunk held this cell; `last`: no later one will.
template <bool kDebug, int kFast>
__device__ __forceinline__ void band_segment(const PassArgs &a, int m, int phys, int s0, int s1, bool first,
                                             bool last, const uint3 *rec_s, const uint16_t *idx_s,
                                             const uint16_t *fin_s, const unsigned *ridx_s, unsigned (&cnt)[8]) {
  const Geometry &g = a.geo;
  const long long BHW = g.BHW;
  const long long gc = (long long)m * g.HW + phys;
  float *vals = reinterpret_cast<float *>(a.st.words);
  float *elev = vals + (long long)kWordElev * BHW, *var = vals + (long long)kWordVar * BHW;
  uint8_t *validp = a.st.flags + (long long)kFlagValid * BHW;
  unsigned long long *cw = a.scr + gc * a.R;  // this cell's carry words (multi-chunk bands only)
  // pre-frame state: the Mahalanobis test of every point of the frame uses it (D10)
  float h = elev[gc], s2 = var[gc];
  const float tau2 = a.np.tau2;
  double P = 0.0, S = 0.0;
  unsigned nin = 0u, nout = 0u;
  unsigned cr = 0u, cg = 0u, cb = 0u, na = 0u;  // colour sums and count / average count
  double X = 0.0;                               // 1-channel average sum
  if (!first) {
    P = __longlong_as_double((long long)cw[0]);
    S = __longlong_as_double((long long)cw[1]);
    nin = (unsigned)(cw[2] & 0xffffffffull);
    nout = (unsigned)(cw[2] >> 32);
    if (kFast == 1) {
      cr = (unsigned)(cw[3] & 0xffffffffull);
      cg = (unsigned)(cw[3] >> 32);
      cb = (unsigned)(cw[4] & 0xffffffffull);
      na = (unsigned)(cw[4] >> 32);
    } else if (kFast == 2) {
      na = (unsigned)cw[3];
      X = __longlong_as_double((long long)cw[4]);
    }
  }
  unsigned fin_in = 0u, fout = 0u;
  for (int r = s0; r < s1; ++r) {
    const int j = idx_s[r];
    const uint3 q = rec_s[j];
    const float z = __uint_as_float(q.x), v = __uint_as_float(q.y);
    const float d = z - h;  // a7 (D10): NaN state (invalid cell) compares false
    const bool outl = d * d > tau2 * (s2 + v);
    if (outl) {
      ++fout;
    } else {
      ++fin_in;
      const float w = 1.0f / v;  // a8: the oracle's fp32 terms, summed in fp64 in input order
      P += (double)w;
      S += (double)(z * w);
    }
    if (kFast == 1) {  // D20: packed 0x00RRGGBB, exact integer sums
      cr += (q.z >> 16) & 255u;
      cg += (q.z >> 8) & 255u;
      cb += q.z & 255u;
      ++na;
    } else if (kFast == 2) {  // D31: a non-finite channel skips the group
      const float c = __uint_as_float(q.z);
      if (isfinite(c)) {
        ++na;
        X += (double)c;
      }
    }
    if (kDebug) a.dbg_code[ridx_s[j]] = (uint8_t)(outl ? MEM_CODE_OUTLIER : MEM_CODE_INLIER);
  }
  cnt[5] += fin_in;
  cnt[6] += fout;
  nin += fin_in;
  nout += fout;
  if (kFast == 0) {  // generic groups: per group, per channel, in input order
    for (int bi = 0; bi < a.nb; ++bi) {
      const BindDesc &b = a.b[bi];
      const GroupDesc &gd = b.g;
      unsigned long long *gw = cw + gd.acc0;
      if (gd.rule == MEM_COLOR) {
        unsigned r_ = 0u, g_ = 0u, b_ = 0u, n_ = 0u;
        if (!first) {
          r_ = (unsigned)(gw[0] & 0xffffffffull);
          g_ = (unsigned)(gw[0] >> 32);
          b_ = (unsigned)(gw[1] & 0xffffffffull);
          n_ = (unsigned)(gw[1] >> 32);
        }
        for (int r = s0; r < s1; ++r) {
          const uint32_t bits = __float_as_uint(chan_value(a, b, rec_s[idx_s[r]].z, 0));
          r_ += (bits >> 16) & 255u;
          g_ += (bits >> 8) & 255u;
          b_ += bits & 255u;
          ++n_;
        }
        if (!last) {
          gw[0] = (unsigned long long)r_ | ((unsigned long long)g_ << 32);
          gw[1] = (unsigned long long)b_ | ((unsigned long long)n_ << 32);
        } else {
          uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
          const bool ob = *obs != 0;
          const unsigned sums[3] = {r_, g_, b_};
          for (int k = 0; k < 3; ++k) {
            float *th = vals + (long long)(gd.word0 + k) * BHW + gc;
            *th = rule_average(*th, ob, (double)sums[k], (double)n_, gd.w);
          }
          *obs = 1;
        }
        continue;
      }
      if (gd.rule == MEM_CLASS_MAX) {  // D19: the frame's winner, an order-free maximum
        unsigned long long key = first ? 0ull : gw[0];
        for (int r = s0; r < s1; ++r) {
          const int j = idx_s[r];
          if (fin_s[j] >> bi & 1u) {
            const unsigned long long k = chan_key(a, b, rec_s[j].z);
            key = k > key ? k : key;
          }
        }
        if (!last) {
          gw[0] = key;
        } else if (key != 0ull) {
          reinterpret_cast<int *>(a.st.words)[(long long)gd.label * BHW + gc] =
              gd.nch - 1 - (int)(uint32_t)(key & 0xffffffffull);
          vals[(long long)gd.word0 * BHW + gc] = f32_of_ord((uint32_t)(key >> 32));
        }
        continue;
      }
      unsigned ng = first ? 0u : (unsigned)gw[0];
      for (int r = s0; r < s1; ++r) ng += fin_s[idx_s[r]] >> bi & 1u;
      if (last && ng == 0u) continue;  // no finite point: the group is not updated (D31)
      uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
      const bool ob = last ? *obs != 0 : false;
      for (int k = 0; k < gd.nch; ++k) {
        double sum = first ? 0.0 : __longlong_as_double((long long)gw[1 + k]);
        for (int r = s0; r < s1; ++r) {
          const int j = idx_s[r];
          if (fin_s[j] >> bi & 1u) sum += (double)chan_value(a, b, rec_s[j].z, k);
        }
        if (!last) {
          gw[1 + k] = (unsigned long long)__double_as_longlong(sum);
          continue;
        }
        float *th = vals + (long long)(gd.word0 + k) * BHW + gc;
        switch (gd.rule) {
          case MEM_AVERAGE:
          case MEM_CLASS_AVERAGE: *th = rule_average(*th, ob, sum, (double)ng, gd.w); break;
          case MEM_GAUSSIAN: {
            float *vr = vals + (long long)(gd.word0 + gd.nch + k) * BHW + gc;
            float mu = *th, vv = *vr;
            rule_gaussian(mu, vv, ob, sum, (double)ng, gd);
            *th = mu;
            *vr = vv;
            break;
          }
          case MEM_CLASS_BAYESIAN: *th = rule_dirichlet(*th, ob, sum, gd.a0); break;
          default: break;
        }
      }
      if (!last) gw[0] = ng;
      else *obs = 1;
    }
  }
  if (!last) {  // partial sums to the carry words; the cell is fused at its last chunk
    cw[0] = (unsigned long long)__double_as_longlong(P);
    cw[1] = (unsigned long long)__double_as_longlong(S);
    cw[2] = (unsigned long long)nin | ((unsigned long long)nout << 32);
    if (kFast == 1) {
      cw[3] = (unsigned long long)cr | ((unsigned long long)cg << 32);
      cw[4] = (unsigned long long)cb | ((unsigned long long)na << 32);
    } else if (kFast == 2) {
      cw[3] = na;
      cw[4] = (unsigned long long)__double_as_longlong(X);
    }
    return;
  }
  // a9: Kalman height fusion (D7, D11)
  uint8_t vd = validp[gc];
  const uint8_t vd0 = vd;
  kalman_height(h, s2, vd, (double)nin, (double)nout, P, S, a.np.v_out);
  if (vd) {
    elev[gc] = h;
    var[gc] = s2;
    if (!vd0) validp[gc] = 1;
  }
  ++cnt[7];
  // a10: the fast groups (Eq.(1)+(2))
  if (kFast == 1 || kFast == 2) {
    const GroupDesc &gd = a.b[0].g;
    if (na != 0u) {
      uint8_t *obs = a.st.flags + (long long)gd.flag * BHW + gc;
      const bool ob = *obs != 0;
      if (kFast == 1) {
        const unsigned sums[3] = {cr, cg, cb};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float *th = vals + (long long)(gd.word0 + k) * BHW + gc;
          *th = rule_average(*th, ob, (double)sums[k], (double)na, gd.w);
        }
      } else {
        float *th = vals + (long long)gd.word0 * BHW + gc;
        *th = rule_average(*th, ob, X, (double)na, gd.w);
      }
      *obs = 1;
    }
  }
}

template <bool kDebug, int kFast>
__global__ void __launch_bounds__(kBandThreads) k_band(const __grid_constant__ PassArgs a) {
  using Sort = cub::BlockRadixSort<uint16_t, kBandThreads, kBandIPT, uint16_t>;
  __shared__ typename Sort::TempStorage s_sort;
  __shared__ unsigned s_part[kBandThreads / 32];
  __shared__ unsigned s_cnt[8];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int tid = threadIdx.x;
  const Geometry &g = a.geo;
  int bb;
  const int m = divmod_fast(blockIdx.x, a.nbands, a.inv_nbands, bb);
  const int c0 = a.cell_lo + bb * a.band_cells;
  const int c1 = c0 + a.band_cells < a.cell_hi ? c0 + a.band_cells : a.cell_hi;
  const int t0 = ts_of(a, m), T = ts_of(a, m + 1) - t0;
  const BandSmem L(a.tmax, a.band_cells);
  uint3 *rec_s = reinterpret_cast<uint3 *>(s_dyn + L.rec);
  uint16_t *key_s = reinterpret_cast<uint16_t *>(s_dyn + L.key);
  uint16_t *idx_s = reinterpret_cast<uint16_t *>(s_dyn + L.idx);
  uint16_t *seg_s = reinterpret_cast<uint16_t *>(s_dyn + L.seg);
  uint16_t *fin_s = reinterpret_cast<uint16_t *>(s_dyn + L.fin);
  unsigned *ridx_s = reinterpret_cast<unsigned *>(s_dyn + L.ridx);
  unsigned *tcnt_s = reinterpret_cast<unsigned *>(s_dyn + L.tcnt);
  unsigned *tpre_s = reinterpret_cast<unsigned *>(s_dyn + L.tpre);
  uint16_t *last_s = reinterpret_cast<uint16_t *>(s_dyn + L.last);
  unsigned *seen_s = reinterpret_cast<unsigned *>(s_dyn + L.seen);
  if (tid < 8) s_cnt[tid] = 0;
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  pdl_wait();
  pdl_trigger();
  const PointFrame f = frame_of(a, m);
  if (bb == 0 && tid == 0) a.ring[m] = make_int2(f.r0, f.c0);
  if (f.sr != 0 || f.sc != 0) {  // lazy ring shift: reset the band's scrolled-in cells (a13)
    for (int phys = c0 + tid; phys < c1; phys += kBandThreads) {
      int pcol;
      const int prow = divmod_fast(phys, g.W, g.inv_W, pcol);
      int row = prow - f.r0, col = pcol - f.c0;
      row += row < 0 ? g.H : 0;
      col += col < 0 ? g.W : 0;
      if (in_strip(row, col, f, g)) reset_cell(a.st, g.BHW, (long long)m * g.HW + phys, a.reset);
    }
  }
  // the runs of this band in the map's tiles, and their prefix (input order)
  unsigned K = 0u;
  for (int tb = 0; tb < T; tb += kBandThreads) {
    const int t = tb + tid;
    const unsigned v = t < T ? __ldcg(a.tinfo + (long long)(t0 + t) * a.nbands + bb) : 0u;
    unsigned tot;
    const unsigned pre = block_excl_scan<kBandThreads>(v >> 16, s_part, &tot);
    if (t < T) {
      tcnt_s[t] = v;
      tpre_s[t] = K + pre;
    }
    K += tot;
  }
  if (tid == 0) tpre_s[T] = K;
  __syncthreads();  // also orders the strip resets before the state loads below
  const int nchunks = (int)((K + kBandChunk - 1) / kBandChunk);
  auto locate = [&](unsigned p) -> const uint4 * {  // the record at band position p
    int lo = 0, hi = T - 1;  // last tile t with tpre[t] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tpre_s[mid] <= p) lo = mid; else hi = mid - 1;
    }
    return a.recs + (long long)(t0 + lo) * kTile + (tcnt_s[lo] & 0xffffu) + (p - tpre_s[lo]);
  };
  if (nchunks > 1) {  // multi-chunk band: each cell's last chunk, and no cell seen yet
    for (int i = tid; i < (a.band_cells + 31) / 32; i += kBandThreads) seen_s[i] = 0u;
    for (int c = 0; c < nchunks; ++c) {
      const unsigned p0 = (unsigned)c * kBandChunk;
      const unsigned n = K - p0 < (unsigned)kBandChunk ? K - p0 : (unsigned)kBandChunk;
      for (unsigned j = tid; j < n; j += kBandThreads) last_s[__ldcg(&locate(p0 + j)->x) & 0xffffu] = (uint16_t)c;
      __syncthreads();  // a later chunk's stores win
    }
  }
  const uint16_t pad = (uint16_t)((1u << a.key_bits) - 1u);
  for (int c = 0; c < nchunks; ++c) {
    const unsigned p0 = (unsigned)c * kBandChunk;
    const int n = (int)(K - p0 < (unsigned)kBandChunk ? K - p0 : (unsigned)kBandChunk);
    for (int j = tid; j < kBandChunk; j += kBandThreads) {  // gather the chunk in input order
      if (j < n) {
        const uint4 *src = locate(p0 + j);
        const uint4 r = __ldcg(src);
        key_s[j] = (uint16_t)(r.x & 0xffffu);
        rec_s[j] = make_uint3(r.y, r.z, r.w);
        if (kDebug) ridx_s[j] = __ldcg(a.ridx + (src - a.recs));
        if (kFast == 0) {  // per bound group: are the point's channels usable (D31, D38)?
          unsigned fb = 0u;
          for (int bi = 0; bi < a.nb; ++bi) fb |= chan_ok(a, a.b[bi], r.w) ? (1u << bi) : 0u;
          fin_s[j] = (uint16_t)fb;
        }
      } else {
        key_s[j] = pad;
      }
    }
    __syncthreads();
    {  // stable sort of (cell, position) by cell: positions are the input order
      uint16_t kk[kBandIPT], vv[kBandIPT];
      const uint4 *kv = reinterpret_cast<const uint4 *>(key_s + tid * kBandIPT);
      static_assert(kBandIPT == 8, "one 16-B load of 8 keys per thread");
      const uint4 k4 = *kv;
      const uint16_t *kp = reinterpret_cast<const uint16_t *>(&k4);
#pragma unroll
      for (int i = 0; i < kBandIPT; ++i) {
        kk[i] = kp[i];
        vv[i] = (uint16_t)(tid * kBandIPT + i);
      }
      Sort(s_sort).Sort(kk, vv, 0, a.key_bits);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kBandIPT; ++i) {
        key_s[tid * kBandIPT + i] = kk[i];
        idx_s[tid * kBandIPT + i] = vv[i];
      }
    }
    __syncthreads();
    {  // segment heads (blocked: positions tid*8 .. tid*8+7), compacted in order
      unsigned hm = 0u;
#pragma unroll
      for (int i = 0; i < kBandIPT; ++i) {
        const int p = tid * kBandIPT + i;
        const uint16_t k = key_s[p];
        if (k != pad && (p == 0 || key_s[p - 1] != k)) hm |= 1u << i;
      }
      unsigned nseg;
      unsigned o = block_excl_scan<kBandThreads>((unsigned)__popc(hm), s_part, &nseg);
#pragma unroll
      for (int i = 0; i < kBandIPT; ++i)
        if (hm >> i & 1u) seg_s[o++] = (uint16_t)(tid * kBandIPT + i);
      if (tid == 0) seg_s[nseg] = (uint16_t)n;  // the pads sort last
      __syncthreads();
      for (int s = tid; s < (int)nseg; s += kBandThreads) {
        const int s0 = seg_s[s], s1 = seg_s[s + 1];
        const int lc = key_s[s0];
        bool first = true, last = true;
        if (nchunks > 1) {
          first = !(seen_s[lc >> 5] >> (lc & 31) & 1u);
          last = last_s[lc] == (uint16_t)c;
          if (!last) atomicOr(&seen_s[lc >> 5], 1u << (lc & 31));
        }
        band_segment<kDebug, kFast>(a, m, c0 + lc, s0, s1, first, last, rec_s, idx_s, fin_s, ridx_s, cnt);
      }
    }
    __syncthreads();  // the chunk buffers are refilled
  }
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
