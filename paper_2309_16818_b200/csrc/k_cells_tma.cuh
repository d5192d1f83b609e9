// k_cells_tma.cuh -- k_cells for the fast paths (a9-a10, lazy a13) with bulk-copy (TMA) staged tiles.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
//
// The cell pass of one average / colour group touches every 32-B sector of the map state at
// the densities of C2 (35% of the cells), so instead of per-lane gathers of the touched cells
// (k_cells: one dependent round trip per 128-cell chunk per warp) persistent CTAs stream whole
// tiles of kTT physical cells through a kTStages-deep shared-memory ring.  Warp 8 is the
// producer: one lane issues cp.async.bulk copies of the tile's counts and staged state layers
// (completion on the stage's "full" mbarrier, expect_tx = the tile's bytes), and once the
// consumers have released a stage ("empty" mbarrier) writes its state layers and the zeroed
// count tile back with bulk stores before refilling it.  Warps 0-7 are the consumers: they
// load the scratch records of the NEXT tile's touched cells into registers (one tile ahead),
// reset the scrolled-in strips and fuse the touched cells in shared memory with the arithmetic
// of fuse_cells_avg (bit-identical results), re-zeroing the touched records with plain stores.
//
// Requirements (checked on the host, else k_cells runs): HW, cell_lo and cell_hi multiples
// of 16 (every bulk copy is 16-B aligned and a multiple of 16 bytes) and 16-B aligned bases.
// Opt-in (env MEM_CELLS_TMA=1): measured slower than k_cells on C2x64.
#pragma once

#ifndef MEM_TMA_TILE
#define MEM_TMA_TILE 512
#endif
#ifndef MEM_TMA_STAGES
#define MEM_TMA_STAGES 4
#endif
#ifndef MEM_TMA_MINB
#define MEM_TMA_MINB 3
#endif
#ifndef MEM_TMA_SUSPEND_NS
#define MEM_TMA_SUSPEND_NS 100000
#endif
constexpr int kTT = MEM_TMA_TILE;         // physical cells per tile
constexpr int kTStages = MEM_TMA_STAGES;  // tiles in flight per CTA

template <int kFast>
struct TmaTile {
  static constexpr int NCH = kFast == 1 ? 3 : 1;  // colour: r, g, b; average: one channel
  static constexpr int NW = 2 + NCH;              // word layers staged: elevation, variance, theta_k
  static constexpr int NF = 2;                    // flag layers staged: valid, observed
  static constexpr int kCnt = 0;                  // u64 counts [kTT]
  static constexpr int kWords = kCnt + 8 * kTT;   // f32 [NW][kTT]
  static constexpr int kFlags = kWords + 4 * NW * kTT;  // u8 [NF][kTT]
  static constexpr int kStage = kFlags + NF * kTT;
  static constexpr int kBytesPerCell = 8 + 4 * NW + NF;
};
constexpr int kTmaConsumers = kThreads;             // 8 consumer warps; warp 8 is the producer
constexpr int kTmaThreads = kTmaConsumers + 32;
constexpr int kTmaCellsPerThread = kTT / kTmaConsumers;

// ---------------------------------------------------------------- bulk copy / mbarrier PTX
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// blocking wait: try_wait with a suspend-time hint parks the warp until the phase completes
// (or the hint expires) instead of spinning on issue slots the fusing warps need
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(MEM_TMA_SUSPEND_NS)
        : "memory");
  } while (!ok);
}

size_t cells_tma_smem_bytes(int fast) {
  return (size_t)kTStages * (fast == 1 ? TmaTile<1>::kStage : TmaTile<2>::kStage);
}

template <int kFast>
__global__ void __launch_bounds__(kTmaThreads, MEM_TMA_MINB) k_cells_tma(const __grid_constant__ PassArgs a) {
  using L = TmaTile<kFast>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long s_full[kTStages], s_empty[kTStages];
  __shared__ int s_dirty[kTStages];
  __shared__ unsigned s_cnt[8];
  const Geometry &g = a.geo;
  const GroupDesc &gd = a.b[0].g;
  const long long BHW = g.BHW;
  float *vals = reinterpret_cast<float *>(a.st.words);
  const int tpm = (a.cell_hi - a.cell_lo + kTT - 1) / kTT;  // tiles per map (band)
  const int total = ABLATE(a, 1u) ? 0 : (a.m1 - a.m0) * tpm;
  const int ntile = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // this CTA's j-th tile: map and first physical cell (newest map first, as k_cells)
  auto tile_of = [&](int j, int &m, int &t0, int &n) {
    const int chunk = total - 1 - ((int)blockIdx.x + j * (int)gridDim.x);
    const int mi = chunk / tpm;
    m = a.m0 + mi;
    t0 = a.cell_lo + (chunk - mi * tpm) * kTT;
    n = min(kTT, a.cell_hi - t0);
  };
  auto word_layer = [&](int w) { return w < 2 ? w : gd.word0 + w - 2; };
  auto flag_layer = [&](int f) { return f == 0 ? kFlagValid : gd.flag; };
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x < kTStages) s_dirty[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(smem_addr(&s_full[s]), 1);
      mbar_init(smem_addr(&s_empty[s]), kTmaConsumers / 32);
    }
    fence_proxy_async_smem();  // the initialised barriers are visible to the bulk-copy unit
  }
  pdl_wait();  // counts and records are k_points' output
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (threadIdx.x >= kTmaConsumers) {
    // ---- producer warp, one lane: store tile t - S from stage t % S, then load tile t into it
    if (threadIdx.x == kTmaConsumers) {
      for (int t = 0; t < ntile + kTStages; ++t) {
        const int s = t % kTStages, d = t - kTStages;
        const unsigned base = smem_addr(smem + s * L::kStage);
        if (d >= 0) {
          mbar_wait(smem_addr(&s_empty[s]), (unsigned)(d / kTStages) & 1u);  // consumers are done with d
          if (s_dirty[s]) {
            int m, t0, n;
            tile_of(d, m, t0, n);
            const long long c = (long long)m * g.HW + t0;
            bulk_store(a.cnt + scratch_base(a, m) + t0, base + L::kCnt, 8u * n);
#pragma unroll
            for (int w = 0; w < L::NW; ++w)
              bulk_store(vals + word_layer(w) * BHW + c, base + L::kWords + 4 * w * kTT, 4u * n);
#pragma unroll
            for (int q = 0; q < L::NF; ++q) bulk_store(a.st.flags + flag_layer(q) * BHW + c, base + L::kFlags + q * kTT, n);
            bulk_commit();
            s_dirty[s] = 0;
            if (t < ntile) bulk_wait_read<0>();  // the stores have read the stage before it is refilled
          }
        }
        if (t < ntile) {
          int m, t0, n;
          tile_of(t, m, t0, n);
          const unsigned bar = smem_addr(&s_full[s]);
          const long long c = (long long)m * g.HW + t0;
          mbar_arrive_expect_tx(bar, (unsigned)(n * L::kBytesPerCell));
          bulk_load(base + L::kCnt, a.cnt + scratch_base(a, m) + t0, 8u * n, bar);
#pragma unroll
          for (int w = 0; w < L::NW; ++w)
            bulk_load(base + L::kWords + 4 * w * kTT, vals + word_layer(w) * BHW + c, 4u * n, bar);
#pragma unroll
          for (int q = 0; q < L::NF; ++q) bulk_load(base + L::kFlags + q * kTT, a.st.flags + flag_layer(q) * BHW + c, n, bar);
        }
      }
      bulk_wait_all();
    }
    __syncwarp();
  } else {
    // ---- consumers: the scratch records of the next tile's touched cells are loaded into
    // registers (one tile ahead) while this tile is fused in shared memory
    constexpr int C = kTmaCellsPerThread;
    ulonglong2 rc[C][2], rn[C][2];
    auto load_recs = [&](int j, ulonglong2 (&r)[C][2]) {
      int m, t0, n;
      tile_of(j, m, t0, n);
      const int s = j % kTStages;
      mbar_wait(smem_addr(&s_full[s]), (unsigned)(j / kTStages) & 1u);
      const unsigned long long *scnt = reinterpret_cast<const unsigned long long *>(smem + s * L::kStage + L::kCnt);
      const ulonglong2 *rec = reinterpret_cast<const ulonglong2 *>(a.rec + (scratch_base(a, m) + t0) * 4);
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int k = threadIdx.x + i * kTmaConsumers;
        r[i][0] = r[i][1] = make_ulonglong2(0ull, 0ull);
        if (k < n && scnt[k] != 0ull) {
          r[i][0] = __ldcg(rec + 2 * k);
          r[i][1] = __ldcg(rec + 2 * k + 1);
        }
      }
    };
    if (ntile > 0) load_recs(0, rn);
    for (int j = 0; j < ntile; ++j) {
#pragma unroll
      for (int i = 0; i < C; ++i) {
        rc[i][0] = rn[i][0];
        rc[i][1] = rn[i][1];
      }
      if (j + 1 < ntile) load_recs(j + 1, rn);
      int m, t0, n;
      tile_of(j, m, t0, n);
      const int s = j % kTStages;
      unsigned char *st = smem + s * L::kStage;
      unsigned long long *scnt = reinterpret_cast<unsigned long long *>(st + L::kCnt);
      float *sw = reinterpret_cast<float *>(st + L::kWords);
      uint8_t *sf = st + L::kFlags;
      const PointFrame f = frame_of(a, m);
      if (t0 == a.cell_lo && threadIdx.x == 0) a.ring[m] = make_int2(f.r0, f.c0);
      const long long sb = scratch_base(a, m);
      const bool shifted = f.sr != 0 || f.sc != 0;
      bool dirty = false;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int k = threadIdx.x + i * kTmaConsumers;
        if (k >= n) continue;
        const int phys = t0 + k;
        const long long c = (long long)m * g.HW + phys;
        if (shifted) {  // lazy ring shift: reset the scrolled-in cells (a13), staged layers in smem
          int pcol;
          const int prow = divmod_fast(phys, g.W, g.inv_W, pcol);
          int row = prow - f.r0, col = pcol - f.c0;
          row += row < 0 ? g.H : 0;
          col += col < 0 ? g.W : 0;
          if (in_strip(row, col, f, g)) {
            dirty = true;
            sw[0 * kTT + k] = __int_as_float(0x7fc00000);
            sw[1 * kTT + k] = __int_as_float(0x7fc00000);
#pragma unroll
            for (int w = 2; w < L::NW; ++w) sw[w * kTT + k] = 0.0f;
#pragma unroll
            for (int q = 0; q < L::NF; ++q) sf[q * kTT + k] = 0;
            for (int w = 2; w < a.reset.n_word; ++w)  // the layers of the other groups
              if (w < gd.word0 || w >= gd.word0 + L::NCH) a.st.words[(long long)w * BHW + c] = 0u;
            for (int l = 0; l < a.reset.n_label; ++l)
              reinterpret_cast<int *>(a.st.words)[(long long)a.reset.label_word[l] * BHW + c] = -1;
            for (int q = 1; q < a.reset.n_flag; ++q)
              if (q != gd.flag) a.st.flags[(long long)q * BHW + c] = 0;
          }
        }
        const unsigned long long cv = scnt[k];
        if (cv == 0ull) continue;  // untouched cells stay bit-identical
        dirty = true;
        ++cnt[7];
        scnt[k] = 0ull;  // the count tile is stored back zeroed
        const ulonglong2 ps = rc[i][0], ww = rc[i][1];
        const double P = __longlong_as_double((long long)ps.x), S = __longlong_as_double((long long)ps.y);
        const float h = sw[0 * kTT + k], s2 = sw[1 * kTT + k];
        const bool vd = sf[k] != 0, ob = sf[kTT + k] != 0;
        // a9: Kalman height fusion (D7), outliers inflate first (D11); fuse_cells_avg's arithmetic
        const double n_in = kFast == 1 ? (P > 0.0 ? 1.0 : 0.0) : (double)(uint32_t)(cv & 0xffffffffull);
        const double n_out = kFast == 1 ? (double)ww.y : (double)(uint32_t)(cv >> 32);
        if (vd) {
          const double sp = (double)s2 + n_out * (double)a.np.v_out;
          if (n_in > 0.0) {
            const double rden = 1.0 / (1.0 + P * sp);
            sw[0 * kTT + k] = __double2float_rn(((double)h + S * sp) * rden);
            sw[1 * kTT + k] = __double2float_rn(sp * rden);
          } else {
            sw[1 * kTT + k] = __double2float_rn(sp);
          }
        } else if (n_in > 0.0) {
          const double rP = 1.0 / P;
          sw[0 * kTT + k] = __double2float_rn(S * rP);
          sw[1 * kTT + k] = __double2float_rn(rP);
          sf[k] = 1;
        }
        // a10: Eq.(1)+(2) per channel
        const unsigned long long nn = kFast == 1 ? (cv >> 32) : ww.x;
        if (nn != 0ull) {
          const double rn_ = 1.0 / (double)nn;
#pragma unroll
          for (int q = 0; q < L::NCH; ++q) {
            double sk;
            if (kFast == 1) {
              const uint32_t v = q == 0 ? (uint32_t)(ww.x & 0xffffffffull)
                                        : q == 1 ? (uint32_t)(ww.x >> 32) : (uint32_t)(cv & 0xffffffffull);
              sk = (double)v;  // exact integer colour sums (D20)
            } else {
              sk = __longlong_as_double((long long)ww.y);
            }
            sw[(2 + q) * kTT + k] = rule_average_r(sw[(2 + q) * kTT + k], ob, sk, rn_, gd.w);
          }
          sf[kTT + k] = 1;
        }
        ulonglong2 *r = reinterpret_cast<ulonglong2 *>(a.rec + (sb + phys) * 4);
        __stcg(r, make_ulonglong2(0ull, 0ull));
        __stcg(r + 1, make_ulonglong2(0ull, 0ull));
      }
      fence_proxy_async_smem();  // this thread's shared-memory writes -> the producer's bulk stores
      if (__any_sync(0xffffffffu, dirty) && (threadIdx.x & 31) == 0) s_dirty[s] = 1;
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(smem_addr(&s_empty[s]));
    }
  }
  __syncthreads();
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
