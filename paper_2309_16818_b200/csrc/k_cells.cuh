// k_cells.cuh -- k_cells (a9-a10, lazy a13).
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- k_cells (a9-a10, lazy a13)
constexpr int kChunkPerLane = 4;                 // cells per lane per chunk
constexpr int kChunk = 32 * kChunkPerLane;        // 128-cell chunk per warp

// Warp-persistent grid-stride over 128-cell chunks of the wave's maps (newest map first: its
// scratch was touched last by k_points and is still in L2).  Each warp, independently of the
// others (no CTA barrier): 4 count loads per lane in flight, the pending shift strips reset,
// its touched cells compacted in its own shared-memory slice, then fused 2 per lane per round.
template <int kFast>
__global__ void __launch_bounds__(kThreads, MEM_CELLS_MINB) k_cells(const __grid_constant__ PassArgs a) {
  __shared__ int s_phys[kThreads / 32][kChunk];
  __shared__ unsigned long long s_cntv[kThreads / 32][kChunk];
  __shared__ unsigned s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Geometry &g = a.geo;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (kThreads / 32);
  const int gw = blockIdx.x * (kThreads / 32) + wid;
  const int cpm = (a.cell_hi - a.cell_lo + kChunk - 1) / kChunk;  // chunks per map (band)
  const int total = ABLATE(a, 1u) ? 0 : (a.m1 - a.m0) * cpm;
  int *sp = s_phys[wid];
  unsigned long long *sc = s_cntv[wid];
  for (int rt = gw; rt < total; rt += nwarps) {
    const int chunk = ABLATE(a, 32u) ? rt : total - 1 - rt;
    const int mi = chunk / cpm;
    const int m = a.m0 + mi;
    const int t0 = a.cell_lo + (chunk - mi * cpm) * kChunk;
    const int sb = (int)scratch_base(a, m);
    unsigned long long cv[kChunkPerLane];
#pragma unroll
    for (int u = 0; u < kChunkPerLane; ++u) {  // counts first (memory-level parallelism)
      const int phys = t0 + u * 32 + lane;
      cv[u] = phys < a.cell_hi ? __ldcg(a.cnt + sb + phys) : 0ull;
    }
    const PointFrame f = frame_of(a, m);
    if (t0 == a.cell_lo && lane == 0) a.ring[m] = make_int2(f.r0, f.c0);
    int n = 0;
#pragma unroll
    for (int u = 0; u < kChunkPerLane; ++u) {
      const int phys = t0 + u * 32 + lane;
      if (phys < a.cell_hi && (f.sr != 0 || f.sc != 0)) {  // lazy ring shift: reset the scrolled-in cells (a13)
        int pcol;
        const int prow = divmod_fast(phys, g.W, g.inv_W, pcol);
        int row = prow - f.r0, col = pcol - f.c0;
        row += row < 0 ? g.H : 0;
        col += col < 0 ? g.W : 0;
        if (in_strip(row, col, f, g)) reset_cell(a.st, g.BHW, (long long)m * g.HW + phys, a.reset);
      }
      const bool t = cv[u] != 0ull;  // untouched cells stay bit-identical
      const unsigned b = __ballot_sync(0xffffffffu, t);
      if (t) {
        const int k = n + __popc(b & lanemask_lt());
        sp[k] = phys;
        sc[k] = cv[u];
      }
      n += __popc(b);
    }
    __syncwarp();
    cnt[7] += lane == 0 ? (unsigned)n : 0u;
    for (int k0 = 0; k0 < (ABLATE(a, 512u) ? 0 : n); k0 += 64) {
      int ph[2];
      unsigned long long cc[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u * 32 + lane;
        ph[u] = k < n ? sp[k] : -1;
        cc[u] = k < n ? sc[k] : 0ull;
      }
      if (kFast == 1)
        fuse_cells_avg<2, 3, true>(a, m, sb, ph, cc);
      else if (kFast == 2)
        fuse_cells_avg<2, 1, false>(a, m, sb, ph, cc);
      else
        fuse_cells<2>(a, m, sb, ph, cc);
    }
    __syncwarp();  // this warp's slice is rewritten by its next chunk
  }
  __syncthreads();
  flush_stats(s_cnt, cnt, &a.ctl->stats[a.epoch][0][0]);
}
