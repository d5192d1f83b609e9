// kernels.cu -- the sm_100a kernels of the MEM hot path,
// one translation unit assembled from the .cuh parts included below, plus their launchers.
//
//   point_pass / k_bin  a2-a6: one CTA per 2048-point tile: filters, transform, binning, noise
//                   variance for every point (the oracle's fp32 expressions); the in-window
//                   points split stably by cell band into per-tile runs (16-B records)
//   k_sort          lazy a13 + stable counting sort: one CTA per (map, band): strip reset, the
//                   band's records in input order sorted by cell (input order kept per cell)
//   k_fuse          a7-a10: one thread per touched cell: Mahalanobis test, fp64 sums in input
//                   order, Kalman height update and the group rules -- the oracle's operations
//                   in the oracle's order
//   k_route         sharded big map: route in-window points to their band owner (stable)
//   k_image         a11-a12 (+ NEXT-1 occlusion walk): project, frustum, gather, fuse (N_j = 1)
//   k_post          NEXT-3 plugins: normals, traversability, semantic argmax
//   k_readout       k_shift (eager a13), k_read / k_write (a14), PCA readout (C4)
//
// Everything is stream-ordered; no kernel synchronises the host.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cub/block/block_radix_sort.cuh>

#ifndef MEM_OCC_BATCH
#define MEM_OCC_BATCH 4  // occlusion walk: intermediate cells whose loads are issued together
#endif
#ifndef MEM_PAIR_MIN
#define MEM_PAIR_MIN 4  // colour RED path: pair lanes of the same cell when >= this many repeat
#endif
#ifndef MEM_FULL_ITEMS
#define MEM_FULL_ITEMS 1  // k_points: a variant of the item body without per-lane bounds for full items
#endif

namespace memk {

#include "dev_common.cuh"
#include "point_pass.cuh"
#include "k_bin.cuh"
#include "k_red.cuh"
#include "k_sort.cuh"
#include "k_fuse.cuh"
#include "k_cells.cuh"
#include "k_smap.cuh"
#include "k_route.cuh"
#include "k_post.cuh"
#include "k_image.cuh"
#include "k_readout.cuh"

// ---------------------------------------------------------------- launchers
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// Programmatic dependent launch: k_bin, k_sort and the router may be scheduled while the
// kernel before them on the stream drains (its CTAs retire); each waits on griddepcontrol.wait
// before it reads anything the previous kernel wrote, and lets its own dependent launch early.
template <class K, class... Extra>
static cudaError_t launch_pdl(K kernel, int grid, size_t smem, cudaStream_t s, const PassArgs &a, int threads,
                              const Extra &...extra) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a, extra...);
}

cudaError_t launch_bin(const PassArgs &a, int tiles, cudaStream_t s) {
  const bool dbg = a.dbg_cell != nullptr;
  switch (a.fast) {
    case 1: return dbg ? launch_pdl(k_bin<true, 1>, tiles, 0, s, a, kBinThreads) : launch_pdl(k_bin<false, 1>, tiles, 0, s, a, kBinThreads);
    case 2: return dbg ? launch_pdl(k_bin<true, 2>, tiles, 0, s, a, kBinThreads) : launch_pdl(k_bin<false, 2>, tiles, 0, s, a, kBinThreads);
    case 3: return dbg ? launch_pdl(k_bin<true, 3>, tiles, 0, s, a, kBinThreads) : launch_pdl(k_bin<false, 3>, tiles, 0, s, a, kBinThreads);
    default: return dbg ? launch_pdl(k_bin<true, 0>, tiles, 0, s, a, kBinThreads) : launch_pdl(k_bin<false, 0>, tiles, 0, s, a, kBinThreads);
  }
}

template <bool kDebug>
static cudaError_t launch_sort_t(const PassArgs &a, size_t smem, cudaStream_t s) {
  // the opt-in shared-memory limit is a per-device function attribute: raised once per device
  static bool raised[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!raised[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(k_sort<kDebug>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    raised[dev & 63] = true;
  }
  return launch_pdl(k_sort<kDebug>, a.n_maps * a.nbands, smem, s, a, kSortThreads);
}

cudaError_t launch_sort(const PassArgs &a, cudaStream_t s) {
  const size_t smem = SortSmem(a.tmax, a.band_cells).total;
  return a.dbg_cell ? launch_sort_t<true>(a, smem, s) : launch_sort_t<false>(a, smem, s);
}

template <bool kDebug, int kFast, int kPart>
static cudaError_t launch_fuse_p(const PassArgs &a, cudaStream_t s) {
  static int grid[64] = {};  // resident CTAs per device (persistent grid)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!grid[dev & 63]) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fuse<kDebug, kFast, kPart>, kFuseThreads, 0);
    grid[dev & 63] = std::max(1, sms) * std::max(1, per);
  }
  return launch_pdl(k_fuse<kDebug, kFast, kPart>, grid[dev & 63], 0, s, a, kFuseThreads);
}

template <bool kDebug, int kFast>
static cudaError_t launch_fuse_t(const PassArgs &a, cudaStream_t s) {
  cudaError_t e = launch_fuse_p<kDebug, kFast, 1>(a, s);  // long and mid-size cells
  if (e != cudaSuccess) return e;
  return launch_fuse_p<kDebug, kFast, 0>(a, s);  // short cells
}

cudaError_t launch_fuse(const PassArgs &a, cudaStream_t s) {
  const bool dbg = a.dbg_cell != nullptr;
  switch (a.fast) {
    case 1: return dbg ? launch_fuse_t<true, 1>(a, s) : launch_fuse_t<false, 1>(a, s);
    case 2: return dbg ? launch_fuse_t<true, 2>(a, s) : launch_fuse_t<false, 2>(a, s);
    case 3: return dbg ? launch_fuse_t<true, 3>(a, s) : launch_fuse_t<false, 3>(a, s);
    default: return dbg ? launch_fuse_t<true, 0>(a, s) : launch_fuse_t<false, 0>(a, s);
  }
}

// the RED path (k_points, k_cells, k_refold): persistent grids sized once per device
template <class K>
static int resident_grid(K kernel, int threads, int slot) {
  static int grid[64][16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int &gd = grid[dev & 63][slot];
  if (!gd) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
    gd = std::max(1, sms) * std::max(1, per);
  }
  return gd;
}

template <bool kDebug, int kFast, bool kWave = false>
static cudaError_t launch_points_t(const PassArgs &a, cudaStream_t s) {
  const long long items = (long long)(a.pstart ? 0 : a.psi[a.m1] - a.psi[a.m0]);
  int g = resident_grid(k_points<kDebug, kFast, kWave>, kThreads, kWave ? 10 + kFast : kFast + (kDebug ? 3 : 0));
  if (items > 0) g = (int)std::max(1LL, std::min<long long>(g, (items + 7) / 8));
  return launch_pdl(k_points<kDebug, kFast, kWave>, g, 0, s, a, kThreads);
}

cudaError_t launch_points(const PassArgs &a, cudaStream_t s) {
  const bool dbg = a.dbg_cell != nullptr;
  const int f = a.fast == 3 ? 0 : a.fast;
  if (a.sc_hi > 0) {  // cell waves of one big map (never with debug outputs): their own instantiation,
                      // so that the filter costs the other calls no registers
    if (f == 1) return launch_points_t<false, 1, true>(a, s);
    if (f == 2) return launch_points_t<false, 2, true>(a, s);
    return launch_points_t<false, 0, true>(a, s);
  }
  if (f == 1) return dbg ? launch_points_t<true, 1>(a, s) : launch_points_t<false, 1>(a, s);
  if (f == 2) return dbg ? launch_points_t<true, 2>(a, s) : launch_points_t<false, 2>(a, s);
  return dbg ? launch_points_t<true, 0>(a, s) : launch_points_t<false, 0>(a, s);
}

template <int kFast>
static cudaError_t launch_cells_t(const PassArgs &a, cudaStream_t s) {
  const long long chunks = (long long)(a.m1 - a.m0) * ((a.cell_hi - a.cell_lo + kChunk - 1) / kChunk);
  const int res = resident_grid(k_cells<kFast, kChunkPerLane>, kThreads, 6 + kFast);
  cudaError_t e;
  if (chunks >= (long long)res * (kThreads / 32)) {  // a chunk for every resident warp
    e = launch_pdl(k_cells<kFast, kChunkPerLane>, res, 0, s, a, kThreads);
  } else {  // small calls (C3, single maps): 32-cell chunks
    const long long ch1 = (long long)(a.m1 - a.m0) * ((a.cell_hi - a.cell_lo + 31) / 32);
    const int g = (int)std::max(1LL, std::min<long long>(resident_grid(k_cells<kFast, 1>, kThreads, 13 + kFast),
                                                         (ch1 + 7) / 8));
    e = launch_pdl(k_cells<kFast, 1>, g, 0, s, a, kThreads);
  }
  if (e != cudaSuccess) return e;
  // uncertified cells (none: k_refold returns at once): a cooperative launch (its collect
  // phase and its folds are separated by a grid barrier), every CTA resident
  const size_t smem = refold_smem_bytes<kFast>();
  e = cudaFuncSetAttribute(k_refold<kFast>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  static int coop[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int &grid = coop[dev & 63][kFast];
  if (!grid) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_refold<kFast>, kRefoldThreads, smem);
    grid = std::max(1, sms * std::max(1, std::min(per, 1)));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRefoldThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_refold<kFast>, a);
}

cudaError_t launch_cells(const PassArgs &a, cudaStream_t s) {
  const int f = a.fast == 3 ? 0 : a.fast;
  if (f == 1) return launch_cells_t<1>(a, s);
  if (f == 2) return launch_cells_t<2>(a, s);
  return launch_cells_t<0>(a, s);
}

cudaError_t launch_smap(const PassArgs &a, int grid, size_t smem, cudaStream_t s) {
  // the opt-in shared-memory size is a per-device function attribute: set it for the current
  // device on every launch (a host-side call; maps may live on different devices)
  const bool dbg = a.dbg_cell != nullptr;
  auto k = dbg ? (a.fast == 1 ? k_smap<true, 1> : k_smap<true, 2>) : (a.fast == 1 ? k_smap<false, 1> : k_smap<false, 2>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k, grid, smem, s, a, kSmapThreads);
}

cudaError_t launch_post(const PostArgs &a, cudaStream_t s) {
  k_post<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_route(const PassArgs &a, const RouteArgs &r, cudaStream_t s) {
  if (r.tiles > 0) {
    cudaError_t e = launch_pdl(k_route_count, r.tiles, 0, s, a, kBinThreads, r);
    if (e != cudaSuccess) return e;
  }
  k_route_scan<<<1, kThreads, 0, s>>>(r);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || r.tiles == 0) return e;
  return launch_pdl(k_route_scatter, r.tiles, 0, s, a, kBinThreads, r);
}

cudaError_t launch_code_return(const uint8_t *codes, const unsigned *idx, long long n, uint8_t *dst, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((n + kThreads - 1) / kThreads, 148LL * 8);
  k_code_return<<<(unsigned)blocks, kThreads, 0, s>>>(codes, idx, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_image(const ImageArgs &a, cudaStream_t s) {
  bool simple = !a.occlusion;
  for (int i = 0; i < a.nb && simple; ++i) simple = a.b[i].topk == 0 && a.b[i].g.rule != MEM_GAUSSIAN;
  int nch = 0;  // the widest binding
  for (int i = 0; i < a.nb; ++i) nch = std::max(nch, a.b[i].nch);
  const dim3 grid(cdiv(a.geo.HW, kImgCells), a.geo.n_maps);
  if (simple && nch <= 32 && kImgBatch > 8)  // C3's 20 classes: shorter batches (C3 frame -2 us)
    k_image<true, 8><<<grid, kImgThreads, 0, s>>>(a);
  else if (simple)
    k_image<true, kImgBatch><<<grid, kImgThreads, 0, s>>>(a);
  else
    k_image<false, kImgBatch><<<grid, kImgThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
  const int cnt = a.max_count > 0 ? a.max_count : 1;
  k_shift<<<dim3(cdiv(cnt, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

int pca_parts(int HW) { return (int)std::min<long long>(2 * 148, (HW + kPcaTile - 1) / kPcaTile); }

cudaError_t launch_pca_moments(const PcaArgs &a, cudaStream_t s) {
  const size_t smem = sizeof(double) * pca_ldc(a.d);
  cudaError_t e = cudaFuncSetAttribute(k_pca_moments, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_pca_moments<<<a.nparts, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_eigen(const PcaArgs &a, cudaStream_t s) {
  const int nv = a.d + a.d * (a.d + 1) / 2 + 1;
  k_pca_sum<<<cdiv(nv, 32), kThreads, 0, s>>>(a);
  // A [d][d + 1], eigenvectors [k][d], LU scratch [4][k][d]
  const size_t smem = sizeof(double) * ((size_t)a.d * (a.d + 1) + 5 * (size_t)a.k * a.d);
  cudaError_t e = cudaFuncSetAttribute(k_pca_eigen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_pca_eigen<<<1, kPcaEigThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_project(const PcaArgs &a, int pass, cudaStream_t s) {
  k_pca_project<<<cdiv(a.geo.HW, kThreads), kThreads, 0, s>>>(a, pass);
  return cudaGetLastError();
}

cudaError_t launch_read(const ReadArgs &a, cudaStream_t s) {
  k_read<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_write(const ReadArgs &a, cudaStream_t s) {
  k_write<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace memk
