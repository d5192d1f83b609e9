// kernels.cu -- the sm_100a kernels of the MEM hot path,
// one translation unit assembled from the .cuh parts included below, plus their launchers.
//
//   point_pass / k_points  a2-a8: persistent grid-stride over 128-point warp-items (cp.async
//                   double-buffered float4 stream), filters, transform, bin, noise, one batched
//                   gather for the Mahalanobis test, warp-aggregated native 64-bit REDs into the
//                   per-cell scratch
//   cell_pass / k_cells  a9-a10 + lazy a13: warp-persistent over 128-cell chunks: strip reset,
//                   Kalman height fusion, per-group rules (fp64), scratch re-zeroed
//   k_smap          batches of small maps: one CTA per map sorts its points by cell in shared
//                   memory and fuses every cell in input order (deterministic, oracle order)
//   k_route         sharded big map: route in-window points to their band owner
//   k_image         a11-a12 (+ NEXT-1 occlusion walk): project, frustum, gather, fuse (N_j = 1)
//   k_post          NEXT-3 plugins: normals, traversability, semantic argmax
//   k_readout       k_shift (eager a13), k_read / k_write (a14), PCA readout (C4)
//   k_merge         sharded big map (statistics exchange): typed fold of partial bands
//
// Everything is stream-ordered; no kernel synchronises the host.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

#ifndef MEM_POINTS_MINB
#define MEM_POINTS_MINB 3  // resident CTAs per SM the register allocation of k_points targets
#endif
#ifndef MEM_PAIR_MIN
#define MEM_PAIR_MIN 4  // colour fast path: pair lanes of the same cell when >= this many repeat
#endif
#ifndef MEM_OCC_BATCH
#define MEM_OCC_BATCH 4  // occlusion walk: intermediate cells whose loads are issued together
#endif
// DIAGNOSTICS ONLY: env MEM_ABLATE switches parts of the kernels off (PassArgs::ablate) in a
// build with -DMEM_ABLATION=1; production builds compile the checks out
#ifndef MEM_ABLATION
#define MEM_ABLATION 0
#endif
#define ABLATE(a, bit) (MEM_ABLATION && ((a).ablate & (bit)))
#ifndef MEM_FULL_ITEMS
#define MEM_FULL_ITEMS 1  // k_points: a variant of the item body without per-lane bounds for full items
#endif
#ifndef MEM_CELLS_MINB
#define MEM_CELLS_MINB 3
#endif

namespace memk {

#include "dev_common.cuh"
#include "point_pass.cuh"
#include "cell_pass.cuh"
#include "k_points.cuh"
#include "k_cells.cuh"
#include "k_smap.cuh"
#include "k_route.cuh"
#include "k_post.cuh"
#include "k_image.cuh"
#include "k_readout.cuh"
#include "k_merge.cuh"

// ---------------------------------------------------------------- launchers
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

int points_blocks_per_sm(bool debug) {
  int n = 0;
  if (debug)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_points<true, 0>, kThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_points<false, 0>, kThreads, 0);
  return n > 0 ? n : 1;
}

int cells_blocks_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_cells<0>, kThreads, 0);
  return n > 0 ? n : 1;
}

// Programmatic dependent launch: k_points and k_cells may be scheduled while the
// kernel before them on the stream drains (its CTAs retire); each waits on griddepcontrol.wait
// before it reads anything the previous kernel wrote, and lets its own dependent launch early.
template <class K>
static cudaError_t launch_pdl(K kernel, int grid, size_t smem, cudaStream_t s, const PassArgs &a,
                              int threads = kThreads) {
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
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

cudaError_t launch_points(const PassArgs &a, int grid, cudaStream_t s) {
  // the fast variants need the channel in the float4's w (vec4) and exactly one group bound
  const int f = a.vec4 ? a.fast : 0;
  const size_t fs = 0;  // no dynamic shared memory
  if (a.dbg_cell) {
    if (f == 1) return launch_pdl(k_points<true, 1>, grid, fs, s, a);
    else if (f == 2) return launch_pdl(k_points<true, 2>, grid, fs, s, a);
    else return launch_pdl(k_points<true, 0>, grid, fs, s, a);
  } else {
    if (f == 1) return launch_pdl(k_points<false, 1>, grid, fs, s, a);
    else if (f == 2) return launch_pdl(k_points<false, 2>, grid, fs, s, a);
    else return launch_pdl(k_points<false, 0>, grid, fs, s, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_cells(const PassArgs &a, int grid, cudaStream_t s) {
  if (a.fast == 1)
    return launch_pdl(k_cells<1>, grid, 0, s, a);
  if (a.fast == 2) return launch_pdl(k_cells<2>, grid, 0, s, a);
  return launch_pdl(k_cells<0>, grid, 0, s, a);
}

cudaError_t launch_post(const PostArgs &a, cudaStream_t s) {
  k_post<<<dim3(cdiv(a.geo.HW, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_smap(const PassArgs &a, int grid, size_t smem, cudaStream_t s) {
  // the opt-in shared-memory size is a per-device function attribute: set it for the current
  // device on every launch (a host-side call; maps may live on different devices)
  if (a.dbg_cell)
    cudaFuncSetAttribute(a.fast == 1 ? k_smap<true, 1> : k_smap<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  else
    cudaFuncSetAttribute(a.fast == 1 ? k_smap<false, 1> : k_smap<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSmapThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (a.dbg_cell) return a.fast == 1 ? cudaLaunchKernelEx(&cfg, k_smap<true, 1>, a) : cudaLaunchKernelEx(&cfg, k_smap<true, 2>, a);
  return a.fast == 1 ? cudaLaunchKernelEx(&cfg, k_smap<false, 1>, a) : cudaLaunchKernelEx(&cfg, k_smap<false, 2>, a);
}

cudaError_t launch_route(const PassArgs &a, const RouteArgs &r, int grid, cudaStream_t s) {
  k_route<<<grid, kThreads, 0, s>>>(a, r);
  return cudaGetLastError();
}

cudaError_t launch_image(const ImageArgs &a, cudaStream_t s) {
  k_image<<<dim3(cdiv(a.geo.HW, kImgThreads), a.geo.n_maps), kImgThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
  const int cnt = a.max_count > 0 ? a.max_count : 1;
  k_shift<<<dim3(cdiv(cnt, kThreads), a.geo.n_maps), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_moments(const PcaArgs &a, cudaStream_t s) {
  const int tile = kPcaTileBytes / (4 * a.d);
  k_pca_moments<<<cdiv(a.geo.HW, tile), kThreads, kPcaTileBytes, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pca_project(const PcaArgs &a, int pass, cudaStream_t s) {
  k_pca_project<<<cdiv(a.geo.HW, kThreads), kThreads, 0, s>>>(a, pass);
  return cudaGetLastError();
}

cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s) {
  const long long words = (long long)a.n * (1 + a.R);
  const long long blocks = (words + kThreads - 1) / kThreads;
  k_merge<<<(unsigned)(blocks < 148LL * 16 ? blocks : 148LL * 16), kThreads, 0, s>>>(a);
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
