// kernels.cuh -- launch arguments and host launchers of the libmem kernels.
#pragma once
#include "internal.cuh"

namespace memk {

constexpr int kThreads = 256;           // 8 warps per CTA
#ifndef MEM_WARP_PTS
#define MEM_WARP_PTS 4
#endif
constexpr int kWarpPtsPerLane = MEM_WARP_PTS;  // point warp-item = 128 points (4 float4 loads in flight per lane)
constexpr int kWarpPoints = 32 * kWarpPtsPerLane;
constexpr int kWarpCellsPerLane = 4;    // cell warp-item = 128 physical cells
constexpr int kWarpCells = 32 * kWarpCellsPerLane;
constexpr int kInlineMaps = 128;        // maps whose frames travel in the kernel parameters

// Control block of one point input (zeroed by one cudaMemsetAsync per call).
constexpr int kStatSlots = 64;  // CTAs add their counters to slot blockIdx % 64 (no hot address)
struct Control {  // two epochs: a point input adds to stats[epoch] and clears stats[epoch ^ 1]
  unsigned long long stats[2][kStatSlots][8];  // mem_stats order (n_input is derived on the host)
};

// reset description shared by k_cells (lazy strips) and k_shift
struct ResetInfo {
  int n_word, n_flag, n_label;
  int label_word[kMaxGroups];
};

// Arguments of one wave (maps [m0, m1)) of a point input, shared by k_points and k_cells
// (DESIGN.md §4.2).  Per-cell scratch of map m lives in map-slot scratch_slot(m) of the pool:
// waves alternate between the two halves so that k_cells(w) overlaps k_points(w+1).
struct PassArgs {
  const float *pts;
  int stride;
  int vec4;                    // stride == 4 and 16-B aligned: one float4 per point
  // per-map frames, point offsets [n_maps+1] and prefix sums of point warp-items [n_maps+1]:
  // inline in the kernel parameters (fi, offi, psi) for n_maps <= kInlineMaps (no copy per
  // call), else in a staged device buffer (frames, offsets, pstart non-null)
  const PointFrame *frames;
  const long long *offsets;
  const int *pstart;
  int m0, m1;                  // maps of this wave
  int cell_lo, cell_hi;        // k_cells: physical cells [lo, hi) of each map (a row band when sharded)
  int p_uniform;               // > 0: every map of the wave has exactly this many point warp-items
  double inv_p_uniform;        // 1.0 / p_uniform (divmod_fast)
  int slot0;                   // scratch map-slot of map m0 (map m -> slot slot0 + m - m0)
  int q_per_map;               // cell warp-items per map
  long long SHW;               // scratch map-slots * HW
  unsigned long long *cnt;     // scratch counts [SHW]
  unsigned long long *rec;     // scratch records [SHW][R]
  int R;                       // record words per cell
  int fast;                    // k_cells fast path: 1 = one colour group, 2 = one 1-channel average group
  int2 *ring;                  // device ring offsets, updated to the frames' (r0, c0)
  Geometry geo;
  State st;                    // st.acc: [n_acc][map-slots][HW]
  mem_noise np;
  int nb;
  BindDesc b[kMaxBind];
  Control *ctl;
  int epoch;                   // stats epoch of this call (0/1)
  int pdl;                     // launch with programmatic stream serialization (see launch_pdl)
  int smap_maxpts;             // k_smap: points of the largest map of the call (shared memory layout)
  ResetInfo reset;
  int *dbg_cell;               // optional per-point outputs (MEM_FLAG_DEBUG_POINTS)
  uint8_t *dbg_code;
  PointFrame fi[kInlineMaps];
  long long offi[kInlineMaps + 1];
  int psi[kInlineMaps + 1];
  unsigned ablate;             // DIAGNOSTICS ONLY (env MEM_ABLATE, honoured by builds with -DMEM_ABLATION=1;
                               // results are wrong when != 0):
                               // 1 skip cell updates, 2 skip REDs, 4 skip state gathers, 8 skip point math,
                               // 32 forward (not newest-first) cell tile order, 64 no warp aggregation
};

struct ImageArgs {
  int row_lo, row_hi;          // physical rows fused (the owned band when sharded)
  int occlusion;               // NEXT-1: Bresenham occlusion test of every in-frustum cell
  float eps_occ;
  const float *img;
  int C, IH, IW;
  long long map_stride;        // floats between consecutive maps' images
  const MapFrame *frames;
  MapFrame f0;
  const int2 *ring;
  Geometry geo;
  State st;
  int nb;
  BindDesc b[kMaxBind];
};

struct ShiftArgs {
  Geometry geo;
  State st;
  const ShiftRec *recs;        // device, n_maps (batched) or nullptr (single map: rec0)
  ShiftRec rec0;
  int2 *ring;                  // updated in place to the records' (r0, c0)
  ResetInfo reset;
  int max_count;               // max over maps of the number of cells to reset
};

enum ReadKind { RK_ELEV = 0, RK_VAR = 1, RK_WORD = 2, RK_LABEL = 3, RK_FLAG = 4, RK_THETA = 5 };

struct ReadArgs {
  Geometry geo;
  State st;
  const int2 *ring;
  int kind, idx;               // layer kind and index (word or flag layer)
  int first, K, flag;          // theta: first alpha word layer, class count, observed flag layer
  float *out;                  // read: logical row-major [n_maps][H][W]
  const float *src;            // write
};

// NEXT-3 post-processing plugins: one thread per logical cell
struct PostArgs {
  Geometry geo;
  State st;
  const int2 *ring;
  int op;                      // 0 normals (3 layers), 1 traversability, 2 semantic argmax (2 layers)
  float cos_max, step_max;     // traversability
  int rule, first, K, flag, label;  // argmax: group rule, first value word, classes, observed flag, label word
  float *out;                  // [n_layers][n_maps][H][W] logical row-major
};
cudaError_t launch_post(const PostArgs &a, cudaStream_t s);

// sharded big map, point routing: every in-window point of this rank's shard is
// copied (stride floats) into the bucket of the rank that owns its cell's row band
struct RouteArgs {
  float *buf;                  // [nranks][cap][stride]
  unsigned *cnt;               // [nranks] points appended per destination (zeroed before)
  long long cap;               // points per bucket (= the shard's point count)
  int band_n;                  // cells per band
};
cudaError_t launch_route(const PassArgs &a, const RouteArgs &r, int grid, cudaStream_t s);

cudaError_t launch_points(const PassArgs &a, int grid, cudaStream_t s);
cudaError_t launch_cells(const PassArgs &a, int grid, cudaStream_t s);
size_t smap_smem_bytes(int HW, long long max_pts);
bool smap_eligible(int HW, long long max_pts);
cudaError_t launch_smap(const PassArgs &a, int grid, size_t smem, cudaStream_t s);
cudaError_t launch_image(const ImageArgs &a, cudaStream_t s);
cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s);
// PCA readout: moments of one map's feature group, then projections
struct PcaArgs {
  Geometry geo;
  State st;
  const int2 *ring;
  int map;                     // map index
  int word0, d, flag;          // feature layers [word0, word0 + d), observed flag layer
  double *sums;                // [d] sum x, then [d (d + 1) / 2] sum x_a x_b (a <= b), then count
  int k;                       // components
  const double *mean;          // [d]
  const double *comp;          // [k][d]
  unsigned long long *minmax;  // [k][2] order-preserving keys of min and max projections
  float *out;                  // [k][H][W] logical
};
cudaError_t launch_pca_moments(const PcaArgs &a, cudaStream_t s);
cudaError_t launch_pca_project(const PcaArgs &a, int pass, cudaStream_t s);
// sharded map: fold the partial scratch of the other ranks for this rank's band
struct MergeArgs {
  unsigned long long *cnt;           // own scratch counts (band cells [lo, lo + n))
  unsigned long long *rec;           // own scratch records [HW][R]
  const unsigned long long *src_cnt; // nsrc partial count bands, each n words, contiguous
  const unsigned long long *src_rec; // nsrc partial record bands, each n * R words
  int nsrc, lo, n, R;
  const uint8_t *wtype;              // [R]: 0 f64 sum, 1 u64 sum, 2 u64 max
};
cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s);
cudaError_t launch_read(const ReadArgs &a, cudaStream_t s);
cudaError_t launch_write(const ReadArgs &a, cudaStream_t s);
int points_blocks_per_sm(bool debug);
int cells_blocks_per_sm();

}  // namespace memk
