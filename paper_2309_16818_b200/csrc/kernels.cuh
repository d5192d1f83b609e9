// kernels.cuh -- launch arguments and host launchers of the libmem kernels.
#pragma once
#include "internal.cuh"

namespace memk {

constexpr int kThreads = 256;           // 8 warps per CTA (image, readout, post, shift kernels)
// k_bin: one CTA per tile of kTile consecutive points of one map, 8 points per thread
#ifndef MEM_BIN_THREADS
#define MEM_BIN_THREADS 256
#endif
constexpr int kBinThreads = MEM_BIN_THREADS;
constexpr int kBinPerThread = 8;
constexpr int kTile = kBinThreads * kBinPerThread;  // 2048
constexpr int kMaxBands = 2048;         // bands per map (k_bin's per-warp band counters)
// k_sort: one CTA per (map, band); the band's records counting-sorted kSortCap at a time
#ifndef MEM_SORT_THREADS
#define MEM_SORT_THREADS 256
#endif
constexpr int kSortThreads = MEM_SORT_THREADS;
constexpr int kSortCap = 1024;          // records ranked per window (shared memory)
#ifndef MEM_SORT_BULK_RUN4
#define MEM_SORT_BULK_RUN4 6
#endif
constexpr int kSortBulkRun4 = MEM_SORT_BULK_RUN4;  // k_sort: 4 x the mean run length from which runs are bulk-copied
constexpr int kSortChunk = 2048;        // band sizing: records expected per band
constexpr int kMaxBandCells = 4096;     // cells per band (per-cell arrays in shared memory)
// k_fuse: persistent grid-stride over the touched cells, one thread each
#ifndef MEM_FUSE_THREADS
#define MEM_FUSE_THREADS 128
#endif
constexpr int kFuseThreads = MEM_FUSE_THREADS;
constexpr int kShortSeg = 8;           // cells of at most this many points: a thread each
constexpr int kMidSeg = 64;            // at most this many: 8 lanes each (fast paths); longer: 16 lanes / a warp
constexpr int kMaxTilesPerMap = 8192;   // tiles of one map per call (k_sort keeps their runs in smem)
#ifndef MEM_INLINE_MAPS
#define MEM_INLINE_MAPS 128
#endif
constexpr int kInlineMaps = MEM_INLINE_MAPS;  // maps whose frames travel in the kernel parameters
// k_points: persistent grid-stride over 128-point warp-items (4 points per lane)
#ifndef MEM_WARP_PTS
#define MEM_WARP_PTS 4
#endif
constexpr int kWarpPtsPerLane = MEM_WARP_PTS;
constexpr int kWarpPoints = 32 * kWarpPtsPerLane;

// Control block of one point input (zeroed by one cudaMemsetAsync per call).
constexpr int kStatSlots = 64;  // CTAs add their counters to slot blockIdx % 64 (no hot address)
struct Control {  // two epochs: a point input adds to stats[epoch] and clears stats[epoch ^ 1]
  unsigned long long stats[2][kStatSlots][8];  // mem_stats order (n_input is derived on the host)
  unsigned n_rec, n_seg, n_lseg, n_mseg;       // this call's sorted records, short / long / mid segments (k_sort)
  unsigned n_fb;                               // cells k_cells could not certify (k_refold)
  unsigned n_fbpts;                            // their points (k_refold's list length)
};

// reset description shared by k_cells / k_sort / k_smap (lazy strips) and k_shift
struct ResetInfo {
  int n_word, n_flag, n_label;
  int label_word[kMaxGroups];
};

// Arguments of one point input, shared by the point kernels and the router.
// The call's points are split into tiles of kTile consecutive points of one map (tiles of map
// m: [tstart[m], tstart[m+1])); the physical cells [cell_lo, cell_hi) of every map are split
// into bands of band_cells cells (the last one shorter).
struct PassArgs {
  const float *pts;
  int stride;
  int vec4;                    // stride == 4 and 16-B aligned: one float4 per point
  int vec3;                    // stride == 3, 16-B aligned, every map offset a multiple of 4: 3 float4 per 4 points
  int n_maps;
  // per-map frames, point offsets [n_maps+1] and tile prefix sums [n_maps+1]: inline in the
  // kernel parameters (fi, offi, tsi) for n_maps <= kInlineMaps (no copy per call), else in a
  // staged device buffer (frames, offsets, tstart non-null)
  const PointFrame *frames;
  const long long *offsets;
  const int *tstart;
  const int *pstart;           // k_points: prefix sums of 128-point warp-items per map (staged)
  int m0, m1;                  // k_points / k_smap: maps [m0, m1) = all maps of the call
  int sc_lo, sc_hi;            // RED path, cell waves of one big map: k_points accumulates the points of
                               // the physical cells [sc_lo, sc_hi) only (sc_hi 0: every cell), into scratch
                               // cell (phys - sc_lo); k_cells fuses [cell_lo, cell_hi) = the same range
  int wave_first;               // the first cell wave of the call (counts the dropped points)
  int smap_maxpts;             // k_smap: points of the largest map of the call (shared memory layout)
  int p_uniform;               // > 0: every map has exactly this many warp-items
  double inv_p_uniform;
  unsigned long long *cnt;     // RED path scratch [n_maps][HW]: count word
  unsigned long long *rec;     // [n_maps][HW][4]: P, S, group words
  unsigned *cert;              // [n_maps][HW][2]: certificate slots (bf16x2: S, X; k_red.cuh)
  unsigned long long *fb;      // [2 k]: the k-th cell k_cells could not certify (m * HW + cell);
                               // [2 k + 1]: its list offset | point count << 32 (k_refold)
  int *fbmark;                 // [n_maps][HW]: k of an uncertified cell, else -1 (reset by k_refold)
  unsigned *fbfill;            // [k]: points listed for cell k (k_refold's collect phase) (reset by k_refold)
  unsigned *fbmap;             // [n_maps]: != 0 if the map has an uncertified cell (reset by k_refold)
  unsigned *fblist;            // point indices (relative to the map's first point) of those cells
  int t_uniform;               // > 0: every map has exactly this many tiles
  double inv_t_uniform;        // 1.0 / t_uniform (divmod_fast)
  int tmax;                    // most tiles of one map (k_sort's shared memory)
  int cell_lo, cell_hi;        // physical cells fused (a row band when sharded)
  int band_cells, nbands, key_bits;
  double inv_band, inv_nbands;
  uint4 *recs;                 // [tiles][kTile] records (k_bin -> k_sort)
  unsigned *tinfo;             // [tiles][nbands] offset | count << 16 of each band's run
  unsigned *ridx;              // [tiles][kTile] point index of each record (debug outputs only)
  uint4 *srec;                 // records sorted by cell, input order within a cell (k_sort -> k_fuse)
  unsigned *sridx;             // their point indices (debug outputs only)
  uint4 *segs;                 // one per touched cell: {m * HW + cell, first sorted record, count, 0};
                               // short cells from the front, long cells from the back,
                               // mid-size cells from seg_cap on
  unsigned seg_cap;
  int fast;                    // 1 = one colour group, 2 = one 1-channel average group (float4
                               // points), 3 = no group bound (height only), 0 = generic
  int2 *ring;                  // device ring offsets, updated to the frames' (r0, c0)
  Geometry geo;
  State st;
  mem_noise np;
  float r2lo, r2hi;            // a2: r_min <= sqrtf(r2) <= r_max  <=>  r2lo <= r2 <= r2hi (host, exact)
  int nb;
  BindDesc b[kMaxBind];
  Control *ctl;
  int epoch;                   // stats epoch of this call (0/1)
  int pdl;                     // launch with programmatic stream serialization (see launch_pdl)
  ResetInfo reset;
  int *dbg_cell;               // optional per-point outputs (MEM_FLAG_DEBUG_POINTS)
  uint8_t *dbg_code;
  PointFrame fi[kInlineMaps];
  long long offi[kInlineMaps + 1];
  int tsi[kInlineMaps + 1];
  int psi[kInlineMaps + 1];
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
// copied (stride floats) into the bucket of the rank that owns its cell's row band, in input
// order (two passes over the shard's tiles: counts, then a stable scatter)
struct RouteArgs {
  float *buf;                  // [nranks][cap][stride]
  unsigned *src;               // [nranks][cap] shard index of each routed point (debug outputs), or null
  unsigned *tcnt;              // [tiles][nranks] routed points per tile and owner, then their offsets
  unsigned *cnt;               // [nranks] routed points per owner
  long long cap;               // points per bucket (= the shard's point count)
  int band_n;                  // cells per band
  int nranks;
  int tiles;
};
cudaError_t launch_route(const PassArgs &a, const RouteArgs &r, cudaStream_t s);
cudaError_t launch_code_return(const uint8_t *codes, const unsigned *idx, long long n, uint8_t *dst, cudaStream_t s);

cudaError_t launch_bin(const PassArgs &a, int tiles, cudaStream_t s);
cudaError_t launch_sort(const PassArgs &a, cudaStream_t s);
cudaError_t launch_fuse(const PassArgs &a, cudaStream_t s);
cudaError_t launch_points(const PassArgs &a, cudaStream_t s);
size_t smap_smem_bytes(int HW, long long max_pts);
bool smap_eligible(int HW, long long max_pts);
cudaError_t launch_smap(const PassArgs &a, int grid, size_t smem, cudaStream_t s);
cudaError_t launch_cells(const PassArgs &a, cudaStream_t s);
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
  double *part;                // [nparts][d + d (d + 1) / 2 + 1] partial moments of the CTAs
  int nparts;
  double *proj;                // [k][H*W] projections (pass 0 -> pass 1)
  int k;                       // components
  const double *mean;          // [d]
  const double *comp;          // [k][d]
  unsigned long long *minmax;  // [k][2] order-preserving keys of min and max projections
  float *out;                  // [k][H][W] logical
};
int pca_parts(int HW);
cudaError_t launch_pca_moments(const PcaArgs &a, cudaStream_t s);
cudaError_t launch_pca_eigen(const PcaArgs &a, cudaStream_t s);
cudaError_t launch_pca_project(const PcaArgs &a, int pass, cudaStream_t s);
cudaError_t launch_read(const ReadArgs &a, cudaStream_t s);
cudaError_t launch_write(const ReadArgs &a, cudaStream_t s);

}  // namespace memk
