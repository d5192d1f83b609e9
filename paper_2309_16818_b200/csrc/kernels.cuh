// kernels.cuh -- launch arguments and host launchers of the libmem kernels.
#pragma once
#include "internal.cuh"

namespace memk {

struct PointArgs {
  const float *pts;
  int stride;
  int vec4;                   // 1: stride == 4 and 16-B aligned -> one float4 load per point
  const long long *offsets;   // device, n_maps+1 (batched) or nullptr (single map: [0, n_single))
  long long n_single;
  long long max_n;            // max points of any map (grid x extent)
  const MapFrame *frames;     // device, n_maps (batched) or nullptr (single map: f0)
  MapFrame f0;
  const int2 *ring;           // device ring offsets per map
  Geometry geo;
  State st;
  mem_noise np;
  int nb;
  BindDesc b[kMaxBind];
  unsigned long long *stats;  // [8]: per-code counters (index = code + 1 as in mem_stats minus n_input)
  int *dbg_cell;              // optional, per point
  uint8_t *dbg_code;
};

struct CellArgs {
  Geometry geo;
  State st;
  float v_out;
  int nb;
  BindDesc b[kMaxBind];
  unsigned long long *stats;
};

struct ImageArgs {
  const float *img;
  int C, IH, IW;
  long long map_stride;       // floats between consecutive maps' images
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
  const ShiftRec *recs;       // device, n_maps (batched) or nullptr (single map: rec0)
  ShiftRec rec0;
  int2 *ring;                 // updated in place to the records' (r0, c0)
  int n_word, n_flag;
  int n_label;
  int label_word[kMaxGroups];
  int max_count;              // max over maps of the number of cells to reset
};

enum ReadKind { RK_ELEV = 0, RK_VAR = 1, RK_WORD = 2, RK_LABEL = 3, RK_FLAG = 4, RK_THETA = 5 };

struct ReadArgs {
  Geometry geo;
  State st;
  const int2 *ring;
  int kind, idx;              // layer kind and index (word or flag layer)
  int first, K, flag;         // theta: first alpha word layer, class count, observed flag layer
  float *out;                 // read: logical row-major [n_maps][H][W]
  const float *src;           // write
};

cudaError_t launch_point(const PointArgs &a, cudaStream_t s);
cudaError_t launch_cell(const CellArgs &a, cudaStream_t s);
cudaError_t launch_image(const ImageArgs &a, cudaStream_t s);
cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s);
cudaError_t launch_read(const ReadArgs &a, cudaStream_t s);
cudaError_t launch_write(const ReadArgs &a, cudaStream_t s);

constexpr int kPointThreads = 256;
constexpr int kPointsPerThread = 2;
constexpr int kPointsPerBlock = kPointThreads * kPointsPerThread;

}  // namespace memk
