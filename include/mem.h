/*
 * mem.h -- C-ABI of libmem, the B200 (sm_100a) MEM fusion library.
 *
 * MEM = the multi-modal elevation map of arXiv 2309.16818 (PAPER.md in the reference).
 * The calls follow the paper's statement of the problem:
 *   mem_create(resolution, size, layers, per-layer fusion rule)
 *   mem_input_pointcloud(xyz+channels, R, t, noise params)
 *   mem_input_image(CxHxW channels, K, R, t)
 *   mem_move_to(position)                                             robot-centric
 *   mem_get_layer(name)                                               GridMap publish
 * plus batched variants (many independent maps per call) and test/inspection calls.
 *
 * Conventions (readings D1..D31 of SURVEY.md §8(c)):
 * - Map: `rows` x `cols` cells of `resolution` metres; logical row <-> +x, col <-> +y (D13);
 *   centre = (kx*res, ky*res), (kx, ky) integers snapped by mem_move_to (D14).
 * - Every layer is read/written as logical row-major float32 [rows][cols] (batched:
 *   [n_maps][rows][cols]).  Internally the map is a ring buffer.
 * - Pointers to points, images and layer buffers may be HOST or DEVICE memory (detected
 *   with cudaPointerGetAttributes).  Device pointers are caller-owned and must stay valid
 *   until the stream work completes (stream-ordered, asynchronous).  Host input buffers
 *   are copied before the call returns (pageable) or stream-ordered (pinned: keep them
 *   unchanged until the stream has passed the call).  Host OUTPUT buffers are written
 *   before the call returns (the call synchronises the map's stream).
 * - All device work runs on the map's stream (set at create, changeable with
 *   mem_set_stream).  No call synchronises the device except where stated.
 * - Every call returns a mem_status; out-params are written only on MEM_OK.  On an error
 *   no device work is enqueued.  mem_last_error() returns a thread-local message.
 * - Thread safety: a handle is exclusively owned by one thread during a call.
 * - There is no CPU fallback: without a CUDA device every call returns MEM_ECUDA.
 */
#ifndef MEM_H_
#define MEM_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MEM_API __attribute__((visibility("default")))
#else
#define MEM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mem_map mem_map;       /* opaque; owns all map memory (freed by mem_destroy) */
typedef struct CUstream_st *mem_stream; /* identical to cudaStream_t; NULL = legacy default stream */

typedef enum {
  MEM_OK = 0,
  MEM_EINVAL = -1,    /* bad argument (sizes, offsets, widths, NULL pointers, K matrix ...) */
  MEM_EDUPNAME = -2,  /* duplicate group name or a name equal to elevation/variance/valid */
  MEM_ENOTFOUND = -3, /* unknown layer name */
  MEM_ERULE = -4,     /* rule vs channel semantics mismatch (e.g. class rule on 1 channel) */
  MEM_EPOSE = -5,     /* R not orthonormal within 1e-6 or det(R) != +1 within 1e-6 */
  MEM_ECUDA = -6,     /* CUDA runtime error (no device, launch failure, ...) */
  MEM_ENOMEM = -7,    /* device or host allocation failed */
  MEM_ECOMM = -8      /* collective communication error (reserved for the sharded map) */
} mem_status;

/* Fusion rules. */
typedef enum {
  MEM_AVERAGE = 0,        /* Eq.(1)+(2) PAPER.md:265-292: a = mean of the frame's points; theta = w a + (1-w) theta;
                             first touch theta = a (D3); w = 1 is "Latest" */
  MEM_GAUSSIAN = 1,       /* Eq.(3)-(7) PAPER.md:294-324: conjugate Normal mean/variance per dimension,
                             prior = current posterior, first touch prior (mu0, sigma0_2) (D4) */
  MEM_CLASS_AVERAGE = 2,  /* Eq.(2) on class-probability vectors PAPER.md:290 (D1) */
  MEM_CLASS_BAYESIAN = 3, /* Eq.(8)-(12) PAPER.md:326-357: alpha += sum m_i; theta = alpha/sum(alpha) at readout (D5, D6) */
  MEM_CLASS_MAX = 4,      /* per frame winner (max prob, lowest class on ties) overwrites (label, conf) (D19) */
  MEM_COLOR = 5           /* RGB average(w) (D20): points carry packed 0x00RRGGBB in one float; images 3 channels */
} mem_rule;

/* One fusion GROUP = one rule over n_channels input channels.  Layer names it exposes
 * (mem_get_layer / mem_set_layer):
 *   average, class_average: "name" (n=1) or "name_k"; "name_observed"
 *   gaussian:               "name"/"name_k" (mean), "name_var"/"name_var_k"; "name_observed"
 *   class_bayesian:         "name_k" (theta, read-only, derived), "name_alpha_k"; "name_observed"
 *   class_max:              "name_label" (-1 = unobserved, D15), "name_conf"
 *   color:                  "name_r", "name_g", "name_b" (0..255); "name_observed"
 * Base layers: "elevation", "variance" (NaN where invalid), "valid" (0/1). */
typedef struct {
  const char *name; /* 1..39 chars, unique, not elevation/variance/valid */
  int rule;         /* mem_rule */
  int n_channels;   /* input width: K classes (>= 2 for class rules), d features, 3 for color; <= 256 */
  float w;          /* average / class_average / color: 0 < w <= 1 */
  float sigma_f2;   /* gaussian: known measurement variance > 0 */
  float mu0;        /* gaussian: prior mean */
  float sigma0_2;   /* gaussian: prior variance > 0 */
  float alpha0;     /* class_bayesian: Dirichlet prior per class > 0 */
} mem_layer_spec;

/* Binds an input channel range to a group.  Point clouds: ch_offset counts from float 3 of a
 * point (the first channel after xyz); images: from channel 0.  n_ch must equal the group's
 * input width (color: 1 packed channel for points, 3 for images).  A group may be bound at
 * most once per call; one channel range may feed several groups.
 * Top-k class input ("inputting the top k classes";
 * SPEC.md:144-147, 168-176; reading D38): topk = k > 0 binds n_ch = 2k channels
 * holding (class id, probability) pairs to a class rule group of n_channels = K + 1, whose last
 * class K is the reserved "other" class: the pairs expand to the dense vector
 * dense[id_j] += p_j, dense[K] = 1 - sum_j p_j (fp32, pair order), which is then fused like
 * dense input.  A point/pixel with a non-finite value or an id that is not an integer in
 * [0, K) skips the group (like a non-finite channel, D31).  topk = 0: dense channels. */
typedef struct {
  int ch_offset;
  int n_ch;
  int group; /* index into the mem_layer_spec array given at create */
  int topk;  /* 0 = dense channels; k > 0 = k (id, probability) pairs (see above) */
} mem_binding;

/* Point noise model and filters (readings D8-D11, D30). */
typedef struct {
  float a, b;         /* per-point variance v = a + b r^2, r = sensor-frame range; v must be > 0 */
  float r_min, r_max; /* keep iff r_min <= r <= r_max */
  float h_min, h_max; /* keep iff h_min <= (R p)_z <= h_max (height relative to the sensor) */
  float tau2;         /* outlier iff cell valid and (z - h)^2 > tau2 (sigma^2 + v) */
  float v_out;        /* each outlier inflates the cell variance by v_out before fusion */
} mem_noise;

/* Per-call counters of the last point input (summed over maps).
 * Invariant: n_input = n_nonfinite + n_range + n_height + n_oob + n_inlier + n_outlier. */
typedef struct {
  uint64_t n_input, n_nonfinite, n_range, n_height, n_oob, n_inlier, n_outlier, n_cells_touched;
} mem_stats;

/* Per-point codes written by mem_debug_point_codes (filter order D9). */
enum { MEM_CODE_INLIER = 0, MEM_CODE_OUTLIER = 1, MEM_CODE_NONFINITE = 2, MEM_CODE_RANGE = 3,
       MEM_CODE_HEIGHT = 4, MEM_CODE_OOB = 5 };

#define MEM_FLAG_DEBUG_POINTS 1u /* record per-point (cell, code) of the last point input */
/* Every point input is deterministic and performs the oracle's arithmetic (DESIGN.md reading
 * D39): the per-cell sums are either added in input order (sort-by-cell paths) or with
 * fp64 atomics whose exactness is certified per cell (any order gives the exact sum, hence the
 * sequential one), uncertified cells being recomputed in input order.  The flag is kept for
 * compatibility and has no effect. */
#define MEM_FLAG_DETERMINISTIC 2u
/* Validation: always fuse point inputs by the sort-by-cell pipeline (k_bin, k_sort, k_fuse)
 * instead of the certified-atomic path or the small-map kernel; results are bit-identical
 * either way (tests/test_full_size_gpu.py checks it). */
#define MEM_FLAG_FUSE_SORTED 4u

/* ---- lifetime -------------------------------------------------------------------- */

/* Creates one map: valid = 0, elevation/variance NaN, multimodal 0, observed 0, labels -1,
 * centre (0, 0).  groups may be NULL when n_groups == 0.
 * Errors: EINVAL (resolution <= 0, rows/cols < 1, rows*cols > 2^31, bad spec), EDUPNAME, ERULE,
 * ENOMEM, ECUDA. */
MEM_API mem_status mem_create(float resolution, int rows, int cols, const mem_layer_spec *groups, int n_groups,
                      unsigned flags, mem_stream stream, mem_map **out);

/* Creates n_maps independent maps with identical geometry and groups (one handle). */
MEM_API mem_status mem_create_batch(int n_maps, float resolution, int rows, int cols, const mem_layer_spec *groups,
                            int n_groups, unsigned flags, mem_stream stream, mem_map **out);

/* Synchronises the stream and frees everything.  NULL is a no-op. */
MEM_API mem_status mem_destroy(mem_map *map);

/* Changes the stream (synchronises the old one first). */
MEM_API mem_status mem_set_stream(mem_map *map, mem_stream stream);

/* Blocks until all work enqueued on the map's stream has finished. */
MEM_API mem_status mem_synchronize(mem_map *map);

/* ---- one big map sharded across ranks ----------------------------
 * Rank r owns the physical row band [r*rows/nranks, (r+1)*rows/nranks) (rows divisible by
 * nranks) and every rank takes its own shard of each frame's points.  Point routing: each rank
 * filters and bins its shard, counts its dropped points, and sends every in-window point to the
 * owner of its cell's band (a stable scatter: input order within each destination); the owner
 * tests, accumulates and fuses what it received -- source ranks in order, each in input order,
 * i.e. the global input order -- for its band only, so every cell equals the unsharded map bit
 * for bit.  A rank keeps only its own band current (the readout all-gathers; an image input
 * with occlusion all-gathers elevation and valid first).  With MEM_FLAG_DEBUG_POINTS the
 * owners' inlier / outlier codes are returned to the source ranks.
 * Counters (mem_frame_stats) are per rank and add up to the unsharded counters.  Transport:
 *  - NCCL (nccl_id != NULL, one process per GPU): the per-destination counts all-gathered
 *    (one host synchronisation per point input), the points moved with grouped
 *    ncclSend/ncclRecv, stream-ordered on the map's stream.  Every call on a sharded map is
 *    collective (all ranks, same order); mem_get_layer all-gathers every layer first.
 *  - local (nccl_id == NULL): the nranks shards live in one process on one device (testing
 *    and single-GPU emulation); mem_input_pointcloud only routes, and
 *    mem_shard_local_sync(shards) moves the routed points with device copies and runs the
 *    owners' passes; call it after every point input, with every shard having taken the same
 *    sequence of calls.  All shards must use the same stream.
 * Images: every rank takes the whole image and fuses the cells of its own band (the image
 * fusion is per cell, PAPER §3.3); moves are replicated (every rank calls mem_move_to).
 * Errors: EINVAL (rows % nranks, rank range, shards out of step), ENOMEM, ECOMM (NCCL), ECUDA. */
MEM_API mem_status mem_nccl_unique_id(void *id128);
MEM_API mem_status mem_create_sharded(float resolution, int rows, int cols, const mem_layer_spec *groups,
                                      int n_groups, unsigned flags, mem_stream stream, const void *nccl_id128,
                                      int rank, int nranks, mem_map **out);
MEM_API mem_status mem_shard_local_sync(mem_map **shards, int nranks);

/* ---- inputs ---------------------------------------------------------------------- */

/* Fuses one point cloud: n points of `stride` floats (xyz in the
 * sensor frame, then channels), AoS, host or device.  R (row-major 3x3, sensor->map) and
 * t (sensor position in the map/world frame) are host doubles.  n == 0 is legal and leaves
 * the map unchanged.  Atomic per call: on error nothing is enqueued.  Every result equals the
 * sequential oracle bit for bit whatever the path: one colour group, one
 * 1-channel average group (stride 4, 16-B aligned) or no group take the certified-atomic path
 * when the call's 1/v terms span few binades (colour: at most 131,586 points per map per call);
 * batches of >= 64 small maps the one-CTA-per-map kernel; everything else the sort pipeline.
 * Errors: EINVAL (n < 0, stride < 3, bad binding, a <= 0, b < 0, a + b r_max^2 not finite), EPOSE,
 * ECUDA. */
MEM_API mem_status mem_input_pointcloud(mem_map *map, const float *pts, int64_t n, int stride, const mem_binding *bind,
                                int n_bind, const double R[9], const double t[3], const mem_noise *noise);

/* Batched: map m takes points [offsets[m], offsets[m+1]) of pts; offsets (host, n_maps+1,
 * non-decreasing, offsets[0] = 0), R (host, n_maps x 9), t (host, n_maps x 3). */
MEM_API mem_status mem_input_pointcloud_batch(mem_map *map, const float *pts, const int64_t *offsets, int stride,
                                      const mem_binding *bind, int n_bind, const double *R, const double *t,
                                      const mem_noise *noise);

/* Fuses one image (a11-a12): C x H x W float32 (CHW), host or device; K row-major 3x3 with
 * K[1] = skew, K[3] = K[6] = K[7] = 0, K[8] = 1, fx, fy > 0; R, t camera->map (optical axis
 * +z_c, x right, y down, D17).  Only valid cells are projected; elevation/valid untouched.
 * Errors: EINVAL, EPOSE, ECUDA. */
MEM_API mem_status mem_input_image(mem_map *map, const float *img, int C, int H, int W, const mem_binding *bind,
                           int n_bind, const double K[9], const double R[9], const double t[3]);

/* Batched: img is n_maps x C x H x W; K, R (n_maps x 9), t (n_maps x 3), host. */
MEM_API mem_status mem_input_image_batch(mem_map *map, const float *img, int C, int H, int W, const mem_binding *bind,
                                 int n_bind, const double *K, const double *R, const double *t);

/* ---- post-processing plugins on the fused map (PAPER.md:379-385,
 * Table II rows "normal calculation", "traversability"; DESIGN.md readings
 * D35-D37).  Outputs are logical row-major float32 planes [k][n_maps][rows][cols] into `out`
 * (host or device, like mem_get_layer); no stored layer changes. ---- */

/* 3 planes normal_x, normal_y, normal_z: unit (-gx, -gy, 1)/|.| with gx (rows, +x) and gy
 * (cols, +y) the central difference of the valid neighbours, one-sided when only one is
 * valid; NaN for invalid cells and cells without a valid neighbour along either axis. */
MEM_API mem_status mem_plugin_normals(const mem_map *map, float *out);

/* 1 plane in [0, 1]: clamp(min(slope, step), 0, 1), slope = (n_z - cos(slope_max)) /
 * (1 - cos(slope_max)) with cos rounded once to fp32, step = 1 - max |h_nb - h| / step_max over
 * the valid 8-neighbours; NaN where the normal is invalid.  slope_max in radians.
 * Errors: EINVAL (step_max <= 0, cos(slope_max) >= 1). */
MEM_API mem_status mem_plugin_traversability(const mem_map *map, float slope_max, float step_max, float *out);

/* 2 planes class_id, confidence: argmax_k theta_k of a class group (class_bayesian: alpha /
 * sum alpha as read out; class_average: its values; class_max: its label and conf), ties to
 * the lowest class; -1 and 0 where unobserved.  Errors: ENOTFOUND, ERULE (not a class rule). */
MEM_API mem_status mem_plugin_semantic_argmax(const mem_map *map, const char *group, float *out);

/* Image association with the occlusion test of PAPER.md:234-236, for
 * the following mem_input_image[_batch] calls of this map (default off: frustum only, D18).
 * A valid in-frustum cell is fused only if every intermediate cell of the Bresenham line from
 * the camera's footprint cell to it (8-connected, endpoints excluded; cells outside the map
 * and cells with valid = 0 do not occlude) has elevation <= ray height + eps_occ, the ray
 * height linear in the 2D distance between the camera height and the cell's elevation
 * (readings D32-D34).  eps_occ: metres, >= 0 (1e-4 in SPEC).
 * Errors: EINVAL (eps_occ negative or not finite). */
MEM_API mem_status mem_set_image_occlusion(mem_map *map, int enable, float eps_occ);

/* Recentres on (x, y) snapped to the lattice, k = floor(x/res + 1/2) (D14); scrolled-in
 * cells are reset to the create state.  Errors: EINVAL (non-finite), ECUDA. */
MEM_API mem_status mem_move_to(mem_map *map, double x, double y);

/* Batched: xy host, n_maps x 2. */
MEM_API mem_status mem_move_to_batch(mem_map *map, const double *xy);

/* ---- readout / state -------------------------------------------------------------- */

/* Writes layer `name` as logical row-major float32 (n_maps*rows*cols values) into `out`
 * (host or device).  Elevation/variance are NaN where valid = 0; class_bayesian theta is
 * derived as alpha / sum(alpha) (0 where unobserved); labels as floats.  Errors: ENOTFOUND. */
MEM_API mem_status mem_get_layer(const mem_map *map, const char *name, float *out);

/* Overwrites a stored layer from logical row-major float32 (host or device); flags take
 * value != 0; labels are truncated to int.  Derived layers (class_bayesian theta) give
 * EINVAL.  Used for single-step parity and resume.
 * The variance of a cell with valid = 0 is not stored (it reads as NaN anyway): writing
 * "variance" stores NaN there, writing 0 to "valid" clears the variance.  To restore a
 * state, write "valid" before "variance". */
MEM_API mem_status mem_set_layer(mem_map *map, const char *name, const float *src);

/* PCA readout of a feature group (BASELINE configs[3]):
 * per map, over the cells where the group is observed: covariance of the group's values
 * (average / class_average: theta; gaussian: means) from fp64 moments, top-k eigenvectors
 * (one CTA on the device: Householder tridiagonalisation, Sturm multisection, inverse
 * iteration; each sign makes its largest-|coefficient| positive), projections min-max scaled to [0, 1] (0 when the component is constant or beyond
 * the covariance's rank, and on unobserved cells).  out: n_maps x k x rows x cols float32,
 * logical row-major, host or device.  Stream-ordered: nothing returns to the host (a host
 * `out` is copied back and the stream synchronised).
 * Errors: ENOTFOUND (no such group), EINVAL (rule without values, k < 1, k > n_channels or
 * more than 64 channels). */
MEM_API mem_status mem_pca_readout(mem_map *map, const char *group, int k, float *out);

/* Newline-separated layer names into buf (NUL-terminated); EINVAL if cap is too small. */
MEM_API mem_status mem_get_layer_names(const mem_map *map, char *buf, size_t cap);

/* Bytes of per-cell map state held in device memory (all stored layers and flags, all maps;
 * fp32 layers count 4 B/cell, flags 1 B/cell). */
MEM_API mem_status mem_memory_footprint(const mem_map *map, uint64_t *bytes);

/* Map geometry and centre lattice indices (kxy: host, n_maps x 2). */
MEM_API mem_status mem_get_info(const mem_map *map, int *n_maps, int *rows, int *cols, float *resolution);
MEM_API mem_status mem_get_center(const mem_map *map, int64_t *kxy);

/* Counters of the last point input; synchronises the stream. */
MEM_API mem_status mem_frame_stats(const mem_map *map, mem_stats *out);

/* Per-point (logical cell index row*cols+col or -1, code) of the last point input, for maps
 * created with MEM_FLAG_DEBUG_POINTS; host or device buffers of n (total) entries.
 * EINVAL if the flag was not set. */
MEM_API mem_status mem_debug_point_codes(const mem_map *map, int32_t *cell, uint8_t *code);

/* ---- profiling (Table II-style stage times) ----------------------- */

/* Stages timed by mem_profile_read. */
enum { MEM_STAGE_SHIFT = 0, MEM_STAGE_POINT = 1, MEM_STAGE_CELL = 2, MEM_STAGE_IMAGE = 3, MEM_STAGE_READ = 4,
       MEM_STAGE_WRITE = 5, MEM_STAGE_H2D = 6, MEM_STAGE_D2H = 7, MEM_N_STAGES = 8 };

/* enable != 0: bracket every subsequent kernel launch / staging copy with CUDA events on
 * the map's stream (no host synchronisation).  enable == 0 stops; counters are kept. */
MEM_API mem_status mem_profile(mem_map *map, int enable);

/* Synchronises the stream, then writes per-stage device milliseconds (sum over launches
 * since the last reset) and launch counts (counted whether or not profiling is enabled).
 * reset != 0 clears both afterwards.  ms and counts: host arrays of MEM_N_STAGES (either
 * may be NULL). */
MEM_API mem_status mem_profile_read(mem_map *map, double *ms, uint64_t *counts, int reset);

/* Thread-local description of the last error (never NULL). */
MEM_API const char *mem_last_error(void);

/* Library version string. */
MEM_API const char *mem_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MEM_H_ */
