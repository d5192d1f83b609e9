// mem_api.cu -- host side of the libmem C-ABI (include/mem.h): argument validation, the
// layer registry, device state allocation, per-call parameter staging and kernel launches.
// No compute happens here: every step of the path runs in kernels.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

// host-side checkpoint timing of the point input (diagnostics: -DMEM_HOST_PROF=1, off by default)
#if MEM_HOST_PROF
#include <chrono>
static double g_hp[32];
static long long g_hp_n;
static void hp_report();
static std::chrono::high_resolution_clock::time_point g_hp_t0;
#define HP_START() (g_hp_t0 = std::chrono::high_resolution_clock::now(), ++g_hp_n == 100 ? hp_report() : (void)0)
#define HP(i) (g_hp[i] += std::chrono::duration<double, std::micro>(std::chrono::high_resolution_clock::now() - g_hp_t0).count())
static void hp_report() {
  if (!g_hp_n) return;
  fprintf(stderr, "host prof (%lld calls, us since call start):", g_hp_n);
  for (int i = 0; i < 32; ++i)
    if (g_hp[i] != 0.0) fprintf(stderr, " [%d] %.2f", i, g_hp[i] / g_hp_n);
  fprintf(stderr, "\n");
  for (int i = 0; i < 32; ++i) g_hp[i] = 0.0;
  g_hp_n = 0;
}
#else
#define HP_START() ((void)0)
#define HP(i) ((void)0)
static void hp_report() {}
#endif

#include "kernels.cuh"

using namespace memk;

#ifndef MEM_BAND_RECS
#define MEM_BAND_RECS 768  // records aimed at per band (k_sort)
#endif

namespace {

thread_local std::string g_err = "no error";

mem_status fail(mem_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CU(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return fail(MEM_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

enum LayerKind { LK_ELEV, LK_VAR, LK_VALID, LK_WORD, LK_LABEL, LK_FLAG, LK_THETA };

struct Layer {
  std::string name;
  int kind, idx;          // word or flag layer index
  int first, K, flag;     // theta only
};

// pinned host staging slots with events: the host writes a slot immediately, the H2D copy
// reads it later in stream order, so a slot is reused only after its copy has executed.
struct PinnedRing {
  static constexpr int kSlots = 8;
  void *host[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  size_t cap = 0;
  int next = 0;
};

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[MEM_N_STAGES];
  double ms[MEM_N_STAGES] = {};
  uint64_t count[MEM_N_STAGES] = {};
};

}  // namespace

struct mem_map {
  int B = 1, H = 0, W = 0;
  float res = 0.f;
  unsigned flags = 0;
  cudaStream_t stream = nullptr;
  int device = 0;
  int ng = 0;
  GroupDesc g[kMaxGroups];
  std::string gname[kMaxGroups];
  int n_word = 0, n_flag = 0, n_acc = 0;
  int n_label = 0, label_word[kMaxGroups] = {};
  std::vector<Layer> layers;
  State st{};
  int2 *ring = nullptr;
  std::vector<long long> kx, ky;
  std::vector<int> r0, c0;
  // staging
  void *dparam = nullptr;
  size_t dparam_cap = 0;
  PinnedRing pin;
  unsigned *seen_rec = nullptr;  // pinned: in-window records of a recent point input (band sizing)
  void *din = nullptr;
  size_t din_cap = 0;
  float *dout = nullptr;
  size_t dout_cap = 0;
  void *pca_buf = nullptr;  // PCA readout scratch
  size_t pca_cap = 0;
  Control *ctl = nullptr;   // per-call counters (two epochs) and list lengths
  size_t ctl_bytes = 0;
  int pdl = 1;               // programmatic dependent launch
  int occlusion = 0;         // image association with the Bresenham occlusion test (NEXT-1)
  float eps_occ = 1e-4f;
  int epoch = 1;             // stats epoch of the last point input (the first one uses 0)
  bool stats_empty = true;   // the last point input had no points (all counters 0)
  int sms = 148;            // SMs of the device (band count heuristic)
  // point pass buffers: k_bin records and run table, sorted records, segments,
  // debug point indices
  void *recs = nullptr, *tinfo = nullptr, *ridx = nullptr, *srec = nullptr, *sridx = nullptr, *segs = nullptr;
  size_t recs_cap = 0, tinfo_cap = 0, ridx_cap = 0, srec_cap = 0, sridx_cap = 0, segs_cap = 0;
  // RED path scratch (zeroed once, re-zeroed by k_cells): count words, records, certificates, fallback list
  void *rcnt_s = nullptr, *rrec_s = nullptr, *rcert_s = nullptr, *rfb_s = nullptr;
  void *rmark_s = nullptr, *rfill_s = nullptr, *rmapfb_s = nullptr, *rlist_s = nullptr;
  size_t rlist_cap = 0, red_all = 0;
  size_t red_cells = 0;  // cells the RED scratch holds
  bool pending = false;     // a mem_move_to shift not yet applied (folded into the next point pass)
  // sharded big map: 0 none, 1 NCCL, 2 local (one process, one device)
  int transport = 0, rank = 0, nranks = 1;
  int band_lo = 0, band_n = 0;          // owned physical cells [band_lo, band_lo + band_n)
  ncclComm_t comm = nullptr;
  bool exchange_pending = false;        // local transport: routed, owner passes not yet run
  PassArgs shard_args{};                // the owner pass arguments of the frame being fused
  float *rbuf = nullptr;                // [nranks][cap][stride] outgoing points by owner band, input order
  unsigned *rsrc = nullptr;             // [nranks][cap] their shard indices (debug outputs)
  size_t rsrc_cap = 0;
  unsigned *rtile = nullptr;            // [tiles][nranks] routed points per tile and owner
  size_t rtile_cap = 0;
  int *odbg_cell = nullptr;             // owner pass debug outputs, by received position
  uint8_t *odbg_code = nullptr;
  size_t odbg_cap = 0;
  uint8_t *rcode = nullptr;             // NCCL: codes of this shard's routed points, back from their owners
  size_t rcode_cap = 0;
  std::vector<unsigned> route_all;      // [nranks][nranks] routed counts of the last frame
  size_t rbuf_cap = 0;                  // bytes
  unsigned *rcnt = nullptr;             // [nranks] outgoing counts (device)
  unsigned *rall = nullptr;             // [nranks][nranks] all ranks' counts (device, NCCL)
  float *rin = nullptr;                 // incoming points of this rank's band
  size_t rin_cap = 0;                   // bytes
  long long route_cap = 0;              // points per outgoing bucket of the last frame
  int route_stride = 0;
  std::vector<ShiftRec> pend;
  int *dbg_cell = nullptr;
  uint8_t *dbg_code = nullptr;
  size_t dbg_cap = 0;
  long long dbg_n = 0;
  Prof prof;

  ResetInfo reset_info() const {
    ResetInfo r;
    memset(&r, 0, sizeof r);
    r.n_word = n_word;
    r.n_flag = n_flag;
    r.n_label = n_label;
    for (int i = 0; i < n_label; ++i) r.label_word[i] = label_word[i];
    return r;
  }

  Geometry geo() const {
    Geometry gg;
    gg.H = H;
    gg.W = W;
    gg.HW = H * W;
    gg.n_maps = B;
    gg.BHW = (long long)B * H * W;
    gg.res = res;
    gg.hH = (float)H / 2.0f;
    gg.hW = (float)W / 2.0f;
    gg.inv_W = 1.0 / (double)W;
    return gg;
  }
};

namespace {

cudaEvent_t prof_event(mem_map *m) {
  if (!m->prof.pool.empty()) {
    cudaEvent_t e = m->prof.pool.back();
    m->prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

// runs one launch / copy of `stage`, bracketed by events when profiling is on
template <class F>
mem_status timed(mem_map *m, cudaStream_t st, int stage, const char *what, F &&op) {
  m->prof.count[stage]++;
  cudaEvent_t a = nullptr, b = nullptr;
  if (m->prof.on) {
    a = prof_event(m);
    b = prof_event(m);
    if (!a || !b) return fail(MEM_ECUDA, "cudaEventCreate failed");
    CU(cudaEventRecord(a, st));
  }
  const cudaError_t e = op();
  if (e != cudaSuccess) return fail(MEM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  if (m->prof.on) {
    CU(cudaEventRecord(b, st));
    m->prof.pending[stage].emplace_back(a, b);
  }
  return MEM_OK;
}

#define TIMED_ON(st, stage, expr)                                            \
  do {                                                                       \
    mem_status ts_ = timed(m, st, stage, #expr, [&]() { return (expr); });   \
    if (ts_ != MEM_OK) return ts_;                                           \
  } while (0)
#define TIMED(stage, expr) TIMED_ON(m->stream, stage, expr)

bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

mem_status grow(void **buf, size_t *cap, size_t need, cudaStream_t s) {
  if (need <= *cap) return MEM_OK;
  CU(cudaStreamSynchronize(s));
  if (*buf) CU(cudaFree(*buf));
  *buf = nullptr;
  *cap = 0;
  size_t c = need < 4096 ? 4096 : need + need / 4;
  if (cudaMalloc(buf, c) != cudaSuccess) {
    cudaGetLastError();
    return fail(MEM_ENOMEM, "cudaMalloc(%zu) failed", c);
  }
  *cap = c;
  return MEM_OK;
}

// copies `bytes` of host data to the map's device parameter buffer (stream-ordered).
mem_status stage_params(mem_map *m, const void *src, size_t bytes, void **dptr) {
  mem_status s = grow(&m->dparam, &m->dparam_cap, bytes, m->stream);
  if (s != MEM_OK) return s;
  PinnedRing &p = m->pin;
  if (bytes > p.cap) {
    CU(cudaStreamSynchronize(m->stream));
    for (int i = 0; i < PinnedRing::kSlots; ++i) {
      if (p.host[i]) CU(cudaFreeHost(p.host[i]));
      p.host[i] = nullptr;
    }
    size_t c = bytes < 4096 ? 4096 : bytes + bytes / 4;
    for (int i = 0; i < PinnedRing::kSlots; ++i) {
      if (cudaMallocHost(&p.host[i], c) != cudaSuccess) {
        cudaGetLastError();
        return fail(MEM_ENOMEM, "cudaMallocHost(%zu) failed", c);
      }
      if (!p.ev[i]) CU(cudaEventCreateWithFlags(&p.ev[i], cudaEventDisableTiming));
    }
    p.cap = c;
  }
  const int k = p.next;
  p.next = (p.next + 1) % PinnedRing::kSlots;
  CU(cudaEventSynchronize(p.ev[k]));
  memcpy(p.host[k], src, bytes);
  CU(cudaMemcpyAsync(m->dparam, p.host[k], bytes, cudaMemcpyHostToDevice, m->stream));
  CU(cudaEventRecord(p.ev[k], m->stream));
  *dptr = m->dparam;
  return MEM_OK;
}

// returns a device pointer holding `bytes` of the caller's input (copied if it is host memory).
mem_status stage_input(mem_map *m, const void *src, size_t bytes, const void **dptr) {
  if (bytes == 0 || is_device_ptr(src)) {
    *dptr = src;
    return MEM_OK;
  }
  mem_status s = grow(&m->din, &m->din_cap, bytes, m->stream);
  if (s != MEM_OK) return s;
  TIMED(MEM_STAGE_H2D, cudaMemcpyAsync(m->din, src, bytes, cudaMemcpyHostToDevice, m->stream));
  *dptr = m->din;
  return MEM_OK;
}

// R^T R = I within 1e-6 and det(R) = +1 within 1e-6 (host, fp64).
bool rotation_ok(const double *R) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double d = R[a] * R[b] + R[3 + a] * R[3 + b] + R[6 + a] * R[6 + b];
      double e = (a == b) ? 1.0 : 0.0;
      if (!std::isfinite(d) || std::fabs(d - e) > 1e-6) return false;
    }
  const double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                     R[2] * (R[3] * R[7] - R[4] * R[6]);
  return std::fabs(det - 1.0) <= 1e-6;
}

// ---- exact thresholds of the oracle's fp32 decisions (readings D9, D13).  Every
// float is mapped to an integer key in its numeric order; a monotone predicate over the floats
// is then bisected on the keys.
static long long fkey(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? -(long long)(u & 0x7fffffffu) : (long long)u;
}
static float kfloat(long long k) {
  const uint32_t u = k >= 0 ? (uint32_t)k : (0x80000000u | (uint32_t)(-k));
  float f;
  memcpy(&f, &u, 4);
  return f;
}
// least float in [lo, hi] (keys) where pred turns true (pred monotone false -> true; pred(hi) true)
template <class P>
static float least_true(long long lo, long long hi, P pred) {
  while (lo < hi) {
    const long long mid = lo + (hi - lo) / 2;
    if (pred(kfloat(mid))) hi = mid; else lo = mid + 1;
  }
  return kfloat(lo);
}
// r_min <= sqrtf(r2) <= r_max  <=>  lo <= r2 <= hi over r2 >= +0 (a2, reading D9); an empty
// set gives lo = +inf, hi = -1
static void range_thresholds(float r_min, float r_max, float *lo, float *hi) {
  const long long k0 = fkey(0.0f), kinf = fkey(INFINITY);
  auto ge_min = [&](float x) { volatile float r = std::sqrt(x); return r >= r_min; };
  auto gt_max = [&](float x) { volatile float r = std::sqrt(x); return !(r <= r_max); };
  if (!ge_min(INFINITY) || gt_max(0.0f)) {
    *lo = INFINITY;
    *hi = -1.0f;
    return;
  }
  *lo = least_true(k0, kinf, ge_min);
  if (!gt_max(INFINITY)) {
    *hi = INFINITY;
  } else {
    const float first_out = least_true(k0, kinf, gt_max);
    *hi = kfloat(fkey(first_out) - 1);
  }
}

// a1: frame setup on the host -- t relative to the map centre in fp64, then fp32 (D13)
MapFrame make_frame(const mem_map *m, int map, const double *R, const double *t, const double *K) {
  MapFrame f;
  memset(&f, 0, sizeof f);
  for (int k = 0; k < 9; ++k) f.R[k] = (float)R[k];
  const double cx = (double)m->kx[map] * (double)m->res, cy = (double)m->ky[map] * (double)m->res;
  f.t[0] = (float)(t[0] - cx);
  f.t[1] = (float)(t[1] - cy);
  f.t[2] = (float)t[2];
  if (K) {
    f.K[0] = (float)K[0];
    f.K[1] = (float)K[1];
    f.K[2] = (float)K[2];
    f.K[3] = (float)K[4];
    f.K[4] = (float)K[5];
  }
  return f;
}

mem_status resolve_bindings(const mem_map *m, const mem_binding *bind, int nb, bool image, int stride_or_C,
                            BindDesc *out) {
  if (nb < 0 || nb > kMaxBind) return fail(MEM_EINVAL, "n_bind %d out of [0, %d]", nb, kMaxBind);
  if (nb > 0 && !bind) return fail(MEM_EINVAL, "bindings NULL");
  for (int i = 0; i < nb; ++i) {
    const mem_binding &b = bind[i];
    if (b.group < 0 || b.group >= m->ng) return fail(MEM_EINVAL, "binding %d: group %d out of range", i, b.group);
    const GroupDesc &g = m->g[b.group];
    const int avail = image ? stride_or_C : stride_or_C - 3;
    if (b.ch_offset < 0 || b.n_ch < 1 || b.ch_offset + b.n_ch > avail)
      return fail(MEM_EINVAL, "binding %d: channels [%d, %d) outside the %d input channels", i, b.ch_offset,
                  b.ch_offset + b.n_ch, avail);
    if (b.topk < 0) return fail(MEM_EINVAL, "binding %d: topk %d < 0", i, b.topk);
    if (b.topk > 0) {  // top-k class input (D38)
      if (g.rule != MEM_CLASS_AVERAGE && g.rule != MEM_CLASS_BAYESIAN && g.rule != MEM_CLASS_MAX)
        return fail(MEM_ERULE, "binding %d: top-k input needs a class rule (group '%s')", i,
                    m->gname[b.group].c_str());
      if (b.n_ch != 2 * b.topk)
        return fail(MEM_EINVAL, "binding %d: top-%d input takes %d channels, got %d", i, b.topk, 2 * b.topk, b.n_ch);
    } else {
      const int want = g.rule == MEM_COLOR ? (image ? 3 : 1) : g.nch;
      if (b.n_ch != want)
        return fail(MEM_EINVAL, "binding %d: group '%s' takes %d channel(s), got %d", i,
                    m->gname[b.group].c_str(), want, b.n_ch);
    }
    for (int j = 0; j < i; ++j)
      if (bind[j].group == b.group) return fail(MEM_EINVAL, "group '%s' bound twice", m->gname[b.group].c_str());
    out[i].ch_offset = b.ch_offset;
    out[i].nch = b.n_ch;
    out[i].group = b.group;
    out[i].topk = b.topk;
    out[i].g = g;
  }
  return MEM_OK;
}

mem_status check_map(const mem_map *m) {
  if (!m) return fail(MEM_EINVAL, "map is NULL");
  return MEM_OK;
}

mem_status set_device(const mem_map *m) {
  CU(cudaSetDevice(m->device));
  return MEM_OK;
}

void add_layer(mem_map *m, const std::string &name, int kind, int idx, int first = 0, int K = 0, int flag = 0) {
  Layer l;
  l.name = name;
  l.kind = kind;
  l.idx = idx;
  l.first = first;
  l.K = K;
  l.flag = flag;
  m->layers.push_back(l);
}

mem_status reset_all(mem_map *m) {
  ShiftArgs a;
  memset(&a, 0, sizeof a);
  a.geo = m->geo();
  a.st = m->st;
  a.recs = nullptr;
  a.rec0.sr = m->H;  // |s| >= size: every cell
  a.rec0.sc = 0;
  a.rec0.r0 = 0;
  a.rec0.c0 = 0;
  a.ring = m->ring;
  a.reset = m->reset_info();
  a.max_count = m->H * m->W;
  CU(launch_shift(a, m->stream));
  return MEM_OK;
}

// applies a pending (lazy) shift eagerly with k_shift; every call other than a point input
// does this first, so kernels that read the map never see an unapplied shift.
mem_status flush_shift(mem_map *m) {
  if (!m->pending) return MEM_OK;
  m->pending = false;
  ShiftArgs a;
  memset(&a, 0, sizeof a);
  a.geo = m->geo();
  a.st = m->st;
  a.ring = m->ring;
  a.reset = m->reset_info();
  int max_count = 0;
  for (const ShiftRec &r : m->pend) {
    const int ar = r.sr < 0 ? -r.sr : r.sr, ac = r.sc < 0 ? -r.sc : r.sc;
    const int cnt = (ar >= m->H || ac >= m->W) ? m->H * m->W : ar * m->W + ac * m->H;
    if (cnt > max_count) max_count = cnt;
  }
  a.max_count = max_count;
  if (m->B == 1) {
    a.rec0 = m->pend[0];
  } else {
    void *d = nullptr;
    mem_status s = stage_params(m, m->pend.data(), sizeof(ShiftRec) * m->B, &d);
    if (s != MEM_OK) return s;
    a.recs = reinterpret_cast<const ShiftRec *>(d);
  }
  TIMED(MEM_STAGE_SHIFT, launch_shift(a, m->stream));
  return MEM_OK;
}

void free_map(mem_map *m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  cudaFree(m->st.words);
  cudaFree(m->st.flags);
  cudaFree(m->st.acc);
  cudaFree(m->ring);
  cudaFree(m->dparam);
  cudaFree(m->din);
  cudaFree(m->dout);
  cudaFree(m->pca_buf);
  cudaFree(m->recs);
  cudaFree(m->tinfo);
  cudaFree(m->ridx);
  cudaFree(m->srec);
  cudaFree(m->sridx);
  cudaFree(m->segs);
  cudaFree(m->rcnt_s);
  cudaFree(m->rrec_s);
  cudaFree(m->rcert_s);
  cudaFree(m->rfb_s);
  cudaFree(m->rmark_s);
  cudaFree(m->rfill_s);
  cudaFree(m->rmapfb_s);
  cudaFree(m->rlist_s);
  cudaFree(m->rsrc);
  cudaFree(m->rtile);
  cudaFree(m->odbg_cell);
  cudaFree(m->odbg_code);
  cudaFree(m->rcode);
  cudaFree(m->rbuf);
  cudaFree(m->rcnt);
  cudaFree(m->rall);
  cudaFree(m->rin);
  if (m->comm) ncclCommDestroy(m->comm);
  cudaFree(m->ctl);
  cudaFree(m->dbg_cell);
  cudaFree(m->dbg_code);
  if (m->seen_rec) cudaFreeHost(m->seen_rec);
  for (int i = 0; i < PinnedRing::kSlots; ++i) {
    if (m->pin.host[i]) cudaFreeHost(m->pin.host[i]);
    if (m->pin.ev[i]) cudaEventDestroy(m->pin.ev[i]);
  }
  for (cudaEvent_t e : m->prof.pool) cudaEventDestroy(e);
  for (auto &v : m->prof.pending)
    for (auto &pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  cudaGetLastError();
  delete m;
}

}  // namespace

extern "C" {

const char *mem_last_error(void) { return g_err.c_str(); }

const char *mem_version(void) { return "libmem 0.1.0 (sm_100a)"; }

mem_status mem_create_batch(int n_maps, float resolution, int rows, int cols, const mem_layer_spec *groups,
                            int n_groups, unsigned flags, mem_stream stream, mem_map **out) {
  if (!out) return fail(MEM_EINVAL, "out is NULL");
  if (n_maps < 1 || n_maps > 65535) return fail(MEM_EINVAL, "n_maps %d out of [1, 65535]", n_maps);
  if (!(resolution > 0.0f) || !std::isfinite(resolution)) return fail(MEM_EINVAL, "resolution must be > 0");
  if (rows < 1 || cols < 1 || (long long)n_maps * rows * cols > (1LL << 31) - 1)
    return fail(MEM_EINVAL, "n_maps x rows x cols = %d x %d x %d invalid (must be < 2^31 cells)", n_maps, rows, cols);
  if (n_groups < 0 || n_groups > kMaxGroups) return fail(MEM_EINVAL, "n_groups %d out of [0, %d]", n_groups, kMaxGroups);
  if (n_groups > 0 && !groups) return fail(MEM_EINVAL, "groups is NULL");
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    cudaGetLastError();
    return fail(MEM_ECUDA, "no CUDA device (libmem has no CPU fallback)");
  }
  // validate every spec before allocating anything
  for (int i = 0; i < n_groups; ++i) {
    const mem_layer_spec &s = groups[i];
    if (!s.name || !s.name[0] || strlen(s.name) >= 40) return fail(MEM_EINVAL, "group %d: name must be 1..39 chars", i);
    if (!strcmp(s.name, "elevation") || !strcmp(s.name, "variance") || !strcmp(s.name, "valid"))
      return fail(MEM_EDUPNAME, "group name '%s' is reserved", s.name);
    for (int j = 0; j < i; ++j)
      if (!strcmp(groups[j].name, s.name)) return fail(MEM_EDUPNAME, "duplicate group name '%s'", s.name);
    if (s.rule < MEM_AVERAGE || s.rule > MEM_COLOR) return fail(MEM_ERULE, "group '%s': unknown rule %d", s.name, s.rule);
    if (s.rule == MEM_COLOR) {
      if (s.n_channels != 3) return fail(MEM_EINVAL, "group '%s': color takes n_channels = 3", s.name);
    } else if (s.n_channels < 1 || s.n_channels > kMaxCh) {
      return fail(MEM_EINVAL, "group '%s': n_channels %d out of [1, %d]", s.name, s.n_channels, kMaxCh);
    }
    if ((s.rule == MEM_CLASS_AVERAGE || s.rule == MEM_CLASS_BAYESIAN || s.rule == MEM_CLASS_MAX) && s.n_channels < 2)
      return fail(MEM_ERULE, "group '%s': class rules need >= 2 classes", s.name);
    if ((s.rule == MEM_AVERAGE || s.rule == MEM_CLASS_AVERAGE || s.rule == MEM_COLOR) && !(s.w > 0.0f && s.w <= 1.0f))
      return fail(MEM_EINVAL, "group '%s': w must be in (0, 1]", s.name);
    if (s.rule == MEM_GAUSSIAN && !(s.sigma_f2 > 0.0f && s.sigma0_2 > 0.0f))
      return fail(MEM_EINVAL, "group '%s': variances must be > 0", s.name);
    if (s.rule == MEM_CLASS_BAYESIAN && !(s.alpha0 > 0.0f)) return fail(MEM_EINVAL, "group '%s': alpha0 must be > 0", s.name);
  }
  mem_map *m = new mem_map();
  m->B = n_maps;
  m->H = rows;
  m->W = cols;
  m->res = resolution;
  m->flags = flags;
  m->stream = (cudaStream_t)stream;
  if (cudaGetDevice(&m->device) != cudaSuccess) {
    cudaGetLastError();
    delete m;
    return fail(MEM_ECUDA, "cudaGetDevice failed");
  }
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
    if (sms > 0) m->sms = sms;
    cudaGetLastError();
  }
  m->pend.assign(n_maps, ShiftRec{0, 0, 0, 0});
  m->kx.assign(n_maps, 0);
  m->ky.assign(n_maps, 0);
  m->r0.assign(n_maps, 0);
  m->c0.assign(n_maps, 0);
  // layer registry (names: include/mem.h)
  m->n_word = 2;
  m->n_flag = 1;
  m->n_acc = 3;  // (per-cell statistic words: P, S, n_in | n_out << 32, then the groups' fields)
  add_layer(m, "elevation", LK_ELEV, kWordElev);
  add_layer(m, "variance", LK_VAR, kWordVar);
  add_layer(m, "valid", LK_VALID, kFlagValid);
  m->ng = n_groups;
  for (int i = 0; i < n_groups; ++i) {
    const mem_layer_spec &s = groups[i];
    GroupDesc &g = m->g[i];
    g.rule = s.rule;
    g.nch = s.n_channels;
    g.w = s.w;
    g.sf2 = s.sigma_f2;
    g.mu0 = s.mu0;
    g.s02 = s.sigma0_2;
    g.a0 = s.alpha0;
    g.word0 = m->n_word;
    g.label = -1;
    g.flag = -1;
    g.acc0 = m->n_acc;
    const std::string nm = s.name;
    m->gname[i] = nm;
    auto sfx = [&](int k) { return g.nch == 1 ? nm : nm + "_" + std::to_string(k); };
    switch (s.rule) {
      case MEM_AVERAGE:
      case MEM_CLASS_AVERAGE:
        for (int k = 0; k < g.nch; ++k) add_layer(m, sfx(k), LK_WORD, g.word0 + k);
        m->n_word += g.nch;
        m->n_acc += 1 + g.nch;
        break;
      case MEM_GAUSSIAN:
        for (int k = 0; k < g.nch; ++k) add_layer(m, sfx(k), LK_WORD, g.word0 + k);
        for (int k = 0; k < g.nch; ++k)
          add_layer(m, g.nch == 1 ? nm + "_var" : nm + "_var_" + std::to_string(k), LK_WORD, g.word0 + g.nch + k);
        m->n_word += 2 * g.nch;
        m->n_acc += 1 + g.nch;
        break;
      case MEM_CLASS_BAYESIAN:
        for (int k = 0; k < g.nch; ++k) add_layer(m, nm + "_" + std::to_string(k), LK_THETA, g.word0 + k, g.word0, g.nch, m->n_flag);
        for (int k = 0; k < g.nch; ++k) add_layer(m, nm + "_alpha_" + std::to_string(k), LK_WORD, g.word0 + k);
        m->n_word += g.nch;
        m->n_acc += 1 + g.nch;
        break;
      case MEM_CLASS_MAX:
        g.label = m->n_word + 1;
        add_layer(m, nm + "_label", LK_LABEL, g.label);
        add_layer(m, nm + "_conf", LK_WORD, g.word0);
        m->label_word[m->n_label++] = g.label;
        m->n_word += 2;
        m->n_acc += 1;
        break;
      case MEM_COLOR:
        add_layer(m, nm + "_r", LK_WORD, g.word0);
        add_layer(m, nm + "_g", LK_WORD, g.word0 + 1);
        add_layer(m, nm + "_b", LK_WORD, g.word0 + 2);
        m->n_word += 3;
        m->n_acc += 2;
        break;
    }
    if (s.rule != MEM_CLASS_MAX) {
      g.flag = m->n_flag++;
      add_layer(m, nm + "_observed", LK_FLAG, g.flag);
    }
  }
  // device state
  const long long BHW = (long long)n_maps * rows * cols;
  auto alloc = [&](void **p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  };
  if (!alloc((void **)&m->st.words, sizeof(uint32_t) * BHW * m->n_word) ||
      !alloc((void **)&m->st.flags, (size_t)BHW * m->n_flag) ||
      !alloc((void **)&m->ring, sizeof(int2) * n_maps) ||
      !alloc((void **)&m->ctl, m->ctl_bytes = sizeof(Control))) {
    free_map(m);
    return fail(MEM_ENOMEM, "device allocation of the map state failed");
  }
  mem_status s = MEM_OK;
  if (cudaMemsetAsync(m->ctl, 0, m->ctl_bytes, m->stream) != cudaSuccess) {
    s = fail(MEM_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(cudaGetLastError()));
  }
  if (s == MEM_OK) s = reset_all(m);
  if (s == MEM_OK && cudaStreamSynchronize(m->stream) != cudaSuccess)
    s = fail(MEM_ECUDA, "create: %s", cudaGetErrorString(cudaGetLastError()));
  if (s != MEM_OK) {
    free_map(m);
    return s;
  }
  *out = m;
  return MEM_OK;
}

mem_status mem_create(float resolution, int rows, int cols, const mem_layer_spec *groups, int n_groups,
                      unsigned flags, mem_stream stream, mem_map **out) {
  return mem_create_batch(1, resolution, rows, cols, groups, n_groups, flags, stream, out);
}

mem_status mem_destroy(mem_map *m) {
  hp_report();
  free_map(m);
  return MEM_OK;
}

mem_status mem_set_stream(mem_map *m, mem_stream s) {
  if (check_map(m)) return MEM_EINVAL;
  CU(cudaStreamSynchronize(m->stream));
  m->stream = (cudaStream_t)s;
  return MEM_OK;
}

mem_status mem_synchronize(mem_map *m) {
  if (check_map(m)) return MEM_EINVAL;
  CU(cudaStreamSynchronize(m->stream));
  return MEM_OK;
}

#define NC(expr)                                                                            \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess) return fail(MEM_ECOMM, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

// all-gather every stored layer (readout of a sharded NCCL map)
static mem_status shard_gather_all(mem_map *m) {
  if (m->transport != 1 || m->nranks == 1) return MEM_OK;
  const int HW = m->H * m->W, bn = m->band_n;
  NC(ncclGroupStart());
  for (int w = 0; w < m->n_word; ++w)
    NC(ncclAllGather(m->st.words + (size_t)w * HW + m->band_lo, m->st.words + (size_t)w * HW, bn, ncclUint32,
                     m->comm, m->stream));
  for (int f = 0; f < m->n_flag; ++f)
    NC(ncclAllGather(m->st.flags + (size_t)f * HW + m->band_lo, m->st.flags + (size_t)f * HW, bn, ncclUint8,
                     m->comm, m->stream));
  NC(ncclGroupEnd());
  return MEM_OK;
}

// P = sum 1/v is certified exact for every cell of a call at once: its terms lie in
// [fl(1/v_max), fl(1/v_min)], v_min / v_max from the range bounds of r2, and the certificate
// e_max - e_min + ceil(log2(max points per cell)) <= 29 (k_red.cuh) holds for all cells
static bool p_certified(const PassArgs &a, long long max_n) {
  if (!(a.r2lo <= a.r2hi)) return true;  // no point passes the range filter
  const float vlo = a.np.a + a.np.b * a.r2lo, vhi = a.np.a + a.np.b * a.r2hi;
  if (!std::isfinite(vhi) || !(vlo > 0.0f)) return false;
  const float wmax = 1.0f / vlo, wmin = 1.0f / vhi;
  uint32_t bmax, bmin;
  memcpy(&bmax, &wmax, 4);
  memcpy(&bmin, &wmin, 4);
  const int emax = std::max<int>((bmax >> 23) & 255, 1), emin = std::max<int>((bmin >> 23) & 255, 1);
  int lg = 0;
  while ((1LL << lg) < max_n) ++lg;
  return emax - emin + lg <= 29;
}

// the RED path for the fast groups: k_points (certified REDs), k_cells (fuse
// the certified cells, list the others), k_refold (the others, in input order)
#ifndef MEM_WAVE_MB
#define MEM_WAVE_MB 0  // RED scratch budget: 0 = all maps of a call in one wave
#endif
#ifndef MEM_CELL_WAVE_MB
#define MEM_CELL_WAVE_MB 64  // one big map: RED scratch per cell wave (0 = one wave; C5b: 48 / 64 / 100 MB -> 389 / 325 / 330 us)
#endif
static mem_status fuse_points_red(mem_map *m, PassArgs &a, const int64_t *offsets, long long total) {
  const int B = a.n_maps;
  const size_t HW = (size_t)m->H * m->W;
  // waves of maps whose scratch (count word + record (+ certificate)) fits the budget; the
  // scratch is reused by every wave
  const size_t per_cell = 8 + 32 + (a.fast == 2 ? 8 : 0);
  int wmaps = B;
  if (MEM_WAVE_MB > 0) wmaps = (int)std::max<size_t>(1, std::min<size_t>(B, (size_t)MEM_WAVE_MB * 1048576 / (per_cell * HW)));
  // one big map (C5b): waves of cells whose scratch stays in L2 between the cell pass that
  // zeroes it and the next wave's REDs; every wave re-reads the points
  const int clo = a.cell_lo, chi = a.cell_hi;
  const size_t band = (size_t)(chi - clo);
  int wcells = 0;
  if (B == 1 && a.dbg_cell == nullptr && MEM_CELL_WAVE_MB > 0 && per_cell * band > (size_t)MEM_CELL_WAVE_MB * 1048576) {
    const size_t nw = (per_cell * band + (size_t)MEM_CELL_WAVE_MB * 1048576 - 1) / ((size_t)MEM_CELL_WAVE_MB * 1048576);
    wcells = (int)(((band + nw - 1) / nw + 1023) / 1024 * 1024);
  }
  const size_t cells = wcells ? (size_t)wcells : (size_t)wmaps * HW, all = (size_t)B * HW;
  if (cells > m->red_cells || all > m->red_all) {
    CU(cudaStreamSynchronize(m->stream));
    void **bufs[] = {&m->rcnt_s, &m->rrec_s, &m->rcert_s, &m->rfb_s, &m->rmark_s, &m->rfill_s, &m->rmapfb_s};
    const size_t nc = std::max(cells, m->red_cells), na = std::max(all, m->red_all);
    const size_t bytes[] = {8 * nc, 32 * nc, 8 * nc, 16 * nc, 4 * na, 4 * nc, 4 * (na / HW + 1)};
    for (void **b : bufs) {
      cudaFree(*b);
      *b = nullptr;
    }
    m->red_cells = m->red_all = 0;
    for (int i = 0; i < 7; ++i)
      if (cudaMalloc(bufs[i], bytes[i]) != cudaSuccess) {
        cudaGetLastError();
        return fail(MEM_ENOMEM, "RED scratch (%zu cells)", nc);
      }
    CU(cudaMemsetAsync(m->rcnt_s, 0, bytes[0], m->stream));
    CU(cudaMemsetAsync(m->rrec_s, 0, bytes[1], m->stream));
    CU(cudaMemsetAsync(m->rcert_s, 0, bytes[2], m->stream));
    CU(cudaMemsetAsync(m->rmark_s, 0xff, bytes[4], m->stream));  // -1: no uncertified cell
    CU(cudaMemsetAsync(m->rfill_s, 0, bytes[5], m->stream));
    CU(cudaMemsetAsync(m->rmapfb_s, 0, bytes[6], m->stream));
    m->red_cells = nc;
    m->red_all = na;
  }
  // the point list of the uncertified cells: at most every point of the call
  HP(7);
  const long long npts = offsets ? offsets[B] - offsets[0] : total;
  if (grow(&m->rlist_s, &m->rlist_cap, 4 * (size_t)std::max(1LL, npts), m->stream) != MEM_OK) return MEM_ENOMEM;
  a.cnt = reinterpret_cast<unsigned long long *>(m->rcnt_s);
  a.rec = reinterpret_cast<unsigned long long *>(m->rrec_s);
  a.cert = reinterpret_cast<unsigned *>(m->rcert_s);
  a.fb = reinterpret_cast<unsigned long long *>(m->rfb_s);
  a.fbmark = reinterpret_cast<int *>(m->rmark_s);
  a.fbfill = reinterpret_cast<unsigned *>(m->rfill_s);
  a.fbmap = reinterpret_cast<unsigned *>(m->rmapfb_s);
  a.fblist = reinterpret_cast<unsigned *>(m->rlist_s);
  a.st = m->st;
  // warp-items of 128 points per map (inline prefix sums; staged ones ride in a second blob)
  std::vector<int> ps(B + 1, 0);
  for (int i = 0; i < B; ++i) {
    const long long ni = offsets ? offsets[i + 1] - offsets[i] : total;
    ps[i + 1] = ps[i] + (int)((ni + kWarpPoints - 1) / kWarpPoints);
  }
  a.p_uniform = ps[1] - ps[0];
  for (int i = 1; i < B && a.p_uniform > 0; ++i)
    if (ps[i + 1] - ps[i] != a.p_uniform) a.p_uniform = 0;
  a.inv_p_uniform = a.p_uniform > 0 ? 1.0 / (double)a.p_uniform : 0.0;
  if (B <= kInlineMaps) {
    for (int i = 0; i <= B; ++i) a.psi[i] = ps[i];
    a.pstart = nullptr;
  }  // else: a.pstart points into the staged parameter blob (input_points)
  HP(8);
  if (wcells) {
    a.m0 = 0;
    a.m1 = 1;
    for (int lo = clo; lo < chi; lo += wcells) {
      a.sc_lo = a.cell_lo = lo;
      a.sc_hi = a.cell_hi = std::min(chi, lo + wcells);
      a.wave_first = lo == clo;
      if (ps[1] > ps[0]) TIMED(MEM_STAGE_POINT, launch_points(a, m->stream));
      else CU(cudaMemsetAsync(&m->ctl->n_fb, 0, sizeof(unsigned) * 2, m->stream));
      TIMED(MEM_STAGE_CELL, launch_cells(a, m->stream));
    }
    a.sc_lo = a.sc_hi = 0;
    a.cell_lo = clo;
    a.cell_hi = chi;
    HP(10);
    return MEM_OK;
  }
  for (int w0 = 0; w0 < B; w0 += wmaps) {
    a.m0 = w0;
    a.m1 = std::min(B, w0 + wmaps);
    if (ps[a.m1] > ps[a.m0]) TIMED(MEM_STAGE_POINT, launch_points(a, m->stream));
    else CU(cudaMemsetAsync(&m->ctl->n_fb, 0, sizeof(unsigned) * 2, m->stream));  // k_points clears them
    TIMED(MEM_STAGE_CELL, launch_cells(a, m->stream));
  }
  HP(10);
  return MEM_OK;
}

// tiles of every map, bands of the physical cells [cell_lo, cell_hi), buffers; then k_bin and
// k_sort.  `a` carries the frames, the point offsets and the tile prefix sums
// (inline or staged); `tiles` = all tiles of the call, `tmax` = most tiles of one map.
static mem_status fuse_points(mem_map *m, PassArgs &a, int tiles, long long tmax, long long max_n,
                              const int64_t *offsets = nullptr, long long total = 0) {
  const int B = a.n_maps;
  // batches of small maps with one colour / 1-channel average group (C5a): one CTA per map
  // sorts its points by cell in shared memory and sums them in input order (k_smap)
  const bool sorted = (m->flags & MEM_FLAG_FUSE_SORTED) != 0;
  if (!sorted && (a.fast == 1 || a.fast == 2) && a.vec4 && B >= 64 && a.cell_lo == 0 && a.cell_hi == m->H * m->W &&
      smap_eligible(m->H * m->W, max_n)) {
    a.st = m->st;
    a.m0 = 0;
    a.m1 = B;
    a.smap_maxpts = (int)max_n;
    const int grid = std::max(1, std::min(B, m->sms));
    TIMED(MEM_STAGE_POINT, launch_smap(a, grid, smap_smem_bytes(m->H * m->W, max_n), m->stream));
    return MEM_OK;
  }
  // the fast groups (one colour / one 1-channel average group on float4 points, or height
  // only) take the RED path when the call's P sums are certified; everything else sorts
  if (!sorted && a.fast != 0 && p_certified(a, max_n) && (a.fast != 1 || max_n <= kColourMaxPts))
    return fuse_points_red(m, a, offsets, total);
  const int cells = a.cell_hi - a.cell_lo;
  if (tmax > kMaxTilesPerMap)
    return fail(MEM_EINVAL, "a map takes at most %lld points per call", (long long)kMaxTilesPerMap * kTile);
  // bands: about MEM_BAND_RECS in-window records each, estimated from a recent call of this
  // map (its record count comes back to pinned host memory asynchronously; the first call
  // assumes half of the points in the window) -- the sizing changes speed, never results --
  // at least two CTAs per SM over the call, at most kMaxBandCells cells and kMaxBands bands
  double recs_per_map = 0.5 * (double)max_n;
  if (m->seen_rec && *(volatile unsigned *)m->seen_rec > 0u)
    recs_per_map = std::min(recs_per_map * 2.0, 1.25 * (double)*(volatile unsigned *)m->seen_rec / B);
  long long nb = (long long)std::ceil(recs_per_map / MEM_BAND_RECS);
  nb = std::max(nb, (2LL * m->sms + B - 1) / B);
  nb = std::max(nb, ((long long)cells + kMaxBandCells - 1) / kMaxBandCells);
  nb = std::min<long long>(std::min<long long>(nb, kMaxBands), std::max(1, cells));
  const int bc = (int)(((cells + nb - 1) / nb + 15) / 16 * 16);  // 16-B aligned state slices (bulk copies)
  if (bc > kMaxBandCells) return fail(MEM_EINVAL, "%d cells per map exceed the %d-band limit", cells, kMaxBands);
  a.band_cells = bc;
  a.nbands = (cells + bc - 1) / bc;
  a.inv_band = 1.0 / (double)bc;
  a.inv_nbands = 1.0 / (double)a.nbands;
  int kb = 1;
  while ((1 << kb) - 1 < bc) ++kb;
  a.key_bits = kb;
  a.tmax = (int)tmax;
  const bool dbg = a.dbg_cell != nullptr;
  const size_t nrec = (size_t)std::max(1, tiles) * kTile;
  const size_t nseg = std::min(nrec, (size_t)B * cells);
  if (grow(&m->recs, &m->recs_cap, sizeof(uint4) * nrec, m->stream) != MEM_OK ||
      grow(&m->srec, &m->srec_cap, sizeof(uint4) * nrec, m->stream) != MEM_OK ||
      grow(&m->segs, &m->segs_cap, 2 * sizeof(uint4) * nseg, m->stream) != MEM_OK ||
      grow(&m->tinfo, &m->tinfo_cap, sizeof(unsigned) * (size_t)std::max(1, tiles) * a.nbands, m->stream) != MEM_OK ||
      (dbg && (grow(&m->ridx, &m->ridx_cap, sizeof(unsigned) * nrec, m->stream) != MEM_OK ||
               grow(&m->sridx, &m->sridx_cap, sizeof(unsigned) * nrec, m->stream) != MEM_OK)))
    return fail(MEM_ENOMEM, "point pass buffers (%d tiles)", tiles);
  a.recs = reinterpret_cast<uint4 *>(m->recs);
  a.srec = reinterpret_cast<uint4 *>(m->srec);
  a.segs = reinterpret_cast<uint4 *>(m->segs);
  a.seg_cap = (unsigned)nseg;
  a.tinfo = reinterpret_cast<unsigned *>(m->tinfo);
  a.ridx = dbg ? reinterpret_cast<unsigned *>(m->ridx) : nullptr;
  a.sridx = dbg ? reinterpret_cast<unsigned *>(m->sridx) : nullptr;
  a.st = m->st;
  if (tiles > 0) TIMED(MEM_STAGE_POINT, launch_bin(a, tiles, m->stream));
  TIMED(MEM_STAGE_CELL, launch_sort(a, m->stream));
  if (tiles > 0) TIMED(MEM_STAGE_CELL, launch_fuse(a, m->stream));
  if (!m->seen_rec && cudaMallocHost((void **)&m->seen_rec, sizeof(unsigned)) == cudaSuccess) *m->seen_rec = 0u;
  cudaGetLastError();
  if (m->seen_rec) CU(cudaMemcpyAsync(m->seen_rec, &m->ctl->n_rec, sizeof(unsigned), cudaMemcpyDeviceToHost, m->stream));
  return MEM_OK;
}

// inline parameters of a one-map pass over n points
static void one_map_params(PassArgs &b, long long n, int *tiles, long long *tmax) {
  b.frames = nullptr;
  b.offsets = nullptr;
  b.tstart = nullptr;
  b.n_maps = 1;
  const long long t = (n + kTile - 1) / kTile;
  b.offi[0] = 0;
  b.offi[1] = n;
  b.tsi[0] = 0;
  b.tsi[1] = (int)t;
  b.t_uniform = 0;
  b.inv_t_uniform = 0.0;
  *tiles = (int)t;
  *tmax = t;
}

// point routing: the owner of a band fuses the in-window points it received (all in its band,
// in global input order: by source rank, each source's in input order)
static mem_status owner_pass(mem_map *m, const float *pts, long long n) {
  PassArgs b = m->shard_args;
  b.pts = pts;
  b.vec4 = (b.stride == 4 && ((uintptr_t)pts & 15) == 0) ? 1 : 0;
  if (!b.vec4 && (b.fast == 1 || b.fast == 2)) b.fast = 0;
  int tiles;
  long long tmax;
  one_map_params(b, n, &tiles, &tmax);
  if (m->flags & MEM_FLAG_DEBUG_POINTS) {  // owner-side outputs by received position
    if ((size_t)n > m->odbg_cap) {
      CU(cudaStreamSynchronize(m->stream));
      cudaFree(m->odbg_cell);
      cudaFree(m->odbg_code);
      m->odbg_cell = nullptr;
      m->odbg_code = nullptr;
      m->odbg_cap = 0;
      const size_t c = n + n / 4 + 1024;
      if (cudaMalloc(&m->odbg_cell, c * sizeof(int)) != cudaSuccess || cudaMalloc(&m->odbg_code, c) != cudaSuccess) {
        cudaGetLastError();
        return fail(MEM_ENOMEM, "owner debug buffers");
      }
      m->odbg_cap = c;
    }
    b.dbg_cell = m->odbg_cell;
    b.dbg_code = m->odbg_code;
  } else {
    b.dbg_cell = nullptr;
    b.dbg_code = nullptr;
  }
  return fuse_points(m, b, tiles, tmax, n, nullptr, n);
}

static mem_status grow_floats(float **buf, size_t *cap_bytes, size_t need_floats, cudaStream_t s) {
  return grow((void **)buf, cap_bytes, need_floats * sizeof(float), s);
}

// NCCL transport of the routed points: counts all-gathered (one host sync), grouped send/recv
// of the buckets into one contiguous buffer ordered by source rank, then the owner pass; with
// debug outputs the owners send every routed point's in/out code back to its source rank
static mem_status shard_route_nccl(mem_map *m) {
  const int G = m->nranks, st = m->route_stride;
  std::vector<unsigned> &all = m->route_all;
  all.assign((size_t)G * G, 0u);
  if (G > 1) {
    NC(ncclAllGather(m->rcnt, m->rall, G, ncclUint32, m->comm, m->stream));
    CU(cudaMemcpyAsync(all.data(), m->rall, sizeof(unsigned) * G * G, cudaMemcpyDeviceToHost, m->stream));
  } else {
    CU(cudaMemcpyAsync(all.data(), m->rcnt, sizeof(unsigned) * G, cudaMemcpyDeviceToHost, m->stream));
  }
  CU(cudaStreamSynchronize(m->stream));
  std::vector<long long> off(G + 1, 0);
  for (int p = 0; p < G; ++p) off[p + 1] = off[p] + all[(size_t)p * G + m->rank];
  if (grow_floats(&m->rin, &m->rin_cap, (size_t)std::max(1LL, off[G]) * st, m->stream) != MEM_OK)
    return fail(MEM_ENOMEM, "routed points (%lld)", off[G]);
  const size_t own = all[(size_t)m->rank * G + m->rank];
  if (own)
    CU(cudaMemcpyAsync(m->rin + (size_t)off[m->rank] * st, m->rbuf + (size_t)m->rank * m->route_cap * st,
                       sizeof(float) * own * st, cudaMemcpyDeviceToDevice, m->stream));
  if (G > 1) {
    NC(ncclGroupStart());
    for (int p = 0; p < G; ++p) {
      if (p == m->rank) continue;
      const size_t ns = all[(size_t)m->rank * G + p], nr = all[(size_t)p * G + m->rank];
      if (ns) NC(ncclSend(m->rbuf + (size_t)p * m->route_cap * st, ns * st, ncclFloat32, p, m->comm, m->stream));
      if (nr) NC(ncclRecv(m->rin + (size_t)off[p] * st, nr * st, ncclFloat32, p, m->comm, m->stream));
    }
    NC(ncclGroupEnd());
  }
  mem_status s = owner_pass(m, m->rin, off[G]);
  if (s != MEM_OK || !(m->flags & MEM_FLAG_DEBUG_POINTS)) return s;
  // codes back: owner slice [off[p], off[p+1]) -> source p, which scatters them to its points
  if (grow((void **)&m->rcode, &m->rcode_cap, (size_t)G * std::max(1LL, m->route_cap), m->stream) != MEM_OK)
    return fail(MEM_ENOMEM, "returned codes");
  if (own)
    CU(cudaMemcpyAsync(m->rcode + (size_t)m->rank * m->route_cap, m->odbg_code + off[m->rank], own,
                       cudaMemcpyDeviceToDevice, m->stream));
  if (G > 1) {
    NC(ncclGroupStart());
    for (int p = 0; p < G; ++p) {
      if (p == m->rank) continue;
      const size_t ns = all[(size_t)m->rank * G + p], nr = all[(size_t)p * G + m->rank];
      if (nr) NC(ncclSend(m->odbg_code + off[p], nr, ncclUint8, p, m->comm, m->stream));
      if (ns) NC(ncclRecv(m->rcode + (size_t)p * m->route_cap, ns, ncclUint8, p, m->comm, m->stream));
    }
    NC(ncclGroupEnd());
  }
  for (int p = 0; p < G; ++p) {
    const size_t ns = all[(size_t)m->rank * G + p];
    CU(launch_code_return(m->rcode + (size_t)p * m->route_cap, m->rsrc + (size_t)p * m->route_cap, ns, m->dbg_code,
                          m->stream));
  }
  return MEM_OK;
}

// this rank's shard: drop / count / route in input order (k_route_count, _scan, _scatter)
static mem_status route_points(mem_map *m, PassArgs &a, long long n, int stride) {
  const int G = m->nranks;
  const long long cap = std::max(1LL, n);
  const int tiles = (int)((n + kTile - 1) / kTile);
  const bool dbg = (m->flags & MEM_FLAG_DEBUG_POINTS) != 0;
  if (grow_floats(&m->rbuf, &m->rbuf_cap, (size_t)G * cap * stride, m->stream) != MEM_OK ||
      grow((void **)&m->rtile, &m->rtile_cap, sizeof(unsigned) * (size_t)std::max(1, tiles) * G, m->stream) != MEM_OK ||
      (dbg && grow((void **)&m->rsrc, &m->rsrc_cap, sizeof(unsigned) * (size_t)G * cap, m->stream) != MEM_OK))
    return fail(MEM_ENOMEM, "route buckets");
  RouteArgs r;
  r.buf = m->rbuf;
  r.src = dbg ? m->rsrc : nullptr;
  r.tcnt = m->rtile;
  r.cnt = m->rcnt;
  r.cap = cap;
  r.band_n = m->band_n;
  r.nranks = G;
  r.tiles = tiles;
  m->route_cap = cap;
  m->route_stride = stride;
  TIMED(MEM_STAGE_POINT, launch_route(a, r, m->stream));
  a.cell_lo = m->band_lo;
  a.cell_hi = m->band_lo + m->band_n;
  m->shard_args = a;
  m->pending = false;
  if (m->transport == 2) {
    m->exchange_pending = true;
    return MEM_OK;
  }
  return shard_route_nccl(m);
}

static mem_status input_points(mem_map *m, const float *pts, const int64_t *offsets, int64_t n_single, int stride,
                               const mem_binding *bind, int nb, const double *R, const double *t,
                               const mem_noise *np) {
  HP_START();
  if (check_map(m)) return MEM_EINVAL;
  if (stride < 3) return fail(MEM_EINVAL, "stride %d < 3", stride);
  if (!R || !t || !np) return fail(MEM_EINVAL, "R, t and noise must be non-NULL");
  if (!(np->a > 0.0f) || !(np->b >= 0.0f))
    return fail(MEM_EINVAL, "noise: need a > 0 and b >= 0 (v = a + b r^2 > 0)");
  if (np->b > 0.0f && std::isfinite(np->r_max) && !std::isfinite(np->a + np->b * (np->r_max * np->r_max)))
    return fail(MEM_EINVAL, "noise: v = a + b r_max^2 overflows fp32");  // every 1/v must be > 0
  const int B = m->B;
  long long total = 0, max_n = 0;
  if (offsets) {
    if (offsets[0] != 0) return fail(MEM_EINVAL, "offsets[0] must be 0");
    for (int i = 0; i < B; ++i) {
      const long long c = offsets[i + 1] - offsets[i];
      if (c < 0) return fail(MEM_EINVAL, "offsets must be non-decreasing");
      if (c > max_n) max_n = c;
    }
    total = offsets[B];
  } else {
    if (B != 1) return fail(MEM_EINVAL, "batched map: use mem_input_pointcloud_batch");
    if (n_single < 0) return fail(MEM_EINVAL, "n = %lld < 0", (long long)n_single);
    total = max_n = n_single;
  }
  if (total > 0 && !pts) return fail(MEM_EINVAL, "pts is NULL");
  for (int i = 0; i < B; ++i)
    if (!rotation_ok(R + 9 * i)) return fail(MEM_EPOSE, "map %d: R is not a rotation (SPEC.md:128)", i);
  for (int i = 0; i < 3 * B; ++i)
    if (!std::isfinite(t[i])) return fail(MEM_EINVAL, "t must be finite");
  HP(0);
  PassArgs a;
  memset(&a, 0, sizeof a);
  HP(1);
  mem_status s = resolve_bindings(m, bind, nb, false, stride, a.b);
  if (s != MEM_OK) return s;
  HP(2);
  if (set_device(m)) return MEM_ECUDA;
  HP(3);
  if (m->flags & MEM_FLAG_DEBUG_POINTS) {
    if ((size_t)total > m->dbg_cap) {
      CU(cudaStreamSynchronize(m->stream));
      cudaFree(m->dbg_cell);
      cudaFree(m->dbg_code);
      m->dbg_cell = nullptr;
      m->dbg_code = nullptr;
      m->dbg_cap = 0;
      const size_t c = total + total / 4 + 1024;
      if (cudaMalloc(&m->dbg_cell, c * sizeof(int)) != cudaSuccess || cudaMalloc(&m->dbg_code, c) != cudaSuccess) {
        cudaGetLastError();
        return fail(MEM_ENOMEM, "debug buffers");
      }
      m->dbg_cap = c;
    }
    m->dbg_n = total;
  }
  // legal; only a pending shift changes the map -- except that a shard of a sharded map
  // still takes part in the band exchange with its empty statistics
  if (total == 0 && m->transport == 0) {
    m->stats_empty = true;
    return flush_shift(m);
  }
  // counters: this call adds to stats[epoch], its k_points clears the other epoch for the next
  m->epoch ^= 1;
  m->stats_empty = false;
  const void *dpts = nullptr;
  if (total > 0) {
    s = stage_input(m, pts, sizeof(float) * (size_t)total * stride, &dpts);
    if (s != MEM_OK) return s;
  }
  HP(4);
  a.pts = (const float *)dpts;
  a.stride = stride;
  a.n_maps = B;
  a.ring = m->ring;
  a.geo = m->geo();
  a.st = m->st;
  a.np = *np;
  range_thresholds(np->r_min, np->r_max, &a.r2lo, &a.r2hi);
  HP(5);
  a.nb = nb;
  a.ctl = m->ctl;
  a.epoch = m->epoch;
  a.pdl = m->pdl;
  a.reset = m->reset_info();
  const int HW = m->H * m->W;
  a.cell_lo = 0;
  a.cell_hi = HW;
  if (m->flags & MEM_FLAG_DEBUG_POINTS) {
    a.dbg_cell = m->dbg_cell;
    a.dbg_code = m->dbg_code;
  }
  if (total > 0xffffffffLL) return fail(MEM_EINVAL, "at most 2^32 - 1 points per call");
  auto frame = [&](int i) {
    const MapFrame mf = make_frame(m, i, R + 9 * i, t + 3 * i, nullptr);
    PointFrame f;
    memcpy(f.R, mf.R, sizeof f.R);
    memcpy(f.t, mf.t, sizeof f.t);
    // fold the pending shift of the preceding mem_move_to into this launch (lazy a13)
    f.sr = m->pending ? m->pend[i].sr : 0;
    f.sc = m->pending ? m->pend[i].sc : 0;
    f.r0 = m->r0[i];
    f.c0 = m->c0[i];
    return f;
  };
  a.vec4 = (stride == 4 && ((uintptr_t)dpts & 15) == 0) ? 1 : 0;
  a.vec3 = (stride == 3 && ((uintptr_t)dpts & 15) == 0) ? 1 : 0;
  for (int i = 0; i <= B && a.vec3 && offsets; ++i)
    if (offsets[i] & 3) a.vec3 = 0;
  // fast paths (k_bin carries the channel word in the record): one colour or 1-channel average
  // group bound to the float4's w (never for other strides or unaligned buffers);
  // no binding at all: height only
  a.fast = 0;
  if (nb == 0) {
    a.fast = 3;
  } else if (nb == 1 && a.vec4 && a.b[0].topk == 0 && a.b[0].ch_offset == 0) {
    if (a.b[0].g.rule == MEM_COLOR) a.fast = 1;
    else if (a.b[0].g.rule == MEM_AVERAGE && a.b[0].g.nch == 1) a.fast = 2;
  }
  // tiles of kTile points per map
  std::vector<int> tstart(B + 1);
  tstart[0] = 0;
  long long tmax = 0;
  for (int i = 0; i < B; ++i) {
    const long long ni = offsets ? offsets[i + 1] - offsets[i] : total;
    const long long ti = (ni + kTile - 1) / kTile;
    tmax = std::max(tmax, ti);
    if (tstart[i] + ti > 0x7fffffffLL) return fail(MEM_EINVAL, "too many points in one call");
    tstart[i + 1] = (int)(tstart[i] + ti);
  }
  a.t_uniform = tstart[1] - tstart[0];
  for (int i = 1; i < B && a.t_uniform > 0; ++i)
    if (tstart[i + 1] - tstart[i] != a.t_uniform) a.t_uniform = 0;
  a.inv_t_uniform = a.t_uniform > 0 ? 1.0 / (double)a.t_uniform : 0.0;
  if (B <= kInlineMaps) {  // frames, offsets and tile prefix sums ride in the kernel parameters
    for (int i = 0; i < B; ++i) a.fi[i] = frame(i);
    for (int i = 0; i <= B; ++i) {
      a.offi[i] = offsets ? offsets[i] : (i == 0 ? 0 : total);
      a.tsi[i] = tstart[i];
    }
  } else {
    // parameter blob: frames [B] | offsets [B+1] (i64) | tstart [B+1] (i32)
    const size_t off_at = (sizeof(PointFrame) * B + 15) & ~(size_t)15;  // int64 alignment
    const size_t ts_at = off_at + sizeof(long long) * (B + 1);
    const size_t ps_at = ts_at + sizeof(int) * (B + 1);
    std::vector<unsigned char> blob(ps_at + sizeof(int) * (B + 1));
    {  // k_points' warp-item prefix sums ride in the same blob (no second staging, no sync)
      int *ps = reinterpret_cast<int *>(blob.data() + ps_at);
      ps[0] = 0;
      for (int i = 0; i < B; ++i) ps[i + 1] = ps[i] + (int)((offsets[i + 1] - offsets[i] + kWarpPoints - 1) / kWarpPoints);
    }
    PointFrame *fr = reinterpret_cast<PointFrame *>(blob.data());
    for (int i = 0; i < B; ++i) fr[i] = frame(i);
    memcpy(blob.data() + off_at, offsets, sizeof(long long) * (B + 1));
    memcpy(blob.data() + ts_at, tstart.data(), sizeof(int) * (B + 1));
    void *d = nullptr;
    s = stage_params(m, blob.data(), blob.size(), &d);
    if (s != MEM_OK) return s;
    a.frames = reinterpret_cast<const PointFrame *>(d);
    a.offsets = reinterpret_cast<const long long *>((char *)d + off_at);
    a.tstart = reinterpret_cast<const int *>((char *)d + ts_at);
    a.pstart = reinterpret_cast<const int *>((char *)d + ps_at);
  }
  HP(6);
  if (m->transport != 0 && m->nranks > 1) {  // sharded map: route the shard's points to their owners
    a.fast = a.fast == 3 ? 3 : 0;             // (the owner pass re-checks the float4 fast paths)
    if (nb == 1 && (a.b[0].g.rule == MEM_COLOR || (a.b[0].g.rule == MEM_AVERAGE && a.b[0].g.nch == 1)) &&
        a.b[0].topk == 0 && a.b[0].ch_offset == 0 && stride == 4)
      a.fast = a.b[0].g.rule == MEM_COLOR ? 1 : 2;
    return route_points(m, a, total, stride);
  }
  if (m->transport != 0) {  // one rank: the whole map is this rank's band
    a.cell_lo = m->band_lo;
    a.cell_hi = m->band_lo + m->band_n;
  }
  m->pending = false;
  s = fuse_points(m, a, tstart[B], tmax, max_n, offsets, total);
  HP(11);
  return s;
}

mem_status mem_input_pointcloud(mem_map *m, const float *pts, int64_t n, int stride, const mem_binding *bind,
                                int n_bind, const double R[9], const double t[3], const mem_noise *np) {
  return input_points(m, pts, nullptr, n, stride, bind, n_bind, R, t, np);
}

mem_status mem_input_pointcloud_batch(mem_map *m, const float *pts, const int64_t *offsets, int stride,
                                      const mem_binding *bind, int n_bind, const double *R, const double *t,
                                      const mem_noise *np) {
  if (!offsets) return fail(MEM_EINVAL, "offsets is NULL");
  return input_points(m, pts, offsets, 0, stride, bind, n_bind, R, t, np);
}

static mem_status input_image(mem_map *m, const float *img, int C, int IH, int IW, const mem_binding *bind, int nb,
                              const double *K, const double *R, const double *t, bool batched) {
  if (check_map(m)) return MEM_EINVAL;
  if (C < 1 || IH < 1 || IW < 1) return fail(MEM_EINVAL, "image size %d x %d x %d invalid", C, IH, IW);
  if (!img || !K || !R || !t) return fail(MEM_EINVAL, "img, K, R, t must be non-NULL");
  if (!batched && m->B != 1) return fail(MEM_EINVAL, "batched map: use mem_input_image_batch");
  const int B = m->B;
  for (int i = 0; i < B; ++i) {
    const double *k = K + 9 * i;
    if (!(k[0] > 0.0 && k[4] > 0.0) || k[3] != 0.0 || k[6] != 0.0 || k[7] != 0.0 || k[8] != 1.0 ||
        !std::isfinite(k[1]) || !std::isfinite(k[2]) || !std::isfinite(k[5]))
      return fail(MEM_EINVAL, "map %d: K must be [[fx,s,cx],[0,fy,cy],[0,0,1]] with fx, fy > 0", i);
    if (!rotation_ok(R + 9 * i)) return fail(MEM_EPOSE, "map %d: R is not a rotation (SPEC.md:128)", i);
  }
  for (int i = 0; i < 3 * B; ++i)
    if (!std::isfinite(t[i])) return fail(MEM_EINVAL, "t must be finite");
  ImageArgs a;
  memset(&a, 0, sizeof a);
  mem_status s = resolve_bindings(m, bind, nb, true, C, a.b);
  if (s != MEM_OK) return s;
  if (set_device(m)) return MEM_ECUDA;
  s = flush_shift(m);
  if (s != MEM_OK) return s;
  const long long per = (long long)C * IH * IW;
  const void *dimg = nullptr;
  s = stage_input(m, img, sizeof(float) * (size_t)per * B, &dimg);
  if (s != MEM_OK) return s;
  a.img = (const float *)dimg;
  a.occlusion = m->occlusion;
  a.eps_occ = m->eps_occ;
  if (m->transport == 1 && m->occlusion && m->nranks > 1) {
    // routed NCCL shards only keep their own band current: the occlusion walk needs the rest
    const int HW = m->H * m->W, bn = m->band_n;
    float *vals = reinterpret_cast<float *>(m->st.words);
    NC(ncclGroupStart());
    NC(ncclAllGather(vals + (size_t)kWordElev * HW + m->band_lo, vals + (size_t)kWordElev * HW, bn, ncclFloat32,
                     m->comm, m->stream));
    NC(ncclAllGather(m->st.flags + m->band_lo, m->st.flags, bn, ncclUint8, m->comm, m->stream));
    NC(ncclGroupEnd());
  }
  a.row_lo = m->transport ? m->band_lo / m->W : 0;  // sharded: fuse the owned band only
  a.row_hi = m->transport ? (m->band_lo + m->band_n) / m->W : m->H;
  a.C = C;
  a.IH = IH;
  a.IW = IW;
  a.map_stride = per;
  a.ring = m->ring;
  a.geo = m->geo();
  a.st = m->st;
  a.nb = nb;
  if (B == 1) {
    a.f0 = make_frame(m, 0, R, t, K);
  } else {
    std::vector<MapFrame> fr(B);
    for (int i = 0; i < B; ++i) fr[i] = make_frame(m, i, R + 9 * i, t + 3 * i, K + 9 * i);
    void *d = nullptr;
    s = stage_params(m, fr.data(), sizeof(MapFrame) * B, &d);
    if (s != MEM_OK) return s;
    a.frames = reinterpret_cast<const MapFrame *>(d);
  }
  TIMED(MEM_STAGE_IMAGE, launch_image(a, m->stream));
  return MEM_OK;
}

mem_status mem_input_image(mem_map *m, const float *img, int C, int H, int W, const mem_binding *bind, int n_bind,
                           const double K[9], const double R[9], const double t[3]) {
  return input_image(m, img, C, H, W, bind, n_bind, K, R, t, false);
}

mem_status mem_input_image_batch(mem_map *m, const float *img, int C, int H, int W, const mem_binding *bind,
                                 int n_bind, const double *K, const double *R, const double *t) {
  return input_image(m, img, C, H, W, bind, n_bind, K, R, t, true);
}

static mem_status move_to(mem_map *m, const double *xy) {
  if (check_map(m)) return MEM_EINVAL;
  if (!xy) return fail(MEM_EINVAL, "xy is NULL");
  const int B = m->B;
  for (int i = 0; i < 2 * B; ++i)
    if (!std::isfinite(xy[i])) return fail(MEM_EINVAL, "position must be finite");
  if (set_device(m)) return MEM_ECUDA;
  // two shifts cannot be composed into one strip reset (data scrolled out is gone), so an
  // earlier pending shift is applied first
  mem_status st = flush_shift(m);
  if (st != MEM_OK) return st;
  bool any = false;
  for (int i = 0; i < B; ++i) {
    // D14: k = floor(x/res + 1/2) in fp64
    const long long kx = (long long)std::floor(xy[2 * i] / (double)m->res + 0.5);
    const long long ky = (long long)std::floor(xy[2 * i + 1] / (double)m->res + 0.5);
    long long sr = kx - m->kx[i], sc = ky - m->ky[i];
    m->kx[i] = kx;
    m->ky[i] = ky;
    const bool all = sr >= m->H || -sr >= m->H || sc >= m->W || -sc >= m->W;
    if (all) {  // |s| >= size: every cell scrolls in
      sr = m->H;
      sc = 0;
      m->r0[i] = 0;
      m->c0[i] = 0;
    } else {
      m->r0[i] = (int)(((m->r0[i] + sr) % m->H + m->H) % m->H);
      m->c0[i] = (int)(((m->c0[i] + sc) % m->W + m->W) % m->W);
    }
    m->pend[i] = ShiftRec{(int)sr, (int)sc, m->r0[i], m->c0[i]};
    any |= (sr != 0 || sc != 0);
  }
  // s = 0 everywhere: bit-identical, nothing to do.  Otherwise the strip reset is applied
  // lazily by the next point input's point pass (or eagerly by flush_shift before any other call).
  m->pending = any;
  return MEM_OK;
}

mem_status mem_move_to(mem_map *m, double x, double y) {
  if (check_map(m)) return MEM_EINVAL;
  if (m->B != 1) return fail(MEM_EINVAL, "batched map: use mem_move_to_batch");
  const double xy[2] = {x, y};
  return move_to(m, xy);
}

mem_status mem_move_to_batch(mem_map *m, const double *xy) { return move_to(m, xy); }

static const Layer *find_layer(const mem_map *m, const char *name) {
  if (!name) return nullptr;
  for (const Layer &l : m->layers)
    if (l.name == name) return &l;
  return nullptr;
}

static ReadArgs read_args(const mem_map *m, const Layer &l) {
  ReadArgs a;
  memset(&a, 0, sizeof a);
  a.geo = m->geo();
  a.st = m->st;
  a.ring = m->ring;
  a.idx = l.idx;
  a.first = l.first;
  a.K = l.K;
  a.flag = l.flag;
  switch (l.kind) {
    case LK_ELEV: a.kind = RK_ELEV; break;
    case LK_VAR: a.kind = RK_VAR; break;
    case LK_VALID: a.kind = RK_FLAG; break;
    case LK_WORD: a.kind = RK_WORD; break;
    case LK_LABEL: a.kind = RK_LABEL; break;
    case LK_FLAG: a.kind = RK_FLAG; break;
    case LK_THETA: a.kind = RK_THETA; break;
  }
  return a;
}

mem_status mem_get_layer(const mem_map *cm, const char *name, float *out) {
  mem_map *m = const_cast<mem_map *>(cm);
  if (check_map(m)) return MEM_EINVAL;
  if (!out) return fail(MEM_EINVAL, "out is NULL");
  const Layer *l = find_layer(m, name);
  if (!l) return fail(MEM_ENOTFOUND, "no layer named '%s'", name ? name : "(null)");
  if (set_device(m)) return MEM_ECUDA;
  {
    mem_status fs = flush_shift(m);
    if (fs != MEM_OK) return fs;
    fs = shard_gather_all(m);
    if (fs != MEM_OK) return fs;
  }
  ReadArgs a = read_args(m, *l);
  const size_t bytes = sizeof(float) * (size_t)m->B * m->H * m->W;
  const bool dev = is_device_ptr(out);
  if (dev) {
    a.out = out;
  } else {
    mem_status s = grow((void **)&m->dout, &m->dout_cap, bytes, m->stream);
    if (s != MEM_OK) return s;
    a.out = m->dout;
  }
  TIMED(MEM_STAGE_READ, launch_read(a, m->stream));
  if (!dev) {
    TIMED(MEM_STAGE_D2H, cudaMemcpyAsync(out, m->dout, bytes, cudaMemcpyDeviceToHost, m->stream));
    CU(cudaStreamSynchronize(m->stream));
  }
  return MEM_OK;
}

mem_status mem_set_layer(mem_map *m, const char *name, const float *src) {
  if (check_map(m)) return MEM_EINVAL;
  if (!src) return fail(MEM_EINVAL, "src is NULL");
  const Layer *l = find_layer(m, name);
  if (!l) return fail(MEM_ENOTFOUND, "no layer named '%s'", name ? name : "(null)");
  if (l->kind == LK_THETA) return fail(MEM_EINVAL, "layer '%s' is derived (alpha / sum alpha)", name);
  if (set_device(m)) return MEM_ECUDA;
  {
    mem_status fs = flush_shift(m);
    if (fs != MEM_OK) return fs;
  }
  ReadArgs a = read_args(m, *l);
  const void *d = nullptr;
  mem_status s = stage_input(m, src, sizeof(float) * (size_t)m->B * m->H * m->W, &d);
  if (s != MEM_OK) return s;
  a.src = (const float *)d;
  TIMED(MEM_STAGE_WRITE, launch_write(a, m->stream));
  return MEM_OK;
}

mem_status mem_pca_readout(mem_map *m, const char *group, int k, float *out) {
  if (check_map(m)) return MEM_EINVAL;
  if (!group || !out) return fail(MEM_EINVAL, "group and out must be non-NULL");
  int gi = -1;
  for (int i = 0; i < m->ng; ++i)
    if (m->gname[i] == group) gi = i;
  if (gi < 0) return fail(MEM_ENOTFOUND, "no group named '%s'", group);
  const GroupDesc &gd = m->g[gi];
  if (!(gd.rule == MEM_AVERAGE || gd.rule == MEM_CLASS_AVERAGE || gd.rule == MEM_GAUSSIAN))
    return fail(MEM_EINVAL, "group '%s' has no feature values for PCA", group);
  const int d = gd.nch;
  if (k < 1 || k > d) return fail(MEM_EINVAL, "k = %d out of [1, %d]", k, d);
  if (set_device(m)) return MEM_ECUDA;
  mem_status st = flush_shift(m);
  if (st != MEM_OK) return st;
  const int HW = m->H * m->W;
  const int pairs = d * (d + 1) / 2;
  const size_t nsums = (size_t)d + pairs + 1;
  // device scratch: sums | mean | comp | minmax | partial moments | projections
  const int nparts = pca_parts(HW);
  const size_t need = sizeof(double) * (nsums + d + (size_t)k * d) + sizeof(unsigned long long) * 2 * k +
                      sizeof(double) * ((size_t)nparts * nsums + (size_t)k * HW) + 64;
  st = grow(&m->pca_buf, &m->pca_cap, need, m->stream);
  if (st != MEM_OK) return st;
  double *dsums = reinterpret_cast<double *>(m->pca_buf);
  double *dmean = dsums + nsums;
  double *dcomp = dmean + d;
  unsigned long long *dmm = reinterpret_cast<unsigned long long *>(dcomp + (size_t)k * d);
  const bool dev = is_device_ptr(out);
  const size_t out_bytes = sizeof(float) * (size_t)m->B * k * HW;
  float *dout = out;
  if (!dev) {
    st = grow((void **)&m->dout, &m->dout_cap, out_bytes, m->stream);
    if (st != MEM_OK) return st;
    dout = m->dout;
  }
  PcaArgs a;
  memset(&a, 0, sizeof a);
  a.geo = m->geo();
  a.st = m->st;
  a.ring = m->ring;
  a.word0 = gd.word0;
  a.d = d;
  a.flag = gd.flag;
  a.sums = dsums;
  a.k = k;
  a.mean = dmean;
  a.comp = dcomp;
  a.minmax = dmm;
  a.part = reinterpret_cast<double *>(dmm + 2 * k);
  a.nparts = nparts;
  a.proj = a.part + (size_t)nparts * nsums;
  if ((d + 1) / 2 * 2 > 64) return fail(MEM_EINVAL, "PCA on the device takes at most 64 channels (got %d)", d);
  // per map: moments -> eigen-solve (one CTA) -> projection and min-max scaling, all on the
  // stream; nothing returns to the host
  for (int b = 0; b < m->B; ++b) {
    a.map = b;
    a.out = dout + (size_t)b * k * HW;
    TIMED(MEM_STAGE_READ, launch_pca_moments(a, m->stream));
    TIMED(MEM_STAGE_READ, launch_pca_eigen(a, m->stream));
    TIMED(MEM_STAGE_READ, launch_pca_project(a, 0, m->stream));
    TIMED(MEM_STAGE_READ, launch_pca_project(a, 1, m->stream));
  }
  if (!dev) {
    CU(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, m->stream));
    CU(cudaStreamSynchronize(m->stream));
  }
  return MEM_OK;
}

mem_status mem_get_layer_names(const mem_map *m, char *buf, size_t cap) {
  if (!m || !buf) return fail(MEM_EINVAL, "NULL argument");
  std::string s;
  for (const Layer &l : m->layers) s += l.name + "\n";
  if (s.size() + 1 > cap) return fail(MEM_EINVAL, "buffer too small: need %zu bytes", s.size() + 1);
  memcpy(buf, s.c_str(), s.size() + 1);
  return MEM_OK;
}

mem_status mem_memory_footprint(const mem_map *m, uint64_t *bytes) {
  if (!m || !bytes) return fail(MEM_EINVAL, "NULL argument");
  const uint64_t cells = (uint64_t)m->B * m->H * m->W;
  *bytes = cells * (4ull * m->n_word + (uint64_t)m->n_flag);
  return MEM_OK;
}

mem_status mem_get_info(const mem_map *m, int *n_maps, int *rows, int *cols, float *resolution) {
  if (!m) return fail(MEM_EINVAL, "map is NULL");
  if (n_maps) *n_maps = m->B;
  if (rows) *rows = m->H;
  if (cols) *cols = m->W;
  if (resolution) *resolution = m->res;
  return MEM_OK;
}

mem_status mem_get_center(const mem_map *m, int64_t *kxy) {
  if (!m || !kxy) return fail(MEM_EINVAL, "NULL argument");
  for (int i = 0; i < m->B; ++i) {
    kxy[2 * i] = m->kx[i];
    kxy[2 * i + 1] = m->ky[i];
  }
  return MEM_OK;
}

mem_status mem_frame_stats(const mem_map *m, mem_stats *out) {
  if (!m || !out) return fail(MEM_EINVAL, "NULL argument");
  if (set_device(m)) return MEM_ECUDA;
  unsigned long long hs[kStatSlots][8], h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  CU(cudaMemcpyAsync(hs, m->ctl->stats[m->epoch], sizeof hs, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  if (m->stats_empty) memset(hs, 0, sizeof hs);
  for (int i = 0; i < kStatSlots; ++i)
    for (int k = 0; k < 8; ++k) h[k] += hs[i][k];
  h[0] = h[1] + h[2] + h[3] + h[4] + h[5] + h[6];
  out->n_input = h[0];
  out->n_nonfinite = h[1];
  out->n_range = h[2];
  out->n_height = h[3];
  out->n_oob = h[4];
  out->n_inlier = h[5];
  out->n_outlier = h[6];
  out->n_cells_touched = h[7];
  return MEM_OK;
}

// NEXT-3 plugins: one k_post launch into `layers` output planes (host or device `out`)
static mem_status run_post(mem_map *m, PostArgs &a, int layers, float *out) {
  if (!out) return fail(MEM_EINVAL, "out is NULL");
  if (set_device(m)) return MEM_ECUDA;
  mem_status fs = flush_shift(m);
  if (fs == MEM_OK) fs = shard_gather_all(m);
  if (fs != MEM_OK) return fs;
  a.geo = m->geo();
  a.st = m->st;
  a.ring = m->ring;
  const size_t bytes = sizeof(float) * (size_t)layers * m->B * m->H * m->W;
  const bool dev = is_device_ptr(out);
  if (dev) {
    a.out = out;
  } else {
    mem_status s = grow((void **)&m->dout, &m->dout_cap, bytes, m->stream);
    if (s != MEM_OK) return s;
    a.out = m->dout;
  }
  TIMED(MEM_STAGE_READ, launch_post(a, m->stream));
  if (!dev) {
    TIMED(MEM_STAGE_D2H, cudaMemcpyAsync(out, m->dout, bytes, cudaMemcpyDeviceToHost, m->stream));
    CU(cudaStreamSynchronize(m->stream));
  }
  return MEM_OK;
}

mem_status mem_plugin_normals(const mem_map *cm, float *out) {
  mem_map *m = const_cast<mem_map *>(cm);
  if (check_map(m)) return MEM_EINVAL;
  PostArgs a;
  memset(&a, 0, sizeof a);
  a.op = 0;
  return run_post(m, a, 3, out);
}

mem_status mem_plugin_traversability(const mem_map *cm, float slope_max, float step_max, float *out) {
  mem_map *m = const_cast<mem_map *>(cm);
  if (check_map(m)) return MEM_EINVAL;
  const float cos_max = (float)std::cos((double)slope_max);  // rounded once to fp32 (D36)
  if (!(step_max > 0.0f) || !std::isfinite(step_max) || !(cos_max < 1.0f))
    return fail(MEM_EINVAL, "traversability: need step_max > 0 and cos(slope_max) < 1");
  PostArgs a;
  memset(&a, 0, sizeof a);
  a.op = 1;
  a.cos_max = cos_max;
  a.step_max = step_max;
  return run_post(m, a, 1, out);
}

mem_status mem_plugin_semantic_argmax(const mem_map *cm, const char *group, float *out) {
  mem_map *m = const_cast<mem_map *>(cm);
  if (check_map(m)) return MEM_EINVAL;
  if (!group) return fail(MEM_EINVAL, "group is NULL");
  int gi = -1;
  for (int k = 0; k < m->ng; ++k)
    if (m->gname[k] == group) gi = k;
  if (gi < 0) return fail(MEM_ENOTFOUND, "no group named '%s'", group);
  const GroupDesc &gd = m->g[gi];
  if (gd.rule != MEM_CLASS_BAYESIAN && gd.rule != MEM_CLASS_AVERAGE && gd.rule != MEM_CLASS_MAX)
    return fail(MEM_ERULE, "semantic argmax needs a class rule (group '%s')", group);
  PostArgs a;
  memset(&a, 0, sizeof a);
  a.op = 2;
  a.rule = gd.rule;
  a.first = gd.word0;
  a.K = gd.nch;
  a.flag = gd.flag;
  a.label = gd.label;
  return run_post(m, a, 2, out);
}

mem_status mem_set_image_occlusion(mem_map *m, int enable, float eps_occ) {
  if (check_map(m)) return MEM_EINVAL;
  if (!(eps_occ >= 0.0f) || !std::isfinite(eps_occ)) return fail(MEM_EINVAL, "eps_occ must be finite and >= 0");
  m->occlusion = enable != 0;
  m->eps_occ = eps_occ;
  return MEM_OK;
}

mem_status mem_nccl_unique_id(void *id128) {
  if (!id128) return fail(MEM_EINVAL, "id is NULL");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  memcpy(id128, &id, sizeof id);
  return MEM_OK;
}

mem_status mem_create_sharded(float resolution, int rows, int cols, const mem_layer_spec *groups, int n_groups,
                              unsigned flags, mem_stream stream, const void *nccl_id128, int rank, int nranks,
                              mem_map **out) {
  if (!out) return fail(MEM_EINVAL, "out is NULL");
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks)
    return fail(MEM_EINVAL, "rank %d / nranks %d invalid", rank, nranks);
  if (rows % nranks != 0) return fail(MEM_EINVAL, "rows (%d) must be divisible by nranks (%d)", rows, nranks);
  mem_map *m = nullptr;
  mem_status s = mem_create_batch(1, resolution, rows, cols, groups, n_groups, flags, stream, &m);
  if (s != MEM_OK) return s;
  m->transport = nccl_id128 ? 1 : 2;
  m->rank = rank;
  m->nranks = nranks;
  m->band_n = rows / nranks * cols;
  m->band_lo = rank * m->band_n;
  // every point input routes the shard's in-window points to their band owners
  if (cudaMalloc((void **)&m->rcnt, sizeof(unsigned) * nranks) != cudaSuccess ||
      cudaMalloc((void **)&m->rall, sizeof(unsigned) * nranks * nranks) != cudaSuccess) {
    cudaGetLastError();
    free_map(m);
    return fail(MEM_ENOMEM, "route counters");
  }
  if (m->transport == 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id128, sizeof id);
    ncclResult_t r = ncclCommInitRank(&m->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      free_map(m);
      return fail(MEM_ECOMM, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = m;
  return MEM_OK;
}

mem_status mem_shard_local_sync(mem_map **sh, int G) {
  if (!sh || G < 1) return fail(MEM_EINVAL, "shards");
  for (int r = 0; r < G; ++r) {
    if (!sh[r] || sh[r]->transport != 2 || sh[r]->nranks != G || sh[r]->rank != r)
      return fail(MEM_EINVAL, "shard %d is not local rank %d of %d", r, r, G);
    if (sh[r]->stream != sh[0]->stream) return fail(MEM_EINVAL, "local shards must share one stream");
  }
  for (int r = 1; r < G; ++r)
    if (sh[r]->exchange_pending != sh[0]->exchange_pending)
      return fail(MEM_EINVAL, "shard %d did not take the same inputs as shard 0", r);
  mem_map *m0 = sh[0];
  if (set_device(m0)) return MEM_ECUDA;
  const int HW = m0->H * m0->W, bn = m0->band_n;
  if (m0->exchange_pending) {  // point routing: buckets to their owners, owner passes
    const int st = m0->route_stride;
    std::vector<unsigned> cnt((size_t)G * G);
    for (int p = 0; p < G; ++p)
      CU(cudaMemcpyAsync(cnt.data() + (size_t)p * G, sh[p]->rcnt, sizeof(unsigned) * G, cudaMemcpyDeviceToHost,
                         m0->stream));
    CU(cudaStreamSynchronize(m0->stream));
    for (int r = 0; r < G; ++r) {
      long long n_in = 0;
      for (int p = 0; p < G; ++p) n_in += cnt[(size_t)p * G + r];
      if (grow_floats(&sh[r]->rin, &sh[r]->rin_cap, (size_t)std::max(1LL, n_in) * st, m0->stream) != MEM_OK)
        return fail(MEM_ENOMEM, "routed points");
      long long off = 0;
      for (int p = 0; p < G; ++p) {
        const size_t k = cnt[(size_t)p * G + r];
        if (k)
          CU(cudaMemcpyAsync(sh[r]->rin + (size_t)off * st, sh[p]->rbuf + (size_t)r * sh[p]->route_cap * st,
                             sizeof(float) * k * st, cudaMemcpyDeviceToDevice, m0->stream));
        off += (long long)k;
      }
      mem_status s = owner_pass(sh[r], sh[r]->rin, n_in);
      if (s != MEM_OK) return s;
      if (sh[r]->flags & MEM_FLAG_DEBUG_POINTS) {  // the owner's in/out codes back to the sources
        off = 0;
        for (int p = 0; p < G; ++p) {
          const long long k = cnt[(size_t)p * G + r];
          if (sh[p]->flags & MEM_FLAG_DEBUG_POINTS)
            CU(launch_code_return(sh[r]->odbg_code + off, sh[p]->rsrc + (size_t)r * sh[p]->route_cap, k,
                                  sh[p]->dbg_code, m0->stream));
          off += k;
        }
      }
    }
  }
  for (int r = 0; r < G; ++r) sh[r]->exchange_pending = false;
  // full replication (after point clouds and images alike): every layer's band r from shard r to all others
  for (int r = 0; r < G; ++r)
    for (int p = 0; p < G; ++p) {
      if (p == r) continue;
      for (int w = 0; w < m0->n_word; ++w)
        CU(cudaMemcpyAsync(sh[p]->st.words + (size_t)w * HW + sh[r]->band_lo,
                           sh[r]->st.words + (size_t)w * HW + sh[r]->band_lo, 4 * (size_t)bn,
                           cudaMemcpyDeviceToDevice, m0->stream));
      for (int f = 0; f < m0->n_flag; ++f)
        CU(cudaMemcpyAsync(sh[p]->st.flags + (size_t)f * HW + sh[r]->band_lo,
                           sh[r]->st.flags + (size_t)f * HW + sh[r]->band_lo, bn, cudaMemcpyDeviceToDevice,
                           m0->stream));
    }
  return MEM_OK;
}

mem_status mem_profile(mem_map *m, int enable) {
  if (check_map(m)) return MEM_EINVAL;
  m->prof.on = enable != 0;
  return MEM_OK;
}

mem_status mem_profile_read(mem_map *m, double *ms, uint64_t *counts, int reset) {
  if (check_map(m)) return MEM_EINVAL;
  if (set_device(m)) return MEM_ECUDA;
  CU(cudaStreamSynchronize(m->stream));
  for (int st = 0; st < MEM_N_STAGES; ++st) {
    for (auto &pr : m->prof.pending[st]) {
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, pr.first, pr.second));
      m->prof.ms[st] += t;
      m->prof.pool.push_back(pr.first);
      m->prof.pool.push_back(pr.second);
    }
    m->prof.pending[st].clear();
    if (ms) ms[st] = m->prof.ms[st];
    if (counts) counts[st] = m->prof.count[st];
    if (reset) {
      m->prof.ms[st] = 0.0;
      m->prof.count[st] = 0;
    }
  }
  return MEM_OK;
}

mem_status mem_debug_point_codes(const mem_map *m, int32_t *cell, uint8_t *code) {
  if (!m) return fail(MEM_EINVAL, "map is NULL");
  if (!(m->flags & MEM_FLAG_DEBUG_POINTS)) return fail(MEM_EINVAL, "map created without MEM_FLAG_DEBUG_POINTS");
  if (set_device(m)) return MEM_ECUDA;
  if (m->dbg_n == 0) return MEM_OK;
  if (cell) CU(cudaMemcpyAsync(cell, m->dbg_cell, sizeof(int) * m->dbg_n, cudaMemcpyDefault, m->stream));
  if (code) CU(cudaMemcpyAsync(code, m->dbg_code, m->dbg_n, cudaMemcpyDefault, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return MEM_OK;
}

}  // extern "C"
