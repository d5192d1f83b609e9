/*
 * mem_oracle.c -- the CPU ORACLE for the MEM fusion hot path (arXiv 2309.16818).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2309_16818_b200/, libmem) never links, imports or calls it, and it shares
 * no code, header, constant table or helper with the CUDA path.
 *
 * Plain, slow, single-threaded C, written step by step from
 *   PAPER.md  = /root/reference/PAPER.md  (the paper; its LaTeX body)
 *   SURVEY    = SURVEY.md §8(c) N2 (the step list) and N4 (readings D1..D31)
 * in the order and notation of those passages.  One map, logical row-major storage
 * (no ring buffer: move_to is a naive copy into a new map).
 *
 * Numerics (reading D29): every fp32 operation is IEEE round-to-nearest in the
 * written order, no FMA contraction (compile with -ffp-contract=off, never with
 * -ffast-math); per-cell sums and closed forms in fp64, stored as (float).
 *
 * Parity pins: tests/test_oracle_pins.py (list in DESIGN.md §3).  Every function has a
 * pin that is not a re-typing of its own formula.  Where the paper is silent and the
 * oracle follows the north_star / SPEC.md reading, the pin checks that reading by
 * independent means:
 *   - noise model v = a + b r^2 (D8): a single point into an empty cell gives height z
 *     and variance a + b r^2 exactly (dyadic values; test_single_point_empty_cell);
 *   - Mahalanobis gate (D10) and outlier inflation sigma2 + n_out v_out (D11): the
 *     equality / next-float boundary cases and the inflated variance
 *     (test_outlier_boundary);
 *   - class_max's frame winner (D19): brute force with ties and input permutations
 *     (test_class_max_brute_force_ties_permutation);
 *   - colour rule (D20): brute-force per-cell RGB means (test_color_brute_force).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#define OM_OK 0
#define OM_EINVAL (-1)
#define OM_EDUPNAME (-2)
#define OM_ENOTFOUND (-3)
#define OM_ERULE (-4)
#define OM_EPOSE (-5)
#define OM_ENOMEM (-7)

/* fusion rules */
#define OM_AVERAGE 0        /* PAPER.md:265-292 Eq.(1)+(2); w = 1 is "Latest"          */
#define OM_GAUSSIAN 1       /* PAPER.md:294-324 Eq.(3)-(7)                              */
#define OM_CLASS_AVERAGE 2  /* PAPER.md:290 Eq.(2) on class-probability vectors        */
#define OM_CLASS_BAYESIAN 3 /* PAPER.md:326-357 Eq.(8)-(12), Dirichlet                  */
#define OM_CLASS_MAX 4      /* PAPER.md:251-252, 514; reading D19                       */
#define OM_COLOR 5          /* PAPER.md:488-505; reading D20                            */

/* per-point codes (SURVEY §8(b) mem_debug_point_codes; filter order D9) */
#define OM_INLIER 0
#define OM_OUTLIER 1
#define OM_NONFINITE 2
#define OM_RANGE 3
#define OM_HEIGHT 4
#define OM_OOB 5

typedef struct {
  const char *name;
  int rule;
  int n_channels;
  float w;        /* Eq.(2) weight, 0 < w <= 1 */
  float sigma_f2; /* Eq.(3) known measurement variance */
  float mu0;      /* Eq.(4) prior mean */
  float sigma0_2; /* Eq.(4) prior variance */
  float alpha0;   /* Eq.(8) Dirichlet prior (D6) */
} om_group_spec;

typedef struct {
  int ch_offset; /* point clouds: channel index counted from float 3; images: from channel 0 */
  int n_ch;
  int group;
  int topk;      /* > 0: n_ch = 2 topk channels (class id, probability) pairs (NEXT-2, D38) */
} om_binding;

typedef struct {
  float a, b;         /* v = a + b r^2 (D8) */
  float r_min, r_max; /* range filter, inclusive (D9) */
  float h_min, h_max; /* height filter on q_z, inclusive (D9) */
  float tau2;         /* Mahalanobis gate (D10) */
  float v_out;        /* outlier inflation (D11) */
} om_noise;

typedef struct {
  char name[64];
  int rule, nch;  /* nch = input width: class count K, feature dim d, 3 for colour */
  float w, sigma_f2, mu0, sigma0_2, alpha0;
  float *val;     /* [nval][cells]; average/class_average/colour: theta; gaussian: mu then var;
                     class_bayesian: alpha; class_max: conf */
  int *label;     /* class_max only: label, -1 = unobserved (D15) */
  unsigned char *observed; /* [cells] first-touch flag (D3); unused for class_max */
} om_group;

typedef struct om_map {
  float res;
  int rows, cols; /* rows <-> +x, cols <-> +y (D13) */
  long long kx, ky; /* centre = (kx*res, ky*res) (D13, D14) */
  float *h, *s2;  /* elevation, variance: NaN where invalid (D15) */
  unsigned char *valid;
  int ng;
  om_group g[32];
  unsigned long long stats[8];
  int occlusion;   /* image association with the Bresenham occlusion test (NEXT-1) */
  float eps_occ;   /* occlusion tolerance, default 1e-4 m */
} om_map;

static int nval_of(int rule, int nch) {
  if (rule == OM_GAUSSIAN) return 2 * nch;
  if (rule == OM_CLASS_MAX) return 1;
  return nch;
}

static long ncells(const om_map *m) { return (long)m->rows * (long)m->cols; }

static void reset_cell(om_map *m, long j) {
  /* the state of a never-observed cell (D15) */
  m->h[j] = NAN;
  m->s2[j] = NAN;
  m->valid[j] = 0;
  for (int gi = 0; gi < m->ng; ++gi) {
    om_group *g = &m->g[gi];
    for (int k = 0; k < nval_of(g->rule, g->nch); ++k) g->val[(long)k * ncells(m) + j] = 0.0f;
    if (g->label) g->label[j] = -1;
    g->observed[j] = 0;
  }
}

void om_destroy(om_map *m) {
  if (!m) return;
  free(m->h); free(m->s2); free(m->valid);
  for (int i = 0; i < m->ng; ++i) { free(m->g[i].val); free(m->g[i].label); free(m->g[i].observed); }
  free(m);
}

om_map *om_create(float res, int rows, int cols, const om_group_spec *gs, int ng, int *status) {
  *status = OM_EINVAL;
  if (!(res > 0.0f) || rows < 1 || cols < 1 || ng < 0 || ng > 32) return NULL;
  for (int i = 0; i < ng; ++i) {
    const om_group_spec *s = &gs[i];
    if (!s->name || !s->name[0] || strlen(s->name) >= 40) return NULL;
    if (s->rule < 0 || s->rule > 5) { *status = OM_ERULE; return NULL; }
    if (s->rule == OM_COLOR) { if (s->n_channels != 3) return NULL; }
    else if (s->n_channels < 1 || s->n_channels > 256) return NULL;
    if ((s->rule == OM_CLASS_AVERAGE || s->rule == OM_CLASS_BAYESIAN || s->rule == OM_CLASS_MAX) &&
        s->n_channels < 2) { *status = OM_ERULE; return NULL; }
    if ((s->rule == OM_AVERAGE || s->rule == OM_CLASS_AVERAGE || s->rule == OM_COLOR) &&
        !(s->w > 0.0f && s->w <= 1.0f)) return NULL;
    if (s->rule == OM_GAUSSIAN && !(s->sigma_f2 > 0.0f && s->sigma0_2 > 0.0f)) return NULL;
    if (s->rule == OM_CLASS_BAYESIAN && !(s->alpha0 > 0.0f)) return NULL;
    if (!strcmp(s->name, "elevation") || !strcmp(s->name, "variance") || !strcmp(s->name, "valid")) {
      *status = OM_EDUPNAME; return NULL;
    }
    for (int k = 0; k < i; ++k)
      if (!strcmp(gs[k].name, s->name)) { *status = OM_EDUPNAME; return NULL; }
  }
  om_map *m = (om_map *)calloc(1, sizeof(om_map));
  if (!m) { *status = OM_ENOMEM; return NULL; }
  m->res = res; m->rows = rows; m->cols = cols; m->kx = 0; m->ky = 0;
  m->occlusion = 0; m->eps_occ = 1e-4f;
  long n = ncells(m);
  m->h = (float *)malloc(sizeof(float) * n);
  m->s2 = (float *)malloc(sizeof(float) * n);
  m->valid = (unsigned char *)malloc(n);
  m->ng = ng;
  for (int i = 0; i < ng; ++i) {
    om_group *g = &m->g[i];
    snprintf(g->name, sizeof g->name, "%s", gs[i].name);
    g->rule = gs[i].rule; g->nch = gs[i].n_channels;
    g->w = gs[i].w; g->sigma_f2 = gs[i].sigma_f2; g->mu0 = gs[i].mu0;
    g->sigma0_2 = gs[i].sigma0_2; g->alpha0 = gs[i].alpha0;
    g->val = (float *)malloc(sizeof(float) * n * nval_of(g->rule, g->nch));
    g->label = g->rule == OM_CLASS_MAX ? (int *)malloc(sizeof(int) * n) : NULL;
    g->observed = (unsigned char *)malloc(n);
  }
  for (long j = 0; j < n; ++j) reset_cell(m, j);
  *status = OM_OK;
  return m;
}

/* R^T R = I within 1e-6 and det(R) = +1 within 1e-6. */
static int pose_ok(const double R[9]) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double d = 0.0;
      for (int k = 0; k < 3; ++k) d += R[k * 3 + a] * R[k * 3 + b];
      if (!isfinite(d) || fabs(d - (a == b ? 1.0 : 0.0)) > 1e-6) return 0;
    }
  double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
               R[2] * (R[3] * R[7] - R[4] * R[6]);
  return fabs(det - 1.0) <= 1e-6;
}

/* top-k class input ("inputting the top k classes", SPEC.md:144-147,
 * 168-176 expand_topk; reading D38): the group's last class (index K = nch - 1) is the
 * reserved "other" class.  dense[id_j] += p_j, dense[K] = 1 - sum_j p_j (fp32, pair order);
 * returns 0 (the group skips this point / pixel, like a non-finite channel, D31) if a value is
 * non-finite or an id is not an integer in [0, K). */
static int expand_topk(const float *ch, long step, int k, int nch, float *dense) {
  const int K = nch - 1;
  for (int c = 0; c < nch; ++c) dense[c] = 0.0f;
  float sp = 0.0f;
  for (int j = 0; j < k; ++j) {
    const float id = ch[(long)(2 * j) * step], pj = ch[(long)(2 * j + 1) * step];
    if (!isfinite(id) || !isfinite(pj) || id != floorf(id) || id < 0.0f || id >= (float)K) return 0;
    dense[(int)id] += pj;
    sp += pj;
  }
  dense[K] = 1.0f - sp;
  return 1;
}

static int topk_binding_ok(const om_group *g, const om_binding *b) {
  if (b->topk <= 0) return 1;
  return (g->rule == OM_CLASS_AVERAGE || g->rule == OM_CLASS_BAYESIAN || g->rule == OM_CLASS_MAX) &&
         b->n_ch == 2 * b->topk;
}

static int binding_width_ok(const om_group *g, int n_ch, int is_image) {
  if (g->rule == OM_COLOR) return is_image ? n_ch == 3 : n_ch == 1; /* D20 */
  return n_ch == g->nch;
}

/* ---- per-cell fusion rules, fp64 in, (float) out.  `n` = N_j this frame,
 *      `sum[k]` = sum_i m_{i,k} over the cell's points (Eq.(1) numerator). ---- */

/* Eq.(1) + Eq.(2): a = sum/N_j; theta' = w a + (1-w) theta; first touch theta' = a (D3). */
static void fuse_average(om_group *g, long j, long cells, long n, const double *sum) {
  for (int k = 0; k < g->nch; ++k) {
    double a = sum[k] / (double)n;
    float *th = &g->val[(long)k * cells + j];
    double out;
    if (g->observed[j]) out = (double)g->w * a + (1.0 - (double)g->w) * (double)(*th);
    else out = a;
    *th = (float)out;
  }
  g->observed[j] = 1;
}

/* Eq.(6)-(7) with prior = current posterior (first touch: (mu0, sigma0^2)), N = N_j (D4). */
static void fuse_gaussian(om_group *g, long j, long cells, long n, const double *sum) {
  for (int k = 0; k < g->nch; ++k) {
    float *mu = &g->val[(long)k * cells + j];
    float *var = &g->val[(long)(g->nch + k) * cells + j];
    double mu_p = g->observed[j] ? (double)(*mu) : (double)g->mu0;
    double s2_p = g->observed[j] ? (double)(*var) : (double)g->sigma0_2;
    double sf2 = (double)g->sigma_f2;
    double N = (double)n;
    double mu_ml = sum[k] / N;
    double den = N * s2_p + sf2;
    double mu_n = (sf2 / den) * mu_p + ((N * s2_p) / den) * mu_ml; /* Eq.(6) */
    double s2_n = (sf2 * s2_p) / den;                               /* Eq.(7) */
    *mu = (float)mu_n;
    *var = (float)s2_n;
  }
  g->observed[j] = 1;
}

/* Eq.(12): alpha_t = alpha_{t-1} + sum_i m_i; first touch alpha_{t-1} = alpha0 (D6). */
static void fuse_dirichlet(om_group *g, long j, long cells, const double *sum) {
  for (int k = 0; k < g->nch; ++k) {
    float *al = &g->val[(long)k * cells + j];
    double prior = g->observed[j] ? (double)(*al) : (double)g->alpha0;
    *al = (float)(prior + sum[k]);
  }
  g->observed[j] = 1;
}

/* D19: monotone map of a float's bits to u32 (order-preserving for all finite floats). */
static uint32_t ord_of_float(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
static float float_of_ord(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
/* D19: one observation's key: (conf, -k*) with k* the lowest index among maximal m_k. */
static uint64_t class_max_key(const float *m, int K, long step) {
  int best = 0;
  float bv = m[0];
  for (int k = 1; k < K; ++k)
    if (m[k * step] > bv) { bv = m[k * step]; best = k; }
  return ((uint64_t)ord_of_float(bv) << 32) | (uint64_t)(uint32_t)(K - 1 - best);
}
static void store_class_max(om_group *g, long j, uint64_t key) {
  g->label[j] = g->nch - 1 - (int)(uint32_t)(key & 0xffffffffu);
  g->val[j] = float_of_ord((uint32_t)(key >> 32));
}

/* ---- point-cloud input: SURVEY §8(c) N2 steps 1-3 ----
 * Split in two so that the sharded big map can be checked on CPU:
 * om_accumulate runs steps 1-2 and returns the frame's per-cell sufficient statistics;
 * om_fuse_rows runs step 3 on the rows [row_lo, row_hi).  om_input_pointcloud is the two
 * in sequence over all rows.  The statistics are plain sums / counts / maxima of
 * per-point terms, so statistics of disjoint point subsets add up (max for class_max keys). */
typedef struct om_frame {
  long cells;
  int nb;
  om_binding bind[16];
  om_noise noise;
  unsigned long long *n_in, *n_out;
  double *P, *S;
  unsigned long long *ng[16];
  double *gsum[16];
  unsigned long long *gkey[16];
  int nsum[16]; /* sums per cell of binding b = the group's width (3 for colour) */
  unsigned long long st[8];
} om_frame;

void om_frame_free(om_frame *f) {
  if (!f) return;
  free(f->n_in); free(f->n_out); free(f->P); free(f->S);
  for (int b = 0; b < f->nb; ++b) { free(f->ng[b]); free(f->gsum[b]); free(f->gkey[b]); }
  free(f);
}

/* raw access to a frame's statistics (field 0 n_in, 1 n_out, 2 P, 3 S, 4 group count,
   5 group sums [n_ch][cells], 6 class_max keys, 7 the 8 counters); *len = element count */
void *om_frame_array(om_frame *f, int field, int b, long *len) {
  *len = f->cells;
  switch (field) {
    case 0: return f->n_in;
    case 1: return f->n_out;
    case 2: return f->P;
    case 3: return f->S;
    case 4: return f->ng[b];
    case 5: *len = f->cells * f->nsum[b]; return f->gsum[b];
    case 6: if (!f->gkey[b]) *len = 0; return f->gkey[b];
    case 7: *len = 8; return f->st;
  }
  *len = 0;
  return NULL;
}

om_frame *om_accumulate(om_map *m, const float *pts, long n, int stride, const om_binding *bind, int nb,
                        const double R[9], const double t[3], const om_noise *np, int *cell_out,
                        unsigned char *code_out, int *status) {
  *status = OM_EINVAL;
  if (n < 0 || stride < 3 || nb < 0 || nb > 16 || !np) return NULL;
  if (!pose_ok(R)) { *status = OM_EPOSE; return NULL; }
  for (int b = 0; b < nb; ++b) {
    if (bind[b].group < 0 || bind[b].group >= m->ng) return NULL;
    if (bind[b].ch_offset < 0 || 3 + bind[b].ch_offset + bind[b].n_ch > stride) return NULL;
    if (bind[b].topk > 0 ? !topk_binding_ok(&m->g[bind[b].group], &bind[b])
                         : !binding_width_ok(&m->g[bind[b].group], bind[b].n_ch, 0)) return NULL;
    for (int c = 0; c < b; ++c) if (bind[c].group == bind[b].group) return NULL;
  }
  const long cells = ncells(m);
  const int H = m->rows, W = m->cols;
  /* step 1: host frame setup -- t relative to the map centre in fp64, then fp32 (D13) */
  const float Rf[9] = {(float)R[0], (float)R[1], (float)R[2], (float)R[3], (float)R[4],
                       (float)R[5], (float)R[6], (float)R[7], (float)R[8]};
  const double cx = (double)m->kx * (double)m->res, cy = (double)m->ky * (double)m->res;
  const float tx = (float)(t[0] - cx), ty = (float)(t[1] - cy), tz = (float)t[2];
  const float hH = (float)H / 2.0f, hW = (float)W / 2.0f;
  const float res = m->res;

  /* per-cell, per-frame sufficient statistics */
  om_frame *f = (om_frame *)calloc(1, sizeof(om_frame));
  f->cells = cells;
  f->nb = nb;
  memcpy(f->bind, bind, sizeof(om_binding) * (size_t)nb);
  f->noise = *np;
  unsigned long long *n_in = f->n_in = calloc(cells, sizeof *n_in), *n_out = f->n_out = calloc(cells, sizeof *n_out);
  double *P = f->P = calloc(cells, sizeof *P), *S = f->S = calloc(cells, sizeof *S);
  unsigned long long **ng = f->ng;
  double **gsum = f->gsum;
  unsigned long long **gkey = f->gkey;
  for (int b = 0; b < nb; ++b) {
    const om_group *g = &m->g[bind[b].group];
    ng[b] = calloc(cells, sizeof(unsigned long long));
    gsum[b] = calloc((size_t)cells * g->nch, sizeof(double));
    gkey[b] = g->rule == OM_CLASS_MAX ? calloc(cells, sizeof(unsigned long long)) : NULL;
    f->nsum[b] = g->nch;
  }
  unsigned long long *st = f->st;
  st[0] = (unsigned long long)n;

  /* step 2: for each point, in input order */
  for (long i = 0; i < n; ++i) {
    const float *p = pts + (size_t)i * stride;
    const float px = p[0], py = p[1], pz = p[2];
    int code, cell = -1;
    long j = -1;
    float z = 0.0f, v = 0.0f;
    if (!isfinite(px) || !isfinite(py) || !isfinite(pz)) {
      code = OM_NONFINITE; /* 2.1 */
    } else {
      /* 2.2: range filter r_min <= r <= r_max on the sensor-frame range (reading D9) */
      const float r2 = (px * px + py * py) + pz * pz;
      const float r = sqrtf(r2);
      if (!(np->r_min <= r && r <= np->r_max)) {
        code = OM_RANGE;
      } else {
        /* 2.3: q = R p ("point trsf.") */
        const float qx = (Rf[0] * px + Rf[1] * py) + Rf[2] * pz;
        const float qy = (Rf[3] * px + Rf[4] * py) + Rf[5] * pz;
        const float qz = (Rf[6] * px + Rf[7] * py) + Rf[8] * pz;
        if (!(np->h_min <= qz && qz <= np->h_max)) {
          code = OM_HEIGHT;
        } else {
          /* 2.4 */
          const float x = qx + tx, y = qy + ty;
          z = qz + tz;
          /* 2.5: bin by horizontal coordinates, half-open cells */
          const float fr = x / res + hH, fc = y / res + hW; /* reading D13 */
          if (!(0.0f <= fr && fr < (float)H && 0.0f <= fc && fc < (float)W)) {
            code = OM_OOB;
          } else {
            const int row = (int)floorf(fr), col = (int)floorf(fc);
            cell = row * W + col;
            j = cell;
            v = np->a + np->b * r2; /* 2.6 (D8) */
            /* 2.7: Mahalanobis test against the pre-frame cell state (D10) */
            int outlier = 0;
            if (m->valid[j]) {
              const float d = z - m->h[j];
              outlier = d * d > np->tau2 * (m->s2[j] + v);
            }
            code = outlier ? OM_OUTLIER : OM_INLIER;
          }
        }
      }
    }
    if (cell_out) cell_out[i] = cell;
    if (code_out) code_out[i] = (unsigned char)code;
    st[code == OM_INLIER ? 5 : code == OM_OUTLIER ? 6 : code - 1]++;
    if (j < 0) continue;
    /* 2.8: accumulate */
    if (code == OM_OUTLIER) {
      n_out[j]++;
    } else {
      n_in[j]++;
      const float w = 1.0f / v;
      P[j] += (double)w;
      S[j] += (double)(z * w);
    }
    for (int b = 0; b < nb; ++b) { /* every filtered in-bounds point feeds the groups (D12) */
      const om_group *g = &m->g[bind[b].group];
      const float *ch = p + 3 + bind[b].ch_offset;
      if (g->rule == OM_COLOR) { /* D20: 0x00RRGGBB bit-cast into the float */
        uint32_t bits;
        memcpy(&bits, ch, 4);
        ng[b][j]++;
        gsum[b][(long)0 * cells + j] += (double)((bits >> 16) & 255u);
        gsum[b][(long)1 * cells + j] += (double)((bits >> 8) & 255u);
        gsum[b][(long)2 * cells + j] += (double)(bits & 255u);
        continue;
      }
      float dense[257];
      const float *src = ch;
      if (bind[b].topk > 0) { /* NEXT-2: expand the top-k pairs first (D38) */
        if (!expand_topk(ch, 1, bind[b].topk, g->nch, dense)) continue;
        src = dense;
      }
      int finite = 1;
      for (int k = 0; k < g->nch; ++k) finite &= isfinite(src[k]) ? 1 : 0;
      if (!finite) continue; /* D31 */
      ng[b][j]++;
      for (int k = 0; k < g->nch; ++k) gsum[b][(long)k * cells + j] += (double)src[k];
      if (g->rule == OM_CLASS_MAX) {
        uint64_t key = class_max_key(src, g->nch, 1);
        if (key > gkey[b][j]) gkey[b][j] = key;
      }
    }
  }

  *status = OM_OK;
  return f;
}

int om_fuse_rows(om_map *m, om_frame *f, int row_lo, int row_hi) {
  if (row_lo < 0 || row_hi > m->rows || row_lo > row_hi || f->cells != ncells(m)) return OM_EINVAL;
  const long cells = f->cells;
  const int nb = f->nb;
  const om_binding *bind = f->bind;
  const om_noise *np = &f->noise;
  const unsigned long long *n_in = f->n_in, *n_out = f->n_out;
  const double *P = f->P, *S = f->S;
  unsigned long long st[8];
  memcpy(st, f->st, sizeof st);
  /* step 3: per cell; cells with no points stay bit-untouched */
  double sums[256];
  for (long j = (long)row_lo * m->cols; j < (long)row_hi * m->cols; ++j) {
    if (n_in[j] + n_out[j] == 0) continue;
    st[7]++;
    /* a9: Kalman height fusion in information form (D7, D11) */
    if (m->valid[j]) {
      const double sp = (double)m->s2[j] + (double)n_out[j] * (double)np->v_out;
      if (n_in[j] > 0) {
        /* information form h' = (h/sp + S)/(1/sp + P), sigma2' = 1/(1/sp + P) (reading D7) */
        const double den = 1.0 / sp + P[j];
        m->h[j] = (float)(((double)m->h[j] / sp + S[j]) / den);
        m->s2[j] = (float)(1.0 / den);
      } else {
        m->s2[j] = (float)sp;
      }
    } else if (n_in[j] > 0) { /* first touch: h = S/P, sigma^2 = 1/P */
      m->h[j] = (float)(S[j] / P[j]);
      m->s2[j] = (float)(1.0 / P[j]);
      m->valid[j] = 1;
    }
    /* a10: each bound group by its rule */
    for (int b = 0; b < nb; ++b) {
      om_group *g = &m->g[bind[b].group];
      if (f->ng[b][j] == 0) continue;
      for (int k = 0; k < g->nch; ++k) sums[k] = f->gsum[b][(long)k * cells + j];
      switch (g->rule) {
        case OM_AVERAGE:
        case OM_CLASS_AVERAGE:
        case OM_COLOR: fuse_average(g, j, cells, (long)f->ng[b][j], sums); break;
        case OM_GAUSSIAN: fuse_gaussian(g, j, cells, (long)f->ng[b][j], sums); break;
        case OM_CLASS_BAYESIAN: fuse_dirichlet(g, j, cells, sums); break;
        case OM_CLASS_MAX: store_class_max(g, j, f->gkey[b][j]); break;
      }
    }
  }
  memcpy(m->stats, st, sizeof st);
  return OM_OK;
}

int om_input_pointcloud(om_map *m, const float *pts, long n, int stride, const om_binding *bind, int nb,
                        const double R[9], const double t[3], const om_noise *np, int *cell_out,
                        unsigned char *code_out) {
  int status;
  om_frame *f = om_accumulate(m, pts, n, stride, bind, nb, R, t, np, cell_out, code_out, &status);
  if (!f) return status;
  status = om_fuse_rows(m, f, 0, m->rows);
  om_frame_free(f);
  return status;
}

/* ---- Bresenham line ("computed using Bresenham's algorithm").
 * The intermediate cells (both endpoints excluded) of the 8-connected line between integer
 * cells a and b, written to out (capacity cap), returns their count.  Standard all-octant
 * integer form (err = dx + dy with dy = -|y1-y0|; step x when 2 err >= dy, y when 2 err <= dx),
 * always walked from the lexicographically smaller endpoint so that (a, b) and (b, a) give the
 * same cell set (reading D33). ---- */
int om_bresenham(int r0, int c0, int r1, int c1, int *out_r, int *out_c, int cap) {
  if (r1 < r0 || (r1 == r0 && c1 < c0)) { int t = r0; r0 = r1; r1 = t; t = c0; c0 = c1; c1 = t; }
  const int dx = abs(r1 - r0), dy = -abs(c1 - c0);
  const int sx = r0 < r1 ? 1 : -1, sy = c0 < c1 ? 1 : -1;
  int err = dx + dy, x = r0, y = c0, n = 0;
  for (;;) {
    if (x == r1 && y == c1) break;
    const int e2 = 2 * err;
    if (e2 >= dy) { err += dy; x += sx; }
    if (e2 <= dx) { err += dx; y += sy; }
    if (x == r1 && y == c1) break;
    if (n < cap) { out_r[n] = x; out_c[n] = y; }
    ++n;
  }
  return n;
}

void om_set_occlusion(om_map *m, int enable, float eps_occ) {
  m->occlusion = enable != 0;
  m->eps_occ = eps_occ;
}

/* the occlusion test of one target cell (readings
 * D32-D34): every valid in-map intermediate cell on the line from the camera's footprint cell
 * to the target must have elevation <= the ray height + eps_occ, the ray height interpolated
 * linearly between the camera height and the target elevation by 2D distance fraction */
static int om_visible(const om_map *m, int row, int col, float tx, float ty, float tz, float hb) {
  const int H = m->rows, W = m->cols;
  const float hH = (float)H / 2.0f, hW = (float)W / 2.0f;
  const int rc = (int)floorf(tx / m->res + hH), cc = (int)floorf(ty / m->res + hW); /* binned like a point (D13) */
  const float xb = ((float)row + 0.5f - hH) * m->res, yb = ((float)col + 0.5f - hW) * m->res;
  const float dxb = xb - tx, dyb = yb - ty;
  const float db = sqrtf(dxb * dxb + dyb * dyb);
  static int rr[1 << 16], cr[1 << 16];
  const int n = om_bresenham(rc, cc, row, col, rr, cr, 1 << 16);
  for (int k = 0; k < n && k < (1 << 16); ++k) {
    const int i = rr[k], jj = cr[k];
    if (i < 0 || i >= H || jj < 0 || jj >= W) continue; /* outside the map: no occluder */
    const long j = (long)i * W + jj;
    if (!m->valid[j]) continue;                          /* unknown terrain does not occlude */
    const float xi = ((float)i + 0.5f - hH) * m->res, yi = ((float)jj + 0.5f - hW) * m->res;
    const float dxi = xi - tx, dyi = yi - ty;
    const float di = sqrtf(dxi * dxi + dyi * dyi);
    const float ray = tz + (di / db) * (hb - tz);
    if (m->h[j] > ray + m->eps_occ) return 0;
  }
  return 1;
}

/* ---- image input: SURVEY §8(c) N2 step 4 (a11 + a12), PAPER.md:232-239 ---- */
int om_input_image(om_map *m, const float *img, int C, int IH, int IW, const om_binding *bind, int nb,
                   const double K[9], const double R[9], const double t[3]) {
  if (C < 1 || IH < 1 || IW < 1 || nb < 0 || nb > 16) return OM_EINVAL;
  if (!(K[0] > 0.0 && K[4] > 0.0) || K[3] != 0.0 || K[6] != 0.0 || K[7] != 0.0 || K[8] != 1.0)
    return OM_EINVAL;
  if (!pose_ok(R)) return OM_EPOSE;
  for (int b = 0; b < nb; ++b) {
    if (bind[b].group < 0 || bind[b].group >= m->ng) return OM_EINVAL;
    if (bind[b].ch_offset < 0 || bind[b].ch_offset + bind[b].n_ch > C) return OM_EINVAL;
    if (bind[b].topk > 0 ? !topk_binding_ok(&m->g[bind[b].group], &bind[b])
                         : !binding_width_ok(&m->g[bind[b].group], bind[b].n_ch, 1)) return OM_EINVAL;
    for (int c = 0; c < b; ++c) if (bind[c].group == bind[b].group) return OM_EINVAL;
  }
  const long cells = ncells(m);
  const int H = m->rows, W = m->cols;
  const float Rf[9] = {(float)R[0], (float)R[1], (float)R[2], (float)R[3], (float)R[4],
                       (float)R[5], (float)R[6], (float)R[7], (float)R[8]};
  const double cxm = (double)m->kx * (double)m->res, cym = (double)m->ky * (double)m->res;
  const float tx = (float)(t[0] - cxm), ty = (float)(t[1] - cym), tz = (float)t[2];
  const float fx = (float)K[0], sk = (float)K[1], ccx = (float)K[2], fy = (float)K[4], ccy = (float)K[5];
  const float hH = (float)H / 2.0f, hW = (float)W / 2.0f;
  const long plane = (long)IH * (long)IW;
  double sums[256];
  for (int row = 0; row < H; ++row)
    for (int col = 0; col < W; ++col) {
      const long j = (long)row * W + col;
      if (!m->valid[j]) continue; /* only cells with an elevation are candidates */
      /* a11: cell centre at its elevation, relative to the map centre (D13) */
      const float xc = ((float)row + 0.5f - hH) * m->res;
      const float yc = ((float)col + 0.5f - hW) * m->res;
      const float dx = xc - tx, dy = yc - ty, dz = m->h[j] - tz;
      /* p_c = R^T (p - t) (D17) */
      const float pcx = (Rf[0] * dx + Rf[3] * dy) + Rf[6] * dz;
      const float pcy = (Rf[1] * dx + Rf[4] * dy) + Rf[7] * dz;
      const float pcz = (Rf[2] * dx + Rf[5] * dy) + Rf[8] * dz;
      if (!(pcz > 1e-6f)) continue; /* behind the camera */
      const float ux = pcx / pcz, uy = pcy / pcz;
      const float u = (fx * ux + sk * uy) + ccx; /* pinhole */
      const float v = fy * uy + ccy;
      const float fu = floorf(u + 0.5f), fv = floorf(v + 0.5f); /* nearest pixel (D16) */
      if (!(0.0f <= fu && fu < (float)IW && 0.0f <= fv && fv < (float)IH)) continue; /* frustum */
      if (m->occlusion && !om_visible(m, row, col, tx, ty, tz, m->h[j])) continue; /* NEXT-1 */
      const long pix = (long)(int)fv * IW + (long)(int)fu;
      /* a12: sample the bound channels and fuse with N_j = 1 (D21) */
      for (int b = 0; b < nb; ++b) {
        om_group *g = &m->g[bind[b].group];
        const float *ch = img + (long)bind[b].ch_offset * plane + pix;
        float dense[257];
        long step = plane;
        if (bind[b].topk > 0) { /* NEXT-2: expand the top-k pairs first (D38) */
          if (!expand_topk(ch, plane, bind[b].topk, g->nch, dense)) continue;
          ch = dense;
          step = 1;
        }
        const int width = bind[b].topk > 0 ? g->nch : bind[b].n_ch;
        int finite = 1;
        for (int k = 0; k < width; ++k) finite &= isfinite(ch[(long)k * step]) ? 1 : 0;
        if (!finite) continue;
        for (int k = 0; k < width; ++k) sums[k] = (double)ch[(long)k * step];
        switch (g->rule) {
          case OM_AVERAGE:
          case OM_CLASS_AVERAGE:
          case OM_COLOR: fuse_average(g, j, cells, 1, sums); break;
          case OM_GAUSSIAN: fuse_gaussian(g, j, cells, 1, sums); break;
          case OM_CLASS_BAYESIAN: fuse_dirichlet(g, j, cells, sums); break;
          case OM_CLASS_MAX: store_class_max(g, j, class_max_key(ch, g->nch, step)); break;
        }
      }
    }
  return OM_OK;
}

/* ---- move_to: a13 as a NAIVE COPY INTO A NEW MAP (D14) ---- */
int om_move_to(om_map *m, double x, double y) {
  if (!isfinite(x) || !isfinite(y)) return OM_EINVAL;
  const long long kx = (long long)floor(x / (double)m->res + 0.5);
  const long long ky = (long long)floor(y / (double)m->res + 0.5);
  const long long sr = kx - m->kx, sc = ky - m->ky;
  const long cells = ncells(m);
  /* deep copy of the old layers */
  float *oh = malloc(sizeof(float) * cells), *os2 = malloc(sizeof(float) * cells);
  unsigned char *ov = malloc(cells);
  memcpy(oh, m->h, sizeof(float) * cells); memcpy(os2, m->s2, sizeof(float) * cells);
  memcpy(ov, m->valid, cells);
  float *oval[32]; int *olab[32]; unsigned char *oobs[32];
  for (int gi = 0; gi < m->ng; ++gi) {
    om_group *g = &m->g[gi];
    long nv = (long)nval_of(g->rule, g->nch) * cells;
    oval[gi] = malloc(sizeof(float) * nv); memcpy(oval[gi], g->val, sizeof(float) * nv);
    olab[gi] = NULL;
    if (g->label) { olab[gi] = malloc(sizeof(int) * cells); memcpy(olab[gi], g->label, sizeof(int) * cells); }
    oobs[gi] = malloc(cells); memcpy(oobs[gi], g->observed, cells);
  }
  /* new map: every cell reset, then copy the cells whose footprint stays in the window.
     New logical row i covers the old logical row i + sr (moving +x scrolls rows down). */
  for (long j = 0; j < cells; ++j) reset_cell(m, j);
  for (long long i = 0; i < m->rows; ++i)
    for (long long c = 0; c < m->cols; ++c) {
      const long long oi = i + sr, oc = c + sc;
      if (oi < 0 || oi >= m->rows || oc < 0 || oc >= m->cols) continue;
      const long dst = (long)(i * m->cols + c), src = (long)(oi * m->cols + oc);
      m->h[dst] = oh[src]; m->s2[dst] = os2[src]; m->valid[dst] = ov[src];
      for (int gi = 0; gi < m->ng; ++gi) {
        om_group *g = &m->g[gi];
        for (int k = 0; k < nval_of(g->rule, g->nch); ++k)
          g->val[(long)k * cells + dst] = oval[gi][(long)k * cells + src];
        if (g->label) g->label[dst] = olab[gi][src];
        g->observed[dst] = oobs[gi][src];
      }
    }
  m->kx = kx; m->ky = ky;
  free(oh); free(os2); free(ov);
  for (int gi = 0; gi < m->ng; ++gi) { free(oval[gi]); free(olab[gi]); free(oobs[gi]); }
  return OM_OK;
}

/* ---- layers by name (SURVEY §8(b) naming) ---- */
typedef struct { int kind; int group; int k; } om_layer_ref;
enum { L_ELEV, L_VAR, L_VALID, L_VAL, L_THETA, L_LABEL, L_OBS };

static int parse_int_suffix(const char *s, int *k) {
  if (!*s) return 0;
  int v = 0;
  for (const char *c = s; *c; ++c) { if (*c < '0' || *c > '9') return 0; v = v * 10 + (*c - '0'); }
  *k = v;
  return 1;
}

static int find_layer(const om_map *m, const char *name, om_layer_ref *ref) {
  if (!strcmp(name, "elevation")) { ref->kind = L_ELEV; return 1; }
  if (!strcmp(name, "variance")) { ref->kind = L_VAR; return 1; }
  if (!strcmp(name, "valid")) { ref->kind = L_VALID; return 1; }
  for (int gi = 0; gi < m->ng; ++gi) {
    const om_group *g = &m->g[gi];
    size_t L = strlen(g->name);
    if (strncmp(name, g->name, L)) continue;
    const char *s = name + L;
    ref->group = gi;
    int k;
    if (g->rule == OM_CLASS_MAX) {
      if (!strcmp(s, "_label")) { ref->kind = L_LABEL; return 1; }
      if (!strcmp(s, "_conf")) { ref->kind = L_VAL; ref->k = 0; return 1; }
      continue;
    }
    if (!strcmp(s, "_observed")) { ref->kind = L_OBS; return 1; }
    if (g->rule == OM_COLOR) {
      if (!strcmp(s, "_r")) { ref->kind = L_VAL; ref->k = 0; return 1; }
      if (!strcmp(s, "_g")) { ref->kind = L_VAL; ref->k = 1; return 1; }
      if (!strcmp(s, "_b")) { ref->kind = L_VAL; ref->k = 2; return 1; }
      continue;
    }
    if (g->rule == OM_GAUSSIAN) {
      if (g->nch == 1 && !strcmp(s, "")) { ref->kind = L_VAL; ref->k = 0; return 1; }
      if (g->nch == 1 && !strcmp(s, "_var")) { ref->kind = L_VAL; ref->k = 1; return 1; }
      if (g->nch > 1 && s[0] == '_' && parse_int_suffix(s + 1, &k) && k < g->nch) { ref->kind = L_VAL; ref->k = k; return 1; }
      if (g->nch > 1 && !strncmp(s, "_var_", 5) && parse_int_suffix(s + 5, &k) && k < g->nch) {
        ref->kind = L_VAL; ref->k = g->nch + k; return 1;
      }
      continue;
    }
    if (g->rule == OM_CLASS_BAYESIAN) {
      if (!strncmp(s, "_alpha_", 7) && parse_int_suffix(s + 7, &k) && k < g->nch) { ref->kind = L_VAL; ref->k = k; return 1; }
      if (s[0] == '_' && parse_int_suffix(s + 1, &k) && k < g->nch) { ref->kind = L_THETA; ref->k = k; return 1; }
      continue;
    }
    /* average / class_average */
    if (g->nch == 1 && !strcmp(s, "")) { ref->kind = L_VAL; ref->k = 0; return 1; }
    if (g->nch > 1 && s[0] == '_' && parse_int_suffix(s + 1, &k) && k < g->nch) { ref->kind = L_VAL; ref->k = k; return 1; }
  }
  return 0;
}

int om_get_layer(const om_map *m, const char *name, float *out) {
  om_layer_ref r;
  if (!find_layer(m, name, &r)) return OM_ENOTFOUND;
  const long cells = ncells(m);
  for (long j = 0; j < cells; ++j) {
    float v = 0.0f;
    switch (r.kind) {
      case L_ELEV: v = m->valid[j] ? m->h[j] : NAN; break;
      case L_VAR: v = m->valid[j] ? m->s2[j] : NAN; break;
      case L_VALID: v = (float)m->valid[j]; break;
      case L_VAL: v = m->g[r.group].val[(long)r.k * cells + j]; break;
      case L_LABEL: v = (float)m->g[r.group].label[j]; break;
      case L_OBS: v = (float)m->g[r.group].observed[j]; break;
      case L_THETA: {
        /* Eq.(11) posterior mean theta = alpha / sum(alpha), derived at readout (D5) */
        const om_group *g = &m->g[r.group];
        if (!g->observed[j]) { v = 0.0f; break; }
        double tot = 0.0;
        for (int k = 0; k < g->nch; ++k) tot += (double)g->val[(long)k * cells + j];
        v = (float)((double)g->val[(long)r.k * cells + j] / tot);
        break;
      }
    }
    out[j] = v;
  }
  return OM_OK;
}

/* state injection for single-step parity: derived layers are read-only */
int om_set_layer(om_map *m, const char *name, const float *src) {
  om_layer_ref r;
  if (!find_layer(m, name, &r)) return OM_ENOTFOUND;
  if (r.kind == L_THETA) return OM_EINVAL;
  const long cells = ncells(m);
  for (long j = 0; j < cells; ++j) {
    switch (r.kind) {
      case L_ELEV: m->h[j] = src[j]; break;
      case L_VAR: m->s2[j] = src[j]; break;
      case L_VALID: m->valid[j] = src[j] != 0.0f; break;
      case L_VAL: m->g[r.group].val[(long)r.k * cells + j] = src[j]; break;
      case L_LABEL: m->g[r.group].label[j] = (int)src[j]; break;
      case L_OBS: m->g[r.group].observed[j] = src[j] != 0.0f; break;
    }
  }
  return OM_OK;
}

void om_get_stats(const om_map *m, unsigned long long out[8]) { memcpy(out, m->stats, sizeof m->stats); }
void om_get_center(const om_map *m, long long out[2]) { out[0] = m->kx; out[1] = m->ky; }

/* ---- PCA readout of a feature group (reading D28) ----
 * Over the cells where the group is observed: mean mu and covariance
 * C = (1/n) sum (x - mu)(x - mu)^T in fp64 (plain loops); eigenvectors by power iteration
 * with deflation in long double (the library uses a different solver); each component's
 * sign makes its largest-|coefficient| positive (D25); projections p = (x - mu) . e in fp64;
 * min-max scaled to [0, 1] over the observed cells, 0 when max == min;
 * unobserved cells and components beyond the rank get 0. out: k x rows x cols. */
int om_pca_readout(const om_map *m, const char *group, int k, float *out) {
  int gi = -1;
  for (int i = 0; i < m->ng; ++i)
    if (!strcmp(m->g[i].name, group)) gi = i;
  if (gi < 0) return OM_ENOTFOUND;
  const om_group *g = &m->g[gi];
  if (!(g->rule == OM_AVERAGE || g->rule == OM_CLASS_AVERAGE || g->rule == OM_GAUSSIAN) || k < 1) return OM_EINVAL;
  const int d = g->nch;
  const long cells = ncells(m);
  double *mu = calloc(d, sizeof(double)), *C = calloc((size_t)d * d, sizeof(double));
  long n = 0;
  for (long j = 0; j < cells; ++j) {
    if (!g->observed[j]) continue;
    ++n;
    for (int a = 0; a < d; ++a) mu[a] += (double)g->val[(long)a * cells + j];
  }
  for (long j = 0; j < (long)k * cells; ++j) out[j] = 0.0f;
  if (n == 0) { free(mu); free(C); return OM_OK; }
  for (int a = 0; a < d; ++a) mu[a] /= (double)n;
  for (long j = 0; j < cells; ++j) {
    if (!g->observed[j]) continue;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b)
        C[a * d + b] += ((double)g->val[(long)a * cells + j] - mu[a]) * ((double)g->val[(long)b * cells + j] - mu[b]);
  }
  for (int a = 0; a < d * d; ++a) C[a] /= (double)n;
  long double *A = malloc(sizeof(long double) * d * d), *v = malloc(sizeof(long double) * d),
              *w = malloc(sizeof(long double) * d);
  for (int a = 0; a < d * d; ++a) A[a] = C[a];
  double *comp = calloc((size_t)k * d, sizeof(double));
  long double lam_max = 0.0L;
  for (int c = 0; c < k && c < d; ++c) {
    for (int a = 0; a < d; ++a) v[a] = 1.0L / sqrtl((long double)d) + (long double)a * 1e-3L;
    long double lam = 0.0L;
    for (int it = 0; it < 200000; ++it) {
      long double nrm = 0.0L;
      for (int a = 0; a < d; ++a) {
        w[a] = 0.0L;
        for (int b = 0; b < d; ++b) w[a] += A[a * d + b] * v[b];
        nrm += w[a] * w[a];
      }
      nrm = sqrtl(nrm);
      if (nrm == 0.0L) { lam = 0.0L; break; }
      long double diff = 0.0L;
      for (int a = 0; a < d; ++a) { const long double x = w[a] / nrm; diff += fabsl(x - v[a]); v[a] = x; }
      lam = nrm;
      if (diff < 1e-16L) break;
    }
    if (c == 0) lam_max = lam;
    /* rank exhausted: components with lambda <= 1e-12 lambda_max stay 0 */
    if (lam <= 0.0L || lam <= 1e-12L * lam_max) break;
    int big = 0;
    for (int a = 1; a < d; ++a) if (fabsl(v[a]) > fabsl(v[big])) big = a;
    const long double sg = v[big] < 0.0L ? -1.0L : 1.0L;
    for (int a = 0; a < d; ++a) comp[(long)c * d + a] = (double)(sg * v[a]);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) A[a * d + b] -= lam * v[a] * v[b];
  }
  for (int c = 0; c < k; ++c) {
    double lo = INFINITY, hi = -INFINITY;
    for (int pass = 0; pass < 2; ++pass)
      for (long j = 0; j < cells; ++j) {
        if (!g->observed[j]) continue;
        double p = 0.0;
        for (int a = 0; a < d; ++a) p += ((double)g->val[(long)a * cells + j] - mu[a]) * comp[(long)c * d + a];
        if (pass == 0) { if (p < lo) lo = p; if (p > hi) hi = p; }
        else out[(long)c * cells + j] = hi > lo ? (float)((p - lo) / (hi - lo)) : 0.0f;
      }
  }
  free(mu); free(C); free(A); free(v); free(w); free(comp);
  return OM_OK;
}

/* ---- NEXT-3 post-processing plugins on the fused map (Table II
 * rows "normal calculation", "traversability"; readings D35-D37) ---- */

/* gradient of the elevation along one axis at a valid cell: central difference when both
 * neighbours are valid, one-sided with the valid one otherwise; 0 = no valid neighbour */
static int om_grad(const om_map *m, int i, int j, int di, int dj, float *g) {
  const int H = m->rows, W = m->cols;
  const long c = (long)i * W + j;
  const int ip = i + di, jp = j + dj, im = i - di, jm = j - dj;
  const int vp = ip >= 0 && ip < H && jp >= 0 && jp < W && m->valid[(long)ip * W + jp];
  const int vm = im >= 0 && im < H && jm >= 0 && jm < W && m->valid[(long)im * W + jm];
  if (vp && vm) *g = (m->h[(long)ip * W + jp] - m->h[(long)im * W + jm]) / (2.0f * m->res);
  else if (vp) *g = (m->h[(long)ip * W + jp] - m->h[c]) / m->res;
  else if (vm) *g = (m->h[c] - m->h[(long)im * W + jm]) / m->res;
  else return 0;
  return 1;
}

/* unit normal (-gx, -gy, 1)/|.| of a cell (x = rows, y = cols, D13); 0 = invalid output */
static int om_normal(const om_map *m, int i, int j, float n[3]) {
  const long c = (long)i * m->cols + j;
  float gx, gy;
  if (!m->valid[c] || !om_grad(m, i, j, 1, 0, &gx) || !om_grad(m, i, j, 0, 1, &gy)) return 0;
  const float norm = sqrtf((gx * gx + gy * gy) + 1.0f);
  n[0] = -gx / norm;
  n[1] = -gy / norm;
  n[2] = 1.0f / norm;
  return 1;
}

/* out: 3 x rows x cols (normal_x, normal_y, normal_z), NaN where invalid */
int om_plugin_normals(const om_map *m, float *out) {
  const long cells = ncells(m);
  for (int i = 0; i < m->rows; ++i)
    for (int j = 0; j < m->cols; ++j) {
      const long c = (long)i * m->cols + j;
      float n[3];
      if (!om_normal(m, i, j, n)) n[0] = n[1] = n[2] = NAN;
      for (int k = 0; k < 3; ++k) out[(long)k * cells + c] = n[k];
    }
  return OM_OK;
}

/* score = clamp(min(slope, step), 0, 1), slope = (n_z - cos_max) / (1 - cos_max),
 * step = 1 - max |h_nb - h| / step_max over the valid 8-neighbours (D36); NaN where invalid.
 * cos_max = cos(slope_max) rounded once to fp32 by the caller. */
int om_plugin_traversability(const om_map *m, float cos_max, float step_max, float *out) {
  if (!(step_max > 0.0f) || !(cos_max < 1.0f)) return OM_EINVAL;
  const int H = m->rows, W = m->cols;
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < W; ++j) {
      const long c = (long)i * W + j;
      float n[3];
      if (!om_normal(m, i, j, n)) { out[c] = NAN; continue; }
      const float slope = (n[2] - cos_max) / (1.0f - cos_max);
      float mx = 0.0f;
      for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj) {
          const int a = i + di, b = j + dj;
          if ((di == 0 && dj == 0) || a < 0 || a >= H || b < 0 || b >= W || !m->valid[(long)a * W + b]) continue;
          const float d = fabsf(m->h[(long)a * W + b] - m->h[c]);
          if (d > mx) mx = d;
        }
      const float step = 1.0f - mx / step_max;
      float s = slope < step ? slope : step;
      s = s < 0.0f ? 0.0f : s;
      out[c] = s > 1.0f ? 1.0f : s;
    }
  return OM_OK;
}

/* per cell argmax of the group's class probabilities theta (class_bayesian: alpha / sum alpha
 * as read out; class_average: the stored values; class_max: its label/conf), ties to the
 * lowest class (D37); out: 2 x rows x cols (class_id, confidence), -1 / 0 where unobserved */
int om_plugin_semantic_argmax(const om_map *m, const char *group, float *out) {
  int gi = -1;
  for (int k = 0; k < m->ng; ++k) if (!strcmp(m->g[k].name, group)) gi = k;
  if (gi < 0) return OM_ENOTFOUND;
  const om_group *g = &m->g[gi];
  if (g->rule != OM_CLASS_BAYESIAN && g->rule != OM_CLASS_AVERAGE && g->rule != OM_CLASS_MAX) return OM_ERULE;
  const long cells = ncells(m);
  for (long c = 0; c < cells; ++c) {
    float id = -1.0f, conf = 0.0f;
    if (g->rule == OM_CLASS_MAX) {
      if (g->label[c] >= 0) { id = (float)g->label[c]; conf = g->val[c]; }
    } else if (g->observed[c]) {
      double tot = 0.0;
      if (g->rule == OM_CLASS_BAYESIAN)
        for (int k = 0; k < g->nch; ++k) tot += (double)g->val[(long)k * cells + c];
      for (int k = 0; k < g->nch; ++k) {
        const float th = g->rule == OM_CLASS_BAYESIAN ? (float)((double)g->val[(long)k * cells + c] / tot)
                                                      : g->val[(long)k * cells + c];
        if (k == 0 || th > conf) { conf = th; id = (float)k; }
      }
    }
    out[c] = id;
    out[cells + c] = conf;
  }
  return OM_OK;
}
