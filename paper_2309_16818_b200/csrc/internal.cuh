// internal.cuh -- device-side data layout and per-cell fusion math of libmem (sm_100a).
//
// Layout in HBM: one allocation per kind, layer-major, map-major, then the
// PHYSICAL (ring-buffered) row-major cell index:
//   words [n_word_layers][n_maps][rows*cols]  fp32 layers (elevation, variance, group values)
//                                               and int32 class_max labels
//   flags [n_flag_layers][n_maps][rows*cols]  u8 (valid, per-group observed)
//   acc   scratch pool of per-frame sufficient statistics for the maps in flight: counts
//         [slots][rows*cols] then records [slots][rows*cols][R] (zero between frames;
//         k_cells re-zeroes what it reads)
// Logical cell (i, j) of map m lives at physical ((i + r0[m]) % rows, (j + c0[m]) % cols).
//
// Numerics (reading D29): the library is compiled with -fmad=false (no FFMA/DFMA
// contraction), IEEE division and sqrt, no FTZ; every fp32 op below is in the order
// DESIGN.md §3 states, every per-cell closed form in fp64 rounded once to fp32.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mem.h"

namespace memk {

constexpr int kMaxGroups = 32;
constexpr int kMaxBind = 16;
constexpr int kMaxCh = 256;

// word layers 0, 1 and flag layer 0 are the base layers
constexpr int kWordElev = 0;
constexpr int kWordVar = 1;
constexpr int kFlagValid = 0;
// per-cell scratch: a count array (SoA, u64 n_in | n_out << 32, scanned
// densely) and one AoS record of R u64 words per cell, so a touched cell's sums share one
// or two 32-B sectors.  Record words 0, 1 are the height statistics:
constexpr int kRecP = 0;    // f64: sum 1/v over inliers
constexpr int kRecS = 1;    // f64: sum z/v over inliers
// colour RED path: count-word fields b (25 bits) | n (18) | n_out (18) hold any cell of a map of
// at most this many points per call (b <= 255 n < 2^25); larger maps take the sort path
constexpr long long kColourMaxPts = 131586;

struct GroupDesc {
  int rule, nch;
  float w, sf2, mu0, s02, a0;
  int word0;  // first word layer (theta / mu then var / alpha / conf)
  int label;  // word layer of class_max labels, -1 otherwise
  int flag;   // observed flag layer, -1 for class_max
  int acc0;   // first record word (average etc.: n then nch sums; color: r|g<<32, b|n<<32; class_max: key)
};

struct BindDesc {  // one binding of a call, resolved against its group
  int ch_offset, nch, group;
  int topk;  // > 0: nch = 2 topk (id, p) pairs expanding to the group's K + 1 classes (D38)
  GroupDesc g;
};

struct __align__(16) PointFrame {  // per-map frame of a point input (64 B)
  float R[9];      // sensor->map rotation (fp32 of the host doubles)
  float t[3];      // t.xy relative to the map centre (fp64 subtraction, then fp32), t.z
  int sr, sc;      // pending (lazy) shift of the preceding mem_move_to: strips to reset first
  int r0, c0;      // ring offsets after that shift
};

struct __align__(16) MapFrame {  // per-map, per-call point/image frame parameters (16-B aligned: vector loads)
  float R[9];      // sensor->map rotation (fp32 of the host doubles)
  float t[3];      // t.xy relative to the map centre (fp64 subtraction, then fp32), t.z
  float K[5];      // images: fx, skew, cx, fy, cy
  int sr, sc;      // pending (lazy) shift of the preceding mem_move_to: strips to reset first
  int r0, c0;      // ring offsets after that shift
};

struct ShiftRec {  // per-map shift of one move_to call
  int sr, sc;      // lattice deltas (clamped to +-size: |s| >= size resets all)
  int r0, c0;      // ring offsets AFTER the move
};

struct Geometry {
  int H, W;
  int HW;
  int n_maps;
  long long BHW;  // n_maps * HW: stride between layers (< 2^31, so cell indices fit in int)
  float res, hH, hW;
  double inv_W;   // 1.0 / W for divmod_w (index arithmetic only)
};

struct State {
  uint32_t *words;
  uint8_t *flags;
  unsigned long long *acc;
};

// ---------------------------------------------------------------- indexing
__device__ __forceinline__ int wrap(int v, int n) { return v >= n ? v - n : v; }

// q = x / d, r = x % d for 0 <= x < 2^31, d >= 1 without the integer-division sequence: the
// fp64 product x * (1/d) is within 2^-21 of x/d, so the truncated quotient is off by at most
// one and one correction step makes it exact.
__device__ __forceinline__ int divmod_fast(int x, int d, double inv_d, int &r) {
  int q = (int)((double)x * inv_d);
  r = x - q * d;
  if (r < 0) { --q; r += d; }
  else if (r >= d) { ++q; r -= d; }
  return q;
}

// ---------------------------------------------------------------- class_max key (D19)
// order-preserving map of finite fp32 to u32, so that u64 atomicMax picks the largest conf,
// then the lowest class index (stored as K-1-k).
__device__ __forceinline__ uint32_t ord_f32(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float f32_of_ord(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// ---------------------------------------------------------------- a9: Kalman height (fp64)
// Information form of SURVEY §8(c) a9 / reading D7, in the oracle's exact expressions: prior
// variance inflated by the outliers first (D11), sp = s2 + n_out v_out; valid cell with
// inliers: den = 1/sp + P, h' = (h/sp + S)/den, s2' = 1/den; first touch h = S/P, s2 = 1/P.
// Returns true when the cell becomes valid.
__device__ __forceinline__ void kalman_height(float &h, float &s2, uint8_t &valid, double n_in, double n_out,
                                              double P, double S, float v_out) {
  if (valid) {
    const double sp = (double)s2 + n_out * (double)v_out;
    if (n_in > 0.0) {
      const double den = 1.0 / sp + P;
      h = __double2float_rn(((double)h / sp + S) / den);
      s2 = __double2float_rn(1.0 / den);
    } else {
      s2 = __double2float_rn(sp);
    }
  } else if (n_in > 0.0) {
    h = __double2float_rn(S / P);
    s2 = __double2float_rn(1.0 / P);
    valid = 1;
  }
}

// ---------------------------------------------------------------- per-cell rules (fp64)
// Eq.(1)+(2): a = sum/n; theta' = w a + (1-w) theta; first touch theta' = a (D3)
__device__ __forceinline__ float rule_average(float theta, bool observed, double sum, double n, float w) {
  const double a = sum / n;
  const double wd = (double)w;
  const double out = observed ? wd * a + (1.0 - wd) * (double)theta : a;
  return __double2float_rn(out);
}

// Eq.(6)-(7): prior (mu_p, s2_p) = current posterior, or (mu0, sigma0^2) on first touch (D4)
__device__ __forceinline__ void rule_gaussian(float &mu, float &var, bool observed, double sum, double n,
                                              const GroupDesc &g) {
  const double mu_p = observed ? (double)mu : (double)g.mu0;
  const double s2_p = observed ? (double)var : (double)g.s02;
  const double sf2 = (double)g.sf2;
  const double mu_ml = sum / n;
  const double ns2 = n * s2_p;
  const double den = ns2 + sf2;
  mu = __double2float_rn((sf2 / den) * mu_p + (ns2 / den) * mu_ml);
  var = __double2float_rn((sf2 * s2_p) / den);
}

// Eq.(12): alpha' = alpha (or alpha0 on first touch, D6) + sum m
__device__ __forceinline__ float rule_dirichlet(float alpha, bool observed, double sum, float a0) {
  const double prior = observed ? (double)alpha : (double)a0;
  return __double2float_rn(prior + sum);
}

// Applies group g's rule to physical cell `cell` (global index m*HW + phys) given the frame's
// count n and a per-channel sum accessor.  class_max takes the frame's winning key instead.
template <class SumFn>
__device__ __forceinline__ void apply_group(const State &st, long long BHW, long long cell, const GroupDesc &g,
                                            double n, SumFn sum_of, unsigned long long key) {
  float *vals = reinterpret_cast<float *>(st.words);
  if (g.rule == MEM_CLASS_MAX) {
    const int k = g.nch - 1 - (int)(uint32_t)(key & 0xffffffffull);
    reinterpret_cast<int *>(st.words)[(long long)g.label * BHW + cell] = k;
    vals[(long long)g.word0 * BHW + cell] = f32_of_ord((uint32_t)(key >> 32));
    return;
  }
  uint8_t *obs = st.flags + (long long)g.flag * BHW + cell;
  const bool observed = *obs != 0;
  switch (g.rule) {
    case MEM_AVERAGE:
    case MEM_CLASS_AVERAGE:
    case MEM_COLOR:
      for (int k = 0; k < g.nch; ++k) {
        float *th = vals + (long long)(g.word0 + k) * BHW + cell;
        *th = rule_average(*th, observed, sum_of(k), n, g.w);
      }
      break;
    case MEM_GAUSSIAN:
      for (int k = 0; k < g.nch; ++k) {
        float *mu = vals + (long long)(g.word0 + k) * BHW + cell;
        float *var = vals + (long long)(g.word0 + g.nch + k) * BHW + cell;
        float m = *mu, v = *var;
        rule_gaussian(m, v, observed, sum_of(k), n, g);
        *mu = m;
        *var = v;
      }
      break;
    case MEM_CLASS_BAYESIAN:
      for (int k = 0; k < g.nch; ++k) {
        float *al = vals + (long long)(g.word0 + k) * BHW + cell;
        *al = rule_dirichlet(*al, observed, sum_of(k), g.a0);
      }
      break;
    default:
      break;
  }
  *obs = 1;
}

}  // namespace memk
