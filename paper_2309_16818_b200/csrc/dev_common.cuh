// dev_common.cuh -- device helpers shared by the kernels: PDL, streaming loads, strip test, cell reset.
// Part of the single translation unit kernels.cu (included inside namespace memk, in order).
#pragma once

// ---------------------------------------------------------------- programmatic dependent launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- memory helpers
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long evict_last_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 16-byte store with an L2 eviction-priority policy
__device__ __forceinline__ void st_hint_u64x2(void *p, unsigned long long x, unsigned long long y,
                                              unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(p), "l"(x), "l"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint_u64(void *p, unsigned long long x, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ float ld_hint_f32(const float *p, unsigned long long pol) {
  float r;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}
// read-once point data: no L1 allocation, evict-first in L2 so the scratch of the maps in
// flight keeps its L2 residency
__device__ __forceinline__ float4 ld_stream_f4(const float *p, unsigned long long pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
// branch-free: |x| < inf is false exactly for +-inf and NaN
__device__ __forceinline__ bool finite3(float a, float b, float c) {
  return (fabsf(a) < INFINITY) & (fabsf(b) < INFINITY) & (fabsf(c) < INFINITY);
}

__device__ __forceinline__ int stat_slot(int code) {
  // mem_stats order: n_input, nonfinite, range, height, oob, inlier, outlier, touched
  return code == MEM_CODE_INLIER ? 5 : code == MEM_CODE_OUTLIER ? 6 : code - 1;
}

// is logical cell (row, col) in the strips that scrolled in with the pending shift (D14)?
template <class F>
__device__ __forceinline__ bool in_strip(int row, int col, const F &f, const Geometry &g) {
  if (f.sr == 0 && f.sc == 0) return false;
  const int ar = f.sr < 0 ? -f.sr : f.sr, ac = f.sc < 0 ? -f.sc : f.sc;
  if (ar >= g.H || ac >= g.W) return true;
  const bool rs = f.sr > 0 ? row >= g.H - f.sr : row < -f.sr;
  const bool cs = f.sc > 0 ? col >= g.W - f.sc : col < -f.sc;
  return rs || cs;
}

// the state of a never-observed cell (D15)
__device__ __forceinline__ void reset_cell(const State &st, long long BHW, long long cell, const ResetInfo &r) {
  float *vals = reinterpret_cast<float *>(st.words);
  vals[(long long)kWordElev * BHW + cell] = __int_as_float(0x7fc00000);
  vals[(long long)kWordVar * BHW + cell] = __int_as_float(0x7fc00000);
  for (int w = 2; w < r.n_word; ++w) st.words[(long long)w * BHW + cell] = 0u;
  for (int l = 0; l < r.n_label; ++l) reinterpret_cast<int *>(st.words)[(long long)r.label_word[l] * BHW + cell] = -1;
  for (int fl = 0; fl < r.n_flag; ++fl) st.flags[(long long)fl * BHW + cell] = 0;
}

// per-lane code counters packed in one u64: 10 bits per code, flushed before they can wrap
__device__ __forceinline__ void count_code(unsigned long long &packed, unsigned &n, int code, unsigned (&cnt)[8]) {
  if (code >= 0) packed += 1ull << (10 * code);
  if (++n == 1000u) {
#pragma unroll
    for (int c = 0; c < 6; ++c) cnt[stat_slot(c)] += (unsigned)(packed >> (10 * c)) & 1023u;
    packed = 0ull;
    n = 0;
  }
}

// per-CTA counters: warp reduce, one smem add per warp, one global add per counter
__device__ __forceinline__ void flush_stats(unsigned *s_cnt, const unsigned (&cnt)[8], unsigned long long *out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const unsigned v = __reduce_add_sync(0xffffffffu, cnt[c]);
    if (lane == 0 && v) atomicAdd(&s_cnt[c], v);
  }
  __syncthreads();
  if (threadIdx.x < 8 && s_cnt[threadIdx.x])
    atomicAdd(&out[(blockIdx.x % kStatSlots) * 8 + threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// ---------------------------------------------------------------- bulk copy (TMA) / mbarrier PTX
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// global -> shared bulk copy (16-B aligned, size a multiple of 16) completing on an mbarrier
__device__ __forceinline__ void bulk_load(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000000)
        : "memory");
  } while (!ok);
}

// block-wide exclusive scan of one value per thread; returns the prefix, *total the sum
template <int kT>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned *s_part, unsigned *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  __syncthreads();  // s_part may still be read by a previous scan
  if (lane == 31) s_part[wid] = incl;
  __syncthreads();
  unsigned wpre = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    const unsigned p = s_part[w];
    wpre += w < wid ? p : 0u;
    tot += p;
  }
  *total = tot;
  return wpre + incl - v;
}

