// Small device helpers shared by the libwl kernels (sm_100a).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace wl {

// 16-byte vector type of T
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int n = 2;
};

template <typename T>
__device__ __forceinline__ void vec_split(const typename Vec16<T>::type &v, T *out);
template <>
__device__ __forceinline__ void vec_split<float>(const float4 &v, float *o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void vec_split<double>(const double2 &v, double *o) {
  o[0] = v.x; o[1] = v.y;
}
template <typename T>
__device__ __forceinline__ typename Vec16<T>::type vec_make(const T *i);
template <>
__device__ __forceinline__ float4 vec_make<float>(const float *i) { return make_float4(i[0], i[1], i[2], i[3]); }
template <>
__device__ __forceinline__ double2 vec_make<double>(const double *i) { return make_double2(i[0], i[1]); }

// Source index of extended position p under the infinite half-point symmetric extension
// (P:82 applied repeatedly): ..., y[1], y[0] | y[0], ..., y[n-1] | y[n-1], y[n-2], ...
__device__ __forceinline__ int refl_inf(int p, int n) {
  if (p >= 0 && p < n) return p;
  if (p < 0 && p >= -n) return -1 - p;  // single reflections (the only ones a plan with n >= h needs)
  if (p >= n && p < 2 * n) return 2 * n - 1 - p;
  const int m = 2 * n;
  p %= m;
  if (p < 0) p += m;
  return p < n ? p : m - 1 - p;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async 16 bytes global -> shared (L2 only, no L1 allocation)
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>  // wait until at most N committed cp.async groups are still pending
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Smallest pitch (elements) >= n whose size in 4-byte words is 4 mod 8: 8 rows read with
// 16-byte loads at the same column then hit 8 distinct 4-bank groups (conflict-free).
template <typename T>
constexpr int conflict_free_pitch(int n) {
  int words_per = (int)sizeof(T) / 4;
  int p = n;
  while (((p * words_per) % 8) != 4) p++;
  return p;
}

constexpr int round_up_c(int v, int a) { return (v + a - 1) / a * a; }

// Smallest row length (elements, a multiple of the 16-byte vector) >= n whose size in 4-byte words
// is 4 mod 8: 16-byte accesses of 8 consecutive rows at one column hit 8 distinct 4-bank groups.
template <typename T>
constexpr int bank_pad(int n) {
  const int vec = 16 / (int)sizeof(T);
  int p = round_up_c(n, vec);
  while (((p * (int)sizeof(T) / 4) % 8) != 4) p += vec;
  return p;
}

// Packed pair arithmetic: float2 maps to FFMA2 / FADD2 (sm_100a), double2 to two FMAs.
template <typename T>
struct Pair;
template <>
struct Pair<float> {
  using t = float2;
};
template <>
struct Pair<double> {
  using t = double2;
};
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ double2 mul2(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <typename P>
__device__ __forceinline__ P zero2() {
  P z;
  z.x = 0;
  z.y = 0;
  return z;
}
template <typename P, typename T>
__device__ __forceinline__ P splat2(T v) {
  P z;
  z.x = v;
  z.y = v;
  return z;
}

}  // namespace wl

namespace wl {

// Structural zeros of the filter pair: the nonzero tap range [l0, l1) of the lowpass
// and [h0, h1) of the highpass array of the L-tap frame.  ZV = 0: every tap; the CDF 9/7 frame
// (reading R4: a_lo = [0, h9], d_lo = [0, 0, h7, 0], unified highpass rule) has zeros at both ends.
template <int L, int ZV>
struct TapRange {
  static constexpr int l0 = 0, l1 = L, h0 = 0, h1 = L;
};
template <>
struct TapRange<10, 1> {  // dual filters (d_lo, d_hi): W* and W
  static constexpr int l0 = 2, l1 = 9, h0 = 0, h1 = 9;
};
template <>
struct TapRange<10, 2> {  // analysis filters (a_lo, a_hi): W-dagger and (W-dagger)*
  static constexpr int l0 = 1, l1 = 10, h0 = 1, h1 = 8;
};

}  // namespace wl

// ---------------------------------------------------------------- mbarrier + TMA (sm_90+)
namespace wl {

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WL_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WL_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Programmatic dependent launch: let the next kernel in the stream start its prologue now;
// wait until the previous kernel's results are visible before touching global memory.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Order this thread's earlier generic-proxy shared-memory accesses before later async-proxy
// (TMA) accesses of the same buffers.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 3-D tiled TMA load of one box into shared memory; completion is signalled on `bar`.
__device__ __forceinline__ void tma_load_3d(void *dst, const void *tmap, uint64_t *bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// L2 eviction-priority policies and stores that carry one (PTX createpolicy / st.L2::cache_hint):
// a level's LL output is read by the next level right away, so it is stored evict_last; the final
// coefficients are not re-read by the chain.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(float2 *ptr, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(ptr), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2 *ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

// Grid-wide barrier of a cooperative launch (gpu-scope fence included).
__device__ __forceinline__ void grid_sync_all() { cooperative_groups::this_grid().sync(); }
// Order this thread's earlier generic-proxy accesses (any state space) before its later
// async-proxy (TMA) accesses: after a grid barrier, before TMA reads of data other CTAs stored.
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;\n" ::: "memory"); }

// 1-D bulk copy global -> shared (16-byte aligned, bytes % 16 == 0); completion on `bar`.
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

}  // namespace wl

// ---------------------------------------------------------------- persistent run map
namespace wl {

// Work decomposition of the streaming kernels: `ncols` columns ((image, strip) pairs, image
// major) of `span` rows, handed out as runs, one per resident CTA when the columns allow it.
//  * banded (bal = 0): each column is cut into bands; the first `extra` columns get nb_lo + 1
//    bands, the rest nb_lo, so the number of runs equals the resident CTAs while neighbouring
//    strips keep the same band boundaries (their halo columns stream through L2 together);
//  * balanced (bal = 1): the columns are laid end to end and cut into `nparts` runs of equal
//    row count (rounded to `align`); a run may continue from the bottom of one column into the
//    top of the next (each piece is a segment with its own priming).  With 132 columns on 444
//    CTAs the banded split leaves bands of 513 and 684 rows; the balanced one gives every CTA
//    the same work -- and measured far slower on B200 (cfg5 W* level 1 170 vs 108 us): strips
//    that stream different rows at the same time lose DRAM page locality.  A/B only.
// Iterate a CTA's segments with:  for (RunIter it(map); it.next(col, r0, r1);) { ... }
struct RunMap {
  int ncols, nb_lo, extra, span, align, bal, nparts;

  __host__ __device__ int nruns() const { return bal ? nparts : extra * (nb_lo + 1) + (ncols - extra) * nb_lo; }

  // banded: run -> (column, first row, end row) with rows in [0, span)
  __device__ __forceinline__ void get(int run, int &col, int &r0, int &r1) const {
    int band, nb;
    const int big = extra * (nb_lo + 1);
    if (run < big) {
      col = run / (nb_lo + 1);
      band = run - col * (nb_lo + 1);
      nb = nb_lo + 1;
    } else {
      const int r = run - big;
      col = extra + r / nb_lo;
      band = r - (col - extra) * nb_lo;
      nb = nb_lo;
    }
    int br = (span + nb - 1) / nb;
    br = (br + align - 1) / align * align;
    r0 = band * br;
    r1 = r0 + br < span ? r0 + br : span;
  }
  // balanced: first row boundary (a multiple of align, < span) at or after unit position s
  __device__ __forceinline__ void locate(long long s, int &col, int &row) const {
    const int units = (span + align - 1) / align;
    int c = (int)(s / units);
    int u = (int)(s - (long long)c * units);
    col = c;
    row = u * align;
  }
  // run -> segments [(col, r0), (ce, re)): (col, r0 .. span), (col + 1, 0 .. span), ..., (ce, 0 .. re)
  __device__ __forceinline__ void bounds(int run, int &col, int &r0, int &ce, int &re) const {
    if (!bal) {
      get(run, col, r0, re);
      ce = col;
      return;
    }
    const long long T = (long long)ncols * ((span + align - 1) / align);
    locate(T * run / nparts, col, r0);
    locate(T * (run + 1) / nparts, ce, re);
  }

  // host: banded split so that nruns() == resident when the columns allow it, bands >= min_rows;
  // balanced: min(resident, ncols * span / min_rows) runs
  static RunMap make(long long ncols, int span, long long resident, int min_rows, int align, bool balanced = false) {
    RunMap m;
    m.ncols = (int)ncols;
    m.span = span;
    m.align = align > 0 ? align : 1;
    m.bal = 0;
    m.nparts = 0;
    const int mr = min_rows > 0 ? min_rows : 1;
    const int max_nb = span / mr > 1 ? span / mr : 1;
    if (ncols >= resident) {
      m.nb_lo = 1;
      m.extra = 0;
    } else {
      m.nb_lo = (int)(resident / ncols);
      m.extra = (int)(resident % ncols);
      if (m.nb_lo >= max_nb) {
        m.nb_lo = max_nb;
        m.extra = 0;
      } else if (balanced && m.extra != 0) {
        // uneven bands: split evenly instead (whole columns when there are enough of them)
        m.bal = 1;
        long long units = ncols * ((span + m.align - 1) / m.align);
        long long parts = resident;
        const long long cap = ncols * span / mr;
        if (parts > cap) parts = cap;
        if (parts > units) parts = units;
        m.nparts = (int)(parts < 1 ? 1 : parts);
      }
    }
    return m;
  }
  // mean rows per run (host: short-run decisions)
  int mean_rows() const {
    return bal ? (int)(((long long)ncols * span + nparts - 1) / nparts) : (span + nb_lo - 1) / nb_lo;
  }
};

// The segments of this CTA's runs (runs blockIdx.x, blockIdx.x + gridDim.x, ...).
struct RunIter {
  const RunMap &m;
  int run, col, r0, ce, re;
  __device__ __forceinline__ explicit RunIter(const RunMap &map) : m(map), run((int)blockIdx.x), col(0), r0(0), ce(-1), re(0) {}
  __device__ __forceinline__ bool next(int &c, int &a, int &b) {
    while (!(col < ce || (col == ce && r0 < re))) {
      if (run >= m.nruns()) return false;
      m.bounds(run, col, r0, ce, re);
      run += gridDim.x;
    }
    c = col;
    a = r0;
    b = col == ce ? re : m.span;
    col++;
    r0 = 0;
    return true;
  }
};

}  // namespace wl
