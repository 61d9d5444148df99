// Small-level kernels (sm_100a, fp32 / fp64): every coarse level whose input fits in one CTA's
// shared memory runs inside ONE launch, one CTA per image, with the LL of each level kept in
// shared memory between levels (north_star "coarse levels run as a persistent
// kernel").  A whole small problem (cfg1, 64^2 fp64) is one launch; for larger images the tail
// of the chain is.  There is no grid-wide barrier: an image's levels depend only on that image.
//
// Analysis (W*, W-dagger; reading R5):
//   out[k] = sum_{j<L} f[j] yhat[2k+1-j]   along axis 1 (rows), then axis 0 (columns),
// yhat = E y with the level's extension (zero / periodic wrap / half-point reflection / the
// (E_sym^dagger)* weights); subband XY = axis-0 filter X, axis-1 filter Y.
// Synthesis (W = (W*)^T under crop or periodic wrap):
//   y[i] = sum_{j<L, i+j-1 even} f[j] c[(i+j-1)/2]   (crop: the index in [0, m); wrap: mod m),
// axis 1 for every coefficient row, then axis 0.  Plain loops (the work is a few kB per level):
// the point is one launch instead of one per level.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

constexpr int kSmallMaxLev = 12;
constexpr int kSmallNT = 512;
constexpr size_t kSmallSmem = 200 * 1024;  // shared memory one small launch may use
// largest level input (analysis) / output (synthesis) taken, in elements: one CTA does a level's
// work alone, so only levels that are latency-bound anyway (A/B on B200: cfg1 64^2 W* 20.7 -> 16.6
// us, W 22.7 -> 14.5 us; cfg2's 133^2 and 70^2 levels on one CTA per image were 3x slower)
constexpr size_t kSmallMaxElems = 80 * 80;

template <typename T>
struct SmallLev {
  int n0, n1, m0, m1;       // input (analysis) / output (synthesis) and coefficient extents
  T *band[4];               // LL, LH, HL, HH (analysis: outputs; synthesis: inputs, LL only at the first)
  long long pitch[4], bstride[4];
};

template <typename T>
struct SmallParams {
  SmallLev<T> lev[kSmallMaxLev];
  int nlev, ext, L;
  const T *in;              // analysis: the first level's input; synthesis: unused
  long long in_pitch, in_bstride;
  T *out;                   // synthesis: the last level's output
  long long out_pitch, out_bstride;
  T lo[kMaxL], hi[kMaxL];
  size_t off_p1, off_t;     // shared-memory regions (elements): LL ping-pong buffer 1, temporaries
};

// source index of extended position t (or -1: zero) and its weight
template <typename T>
__device__ __forceinline__ int small_src(int t, int n, int ext, int Lp, T &w) {
  w = T(1);
  if (t >= 0 && t < n && ext != EXT_SYM_PADJ) return t;
  if (ext == EXT_ZERO) return -1;
  if (ext == EXT_PER) {
    int r = t % n;
    return r < 0 ? r + n : r;
  }
  const int s = refl_inf(t, n);
  if (ext == EXT_SYM_PADJ) w = T(1) / T(1 + (s < Lp ? 1 : 0) + (s >= n - Lp ? 1 : 0));
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kSmallNT) k_ana_small(const __grid_constant__ SmallParams<T> p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sm = reinterpret_cast<T *>(sm_raw);
  const int img = blockIdx.x, tid = threadIdx.x, L = p.L, Lp = L - 1;
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our input
  T *buf[2] = {sm, sm + p.off_p1};
  T *tl = sm + p.off_t;
  {  // the first level's input -> buf[0]
    const SmallLev<T> &v = p.lev[0];
    const T *src = p.in + (long long)img * p.in_bstride;
    for (int i = tid; i < v.n0 * v.n1; i += kSmallNT) {
      const int r = i / v.n1, c = i - r * v.n1;
      buf[0][i] = src[(long long)r * p.in_pitch + c];
    }
  }
  __syncthreads();
  for (int l = 0; l < p.nlev; l++) {
    const SmallLev<T> &v = p.lev[l];
    const T *A = buf[l & 1];
    T *th = tl + v.n0 * v.m1;
    // axis 1: every input row -> lo / hi coefficient rows
    for (int i = tid; i < v.n0 * v.m1; i += kSmallNT) {
      const int r = i / v.m1, k = i - r * v.m1;
      T lo = T(0), hi = T(0);
      for (int j = 0; j < L; j++) {
        T w;
        const int c = small_src<T>(2 * k + 1 - j, v.n1, p.ext, Lp, w);
        if (c < 0) continue;
        const T x = A[r * v.n1 + c] * w;
        lo += p.lo[j] * x;
        hi += p.hi[j] * x;
      }
      tl[i] = lo;
      th[i] = hi;
    }
    __syncthreads();
    // axis 0: (LL, LH) from the lo rows, (HL, HH) from the hi rows; LL of a non-last level stays
    // in shared memory; padding columns [m1, pitch) of the stored rows are written 0
    const bool last = l + 1 == p.nlev;
    T *nxt = buf[(l + 1) & 1];
    const int wcols = (int)v.pitch[1];  // all four pitches are >= m1
    for (int i = tid; i < v.m0 * wcols; i += kSmallNT) {
      const int kr = i / wcols, k = i - kr * wcols;
      T s[4] = {T(0), T(0), T(0), T(0)};
      if (k < v.m1) {
        for (int j = 0; j < L; j++) {
          T w;
          const int r = small_src<T>(2 * kr + 1 - j, v.n0, p.ext, Lp, w);
          if (r < 0) continue;
          const T a = tl[r * v.m1 + k] * w, d = th[r * v.m1 + k] * w;
          s[0] += p.lo[j] * a;
          s[1] += p.lo[j] * d;
          s[2] += p.hi[j] * a;
          s[3] += p.hi[j] * d;
        }
      }
      for (int b = last ? 0 : 1; b < 4; b++)
        if (k < v.pitch[b]) v.band[b][(long long)img * v.bstride[b] + (long long)kr * v.pitch[b] + k] = s[b];
      if (!last && k < v.m1) nxt[kr * v.m1 + k] = s[0];
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kSmallNT) k_syn_small(const __grid_constant__ SmallParams<T> p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T *sm = reinterpret_cast<T *>(sm_raw);
  const int img = blockIdx.x, tid = threadIdx.x, L = p.L;
  const bool wrap = p.ext == EXT_PER;
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our coefficients
  T *buf[2] = {sm, sm + p.off_p1};
  T *vl = sm + p.off_t;
  for (int l = 0; l < p.nlev; l++) {
    const SmallLev<T> &v = p.lev[l];
    T *vh = vl + v.m0 * v.n1;
    const T *LLs = buf[(l + 1) & 1];  // the previous level's output (l > 0)
    auto coef = [&](int b, int kr, int k) -> T {
      if (b == 0 && l > 0) return LLs[kr * v.m1 + k];
      return v.band[b][(long long)img * v.bstride[b] + (long long)kr * v.pitch[b] + k];
    };
    // axis 1: coefficient rows -> VL (from LL, LH) and VH (from HL, HH) of width n1
    for (int i = tid; i < v.m0 * v.n1; i += kSmallNT) {
      const int kr = i / v.n1, c = i - kr * v.n1;
      T a = T(0), d = T(0);
      for (int j = (c + 1) & 1; j < L; j += 2) {  // c + j - 1 even
        int k = (c + j - 1) >> 1;
        if (wrap) {
          k %= v.m1;
          if (k < 0) k += v.m1;
        } else if (k < 0 || k >= v.m1) {
          continue;
        }
        a += p.lo[j] * coef(0, kr, k) + p.hi[j] * coef(1, kr, k);
        d += p.lo[j] * coef(2, kr, k) + p.hi[j] * coef(3, kr, k);
      }
      vl[i] = a;
      vh[i] = d;
    }
    __syncthreads();
    // axis 0: output rows from VL, VH
    const bool last = l + 1 == p.nlev;
    T *y = buf[l & 1];
    for (int i = tid; i < v.n0 * v.n1; i += kSmallNT) {
      const int r = i / v.n1, c = i - r * v.n1;
      T acc = T(0);
      for (int j = (r + 1) & 1; j < L; j += 2) {
        int k = (r + j - 1) >> 1;
        if (wrap) {
          k %= v.m0;
          if (k < 0) k += v.m0;
        } else if (k < 0 || k >= v.m0) {
          continue;
        }
        acc += p.lo[j] * vl[k * v.n1 + c] + p.hi[j] * vh[k * v.n1 + c];
      }
      if (last) p.out[(long long)img * p.out_bstride + (long long)r * p.out_pitch + c] = acc;
      else y[i] = acc;
    }
    __syncthreads();
  }
}

bool small_disabled() {
  static const bool v = getenv("WL_NO_SMALL") != nullptr;  // A/B switch: per-level launches only
  return v;
}

template <typename T>
cudaError_t launch_small(bool analysis, SmallParams<T> &p, int batch, size_t smem, cudaStream_t s) {
  auto kern = analysis ? k_ana_small<T> : k_syn_small<T>;
  static bool attr[2] = {false, false};
  if (!attr[analysis]) {
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(kern),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
    if (e != cudaSuccess) return e;
    attr[analysis] = true;
  }
  cudaError_t e = launch_pdl(kern, batch, kSmallNT, smem, s, p, analysis ? 'a' : 's');
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// analysis levels a[i0 .. n): the LL ping-pong buffers hold the largest input or output of the range
// (zero-padded coefficients grow on tiny images), the temporaries the largest lo / hi row pair
size_t ana_small_ll(const AnalysisArgs *a, int i0, int n) {
  size_t m = 0;
  for (int i = i0; i < n; i++) m = std::max({m, (size_t)a[i].n0 * a[i].n1, (size_t)a[i].m0 * a[i].m1});
  return m;
}
size_t ana_small_tmp(const AnalysisArgs *a, int i0, int n) {
  size_t m = 0;
  for (int i = i0; i < n; i++) m = std::max(m, 2 * (size_t)a[i].n0 * a[i].m1);
  return m;
}
size_t ana_small_bytes(const AnalysisArgs *a, int i0, int n, size_t es) {
  return (2 * ana_small_ll(a, i0, n) + ana_small_tmp(a, i0, n)) * es;
}

// synthesis levels a[0 .. i1) (coarse -> fine): bytes (buffers sized by the largest in-shared output)
size_t syn_small_bytes(const SynthesisArgs *a, int i1, size_t es) {
  size_t ll = 0, v = 0;
  for (int i = 0; i < i1; i++) {
    if (i + 1 < i1) ll = std::max(ll, (size_t)a[i].N0 * a[i].N1);
    v = std::max(v, 2 * (size_t)a[i].m0 * a[i].N1);
  }
  return (2 * ll + v) * es;
}

}  // namespace

int small_analysis_start(int dtype, const AnalysisArgs *a, int n) {
  if (small_disabled() || n < 1 || a[0].fista_mask) return n;
  const size_t es = dtype == WL_F64 ? 8 : 4;
  int i0 = n;
  for (int i = n - 1; i >= 0; i--) {
    bool ok = a[i].L <= kMaxL && ana_small_bytes(a, i, n, es) <= kSmallSmem && n - i <= kSmallMaxLev &&
              (size_t)a[i].n0 * a[i].n1 <= kSmallMaxElems && (size_t)a[i].m0 * a[i].m1 <= kSmallMaxElems &&
              a[i].batch <= 65535 && a[i].out_pitch[1] == a[i].out_pitch[2] && a[i].out_pitch[1] == a[i].out_pitch[3];
    if (!ok) break;
    i0 = i;
  }
  // one level alone gains nothing over the streaming kernel unless it is the whole chain
  return (n - i0 >= 2 || i0 == 0) ? i0 : n;
}

cudaError_t launch_analysis_small(int dtype, const AnalysisArgs *a, int n, cudaStream_t s) {
  auto run = [&](auto zero) -> cudaError_t {
    using T = decltype(zero);
    SmallParams<T> p;
    memset(&p, 0, sizeof p);
    p.nlev = n;
    p.ext = a[0].ext;
    p.L = a[0].L;
    for (int j = 0; j < a[0].L; j++) {
      p.lo[j] = T(a[0].lo[j]);
      p.hi[j] = T(a[0].hi[j]);
    }
    p.in = static_cast<const T *>(a[0].in);
    p.in_pitch = a[0].in_pitch;
    p.in_bstride = a[0].in_bstride;
    for (int l = 0; l < n; l++) {
      SmallLev<T> &v = p.lev[l];
      v.n0 = a[l].n0; v.n1 = a[l].n1; v.m0 = a[l].m0; v.m1 = a[l].m1;
      for (int b = 0; b < 4; b++) {
        v.band[b] = static_cast<T *>(a[l].out[b]);
        v.pitch[b] = a[l].out_pitch[b];
        v.bstride[b] = a[l].out_bstride[b];
      }
    }
    p.off_p1 = ana_small_ll(a, 0, n);
    p.off_t = 2 * p.off_p1;
    return launch_small<T>(true, p, a[0].batch, ana_small_bytes(a, 0, n, sizeof(T)), s);
  };
  return dtype == WL_F64 ? run(double(0)) : run(float(0));
}

int small_synthesis_end(int dtype, const SynthesisArgs *a, int n) {
  if (small_disabled() || n < 1) return 0;
  const size_t es = dtype == WL_F64 ? 8 : 4;
  int i1 = 0;
  for (int i = 0; i < n && i < kSmallMaxLev; i++) {
    const SynthesisArgs &v = a[i];
    if (v.o0 != 0 || v.o1 != 0 || v.L > kMaxL || v.batch > 65535 || syn_small_bytes(a, i + 1, es) > kSmallSmem ||
        (size_t)v.N0 * v.N1 > kSmallMaxElems || (size_t)v.m0 * v.m1 > kSmallMaxElems)
      break;
    i1 = i + 1;
  }
  return (i1 >= 2 || i1 == n) ? i1 : 0;
}

cudaError_t launch_synthesis_small(int dtype, const SynthesisArgs *a, int n, cudaStream_t s) {
  auto run = [&](auto zero) -> cudaError_t {
    using T = decltype(zero);
    SmallParams<T> p;
    memset(&p, 0, sizeof p);
    p.nlev = n;
    p.ext = a[0].coef_mod ? EXT_PER : EXT_ZERO;
    p.L = a[0].L;
    for (int j = 0; j < a[0].L; j++) {
      p.lo[j] = T(a[0].lo[j]);
      p.hi[j] = T(a[0].hi[j]);
    }
    for (int l = 0; l < n; l++) {
      SmallLev<T> &v = p.lev[l];
      v.n0 = a[l].N0; v.n1 = a[l].N1; v.m0 = a[l].m0; v.m1 = a[l].m1;
      for (int b = 0; b < 4; b++) {
        v.band[b] = const_cast<T *>(static_cast<const T *>(a[l].in[b]));
        v.pitch[b] = a[l].in_pitch[b];
        v.bstride[b] = a[l].in_bstride[b];
      }
    }
    p.out = static_cast<T *>(a[n - 1].out);
    p.out_pitch = a[n - 1].out_pitch;
    p.out_bstride = a[n - 1].out_bstride;
    size_t ll = 0;
    for (int l = 0; l + 1 < n; l++) ll = std::max(ll, (size_t)a[l].N0 * a[l].N1);
    p.off_p1 = ll;
    p.off_t = 2 * ll;
    return launch_small<T>(false, p, a[0].batch, syn_small_bytes(a, n, sizeof(T)), s);
  };
  return dtype == WL_F64 ? run(double(0)) : run(float(0));
}

}  // namespace wl
