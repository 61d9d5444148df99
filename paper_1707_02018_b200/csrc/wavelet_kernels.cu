// Wavelet level kernels (sm_100a): one launch = one 2-D level of W-dagger / W* (analysis)
// or of W (synthesis), fused row + column passes in shared memory.
//
// Analysis core (R5):   out[k] = sum_{j<L} f[j] * yhat[2k+1-j]
// applied along axis 1 (rows) then axis 0 (columns); yhat = E y with E chosen per operator
// (P:52-98):  W-dagger: E_bc;  W*: E_zpd / periodisation / (E_sym^dagger)* = E_sym diag(1/c)
// (Eq. (4); reading R1).
// Synthesis (W) lives in synthesis_kernels.cu; the EDAG fold stays here.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

template <typename T>
struct AnaParams {
  const T *in;
  long long in_pitch, in_bstride;
  int n0, n1;
  T *out[4];
  long long out_pitch[4], out_bstride[4];
  int m0, m1;
  int m1s;  // columns stored per row: m1 rounded up to the 16-byte pitch (padding written as 0)
  int ext;
  int chunk;  // coefficient rows per CTA
  int fast;   // 16-byte cp.async path allowed for interior chunks
  T lo[kMaxL], hi[kMaxL];
};

// Source index of extended position t (or -1 for a zero) and its weight.
template <typename T>
__device__ __forceinline__ int ext_src(int t, int n, int ext, int Lp, T &w) {
  w = T(1);
  if (ext == EXT_ZERO) return (t >= 0 && t < n) ? t : -1;
  if (ext == EXT_PER) {
    int r = t % n;
    return r < 0 ? r + n : r;
  }
  int s = t < 0 ? -1 - t : (t >= n ? 2 * n - 1 - t : t);
  if (s < 0 || s >= n) return -1;  // only reached by positions that feed no stored output
  if (ext == EXT_SYM_PADJ) {
    // multiplicity c_s = #{t in [-Lp, n+Lp) : src(t) = s} = 1 + [s < Lp] + [s >= n - Lp]
    int c = 1 + (s < Lp ? 1 : 0) + (s >= n - Lp ? 1 : 0);
    w = T(1) / T(c);
  }
  return s;
}

// ------------------------------------------------------------------ analysis
// Streaming strip kernel.  A CTA owns TN coefficient columns [q0, q0+TN) of one image and a
// chunk of coefficient rows [kc0, kc1); it walks down the rows G at a time:
//   A  cp.async the 2G new extended input rows (2TN+L-2 columns + alignment) into a double
//      buffer, one iteration ahead;
//   B  axis-1 pass: each thread filters one input row into VB coefficient pairs (lo, hi)
//      from a register window (2VB+L-2 samples) and writes them to the lo/hi row rings;
//   C  axis-0 pass: each thread owns one ring column and produces VC coefficient rows of
//      two subbands from a register window of the ring (2VC+L-2 samples), stored straight
//      to global memory (coalesced across the warp).
// Vertical halos are never recomputed inside a chunk (the rings carry L-2 rows over).
template <typename T, int L, int TN, int G>
struct AnaCfg {
  static constexpr int VB = 8, VC = 8;
  static constexpr int VEC = Vec16<T>::n;
  static constexpr int SHIFT = ((2 - L) % VEC + VEC) % VEC;  // smem col of ext col c0 = 2q0+2-L
  static constexpr int CI = 2 * TN + L - 2;
  static constexpr int CL = round_up_c(SHIFT + CI, VEC);      // loaded columns
  static constexpr int NV = CL / VEC;                         // 16-byte chunks per row
  static constexpr int IP = conflict_free_pitch<T>(CL);
  static constexpr int ROWS = 2 * G;
  static constexpr int RING = 64;
  static_assert(ROWS + L - 2 <= RING, "ring too small");
  static_assert(L - 2 <= ROWS, "prologue must fit the input buffer");
  static constexpr int MP = conflict_free_pitch<T>(TN);
  static constexpr int NSEG = TN / VB;
  static constexpr int NT = ROWS * NSEG;
  static_assert(NT == 2 * TN * (G / VC), "stage B and C thread counts differ");
  static constexpr int WB = round_up_c(SHIFT + 2 * VB + L - 2, VEC);  // row-pass window (elements)
  static constexpr int WC = 2 * VC + L - 2;                          // column-pass window
  static constexpr size_t smem_bytes() { return sizeof(T) * (2 * (size_t)ROWS * IP + 2 * (size_t)RING * MP); }
};

template <typename T, int L, int TN, int G>
__device__ __forceinline__ void ana_load_rows(T *buf, const AnaParams<T> &p, const T *in, int e0, int nrows,
                                              int c0, bool fast) {
  using C = AnaCfg<T, L, TN, G>;
  using V = typename Vec16<T>::type;
  for (int idx = threadIdx.x; idx < nrows * C::NV; idx += C::NT) {
    int r = idx / C::NV, v = idx - r * C::NV;
    T wr;
    int sr = ext_src<T>(e0 + r, p.n0, p.ext, L - 1, wr);
    T *dst = buf + r * C::IP + v * C::VEC;
    int cg = c0 - C::SHIFT + v * C::VEC;
    if (sr < 0) {
      T z[C::VEC];
#pragma unroll
      for (int u = 0; u < C::VEC; u++) z[u] = T(0);
      *reinterpret_cast<V *>(dst) = vec_make<T>(z);
    } else if (fast && cg >= 0 && cg + C::VEC <= p.n1) {
      cp_async16(dst, in + (long long)sr * p.in_pitch + cg);
    } else {
      T z[C::VEC];
#pragma unroll
      for (int u = 0; u < C::VEC; u++) {
        T wc;
        int sc = ext_src<T>(cg + u, p.n1, p.ext, L - 1, wc);
        z[u] = sc >= 0 ? in[(long long)sr * p.in_pitch + sc] * (wr * wc) : T(0);
      }
      *reinterpret_cast<V *>(dst) = vec_make<T>(z);
    }
  }
}

template <typename T, int L, int TN, int G>
__device__ __forceinline__ void ana_row_pass(const T *buf, T *ring_lo, T *ring_hi, const AnaParams<T> &p, int e0,
                                             int nrows) {
  using C = AnaCfg<T, L, TN, G>;
  using V = typename Vec16<T>::type;
  const int tid = threadIdx.x;
  const int seg = (tid / 8) % C::NSEG;
  const int row = (tid % 8) + 8 * (tid / (8 * C::NSEG));
  if (row >= nrows) return;
  T w[C::WB];
  const V *src = reinterpret_cast<const V *>(buf + row * C::IP + 2 * C::VB * seg);
#pragma unroll
  for (int i = 0; i < C::WB / C::VEC; i++) vec_split<T>(src[i], w + i * C::VEC);
  T lo[C::VB], hi[C::VB];
#pragma unroll
  for (int k = 0; k < C::VB; k++) {
    T al = T(0), ah = T(0);
#pragma unroll
    for (int j = 0; j < L; j++) {
      T v = w[C::SHIFT + 2 * k + L - 1 - j];
      al = fma(p.lo[j], v, al);
      ah = fma(p.hi[j], v, ah);
    }
    lo[k] = al;
    hi[k] = ah;
  }
  const int slot = (e0 + row) & (C::RING - 1);
  V *dl = reinterpret_cast<V *>(ring_lo + slot * C::MP + C::VB * seg);
  V *dh = reinterpret_cast<V *>(ring_hi + slot * C::MP + C::VB * seg);
#pragma unroll
  for (int i = 0; i < C::VB / C::VEC; i++) {
    dl[i] = vec_make<T>(lo + i * C::VEC);
    dh[i] = vec_make<T>(hi + i * C::VEC);
  }
}

template <typename T, int L, int TN, int G>
__global__ void __launch_bounds__(AnaCfg<T, L, TN, G>::NT, 2) k_analysis(const AnaParams<T> p) {
  using C = AnaCfg<T, L, TN, G>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *inbuf = reinterpret_cast<T *>(smem_raw);  // [2][ROWS][IP]
  T *ring_lo = inbuf + 2 * C::ROWS * C::IP;    // [RING][MP]
  T *ring_hi = ring_lo + C::RING * C::MP;

  const int b = blockIdx.z;
  const int q0 = blockIdx.x * TN;
  const int kc0 = blockIdx.y * p.chunk;
  const int kc1 = min(p.m0, kc0 + p.chunk);
  const int c0 = 2 * q0 + 2 - L;
  const T *in = p.in + (long long)b * p.in_bstride;
  const bool fast = p.fast;
  const int n_it = (kc1 - kc0 + G - 1) / G;

  // prologue: ext rows [2kc0+2-L, 2kc0) -> rings
  {
    const int e0 = 2 * kc0 + 2 - L;
    ana_load_rows<T, L, TN, G>(inbuf, p, in, e0, L - 2, c0, fast);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    ana_row_pass<T, L, TN, G>(inbuf, ring_lo, ring_hi, p, e0, L - 2);
  }
  __syncthreads();
  ana_load_rows<T, L, TN, G>(inbuf + C::ROWS * C::IP, p, in, 2 * kc0, C::ROWS, c0, fast);
  cp_async_commit();

  const int tid = threadIdx.x;
  const int cc = tid % (2 * TN), rs = tid / (2 * TN);
  const T *ring = cc < TN ? ring_lo : ring_hi;
  const int col = cc % TN;
  const int q = q0 + col;
  T *o_lo = cc < TN ? p.out[0] : p.out[1];  // LL or LH
  T *o_hi = cc < TN ? p.out[2] : p.out[3];  // HL or HH
  const long long ps_lo = cc < TN ? p.out_pitch[0] : p.out_pitch[1];
  const long long ps_hi = cc < TN ? p.out_pitch[2] : p.out_pitch[3];
  o_lo += (long long)b * (cc < TN ? p.out_bstride[0] : p.out_bstride[1]) + q;
  o_hi += (long long)b * (cc < TN ? p.out_bstride[2] : p.out_bstride[3]) + q;
  const bool qvalid = q < p.m1s;
  const bool qzero = q >= p.m1;

  for (int it = 0; it < n_it; it++) {
    const int kb = kc0 + it * G;
    cp_async_wait_all();
    __syncthreads();
    const T *cur = inbuf + ((it + 1) & 1) * C::ROWS * C::IP;
    if (it + 1 < n_it) {
      ana_load_rows<T, L, TN, G>(inbuf + (it & 1) * C::ROWS * C::IP, p, in, 2 * (kb + G), C::ROWS, c0, fast);
      cp_async_commit();
    }
    ana_row_pass<T, L, TN, G>(cur, ring_lo, ring_hi, p, 2 * kb, C::ROWS);
    __syncthreads();
    // stage C
    const int k0 = kb + C::VC * rs;
    const int eb = 2 * k0 + 2 - L;
    T w[C::WC];
#pragma unroll
    for (int i = 0; i < C::WC; i++) w[i] = ring[((eb + i) & (C::RING - 1)) * C::MP + col];
#pragma unroll
    for (int k = 0; k < C::VC; k++) {
      T al = T(0), ah = T(0);
#pragma unroll
      for (int j = 0; j < L; j++) {
        T v = w[2 * k + L - 1 - j];
        al = fma(p.lo[j], v, al);
        ah = fma(p.hi[j], v, ah);
      }
      const int kr = k0 + k;
      if (qvalid && kr < kc1) {
        o_lo[(long long)kr * ps_lo] = qzero ? T(0) : al;
        o_hi[(long long)kr * ps_hi] = qzero ? T(0) : ah;
      }
    }
  }
}

// ------------------------------------------------------------- EDAG fold
template <typename T>
__global__ void k_fold_sym_pinv(const T *__restrict__ U, long long upitch, long long ubs, T *__restrict__ y,
                                long long ypitch, long long ybs, int n0, int n1, int Lp) {
  int pcol = blockIdx.x * blockDim.x + threadIdx.x;
  int i = blockIdx.y;
  int b = blockIdx.z;
  if (pcol >= n1) return;
  int t0s[3], t1s[3], c0 = 0, c1 = 0;
  t0s[c0++] = i;
  if (i < Lp) t0s[c0++] = -1 - i;
  if (i >= n0 - Lp) t0s[c0++] = 2 * n0 - 1 - i;
  t1s[c1++] = pcol;
  if (pcol < Lp) t1s[c1++] = -1 - pcol;
  if (pcol >= n1 - Lp) t1s[c1++] = 2 * n1 - 1 - pcol;
  const T *u = U + (long long)b * ubs;
  T acc = T(0);
  for (int a = 0; a < c0; a++)
    for (int c = 0; c < c1; c++) acc += u[(long long)(t0s[a] + Lp) * upitch + (t1s[c] + Lp)];
  y[(long long)b * ybs + (long long)i * ypitch + pcol] = acc / T(c0 * c1);
}

template <typename T, int L>
cudaError_t launch_analysis_t(const AnalysisArgs &a, cudaStream_t s) {
  constexpr int TN = sizeof(T) == 4 ? 64 : 32, G = 16;
  using C = AnaCfg<T, L, TN, G>;
  AnaParams<T> p;
  p.in = static_cast<const T *>(a.in);
  p.in_pitch = a.in_pitch; p.in_bstride = a.in_bstride; p.n0 = a.n0; p.n1 = a.n1;
  for (int i = 0; i < 4; i++) {
    p.out[i] = static_cast<T *>(a.out[i]);
    p.out_pitch[i] = a.out_pitch[i]; p.out_bstride[i] = a.out_bstride[i];
  }
  p.m0 = a.m0; p.m1 = a.m1; p.ext = a.ext;
  p.m1s = (int)((a.m1 + C::VEC - 1) / C::VEC * C::VEC);
  p.fast = (a.ext != EXT_SYM_PADJ) && (a.in_pitch % C::VEC == 0) && (a.in_bstride % C::VEC == 0) &&
           (reinterpret_cast<uintptr_t>(a.in) % 16 == 0);
  for (int j = 0; j < kMaxL; j++) { p.lo[j] = T(j < L ? a.lo[j] : 0); p.hi[j] = T(j < L ? a.hi[j] : 0); }
  // chunking: enough CTAs for ~4 waves of 2 CTAs per SM, chunks a multiple of G rows
  const int strips = (a.m1 + TN - 1) / TN;
  const long long base = (long long)strips * a.batch;
  const long long target = 148LL * 2 * 4;
  int nchunk = (int)std::max(1LL, std::min((long long)((a.m0 + G - 1) / G), (target + base - 1) / base));
  int chunk = (a.m0 + nchunk - 1) / nchunk;
  chunk = (chunk + G - 1) / G * G;
  nchunk = (a.m0 + chunk - 1) / chunk;
  p.chunk = chunk;
  size_t smem = C::smem_bytes();
  auto kern = k_analysis<T, L, TN, G>;
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(kern), C::NT, smem, &resident);
  if (e != cudaSuccess) return e;
  dim3 grid(strips, nchunk, a.batch);
  kern<<<grid, C::NT, smem, s>>>(p);
  g_launches++;
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_analysis(const AnalysisArgs &a, cudaStream_t s) {
  switch (a.L) {
    case 2: return launch_analysis_t<T, 2>(a, s);
    case 4: return launch_analysis_t<T, 4>(a, s);
    case 8: return launch_analysis_t<T, 8>(a, s);
    case 10: return launch_analysis_t<T, 10>(a, s);
    case 16: return launch_analysis_t<T, 16>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_analysis(int dtype, const AnalysisArgs &a, cudaStream_t s) {
  if (a.batch == 0 || a.m0 == 0 || a.m1 == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_analysis<double>(a, s) : dispatch_analysis<float>(a, s);
}

cudaError_t launch_fold(int dtype, const FoldArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  dim3 grid((a.n1 + 127) / 128, a.n0, a.batch);
  if (dtype == WL_F64)
    k_fold_sym_pinv<double><<<grid, 128, 0, s>>>(static_cast<const double *>(a.in), a.in_pitch, a.in_bstride,
                                                 static_cast<double *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                                 a.n1, a.Lp);
  else
    k_fold_sym_pinv<float><<<grid, 128, 0, s>>>(static_cast<const float *>(a.in), a.in_pitch, a.in_bstride,
                                               static_cast<float *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                               a.n1, a.Lp);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace wl
