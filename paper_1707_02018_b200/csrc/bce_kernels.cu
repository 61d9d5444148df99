// Example 2, blind channel estimation, sm_100a.
//
// Every operation is a batched 1-D "valid" cross-correlation  out[i] = sum_{j<T} a[j] b[i+j]:
//   full convolution   x_est = h * s          a = h reversed, b = s zero-padded by K-1
//   S* r (grad_h)      out[n] = sum_k s[k] r[k+n],  n < K
//   H* r (grad_s)      out[k] = sum_n h[n] r[k+n],  k < N
// One CTA owns one batch item (one problem): its operands are staged in shared memory (zero
// padding = the zero-padded boundaries of P:190), each thread produces BV = 8 consecutive outputs
// from a sliding register window of b (2 x BV values, 16-byte shared loads) against 16-byte
// loads of a, so the inner loop issues 64 FFMA per 4 shared loads.  The convolution skips the
// all-zero parts of the padded source (warp-uniform bounds).  These are FP32/FP64 FMA-bound
// (arithmetic intensity ~600 flop/B at the paper's sizes): DESIGN.md §6 "BCE".
//
// k_bce_grad fuses the whole gradient of Eq. (6) for C channels sharing s:
//   r_i = h_i * s - x_i (smem),  grad_{h_i} = 2 S* r_i + (lam_tv/delta) D^T psi(D h_i),
//   grad_s = 2 sum_i H_i* r_i,   F = sum_i ||r_i||^2 + (lam_tv/delta) sum_i L_delta(D h_i)
// (Eq. (6) has no 1/2, hence the 2; reading R24).
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

#ifndef WL_BCE_BV
#define WL_BCE_BV 8
#endif
constexpr int BV = WL_BCE_BV;  // outputs per thread item
constexpr int BNT = 256;  // threads per CTA

__host__ __device__ constexpr int rup(int v, int a) { return (v + a - 1) / a * a; }

// acc[v] += sum_{j in [jlo, jhi)} a[j] * b[i0 + j + v]; jlo, jhi multiples of BV; a and b 16-byte
// aligned, i0 a multiple of BV; a zero beyond its length; b readable up to i0 + jhi + BV.
template <typename T>
__device__ __forceinline__ void xcorr_item(const T *__restrict__ a, const T *__restrict__ b, int i0, int jlo, int jhi,
                                           T (&acc)[BV]) {
  using Vt = typename Vec16<T>::type;
  constexpr int VEC = Vec16<T>::n;
  if (jlo >= jhi) return;
  T lo[BV];
#pragma unroll
  for (int i = 0; i < BV / VEC; i++) vec_split<T>(reinterpret_cast<const Vt *>(b + i0 + jlo)[i], lo + i * VEC);
#pragma unroll 2
  for (int j = jlo; j < jhi; j += BV) {
    T hi[BV], av[BV];
#pragma unroll
    for (int i = 0; i < BV / VEC; i++) {
      vec_split<T>(reinterpret_cast<const Vt *>(b + i0 + j + BV)[i], hi + i * VEC);
      vec_split<T>(reinterpret_cast<const Vt *>(a + j)[i], av + i * VEC);
    }
#pragma unroll
    for (int u = 0; u < BV; u++)
#pragma unroll
      for (int v = 0; v < BV; v++) acc[v] = fma(av[u], (u + v < BV) ? lo[u + v] : hi[u + v - BV], acc[v]);
#pragma unroll
    for (int v = 0; v < BV; v++) lo[v] = hi[v];
  }
}

// j range of an item [i0, i0+BV) whose b is nonzero only on [nz0, nz1): j in
// [nz0 - i0 - BV + 1, nz1 - i0) clipped to [0, ta), rounded out to BV, made warp-uniform
// (a must stay a broadcast read).
__device__ __forceinline__ void nz_range(int i0, int nz0, int nz1, int ta, int &jlo, int &jhi) {
  int lo = max(0, nz0 - i0 - BV + 1), hi = min(ta, nz1 - i0);
  if (hi <= lo) {
    lo = 1 << 30;
    hi = 0;
  } else {
    lo = lo / BV * BV;
    hi = rup(hi, BV);
  }
  const unsigned m = __activemask();
  jlo = __reduce_min_sync(m, lo);
  jhi = __reduce_max_sync(m, hi);
}

template <typename T>
__device__ __forceinline__ void zero_acc(T (&acc)[BV]) {
#pragma unroll
  for (int v = 0; v < BV; v++) acc[v] = T(0);
}

// ------------------------------------------------------------------ standalone operators
template <typename T>
struct XcorrParams {
  const T *a;
  long long a_bstride;
  int ta, a_rev;  // a_b[j] = src[a_rev ? ta-1-j : j], j < ta
  const T *b;
  long long b_bstride;
  int lb, b_off;  // b_b[i] = src[i - b_off] for b_off <= i < b_off + lb, else 0
  T *out;
  long long out_bstride;
  int n_out;
  int ap, bp;     // staged lengths (a: rup(ta) + BV, b: rup(n_out) + rup(ta) + 2 BV)
};

template <typename T>
__global__ void __launch_bounds__(BNT) k_xcorr(const __grid_constant__ XcorrParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *as = reinterpret_cast<T *>(smem_raw);
  T *bs = as + p.ap;
  const int item_b = blockIdx.x;
  const T *ga = p.a + (long long)item_b * p.a_bstride;
  const T *gb = p.b + (long long)item_b * p.b_bstride;
  for (int j = threadIdx.x; j < p.ap; j += BNT) as[j] = j < p.ta ? ga[p.a_rev ? p.ta - 1 - j : j] : T(0);
  for (int i = threadIdx.x; i < p.bp; i += BNT) {
    const int k = i - p.b_off;
    bs[i] = (k >= 0 && k < p.lb) ? gb[k] : T(0);
  }
  __syncthreads();
  T *go = p.out + (long long)item_b * p.out_bstride;
  const int nit = (p.n_out + BV - 1) / BV;
  for (int it = threadIdx.x; it < nit; it += BNT) {
    const int i0 = it * BV;
    int jlo, jhi;
    nz_range(i0, p.b_off, p.b_off + p.lb, p.ta, jlo, jhi);
    T acc[BV];
    zero_acc(acc);
    xcorr_item<T>(as, bs, i0, jlo, jhi, acc);
#pragma unroll
    for (int v = 0; v < BV; v++)
      if (i0 + v < p.n_out) go[i0 + v] = acc[v];
  }
}

// ------------------------------------------------------------------ fused gradient of Eq. (6)
template <typename T>
struct BceParams {
  const T *h, *s, *x;
  long long x_pstride;  // 0: every problem observes the same x
  T *gh, *gs;
  double *f;
  int C, K, N, M;
  T lam_over_delta, delta;
  int spl, np, kp, rp;  // staged lengths
};

template <typename T>
__device__ __forceinline__ T huber_grad(T z, T d) { return z > d ? d : (z < -d ? -d : z); }

template <typename T>
__global__ void __launch_bounds__(BNT) k_bce_grad(const __grid_constant__ BceParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int C = p.C, K = p.K, N = p.N, M = p.M;
  T *sp = reinterpret_cast<T *>(smem_raw);  // [spl]   s at offset K-1 (b of the convolution)
  T *sal = sp + p.spl;                       // [np]    s aligned (a of S* r)
  T *hr = sal + p.np;                        // [C][kp] h reversed (a of the convolution)
  T *hh = hr + C * p.kp;                     // [C][kp] h (a of H* r)
  T *r = hh + C * p.kp;                      // [C][rp] residuals
  __shared__ double red[BNT / 32];
  const int prob = blockIdx.x, tid = threadIdx.x;
  const T *gh_in = p.h + (long long)prob * C * K;
  const T *gs_in = p.s + (long long)prob * N;
  const T *gx = p.x + (long long)prob * p.x_pstride;
  for (int i = tid; i < p.spl; i += BNT) {
    const int k = i - (K - 1);
    sp[i] = (k >= 0 && k < N) ? gs_in[k] : T(0);
  }
  for (int i = tid; i < p.np; i += BNT) sal[i] = i < N ? gs_in[i] : T(0);
  for (int i = tid; i < C * p.kp; i += BNT) {
    const int c = i / p.kp, j = i - c * p.kp;
    hh[i] = j < K ? gh_in[c * K + j] : T(0);
    hr[i] = j < K ? gh_in[c * K + K - 1 - j] : T(0);
  }
  __syncthreads();
  // phase 1: r_c = h_c * s - x_c, and sum r^2
  double fl = 0.0;
  const int nbm = (M + BV - 1) / BV;
  for (int it = tid; it < C * nbm; it += BNT) {
    const int c = it / nbm, i0 = (it - c * nbm) * BV;
    int jlo, jhi;
    nz_range(i0, K - 1, K - 1 + N, K, jlo, jhi);
    T acc[BV];
    zero_acc(acc);
    xcorr_item<T>(hr + c * p.kp, sp, i0, jlo, jhi, acc);
    T *rc = r + c * p.rp;
#pragma unroll
    for (int v = 0; v < BV; v++) {
      const int m = i0 + v;
      const T rv = m < M ? acc[v] - gx[(long long)c * M + m] : T(0);
      rc[m] = rv;
      fl += (double)rv * (double)rv;
    }
  }
  for (int i = tid; i < C * p.rp; i += BNT) {  // the tail beyond the items stays zero
    const int c = i / p.rp, m = i - c * p.rp;
    if (m >= nbm * BV) r[i] = T(0);
  }
  // TV value: sum_c sum_j L_delta(h[j+1] - h[j])
  double tv = 0.0;
  for (int i = tid; i < C * (K - 1); i += BNT) {
    const int c = i / (K - 1), j = i - c * (K - 1);
    const double z = (double)hh[c * p.kp + j + 1] - (double)hh[c * p.kp + j];
    const double a = z < 0 ? -z : z, d = (double)p.delta;
    tv += a <= d ? 0.5 * z * z : d * (a - 0.5 * d);
  }
  __syncthreads();
  // phase 2: grad_h (C x K outputs) and grad_s (N outputs)
  const int nbk = (K + BV - 1) / BV, nbn = (N + BV - 1) / BV;
  const T two = T(2);
  for (int it = tid; it < C * nbk + nbn; it += BNT) {
    T acc[BV];
    zero_acc(acc);
    if (it < C * nbk) {
      const int c = it / nbk, n0 = (it - c * nbk) * BV;
      xcorr_item<T>(sal, r + c * p.rp, n0, 0, rup(N, BV), acc);
      const T *hc = hh + c * p.kp;
      T *out = p.gh + ((long long)prob * C + c) * K;
#pragma unroll
      for (int v = 0; v < BV; v++) {
        const int n = n0 + v;
        if (n >= K) break;
        T tvg = T(0);
        if (n >= 1) tvg += huber_grad<T>(hc[n] - hc[n - 1], p.delta);
        if (n <= K - 2) tvg -= huber_grad<T>(hc[n + 1] - hc[n], p.delta);
        out[n] = two * acc[v] + p.lam_over_delta * tvg;
      }
    } else {
      const int k0 = (it - C * nbk) * BV;
      for (int c = 0; c < C; c++) xcorr_item<T>(hh + c * p.kp, r + c * p.rp, k0, 0, rup(K, BV), acc);
      T *out = p.gs + (long long)prob * N;
#pragma unroll
      for (int v = 0; v < BV; v++)
        if (k0 + v < N) out[k0 + v] = two * acc[v];
    }
  }
  if (p.f) {
    double t = fl + (double)p.lam_over_delta * tv;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0) red[tid >> 5] = t;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int i = 0; i < BNT / 32; i++) s += red[i];
      p.f[prob] = s;
    }
  }
}

template <typename T>
cudaError_t launch_xcorr_t(const XcorrArgs &x, cudaStream_t s) {
  XcorrParams<T> p;
  p.a = static_cast<const T *>(x.a);
  p.a_bstride = x.a_bstride;
  p.ta = x.ta;
  p.a_rev = x.a_rev;
  p.b = static_cast<const T *>(x.b);
  p.b_bstride = x.b_bstride;
  p.lb = x.lb;
  p.b_off = x.b_off;
  p.out = static_cast<T *>(x.out);
  p.out_bstride = x.out_bstride;
  p.n_out = x.n_out;
  p.ap = rup(x.ta, BV) + BV;
  p.bp = rup(x.n_out, BV) + rup(x.ta, BV) + 2 * BV;
  const size_t smem = (size_t)(p.ap + p.bp) * sizeof(T);
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(k_xcorr<T>), BNT, smem, &resident);
  if (e != cudaSuccess) return e;
  k_xcorr<T><<<(unsigned)x.batch, BNT, smem, s>>>(p);
  g_launches++;
  return cudaGetLastError();
}

template <typename T>
BceParams<T> bce_params(const BceArgs &a) {
  BceParams<T> p;
  p.C = a.C;
  p.K = a.K;
  p.N = a.N;
  p.M = a.K + a.N - 1;
  p.spl = rup(p.M, BV) + rup(a.K, BV) + 2 * BV;
  p.np = rup(a.N, BV) + BV;
  p.kp = rup(a.K, BV) + BV;
  p.rp = rup(a.K, BV) + rup(a.N, BV) + 2 * BV;
  return p;
}

template <typename T>
size_t bce_smem(const BceArgs &a) {
  BceParams<T> p = bce_params<T>(a);
  return (size_t)(p.spl + p.np + 2 * a.C * p.kp + a.C * p.rp) * sizeof(T);
}

template <typename T>
cudaError_t launch_bce_t(const BceArgs &a, cudaStream_t s) {
  BceParams<T> p = bce_params<T>(a);
  p.h = static_cast<const T *>(a.h);
  p.s = static_cast<const T *>(a.s);
  p.x = static_cast<const T *>(a.x);
  p.x_pstride = a.x_shared ? 0 : (long long)a.C * p.M;
  p.gh = static_cast<T *>(a.gh);
  p.gs = static_cast<T *>(a.gs);
  p.f = a.f;
  p.lam_over_delta = T(a.lam_tv / a.delta);
  p.delta = T(a.delta);
  const size_t smem = bce_smem<T>(a);
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(k_bce_grad<T>), BNT, smem, &resident);
  if (e != cudaSuccess) return e;
  k_bce_grad<T><<<(unsigned)a.problems, BNT, smem, s>>>(p);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace

size_t xcorr_smem_bytes(int dtype, int ta, int n_out) {
  const size_t es = dtype == WL_F64 ? 8 : 4;
  return (size_t)(rup(ta, BV) + BV + rup(n_out, BV) + rup(ta, BV) + 2 * BV) * es;
}

size_t bce_smem_bytes(int dtype, const BceArgs &a) {
  return dtype == WL_F64 ? bce_smem<double>(a) : bce_smem<float>(a);
}

cudaError_t launch_xcorr(int dtype, const XcorrArgs &x, cudaStream_t s) {
  if (x.batch == 0 || x.n_out == 0) return cudaSuccess;
  return dtype == WL_F64 ? launch_xcorr_t<double>(x, s) : launch_xcorr_t<float>(x, s);
}

cudaError_t launch_bce_grad(int dtype, const BceArgs &a, cudaStream_t s) {
  if (a.problems == 0) return cudaSuccess;
  return dtype == WL_F64 ? launch_bce_t<double>(a, s) : launch_bce_t<float>(a, s);
}

}  // namespace wl
