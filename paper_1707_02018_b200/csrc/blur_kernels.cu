// Separable PSF blur kernels (sm_100a): R, and the fused middle stage of grad f,
// s = R*(R u - b) (= R (R u - b) for the symmetric PSFs the plan accepts), optionally
// with f = 1/2 ||R u - b||^2.
//
// Per axis (R12):  (R_a y)[i] = sum_{t=-h..h} k[t] yhat[i - t],
// yhat = half-point symmetric extension of y:  yhat[-1-i] = y[i], yhat[n+i] = y[n-1-i].
#include <cuda_runtime.h>

#include "wl_internal.h"

namespace wl {
namespace {

template <typename T>
struct BlurParams {
  const T *in;
  const T *b;
  T *out;
  double *f;
  int h, w;
  T k[kMaxTaps];
};

__device__ __forceinline__ int refl(int i, int n) {
  // half-point symmetric source index of extended position i (single reflection, n >= h)
  return i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i);
}

// ------------------------------------------------------------------ R
template <typename T, int HW, int TB, int NT>
__global__ void __launch_bounds__(NT) k_blur(const BlurParams<T> p) {
  constexpr int E = TB + 2 * HW, EP = E + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *xin = reinterpret_cast<T *>(smem_raw);  // [E][EP]
  T *mid = xin + E * EP;                     // [E][TB]
  const int b = blockIdx.z;
  const int i0 = blockIdx.y * TB, j0 = blockIdx.x * TB;
  const T *in = p.in + (long long)b * p.h * p.w;
  for (int idx = threadIdx.x; idx < E * E; idx += NT) {
    int r = idx / E, c = idx - r * E;
    int sr = refl(i0 - HW + r, p.h), sc = refl(j0 - HW + c, p.w);
    T v = T(0);
    if (sr >= 0 && sr < p.h && sc >= 0 && sc < p.w) v = in[(long long)sr * p.w + sc];
    xin[r * EP + c] = v;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < E * TB; idx += NT) {
    int r = idx / TB, c = idx - r * TB;
    T acc = T(0);
#pragma unroll
    for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], xin[r * EP + c + HW - t], acc);
    mid[r * TB + c] = acc;
  }
  __syncthreads();
  T *out = p.out + (long long)b * p.h * p.w;
  for (int idx = threadIdx.x; idx < TB * TB; idx += NT) {
    int r = idx / TB, c = idx - r * TB;
    T acc = T(0);
#pragma unroll
    for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], mid[(r + HW - t) * TB + c], acc);
    if (i0 + r < p.h && j0 + c < p.w) out[(long long)(i0 + r) * p.w + j0 + c] = acc;
  }
}

// ---------------------------------------------------- s = R (R u - b), f
// r is needed on the in-domain positions Q = [max(0, tile-HW), min(n, tile+HW)) per axis
// (the reflected halo of the second blur lands inside Q); u on Q extended by HW, reflected.
template <typename T, int HW, int TB, int NT>
__global__ void __launch_bounds__(NT) k_blur_residual(const BlurParams<T> p) {
  constexpr int QM = TB + 2 * HW;   // max extent of Q
  constexpr int UM = QM + 2 * HW;   // max extent of the u region
  constexpr int UP = UM + 1, QP = QM + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *us = reinterpret_cast<T *>(smem_raw);  // [UM][UP]
  T *m1 = us + UM * UP;                     // [UM][QP]  (rows: u region, cols: Q)
  T *rs = m1 + UM * QP;                     // [QM][QP]  r on Q x Q
  T *m2 = rs + QM * QP;                     // [QM][TB]  (rows: Q, cols: tile)
  __shared__ double red[NT / 32];

  const int b = blockIdx.z;
  const int i0 = blockIdx.y * TB, j0 = blockIdx.x * TB;
  const int qr0 = max(0, i0 - HW), qr1 = min(p.h, i0 + TB + HW);
  const int qc0 = max(0, j0 - HW), qc1 = min(p.w, j0 + TB + HW);
  const int nqr = qr1 - qr0, nqc = qc1 - qc0;
  const int nur = nqr + 2 * HW, nuc = nqc + 2 * HW;
  const T *u = p.in + (long long)b * p.h * p.w;
  const T *bb = p.b + (long long)b * p.h * p.w;

  for (int idx = threadIdx.x; idx < nur * nuc; idx += NT) {
    int r = idx / nuc, c = idx - r * nuc;
    int sr = refl(qr0 - HW + r, p.h), sc = refl(qc0 - HW + c, p.w);
    us[r * UP + c] = u[(long long)sr * p.w + sc];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nur * nqc; idx += NT) {
    int r = idx / nqc, c = idx - r * nqc;
    T acc = T(0);
#pragma unroll
    for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], us[r * UP + c + HW - t], acc);
    m1[r * QP + c] = acc;
  }
  __syncthreads();
  double fsum = 0.0;
  for (int idx = threadIdx.x; idx < nqr * nqc; idx += NT) {
    int r = idx / nqc, c = idx - r * nqc;
    T acc = T(0);
#pragma unroll
    for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], m1[(r + HW - t) * QP + c], acc);
    int gi = qr0 + r, gj = qc0 + c;
    T res = acc - bb[(long long)gi * p.w + gj];
    rs[r * QP + c] = res;
    if (gi >= i0 && gi < i0 + TB && gj >= j0 && gj < j0 + TB) fsum += (double)res * (double)res;
  }
  __syncthreads();
  // second blur: rows of Q, tile columns; r_ext(P) = r(refl(P))
  for (int idx = threadIdx.x; idx < nqr * TB; idx += NT) {
    int r = idx / TB, c = idx - r * TB;
    T acc = T(0);
    if (j0 + c < p.w) {
#pragma unroll
      for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], rs[r * QP + refl(j0 + c - t, p.w) - qc0], acc);
    }
    m2[r * TB + c] = acc;
  }
  __syncthreads();
  T *out = p.out + (long long)b * p.h * p.w;
  for (int idx = threadIdx.x; idx < TB * TB; idx += NT) {
    int r = idx / TB, c = idx - r * TB;
    if (i0 + r >= p.h || j0 + c >= p.w) continue;
    T acc = T(0);
#pragma unroll
    for (int t = -HW; t <= HW; t++) acc = fma(p.k[t + HW], m2[(refl(i0 + r - t, p.h) - qr0) * TB + c], acc);
    out[(long long)(i0 + r) * p.w + j0 + c] = acc;
  }
  if (p.f) {
    for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = fsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < NT / 32; i++) s += red[i];
      atomicAdd(p.f + b, 0.5 * s);
    }
  }
}

template <typename T, int HW>
cudaError_t launch_blur_hw(const BlurArgs &a, cudaStream_t s, bool residual) {
  constexpr int TB = 32, NT = 256;
  BlurParams<T> p;
  p.in = static_cast<const T *>(a.in);
  p.b = static_cast<const T *>(a.b);
  p.out = static_cast<T *>(a.out);
  p.f = a.f;
  p.h = (int)a.h;
  p.w = (int)a.w;
  for (int i = 0; i < kMaxTaps; i++) p.k[i] = T(i < a.ntaps ? a.taps[i] : 0.0);
  dim3 grid((unsigned)((a.w + TB - 1) / TB), (unsigned)((a.h + TB - 1) / TB), (unsigned)a.batch);
  cudaError_t e;
  if (!residual) {
    constexpr int E = TB + 2 * HW;
    size_t smem = sizeof(T) * ((size_t)E * (E + 1) + (size_t)E * TB);
    auto kern = k_blur<T, HW, TB, NT>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, NT, smem, s>>>(p);
  } else {
    constexpr int QM = TB + 2 * HW, UM = QM + 2 * HW;
    size_t smem = sizeof(T) * ((size_t)UM * (UM + 1) + (size_t)UM * (QM + 1) + (size_t)QM * (QM + 1) + (size_t)QM * TB);
    auto kern = k_blur_residual<T, HW, TB, NT>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.f) {
      e = cudaMemsetAsync(a.f, 0, sizeof(double) * (size_t)a.batch, s);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, NT, smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_blur(const BlurArgs &a, cudaStream_t s, bool residual) {
  switch (a.ntaps / 2) {
#define WL_BLUR_CASE(H) \
  case H: return launch_blur_hw<T, H>(a, s, residual);
    WL_BLUR_CASE(0) WL_BLUR_CASE(1) WL_BLUR_CASE(2) WL_BLUR_CASE(3) WL_BLUR_CASE(4) WL_BLUR_CASE(5)
    WL_BLUR_CASE(6) WL_BLUR_CASE(7) WL_BLUR_CASE(8) WL_BLUR_CASE(9) WL_BLUR_CASE(10) WL_BLUR_CASE(11)
    WL_BLUR_CASE(12) WL_BLUR_CASE(13) WL_BLUR_CASE(14) WL_BLUR_CASE(15)
#undef WL_BLUR_CASE
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_blur(int dtype, const BlurArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_blur<double>(a, s, false) : dispatch_blur<float>(a, s, false);
}

cudaError_t launch_blur_residual(int dtype, const BlurArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_blur<double>(a, s, true) : dispatch_blur<float>(a, s, true);
}

}  // namespace wl
