// The symmetric folds after a synthesis onto the extended range [-L', n+L') per axis
// (synthesis_kernels.cu writes U there):
//   weighted   W of the paper-literal variant (SYMMETRIC_EDAG, reading R1): y = E_sym^dagger U
//              = diag(1/c) E_sym^T U;
//   unweighted (W-dagger)* under symmetric BC: y = E_sym^T U (reflect-add).
// Analysis (W*, W-dagger) lives in analysis_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

// ------------------------------------------------------------- EDAG fold
// One thread per 4 consecutive output columns of one row.  Rows and columns at least L' from both
// edges are a plain shifted copy y[i][p] = U[i+L'][p+L'] (the memory-bound bulk); the L'-wide
// border adds the reflected positions (2 or 3 per axis) and, weighted, divides by c_i c_p.
template <typename T>
__global__ void __launch_bounds__(256) k_fold_sym_pinv(const T *__restrict__ U, long long upitch, long long ubs,
                                                       T *__restrict__ y, long long ypitch, long long ybs, int n0,
                                                       int n1, int Lp, int weighted, int vec, long long nrows,
                                                       int coff) {
  const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (p0 >= n1) return;
  // (image, row) pairs flattened over gridDim.y with a stride loop: any batch and height
  for (long long ib = blockIdx.y; ib < nrows; ib += gridDim.y) {
  const int b = (int)(ib / n0), i = (int)(ib - (long long)b * n0);
  const T *u = U + (long long)b * ubs;
  T *yo = y + (long long)b * ybs + (long long)i * ypitch;
  const bool row_in = i >= Lp && i < n0 - Lp;
  if (row_in && p0 >= Lp && p0 + 4 <= n1 - Lp) {
    const T *ur = u + (long long)(i + Lp) * upitch + (p0 + Lp + coff);
    const T v[4] = {ur[0], ur[1], ur[2], ur[3]};
    if (vec) {  // 16-byte aligned output rows (fp32) / 2 x 16 bytes (fp64)
      using Vt = typename Vec16<T>::type;
      constexpr int VEC = Vec16<T>::n;
#pragma unroll
      for (int k = 0; k < 4 / VEC; k++) reinterpret_cast<Vt *>(yo + p0)[k] = vec_make<T>(v + k * VEC);
    } else {
#pragma unroll
      for (int k = 0; k < 4; k++) yo[p0 + k] = v[k];
    }
    continue;
  }
  int t0s[3], c0 = 0;
  t0s[c0++] = i;
  if (i < Lp) t0s[c0++] = -1 - i;
  if (i >= n0 - Lp) t0s[c0++] = 2 * n0 - 1 - i;
  for (int q = 0; q < 4; q++) {
    const int pcol = p0 + q;
    if (pcol >= n1) break;
    int t1s[3], c1 = 0;
    t1s[c1++] = pcol;
    if (pcol < Lp) t1s[c1++] = -1 - pcol;
    if (pcol >= n1 - Lp) t1s[c1++] = 2 * n1 - 1 - pcol;
    T acc = T(0);
    for (int a = 0; a < c0; a++)
      for (int c = 0; c < c1; c++) acc += u[(long long)(t0s[a] + Lp) * upitch + (t1s[c] + Lp + coff)];
    yo[pcol] = weighted ? acc / T(c0 * c1) : acc;
  }
  }
}

// Border-only fold after a split synthesis: y already holds U at every in-image position (the
// synthesis wrote it there), U keeps the frame outside the image; the pixels within L' of an edge
// add their reflected positions from U (2 or 3 per axis) and, weighted, divide by c_i c_p
// (E_sym^dagger = diag(1/c) E_sym^T).  One thread per border pixel (top / bottom rows,
// then the left / right columns of the rows between), grid-stride over the batch.
template <typename T>
struct FoldBorderParams {
  const T *U;
  long long upitch, ubs;
  T *y;
  long long ypitch, ybs;
  int n0, n1, Lp, weighted, coff;
  long long per_img, total;
};

template <typename T>
__global__ void __launch_bounds__(256) k_fold_border(const __grid_constant__ FoldBorderParams<T> p) {
  pdl_launch_dependents();
  pdl_wait();  // the synthesis of this level wrote y and U
  const int n0 = p.n0, n1 = p.n1, Lp = p.Lp;
  const int a = min(Lp, n0), b = max(a, n0 - Lp);   // border rows [0, a) and [b, n0)
  const int ca = min(Lp, n1), cb = max(ca, n1 - Lp);  // border columns [0, ca) and [cb, n1)
  const long long nrow = (long long)(a + n0 - b) * n1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < p.total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long img = idx / p.per_img;
    long long k = idx - img * p.per_img;
    int i, q;
    if (k < nrow) {
      const int r = (int)(k / n1);
      q = (int)(k - (long long)r * n1);
      i = r < a ? r : b + (r - a);
    } else {
      k -= nrow;
      const int w = ca + n1 - cb;
      const int r = (int)(k / w), c = (int)(k - (long long)r * w);
      i = a + r;
      q = c < ca ? c : cb + (c - ca);
    }
    int t0s[3], c0 = 0, t1s[3], c1 = 0;
    t0s[c0++] = i;
    if (i < Lp) t0s[c0++] = -1 - i;
    if (i >= n0 - Lp) t0s[c0++] = 2 * n0 - 1 - i;
    t1s[c1++] = q;
    if (q < Lp) t1s[c1++] = -1 - q;
    if (q >= n1 - Lp) t1s[c1++] = 2 * n1 - 1 - q;
    const T *u = p.U + img * p.ubs;
    T *yp = p.y + img * p.ybs + (long long)i * p.ypitch + q;
    T acc = *yp;  // U(i, q) itself, written to y by the synthesis
    for (int s0 = 0; s0 < c0; s0++)
      for (int s1 = 0; s1 < c1; s1++)
        if (s0 || s1) acc += u[(long long)(t0s[s0] + Lp) * p.upitch + (t1s[s1] + Lp + p.coff)];
    *yp = p.weighted ? acc / T(c0 * c1) : acc;
  }
}

template <typename T>
cudaError_t launch_fold_border_t(const FoldArgs &a, cudaStream_t s) {
  FoldBorderParams<T> p;
  p.U = static_cast<const T *>(a.in);
  p.upitch = a.in_pitch;
  p.ubs = a.in_bstride;
  p.y = static_cast<T *>(a.out);
  p.ypitch = a.out_pitch;
  p.ybs = a.out_bstride;
  p.n0 = a.n0;
  p.n1 = a.n1;
  p.Lp = a.Lp;
  p.weighted = a.weighted;
  p.coff = a.col_off;
  const int A = std::min(a.Lp, a.n0), B = std::max(A, a.n0 - a.Lp);
  const int CA = std::min(a.Lp, a.n1), CB = std::max(CA, a.n1 - a.Lp);
  p.per_img = (long long)(A + a.n0 - B) * a.n1 + (long long)(B - A) * (CA + a.n1 - CB);
  p.total = p.per_img * a.batch;
  if (p.total == 0) return cudaSuccess;
  const int grid = (int)std::min<long long>((p.total + 255) / 256, 148LL * 8);
  cudaError_t e = launch_pdl(k_fold_border<T>, grid, 256, 0, s, p, 'f');
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fold(int dtype, const FoldArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  if (a.border_only) return dtype == WL_F64 ? launch_fold_border_t<double>(a, s) : launch_fold_border_t<float>(a, s);
  const int vec = (a.out_pitch % 4 == 0) && (a.out_bstride % 4 == 0) && (reinterpret_cast<uintptr_t>(a.out) % 16 == 0);
  const long long nrows = (long long)a.n0 * a.batch;
  dim3 grid((a.n1 + 4 * 256 - 1) / (4 * 256), (unsigned)std::min<long long>(nrows, 65535));
  if (dtype == WL_F64)
    k_fold_sym_pinv<double><<<grid, 256, 0, s>>>(static_cast<const double *>(a.in), a.in_pitch, a.in_bstride,
                                                 static_cast<double *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                                 a.n1, a.Lp, a.weighted, vec, nrows, a.col_off);
  else
    k_fold_sym_pinv<float><<<grid, 256, 0, s>>>(static_cast<const float *>(a.in), a.in_pitch, a.in_bstride,
                                               static_cast<float *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                               a.n1, a.Lp, a.weighted, vec, nrows, a.col_off);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace wl
