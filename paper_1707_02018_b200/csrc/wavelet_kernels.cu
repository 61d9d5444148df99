// The symmetric folds after a synthesis onto the extended range [-L', n+L') per axis
// (synthesis_kernels.cu writes U there):
//   weighted   W of the paper-literal variant (SYMMETRIC_EDAG, reading R1): y = E_sym^dagger U
//              = diag(1/c) E_sym^T U;
//   unweighted (W-dagger)* under symmetric BC: y = E_sym^T U (reflect-add).
// Analysis (W*, W-dagger) lives in analysis_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>

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

}  // namespace

cudaError_t launch_fold(int dtype, const FoldArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
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
