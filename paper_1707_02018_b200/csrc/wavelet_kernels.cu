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
template <typename T>
__global__ void k_fold_sym_pinv(const T *__restrict__ U, long long upitch, long long ubs, T *__restrict__ y,
                                long long ypitch, long long ybs, int n0, int n1, int Lp, int weighted) {
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
  y[(long long)b * ybs + (long long)i * ypitch + pcol] = weighted ? acc / T(c0 * c1) : acc;
}

}  // namespace

cudaError_t launch_fold(int dtype, const FoldArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  dim3 grid((a.n1 + 127) / 128, a.n0, a.batch);
  if (dtype == WL_F64)
    k_fold_sym_pinv<double><<<grid, 128, 0, s>>>(static_cast<const double *>(a.in), a.in_pitch, a.in_bstride,
                                                 static_cast<double *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                                 a.n1, a.Lp, a.weighted);
  else
    k_fold_sym_pinv<float><<<grid, 128, 0, s>>>(static_cast<const float *>(a.in), a.in_pitch, a.in_bstride,
                                               static_cast<float *>(a.out), a.out_pitch, a.out_bstride, a.n0,
                                               a.n1, a.Lp, a.weighted);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace wl
