// FISTA around grad f (P:117 and P:174 run 2500 FISTA iterations, Beck &
// Teboulle 2009) and the power iteration for its step 1/L:
//   k_fista_update   x+ = soft(y - g / L, lambda / L);  y+ = x+ + ((t - 1) / t+) (x+ - x)
//                    fused, in place over [batch, p_alloc] (pitch padding stays 0: g = x = y = 0 there)
//   k_dot            per-image <a, b> in fp64 (block partials, one atomic per block and image)
//   k_scale          v *= alpha
//   k_fill_seeded    counter-hash uniform(-1, 1) start vector for the power iteration
//   k_fista_advance_t  t <- t+ for FISTA with a device-resident t (graph-replayable iterations)
// All elementwise kernels are grid-stride, 16-byte vectorised, sized to 4 waves of the SMs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

template <typename T>
__device__ __forceinline__ T soft(T v, T tau) {
  const T a = v > T(0) ? v : -v;
  const T m = a - tau;
  return m > T(0) ? (v > T(0) ? m : -m) : T(0);
}

template <typename T>
__global__ void k_fista_update(const T *__restrict__ g, T *__restrict__ x, T *__restrict__ y, long long n, T inv_lip,
                               T tau, T mom) {
  using Vt = typename Vec16<T>::type;
  constexpr int VEC = Vec16<T>::n;
  const long long nv = n / VEC;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    T gv[VEC], xv[VEC], yv[VEC];
    vec_split<T>(reinterpret_cast<const Vt *>(g)[i], gv);
    vec_split<T>(reinterpret_cast<const Vt *>(x)[i], xv);
    vec_split<T>(reinterpret_cast<const Vt *>(y)[i], yv);
#pragma unroll
    for (int u = 0; u < VEC; u++) {
      const T xn = soft<T>(yv[u] - gv[u] * inv_lip, tau);
      yv[u] = xn + mom * (xn - xv[u]);
      xv[u] = xn;
    }
    reinterpret_cast<Vt *>(x)[i] = vec_make<T>(xv);
    reinterpret_cast<Vt *>(y)[i] = vec_make<T>(yv);
  }
}

// out[img] += <a, b> over n elements per image (out zeroed by the caller)
template <typename T>
__global__ void k_dot(const T *__restrict__ a, const T *__restrict__ b, long long n, double *out) {
  const int img = blockIdx.y;
  const T *pa = a + (long long)img * n, *pb = b + (long long)img * n;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += (double)pa[i] * (double)pb[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += red[i];
    atomicAdd(out + img, t);
  }
}

template <typename T>
__global__ void k_scale(T *__restrict__ v, long long n, T alpha) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] *= alpha;
}

// uniform(-1, 1) from a 64-bit counter hash (splitmix64).  Pitch-padding entries get values too:
// W never reads them and the first power step (v <- W* R* R W v) writes them back as 0.
template <typename T>
__global__ void k_fill_seeded(T *__restrict__ v, long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
    v[i] = T(2.0 * u - 1.0);
  }
}

__global__ void k_fista_advance_t(double *t) { *t = (1.0 + sqrt(1.0 + 4.0 * *t * *t)) / 2.0; }

int grid_for(long long work, int nt) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (work + nt - 1) / nt;
  return (int)std::max<long long>(1, std::min<long long>(blocks, (long long)sms * 8));
}

}  // namespace

cudaError_t launch_fista_update(int dtype, const void *g, void *x, void *y, long long n, double t, double lambda,
                                double lip, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const double t_new = (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0;
  const double mom = (t - 1.0) / t_new;
  const int nt = 256;
  if (dtype == WL_F64) {
    k_fista_update<double><<<grid_for(n / 2, nt), nt, 0, s>>>(static_cast<const double *>(g), static_cast<double *>(x),
                                                              static_cast<double *>(y), n, 1.0 / lip, lambda / lip, mom);
  } else {
    k_fista_update<float><<<grid_for(n / 4, nt), nt, 0, s>>>(static_cast<const float *>(g), static_cast<float *>(x),
                                                             static_cast<float *>(y), n, (float)(1.0 / lip),
                                                             (float)(lambda / lip), (float)mom);
  }
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_fista_advance_t(double *t_dev, cudaStream_t s) {
  k_fista_advance_t<<<1, 1, 0, s>>>(t_dev);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_dot(int dtype, const void *a, const void *b, long long n, int batch, double *out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * (size_t)batch, s);
  if (e != cudaSuccess) return e;
  const int nt = 256;
  dim3 grid((unsigned)std::max(1, grid_for(n, nt) / std::max(1, batch)), (unsigned)batch);
  if (dtype == WL_F64)
    k_dot<double><<<grid, nt, 0, s>>>(static_cast<const double *>(a), static_cast<const double *>(b), n, out);
  else
    k_dot<float><<<grid, nt, 0, s>>>(static_cast<const float *>(a), static_cast<const float *>(b), n, out);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_scale(int dtype, void *v, long long n, double alpha, cudaStream_t s) {
  const int nt = 256;
  if (dtype == WL_F64)
    k_scale<double><<<grid_for(n, nt), nt, 0, s>>>(static_cast<double *>(v), n, alpha);
  else
    k_scale<float><<<grid_for(n, nt), nt, 0, s>>>(static_cast<float *>(v), n, (float)alpha);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_fill_seeded(int dtype, void *v, long long n, unsigned long long seed, cudaStream_t s) {
  const int nt = 256;
  if (dtype == WL_F64)
    k_fill_seeded<double><<<grid_for(n, nt), nt, 0, s>>>(static_cast<double *>(v), n, seed);
  else
    k_fill_seeded<float><<<grid_for(n, nt), nt, 0, s>>>(static_cast<float *>(v), n, seed);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace wl
