// Wavelet level kernels (sm_100a): one launch = one 2-D level of W-dagger / W* (analysis)
// or of W (synthesis), fused row + column passes in shared memory.
//
// Analysis core (R5):   out[k] = sum_{j<L} f[j] * yhat[2k+1-j]
// applied along axis 1 (rows) then axis 0 (columns); yhat = E y with E chosen per operator
// (P:52-98):  W-dagger: E_bc;  W*: E_zpd / periodisation / (E_sym^dagger)* = E_sym diag(1/c)
// (Eq. (4); reading R1).
// Synthesis = exact transpose, written in gather form per axis: the extended-position sample
//   u[t] = sum_{q < L/2} g[2q + 1 - (t & 1)] * c[floor(t/2) + q]
// so one coefficient window feeds the output pair (t = 2s, 2s+1).
#include <cuda_runtime.h>

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
  T lo[kMaxL], hi[kMaxL];
};

template <typename T>
struct SynParams {
  const T *in[4];
  long long in_pitch[4], in_bstride[4];
  int m0, m1;
  int coef_mod;
  T *out;
  long long out_pitch, out_bstride;
  int N0, N1, o0, o1;
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
template <typename T, int L, int TM, int TN>
struct AnaTile {
  static constexpr int RI = 2 * TM + L - 2;  // input rows of one output tile
  static constexpr int CI = 2 * TN + L - 2;  // input cols
  static constexpr int CIP = CI + 1;
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)RI * CIP + 2 * (size_t)RI * TN + RI + CI) + sizeof(int) * (RI + CI);
  }
};

template <typename T, int L, int TM, int TN, int NT>
__global__ void __launch_bounds__(NT) k_analysis(const AnaParams<T> p) {
  using Tile = AnaTile<T, L, TM, TN>;
  constexpr int RI = Tile::RI, CI = Tile::CI, CIP = Tile::CIP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *xin = reinterpret_cast<T *>(smem_raw);
  T *mL = xin + RI * CIP;
  T *mH = mL + RI * TN;
  T *rw = mH + RI * TN;
  T *cw = rw + RI;
  int *rs = reinterpret_cast<int *>(cw + CI);
  int *cs = rs + RI;

  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int k0 = blockIdx.y * TM, q0 = blockIdx.x * TN;
  const int rbase = 2 * k0 + 2 - L, cbase = 2 * q0 + 2 - L;
  const T *in = p.in + (long long)b * p.in_bstride;

  for (int i = tid; i < RI; i += NT) rs[i] = ext_src<T>(rbase + i, p.n0, p.ext, L - 1, rw[i]);
  for (int i = tid; i < CI; i += NT) cs[i] = ext_src<T>(cbase + i, p.n1, p.ext, L - 1, cw[i]);
  __syncthreads();
  for (int idx = tid; idx < RI * CI; idx += NT) {
    int ri = idx / CI, ci = idx - ri * CI;
    int s0 = rs[ri], s1 = cs[ci];
    T v = T(0);
    if (s0 >= 0 && s1 >= 0) v = in[(long long)s0 * p.in_pitch + s1] * (rw[ri] * cw[ci]);
    xin[ri * CIP + ci] = v;
  }
  __syncthreads();
  // axis 1: out col kk uses local input cols 2kk + L-1-j
  for (int idx = tid; idx < RI * TN; idx += NT) {
    int ri = idx / TN, kk = idx - ri * TN;
    const T *xr = xin + ri * CIP + 2 * kk;
    T aL = T(0), aH = T(0);
#pragma unroll
    for (int j = 0; j < L; j++) {
      T v = xr[L - 1 - j];
      aL = fma(p.lo[j], v, aL);
      aH = fma(p.hi[j], v, aH);
    }
    mL[ri * TN + kk] = aL;
    mH[ri * TN + kk] = aH;
  }
  __syncthreads();
  // axis 0
  for (int idx = tid; idx < TM * TN; idx += NT) {
    int kr = idx / TN, kk = idx - kr * TN;
    T LL = T(0), HL = T(0), LH = T(0), HH = T(0);
#pragma unroll
    for (int j = 0; j < L; j++) {
      int r = 2 * kr + L - 1 - j;
      T vL = mL[r * TN + kk], vH = mH[r * TN + kk];
      LL = fma(p.lo[j], vL, LL);
      HL = fma(p.hi[j], vL, HL);
      LH = fma(p.lo[j], vH, LH);
      HH = fma(p.hi[j], vH, HH);
    }
    int k = k0 + kr, q = q0 + kk;
    if (q >= p.m1) LL = LH = HL = HH = T(0);
    if (k < p.m0 && q < p.m1s) {
      p.out[0][(long long)b * p.out_bstride[0] + (long long)k * p.out_pitch[0] + q] = LL;
      p.out[1][(long long)b * p.out_bstride[1] + (long long)k * p.out_pitch[1] + q] = LH;
      p.out[2][(long long)b * p.out_bstride[2] + (long long)k * p.out_pitch[2] + q] = HL;
      p.out[3][(long long)b * p.out_bstride[3] + (long long)k * p.out_pitch[3] + q] = HH;
    }
  }
}

// ----------------------------------------------------------------- synthesis
template <typename T, int L, int TI, int TP>
struct SynTile {
  static constexpr int H = L / 2;
  static constexpr int KR = TI / 2 + H - 1;
  static constexpr int KC = TP / 2 + H - 1;
  static constexpr int KCP = KC + 1;
  static constexpr size_t smem_bytes() {
    return sizeof(T) * (4 * (size_t)KR * KCP + 2 * (size_t)TI * KCP);
  }
};

__device__ __forceinline__ int floor_div2(int t) { return t >> 1; }  // arithmetic shift = floor

template <typename T, int L, int TI, int TP, int NT>
__global__ void __launch_bounds__(NT) k_synthesis(const SynParams<T> p) {
  using Tile = SynTile<T, L, TI, TP>;
  constexpr int H = Tile::H, KR = Tile::KR, KC = Tile::KC, KCP = Tile::KCP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *cf = reinterpret_cast<T *>(smem_raw);  // [4][KR][KCP]
  T *VL = cf + 4 * KR * KCP;                // [TI][KCP]
  T *VH = VL + TI * KCP;

  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  // tiles cover extended positions t in [o, o+N) starting at an even t
  const int T0 = 2 * floor_div2(p.o0) + blockIdx.y * TI;
  const int P0 = 2 * floor_div2(p.o1) + blockIdx.x * TP;
  const int kr0 = T0 / 2, kc0 = P0 / 2;  // T0, P0 even

  for (int idx = tid; idx < 4 * KR * KC; idx += NT) {
    int band = idx / (KR * KC);
    int rem = idx - band * KR * KC;
    int r = rem / KC, c = rem - r * KC;
    int kr = kr0 + r, kc = kc0 + c;
    T v = T(0);
    if (p.coef_mod) {
      kr %= p.m0; if (kr < 0) kr += p.m0;
      kc %= p.m1; if (kc < 0) kc += p.m1;
      v = p.in[band][(long long)b * p.in_bstride[band] + (long long)kr * p.in_pitch[band] + kc];
    } else if (kr >= 0 && kr < p.m0 && kc >= 0 && kc < p.m1) {
      v = p.in[band][(long long)b * p.in_bstride[band] + (long long)kr * p.in_pitch[band] + kc];
    }
    cf[(band * KR + r) * KCP + c] = v;
  }
  __syncthreads();
  // axis 0: (LL, HL) -> VL ; (LH, HH) -> VH ; rows t = 2s (taps 2q+1) and 2s+1 (taps 2q)
  const T *cLL = cf, *cLH = cf + KR * KCP, *cHL = cf + 2 * KR * KCP, *cHH = cf + 3 * KR * KCP;
  for (int idx = tid; idx < (TI / 2) * KC; idx += NT) {
    int s = idx / KC, c = idx - s * KC;
    T eL = T(0), oL = T(0), eH = T(0), oH = T(0);
#pragma unroll
    for (int q = 0; q < H; q++) {
      int o = (s + q) * KCP + c;
      T a = cLL[o], d = cHL[o], a2 = cLH[o], d2 = cHH[o];
      eL = fma(p.lo[2 * q + 1], a, fma(p.hi[2 * q + 1], d, eL));
      oL = fma(p.lo[2 * q], a, fma(p.hi[2 * q], d, oL));
      eH = fma(p.lo[2 * q + 1], a2, fma(p.hi[2 * q + 1], d2, eH));
      oH = fma(p.lo[2 * q], a2, fma(p.hi[2 * q], d2, oH));
    }
    VL[(2 * s) * KCP + c] = eL;
    VL[(2 * s + 1) * KCP + c] = oL;
    VH[(2 * s) * KCP + c] = eH;
    VH[(2 * s + 1) * KCP + c] = oH;
  }
  __syncthreads();
  // axis 1
  T *out = p.out + (long long)b * p.out_bstride;
  for (int idx = tid; idx < TI * (TP / 2); idx += NT) {
    int ii = idx / (TP / 2), s = idx - ii * (TP / 2);
    T e = T(0), o = T(0);
#pragma unroll
    for (int q = 0; q < H; q++) {
      T vL = VL[ii * KCP + s + q], vH = VH[ii * KCP + s + q];
      e = fma(p.lo[2 * q + 1], vL, fma(p.hi[2 * q + 1], vH, e));
      o = fma(p.lo[2 * q], vL, fma(p.hi[2 * q], vH, o));
    }
    int i = T0 + ii - p.o0;
    int c0 = P0 + 2 * s - p.o1;
    if (i >= 0 && i < p.N0) {
      if (c0 >= 0 && c0 < p.N1) out[(long long)i * p.out_pitch + c0] = e;
      if (c0 + 1 >= 0 && c0 + 1 < p.N1) out[(long long)i * p.out_pitch + c0 + 1] = o;
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
  constexpr int TM = sizeof(T) == 4 ? 32 : 16;
  constexpr int TN = TM, NT = 256;
  using Tile = AnaTile<T, L, TM, TN>;
  AnaParams<T> p;
  p.in = static_cast<const T *>(a.in);
  p.in_pitch = a.in_pitch; p.in_bstride = a.in_bstride; p.n0 = a.n0; p.n1 = a.n1;
  for (int i = 0; i < 4; i++) {
    p.out[i] = static_cast<T *>(a.out[i]);
    p.out_pitch[i] = a.out_pitch[i]; p.out_bstride[i] = a.out_bstride[i];
  }
  p.m0 = a.m0; p.m1 = a.m1; p.ext = a.ext;
  p.m1s = (int)((a.m1 + (16 / sizeof(T)) - 1) / (16 / sizeof(T)) * (16 / sizeof(T)));
  for (int j = 0; j < kMaxL; j++) { p.lo[j] = T(j < L ? a.lo[j] : 0); p.hi[j] = T(j < L ? a.hi[j] : 0); }
  size_t smem = Tile::smem_bytes();
  auto kern = k_analysis<T, L, TM, TN, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.m1 + TN - 1) / TN, (a.m0 + TM - 1) / TM, a.batch);
  kern<<<grid, NT, smem, s>>>(p);
  g_launches++;
  return cudaGetLastError();
}

template <typename T, int L>
cudaError_t launch_synthesis_t(const SynthesisArgs &a, cudaStream_t s) {
  constexpr int TI = sizeof(T) == 4 ? 64 : 32;
  constexpr int TP = TI, NT = 256;
  using Tile = SynTile<T, L, TI, TP>;
  SynParams<T> p;
  for (int i = 0; i < 4; i++) {
    p.in[i] = static_cast<const T *>(a.in[i]);
    p.in_pitch[i] = a.in_pitch[i]; p.in_bstride[i] = a.in_bstride[i];
  }
  p.m0 = a.m0; p.m1 = a.m1; p.coef_mod = a.coef_mod;
  p.out = static_cast<T *>(a.out);
  p.out_pitch = a.out_pitch; p.out_bstride = a.out_bstride;
  p.N0 = a.N0; p.N1 = a.N1; p.o0 = a.o0; p.o1 = a.o1;
  for (int j = 0; j < kMaxL; j++) { p.lo[j] = T(j < L ? a.lo[j] : 0); p.hi[j] = T(j < L ? a.hi[j] : 0); }
  size_t smem = Tile::smem_bytes();
  auto kern = k_synthesis<T, L, TI, TP, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // extended span [o, o+N) starting from the even position 2*floor(o/2)
  int span0 = a.o0 + a.N0 - 2 * (a.o0 >> 1), span1 = a.o1 + a.N1 - 2 * (a.o1 >> 1);
  dim3 grid((span1 + TP - 1) / TP, (span0 + TI - 1) / TI, a.batch);
  kern<<<grid, NT, smem, s>>>(p);
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

template <typename T>
cudaError_t dispatch_synthesis(const SynthesisArgs &a, cudaStream_t s) {
  switch (a.L) {
    case 2: return launch_synthesis_t<T, 2>(a, s);
    case 4: return launch_synthesis_t<T, 4>(a, s);
    case 8: return launch_synthesis_t<T, 8>(a, s);
    case 10: return launch_synthesis_t<T, 10>(a, s);
    case 16: return launch_synthesis_t<T, 16>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_analysis(int dtype, const AnalysisArgs &a, cudaStream_t s) {
  if (a.batch == 0 || a.m0 == 0 || a.m1 == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_analysis<double>(a, s) : dispatch_analysis<float>(a, s);
}

cudaError_t launch_synthesis(int dtype, const SynthesisArgs &a, cudaStream_t s) {
  if (a.batch == 0 || a.N0 == 0 || a.N1 == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_synthesis<double>(a, s) : dispatch_synthesis<float>(a, s);
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
