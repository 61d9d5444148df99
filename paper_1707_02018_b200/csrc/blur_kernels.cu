// Separable PSF blur kernels (sm_100a): R, and the fused middle stage of grad f,
// s = R*(R u - b) (= R (R u - b) for the symmetric PSFs the plan accepts), optionally
// with f = 1/2 ||R u - b||^2.
//
// Per axis (reading R12):  (R_a y)[i] = sum_{t=-h..h} k[t] yhat[i - t],
// yhat = half-point symmetric extension of y:  yhat[-1-i] = y[i], yhat[n+i] = y[n-1-i].
//
// Streaming column-strip design (DESIGN.md §6 "k_blur_stream"):
//   A CTA owns TW output columns of one image and a run of output rows; it walks down
//   extended rows G at a time.  Per iteration
//     A  cp.async the next G input rows (TW + 2A columns) into a double buffer;
//     B  horizontal pass from a register window -> h1 history (2h carried rows + G new);
//     C  vertical pass down a column pair (register window over the h1 history) -> output
//        rows (R), or r = V H u - b written over the b rows in bbuf (residual; b rows are
//        cp.async-prefetched one iteration ahead like u);
//     H2 horizontal pass over the r rows -> h2 history;     (residual only)
//     D  vertical pass over the h2 history -> s rows, stored. (residual only)
//   The last 2h rows of each history buffer are copied to its head once per iteration, so
//   every window is addressed with compile-time offsets.
//   Vertical halos live in the histories and are never recomputed inside a run; horizontal
//   halos cost 2*HB/TW extra columns.  Work is scheduled persistently: the flattened
//   (image, strip, row) space is cut into equal contiguous runs, one per resident CTA.
//
// Boundary handling.  With a symmetric PSF, (k * yhat) is itself symmetric about -1/2 and
// n-1/2, so the reflected halo of the second blur equals the first blur evaluated at the
// reflected position: r_ext(q) = (k * u_ext)(q) - b_ext(q) for the infinite symmetric
// extension, which agrees with the single reflection of R on [-n, 2n) (n >= h).  Every
// load therefore reads source index refl(p) and the passes are plain convolutions.
//
// FP32 arithmetic uses packed FFMA2 (fma.rn.f32x2): vertical passes pair adjacent
// columns; horizontal passes split each 2h+1-tap sum into (even, odd) tap pairs over
// naturally aligned sample pairs and add the two halves at the end.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

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
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <typename P>
__device__ __forceinline__ P zero2() {
  P z;
  z.x = 0;
  z.y = 0;
  return z;
}

// Source index of extended position p under the infinite half-point symmetric extension.
__device__ __forceinline__ int refl_inf(int p, int n) {
  if (p >= 0 && p < n) return p;
  const int m = 2 * n;
  p %= m;
  if (p < 0) p += m;
  return p < n ? p : m - 1 - p;
}

template <typename T, int HW, bool RESID>
struct BCfg {
  using P = typename Pair<T>::t;
  static constexpr int VEC = Vec16<T>::n;
  static constexpr int TW = sizeof(T) == 4 ? 128 : 64;  // output columns per strip
  // extended rows per iteration; G >= 2HW keeps the history move [G, G+2HW) -> [0, 2HW) non-overlapping
  static constexpr int G = (2 * HW > 16) ? 32 : 16;
  static constexpr int V = 8;                            // outputs per thread, horizontal passes
  static constexpr int VC = 4;                           // output rows per thread, vertical passes
  static constexpr int HB = RESID ? round_up_c(HW, 4) : 0;  // r columns beyond the tile per side
  static constexpr int NH1 = TW + 2 * HB;                // columns of the first horizontal pass
  static constexpr int A = round_up_c(HB + HW, VEC);     // u columns loaded beyond the tile per side
  static constexpr int UW = TW + 2 * A;
  static constexpr int NV = UW / VEC;                    // 16-byte chunks per u row
  static constexpr int OFF1 = A - HB - HW;               // window offset of pass B
  static constexpr int OFF2 = HB - HW;                   // window offset of pass H2
  static constexpr int NW1 = round_up_c(OFF1 + V + 2 * HW, VEC);
  static constexpr int NW2 = round_up_c(OFF2 + V + 2 * HW, VEC);
  static constexpr int UP = conflict_free_pitch<T>(UW);
  static constexpr int R1P = conflict_free_pitch<T>(NH1);
  static constexpr int R2P = conflict_free_pitch<T>(TW);
  static constexpr int HR = 2 * HW + G;                  // rows of a history buffer (2HW carried + G new)
  static_assert(2 * HW <= G, "history move must not overlap");
  static_assert(NH1 % V == 0 && TW % V == 0, "segments");
  static_assert(8 * (NH1 / V - 1) + NW1 <= UW, "pass B window overruns the u row");
  static_assert(!RESID || 8 * (TW / V - 1) + NW2 <= NH1, "pass H2 window overruns rbuf");
  static constexpr int ITEMS_B = (NH1 / V) * G;
  static constexpr int ITEMS_C = (RESID ? NH1 / 2 : TW / 2) * (G / VC);
  static constexpr int ITEMS_H2 = RESID ? (TW / V) * G : 0;
  static constexpr int ITEMS_D = RESID ? (TW / 2) * (G / VC) : 0;
  static constexpr int NT = round_up_c(std::max(std::max(ITEMS_B, ITEMS_C), std::max(ITEMS_H2, ITEMS_D)), 32);
  static constexpr int NVB = RESID ? NH1 / VEC : 0;                  // 16-byte chunks per b row
  static constexpr int NCHUNK = G * (NV + NVB);                       // chunks loaded per iteration
  static constexpr int NSLOT = (NCHUNK + NT - 1) / NT;                // chunks per thread per iteration
  static constexpr int MV1 = 2 * HW * (NH1 / VEC);                   // 16-byte moves of h1 history
  static constexpr int MV2 = RESID ? 2 * HW * (TW / VEC) : 0;        // 16-byte moves of h2 history
  static constexpr int NM1 = (MV1 + NT - 1) / NT, NM2 = (MV2 + NT - 1) / NT;
  static constexpr size_t smem_bytes() {
    return sizeof(T) * (2 * (size_t)G * UP + (size_t)HR * R1P + (RESID ? 2 * (size_t)G * R1P + (size_t)HR * R2P : 0));
  }
};

template <typename T, int HW>
struct BlurStreamParams {
  using P = typename Pair<T>::t;
  const T *u;
  const T *b;  // residual only
  T *out;
  double *f;   // residual only (nullable)
  int h, w, nstrips;
  long long total_rows, rows_per_cta;
  int fast;                  // 16-byte aligned rows: cp.async / vector paths allowed
  P cc[2 * HW + 1];          // (c[d], c[d]),  c[d] = k[2h - d]: out[i] = sum_d c[d] yhat[i - h + d]
  P ce[HW + 1], co[HW + 1];  // (c[2m], c[2m+1]) and (c[2m-1], c[2m]) (out-of-range taps = 0)
};

// Horizontal pass: V outputs out[j] = sum_d c[d] win[j + OFF + d] from a VEC-aligned row window.
template <typename T, int HW, int V, int OFF, int NW>
__device__ __forceinline__ void hpass(const T *src, const BlurStreamParams<T, HW> &p, T *outv) {
  using P = typename Pair<T>::t;
  using Vt = typename Vec16<T>::type;
  constexpr int VEC = Vec16<T>::n;
  T win[NW];
#pragma unroll
  for (int i = 0; i < NW / VEC; i++) vec_split<T>(reinterpret_cast<const Vt *>(src)[i], win + i * VEC);
#pragma unroll
  for (int j = 0; j < V; j++) {
    const int s = j + OFF;
    P acc = zero2<P>();
    if (s % 2 == 0) {
#pragma unroll
      for (int m = 0; m <= HW; m++) {
        P x;
        x.x = win[s + 2 * m];
        x.y = (2 * m + 1 <= 2 * HW) ? win[s + 2 * m + 1] : T(0);
        acc = fma2(p.ce[m], x, acc);
      }
    } else {
#pragma unroll
      for (int m = 0; m <= HW; m++) {
        P x;
        x.x = (m > 0) ? win[s - 1 + 2 * m] : T(0);
        x.y = win[s + 2 * m];
        acc = fma2(p.co[m], x, acc);
      }
    }
    outv[j] = acc.x + acc.y;
  }
}

// Vertical pass over a column pair: VC outputs from VC + 2HW consecutive rows at `src` (pitch).
template <typename T, int HW, int VC, int PITCH>
__device__ __forceinline__ void vpass(const T *src, const BlurStreamParams<T, HW> &p, typename Pair<T>::t *acc) {
  using P = typename Pair<T>::t;
  P win[VC + 2 * HW];
#pragma unroll
  for (int i = 0; i < VC + 2 * HW; i++) win[i] = *reinterpret_cast<const P *>(src + i * PITCH);
#pragma unroll
  for (int v = 0; v < VC; v++) {  // two independent chains (even / odd taps) per output
    P a = zero2<P>(), b = zero2<P>();
#pragma unroll
    for (int d = 0; d < 2 * HW + 1; d += 2) a = fma2(p.cc[d], win[v + d], a);
#pragma unroll
    for (int d = 1; d < 2 * HW + 1; d += 2) b = fma2(p.cc[d], win[v + d], b);
    acc[v] = add2(a, b);
  }
}

template <typename T>
__device__ __forceinline__ void store_pair(T *row, int col, typename Pair<T>::t v, bool vec_ok, int w) {
  if (vec_ok) {
    *reinterpret_cast<typename Pair<T>::t *>(row + col) = v;
  } else {
    if (col < w) row[col] = v.x;
    if (col + 1 < w) row[col + 1] = v.y;
  }
}

template <typename T, int HW, bool RESID>
__global__ void __launch_bounds__(BCfg<T, HW, RESID>::NT, (sizeof(T) == 4 && BCfg<T, HW, RESID>::NT <= 320) ? 3 : 1)
    k_blur_stream(const BlurStreamParams<T, HW> p) {
  using C = BCfg<T, HW, RESID>;
  using P = typename C::P;
  using Vt = typename Vec16<T>::type;
  constexpr int G = C::G, VC = C::VC, VEC = C::VEC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *ubuf = reinterpret_cast<T *>(smem_raw);  // [2][G][UP]   u rows e .. e+G-1
  T *h1 = ubuf + 2 * G * C::UP;               // [HR][R1P]    h1 rows e-2HW .. e+G-1
  T *bbuf = h1 + C::HR * C::R1P;              // [2][G][R1P]  b, then r, rows e-HW .. e-HW+G-1  (residual)
  T *h2 = bbuf + 2 * G * C::R1P;              // [HR][R2P]    h2 rows e-3HW .. e-HW+G-1     (residual)
  __shared__ double red[C::NT / 32];

  const int tid = threadIdx.x;
  constexpr int HA = RESID ? 2 * HW : HW;  // first loaded row = r0 - HA
  long long g = (long long)blockIdx.x * p.rows_per_cta;
  const long long gend = std::min(p.total_rows, g + p.rows_per_cta);

  // per-thread work items of every stage (fixed for the whole kernel)
  const bool actB = tid < C::ITEMS_B;
  const int rowB = tid % G, segB = tid / G;
  constexpr int NPC = RESID ? C::NH1 / 2 : C::TW / 2;
  const bool actC = tid < C::ITEMS_C;
  const int mC = tid % NPC, grpC = tid / NPC;
  const bool actH2 = RESID && tid < C::ITEMS_H2;
  const bool actD = RESID && tid < C::ITEMS_D;
  const int mD = tid % (C::TW / 2), grpD = tid / (C::TW / 2);
  // chunks of stage A: slot k = row r, 16-byte chunk v of a u row (v < NV) or of a b row
  int slot[C::NSLOT];  // (r << 16) | v, or -1
#pragma unroll
  for (int k = 0; k < C::NSLOT; k++) {
    const int idx = tid + k * C::NT;
    const bool isb = idx >= G * C::NV;
    const int j = isb ? idx - G * C::NV : idx;
    const int per = isb ? C::NVB : C::NV;
    slot[k] = idx < C::NCHUNK ? ((j / per) << 16) | (isb ? C::NV + j % per : j % per) : -1;
  }

  while (g < gend) {
    const int unit = (int)(g / p.h);
    const int r0 = (int)(g - (long long)unit * p.h);
    const int r1 = (int)std::min<long long>(p.h, r0 + (gend - g));
    g += r1 - r0;
    const int img = unit / p.nstrips, strip = unit - img * p.nstrips;
    const int c0 = strip * C::TW;
    const T *u = p.u + (long long)img * p.h * p.w;
    const T *bimg = RESID ? p.b + (long long)img * p.h * p.w : nullptr;
    T *out = p.out + (long long)img * p.h * p.w;
    const int e_begin = r0 - HA;
    // output row = loaded row - 2*HA; n_it iterations cover output rows [r0, r1)
    const int n_it = (r1 - r0 + 2 * HA + G - 1) / G;
    // per-run column facts
    const int colC = RESID ? c0 - C::HB + 2 * mC : c0 + 2 * mC;      // frame column of stage C's pair
    const bool ovecC = p.fast && colC + 1 < p.w;
    P fmask;                                                          // f counts each pixel once
    fmask.x = (colC >= c0 && colC < c0 + C::TW && colC < p.w) ? T(1) : T(0);
    fmask.y = (colC + 1 >= c0 && colC + 1 < c0 + C::TW && colC + 1 < p.w) ? T(1) : T(0);
    const int colD = c0 + 2 * mD;
    const bool ovecD = p.fast && colD + 1 < p.w;
    double fsum = 0.0;

    // stage A: u rows e0 .. e0+G-1 into ubuf slot `ub`; (residual) b rows e0-HW .. into bbuf slot `ub`
    auto load_rows = [&](int ub, int e0) {
#pragma unroll
      for (int k = 0; k < C::NSLOT; k++) {
        if (slot[k] < 0) continue;
        const int sl_r = slot[k] >> 16, sl_v = slot[k] & 0xffff;
        const bool isb = RESID && sl_v >= C::NV;
        const int v = isb ? sl_v - C::NV : sl_v;
        const int sr = refl_inf(e0 + sl_r - (isb ? HW : 0), p.h);
        const int cg = isb ? c0 - C::HB + v * VEC : c0 - C::A + v * VEC;
        T *dst = isb ? bbuf + (ub * G + sl_r) * C::R1P + v * VEC
                     : ubuf + (ub * G + sl_r) * C::UP + v * VEC;
        const T *row = (isb ? bimg : u) + (long long)sr * p.w;
        if (p.fast && cg >= 0 && cg + VEC <= p.w) {
          cp_async16(dst, row + cg);
        } else {
          T z[VEC];
#pragma unroll
          for (int i = 0; i < VEC; i++) z[i] = row[refl_inf(cg + i, p.w)];
          *reinterpret_cast<Vt *>(dst) = vec_make<T>(z);
        }
      }
    };

    __syncthreads();  // previous run's smem readers are done
    load_rows(0, e_begin);
    cp_async_commit();
    for (int it = 0; it < n_it; it++) {
      const int e = e_begin + it * G;
      cp_async_wait_all();
      __syncthreads();  // (1) u rows landed; previous D / moves done
      if (it + 1 < n_it) {
        load_rows((it + 1) & 1, e + G);
        cp_async_commit();
      }
      if (RESID) {
        // carry the last 2HW h2 rows to the head of the h2 history (D of it-1 has finished)
#pragma unroll
        for (int k = 0; k < C::NM2; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV2) {
            const int r = idx / (C::TW / VEC), c = idx % (C::TW / VEC);
            *reinterpret_cast<Vt *>(h2 + r * C::R2P + c * VEC) =
                *reinterpret_cast<const Vt *>(h2 + (r + G) * C::R2P + c * VEC);
          }
        }
      } else if (it > 0) {
        // R: carry the h1 history now (stage C of it-1 finished at barrier (1))
#pragma unroll
        for (int k = 0; k < C::NM1; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV1) {
            const int r = idx / (C::NH1 / VEC), c = idx % (C::NH1 / VEC);
            *reinterpret_cast<Vt *>(h1 + r * C::R1P + c * VEC) =
                *reinterpret_cast<const Vt *>(h1 + (r + G) * C::R1P + c * VEC);
          }
        }
        __syncthreads();
      }
      // B: horizontal pass of u rows e .. e+G-1 -> h1 rows 2HW .. 2HW+G-1
      if (actB) {
        T hv[C::V];
        hpass<T, HW, C::V, C::OFF1, C::NW1>(ubuf + (it & 1) * G * C::UP + rowB * C::UP + C::V * segB, p, hv);
        Vt *dst = reinterpret_cast<Vt *>(h1 + (2 * HW + rowB) * C::R1P + C::V * segB);
#pragma unroll
        for (int i = 0; i < C::V / VEC; i++) dst[i] = vec_make<T>(hv + i * VEC);
      }
      __syncthreads();  // (2)
      // C: vertical pass -> rows x = e - HW + grpC*VC + v  (h1 index of x - HW is grpC*VC + v)
      if (actC) {
        const int xb = e - HW + grpC * VC;
        P acc[VC];
        vpass<T, HW, VC, C::R1P>(h1 + grpC * VC * C::R1P + 2 * mC, p, acc);
        if (RESID) {
          P fa = zero2<P>();
#pragma unroll
          for (int v = 0; v < VC; v++) {
            P *rb = reinterpret_cast<P *>(bbuf + ((it & 1) * G + grpC * VC + v) * C::R1P + 2 * mC);
            const P r = sub2(acc[v], *rb);
            *rb = r;
            const int x = xb + v;
            if (x >= r0 && x < r1) {
              P rm;
              rm.x = r.x * fmask.x;
              rm.y = r.y * fmask.y;
              fa = fma2(rm, r, fa);
            }
          }
          fsum += (double)fa.x + (double)fa.y;
        } else {
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const int x = xb + v;
            if (x >= r0 && x < r1) store_pair<T>(out + (long long)x * p.w, colC, acc[v], ovecC, p.w);
          }
        }
      }
      if (RESID) {
        __syncthreads();  // (3) r rows complete; h1 readers done
        // H2: horizontal pass of r rows -> h2 rows 2HW .. 2HW+G-1
        if (actH2) {
          T hv[C::V];
          hpass<T, HW, C::V, C::OFF2, C::NW2>(bbuf + ((it & 1) * G + rowB) * C::R1P + C::V * segB, p, hv);
          Vt *dst = reinterpret_cast<Vt *>(h2 + (2 * HW + rowB) * C::R2P + C::V * segB);
#pragma unroll
          for (int i = 0; i < C::V / VEC; i++) dst[i] = vec_make<T>(hv + i * VEC);
        }
        // carry the last 2HW h1 rows to the head of the h1 history
#pragma unroll
        for (int k = 0; k < C::NM1; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV1) {
            const int r = idx / (C::NH1 / VEC), c = idx % (C::NH1 / VEC);
            *reinterpret_cast<Vt *>(h1 + r * C::R1P + c * VEC) =
                *reinterpret_cast<const Vt *>(h1 + (r + G) * C::R1P + c * VEC);
          }
        }
        __syncthreads();  // (4)
        // D: vertical pass -> s rows y = e - 2HW + grpD*VC + v (h2 index of y - HW is grpD*VC + v)
        const int yb = e - 2 * HW + grpD * VC;
        if (actD && yb + VC > r0 && yb < r1) {
          P acc[VC];
          vpass<T, HW, VC, C::R2P>(h2 + grpD * VC * C::R2P + 2 * mD, p, acc);
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const int y = yb + v;
            if (y >= r0 && y < r1) store_pair<T>(out + (long long)y * p.w, colD, acc[v], ovecD, p.w);
          }
        }
      }
    }
    if (RESID && p.f) {
      for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
      if ((tid & 31) == 0) red[tid >> 5] = fsum;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < C::NT / 32; i++) s += red[i];
        atomicAdd(p.f + img, 0.5 * s);
      }
    }
  }
}

template <typename T, int HW, bool RESID>
cudaError_t launch_stream(const BlurArgs &a, cudaStream_t s) {
  using C = BCfg<T, HW, RESID>;
  using P = typename C::P;
  BlurStreamParams<T, HW> p;
  p.u = static_cast<const T *>(a.in);
  p.b = static_cast<const T *>(a.b);
  p.out = static_cast<T *>(a.out);
  p.f = RESID ? a.f : nullptr;
  p.h = (int)a.h;
  p.w = (int)a.w;
  p.nstrips = (int)((a.w + C::TW - 1) / C::TW);
  bool fast = (a.w % C::VEC == 0) && (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) &&
              (reinterpret_cast<uintptr_t>(a.out) % 16 == 0);
  if (RESID) fast = fast && (reinterpret_cast<uintptr_t>(a.b) % 16 == 0);
  p.fast = fast;
  double c[2 * HW + 1];
  for (int d = 0; d <= 2 * HW; d++) c[d] = a.taps[2 * HW - d];
  auto cd = [&](int d) { return (d >= 0 && d <= 2 * HW) ? c[d] : 0.0; };
  for (int d = 0; d <= 2 * HW; d++) {
    p.cc[d].x = T(c[d]);
    p.cc[d].y = T(c[d]);
  }
  for (int m = 0; m <= HW; m++) {
    p.ce[m].x = T(cd(2 * m));
    p.ce[m].y = T(cd(2 * m + 1));
    p.co[m].x = T(cd(2 * m - 1));
    p.co[m].y = T(cd(2 * m));
  }
  (void)sizeof(P);
  const size_t smem = C::smem_bytes();
  auto kern = k_blur_stream<T, HW, RESID>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, smem);
  if (e != cudaSuccess) return e;
  occ = std::max(occ, 1);
  p.total_rows = (long long)a.batch * p.nstrips * p.h;
  // one run per resident CTA, but at least 4 iterations of rows per run (halo rows amortised)
  const long long min_rows = 4LL * C::G;
  long long grid = std::min<long long>((long long)sms * occ, (p.total_rows + min_rows - 1) / min_rows);
  grid = std::max<long long>(grid, 1);
  p.rows_per_cta = (p.total_rows + grid - 1) / grid;
  grid = (p.total_rows + p.rows_per_cta - 1) / p.rows_per_cta;
  if (RESID && a.f) {
    e = cudaMemsetAsync(a.f, 0, sizeof(double) * (size_t)a.batch, s);
    if (e != cudaSuccess) return e;
  }
  kern<<<(unsigned)grid, C::NT, smem, s>>>(p);
  g_launches++;
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_blur(const BlurArgs &a, cudaStream_t s, bool residual) {
  switch (a.ntaps / 2) {
#define WL_BLUR_CASE(H) \
  case H: return residual ? launch_stream<T, H, true>(a, s) : launch_stream<T, H, false>(a, s);
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
