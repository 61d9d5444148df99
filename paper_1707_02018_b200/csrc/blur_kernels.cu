// Separable PSF blur kernels (sm_100a): R, and the fused middle stage of grad f,
// s = R*(R u - b) (= R (R u - b) for the symmetric PSFs the plan accepts), optionally
// with f = 1/2 ||R u - b||^2.
//
// Per axis (reading R12):  (R_a y)[i] = sum_{t=-h..h} k[t] yhat[i - t],
// yhat = half-point symmetric extension of y:  yhat[-1-i] = y[i], yhat[n+i] = y[n-1-i].
//
// Streaming column-strip design (DESIGN.md §6 "k_blur_stream"):
//   A CTA owns TW output columns of one image and a band of rows; it walks down the band G
//   extended rows per iteration:
//     A  the next G u rows (and, residual, the G b rows the next iteration subtracts) land
//        in a double buffer: one TMA box each, issued by one thread and completed on an
//        mbarrier (row blocks touching the image top/bottom are gathered row-reflected with
//        cp.async instead);
//     B  horizontal pass from a register window -> h1 history (2h carried rows + G new);
//     C  vertical pass down a column pair (register window over the h1 history) -> output
//        rows (R), or r = V H u - b written over the b rows (residual);
//     H2 horizontal pass over the r rows -> h2 history;        (residual only)
//     D  vertical pass over the h2 history -> s rows, stored.  (residual only)
//   The last 2h rows of each history are copied to its head once per iteration, so every
//   window is addressed with compile-time offsets; vertical halos are never recomputed
//   inside a band.  Runs are ordered (image, band, strip) and handed to persistent CTAs,
//   so CTAs on neighbouring strips stream the same rows together and the horizontal halo
//   columns are shared through L2.
//
// Boundary handling.  With a symmetric PSF, (k * yhat) is itself symmetric about -1/2 and
// n-1/2, so the reflected halo of the second blur equals the first blur evaluated at the
// reflected position: r_ext(q) = (k * u_ext)(q) - b_ext(q) for the infinite symmetric
// extension, which agrees with the single reflection of R on [-n, 2n) (n >= h).  Rows are
// reflected when loaded; columns outside the image (zero-filled by TMA) are never read:
// the horizontal passes read the mirrored column instead (u and r are both symmetric
// about the image edges), and outputs outside the image are skipped.
//
// FP32 arithmetic uses packed FFMA2 (fma.rn.f32x2): vertical passes pair adjacent
// columns; horizontal passes split each 2h+1-tap sum into (even, odd) tap pairs over
// naturally aligned sample pairs and add the two halves at the end.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

template <typename T, int HW, bool RESID>
struct BCfg {
  using P = typename Pair<T>::t;
  static constexpr int VEC = Vec16<T>::n;
  // output columns per strip: the residual frame NH1 = TW + 2HB is a multiple of the 16-item warps
#ifndef WL_BLUR_TWR
#define WL_BLUR_TWR 112
#endif
  static constexpr int TW = sizeof(T) == 4 ? (RESID ? WL_BLUR_TWR : 128) : (RESID ? 48 : 64);
  // extended rows per iteration; G >= 2HW keeps the history move [G, G+2HW) -> [0, 2HW) non-overlapping
#ifndef WL_BLUR_G
#define WL_BLUR_G 16
#endif
  static constexpr int G = (2 * HW > WL_BLUR_G) ? 32 : WL_BLUR_G;
#ifndef WL_BLUR_V
#define WL_BLUR_V 8
#endif
#ifndef WL_BLUR_VC
#define WL_BLUR_VC 4
#endif
  static constexpr int HB_ = RESID ? round_up_c(HW, 4) : 0;
  static constexpr int VR = sizeof(T) == 4 ? WL_BLUR_V : 8;
  static constexpr int V = ((TW + 2 * HB_) % VR == 0 && TW % VR == 0) ? VR : 8;  // outputs per item, horizontal passes
  static constexpr int VC = sizeof(T) == 4 ? WL_BLUR_VC : 4;  // output rows per item, vertical passes
  static constexpr int HB = RESID ? round_up_c(HW, 4) : 0;  // r columns beyond the tile per side
  static constexpr int NH1 = TW + 2 * HB;                   // columns of h1 / r
  static constexpr int A = round_up_c(HB + HW, VEC);        // u columns loaded beyond the tile per side
  static constexpr int UW = TW + 2 * A;                     // u box width
  static constexpr int NV = UW / VEC;                       // 16-byte chunks per u row
  static constexpr int OFF1 = A - HB - HW;                  // window offset of pass B
  static constexpr int OFF2 = HB - HW;                      // window offset of pass H2
  static constexpr int NW1 = round_up_c(OFF1 + V + 2 * HW, VEC);
  static constexpr int NW2 = round_up_c(OFF2 + V + 2 * HW, VEC);
  static constexpr int UP = UW;                             // u rows: dense TMA box
  static constexpr int BP = NH1;                            // b / r rows: dense TMA box
  static constexpr int H1P = conflict_free_pitch<T>(NH1);
  static constexpr int H2P = conflict_free_pitch<T>(TW);
  static constexpr int HR = 2 * HW + G;                     // rows of a history buffer
  static_assert(2 * HW <= G, "history move must not overlap");
  static_assert(NH1 % V == 0 && TW % V == 0, "segments");
  static_assert(V * (NH1 / V - 1) + NW1 <= UW, "pass B window overruns the u row");
  static_assert(!RESID || V * (TW / V - 1) + NW2 <= NH1, "pass H2 window overruns the r row");
  static constexpr int SEG1 = NH1 / V, SEG2 = TW / V;
  static constexpr int ITEMS_B = SEG1 * G;
  static constexpr int ITEMS_C = (RESID ? NH1 / 2 : TW / 2) * (G / VC);
  static constexpr int ITEMS_H2 = RESID ? SEG2 * G : 0;
  static constexpr int ITEMS_D = RESID ? (TW / 2) * (G / VC) : 0;
  static constexpr int NT = round_up_c(std::max(std::max(ITEMS_B, ITEMS_C), std::max(ITEMS_H2, ITEMS_D)), 32);
  static constexpr int NVB = RESID ? NH1 / VEC : 0;         // 16-byte chunks per b row
  static constexpr int NCHUNK = G * (NV + NVB);             // chunks of a gathered (edge) batch
  static constexpr int MV1 = 2 * HW * (NH1 / VEC);          // 16-byte moves of h1 history
  static constexpr int MV2 = RESID ? 2 * HW * (TW / VEC) : 0;  // 16-byte moves of h2 history
  static constexpr int NM1 = (MV1 + NT - 1) / NT, NM2 = (MV2 + NT - 1) / NT;
  static constexpr int HA = RESID ? 2 * HW : HW;            // first loaded row = r0 - HA
  // byte offsets of the shared-memory carve-up (TMA destinations first, 128-byte aligned)
  static constexpr size_t OFF_U = 0;
  static constexpr size_t OFF_B = OFF_U + round_up_c(2 * G * UP * (int)sizeof(T), 128);
  static constexpr size_t OFF_H1 = OFF_B + (RESID ? round_up_c(2 * G * BP * (int)sizeof(T), 128) : 0);
  static constexpr size_t OFF_H2 = OFF_H1 + round_up_c(HR * H1P * (int)sizeof(T), 16);
  static constexpr size_t OFF_BAR = OFF_H2 + (RESID ? round_up_c(HR * H2P * (int)sizeof(T), 16) : 0);
  static constexpr size_t OFF_RED = OFF_BAR + 2 * sizeof(uint64_t);
  static constexpr size_t smem_bytes() { return OFF_RED + (NT / 32) * sizeof(double); }
};

template <typename T, int HW>
struct BlurStreamParams {
  using P = typename Pair<T>::t;
  CUtensorMap tmap_u;        // u: box (UW columns, G rows, 1 image)        (valid if tma)
  CUtensorMap tmap_b;        // b: box (NH1 columns, G rows, 1 image)       (residual)
  const T *u;
  const T *b;  // residual only
  T *out;
  double *f;   // residual only (nullable)
  int h, w, nstrips;
  RunMap runs;               // (image, strip) columns x row bands
  int fast;                  // 16-byte aligned rows: cp.async / vector paths allowed
  int tma;                   // tensor maps valid
  P cc[2 * HW + 1];          // (c[d], c[d]),  c[d] = k[2h - d]: out[i] = sum_d c[d] yhat[i - h + d]
  P ce[HW + 1], co[HW + 1];  // (c[2m], c[2m+1]) and (c[2m-1], c[2m]) (out-of-range taps = 0)
};

// Horizontal pass over a register window: V outputs out[j] = sum_d c[d] win[j + OFF + d].
template <typename T, int HW, int V, int OFF, int NW>
__device__ __forceinline__ void hpass_win(const T *win, const BlurStreamParams<T, HW> &p, T *outv) {
  using P = typename Pair<T>::t;
  // tap-outer: only the (even, odd) tap pairs of one m are live at a time.  The partner of an
  // out-of-range tap is a real window sample times a zero coefficient (no zero moves).
  P acc[V];
#pragma unroll
  for (int j = 0; j < V; j++) acc[j] = zero2<P>();
#pragma unroll
  for (int m = 0; m <= HW; m++) {
    const P ce = p.ce[m], co = p.co[m];
#pragma unroll
    for (int j = 0; j < V; j++) {
      const int s = j + OFF;
      P x;
      if (s % 2 == 0) {
        x.x = win[s + 2 * m];
        x.y = (s + 2 * m + 1 < NW) ? win[s + 2 * m + 1] : T(0);
        acc[j] = fma2(ce, x, acc[j]);
      } else {
        x.x = win[s - 1 + 2 * m];
        x.y = win[s + 2 * m];
        acc[j] = fma2(co, x, acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < V; j++) outv[j] = acc[j].x + acc[j].y;
}

// Window of a horizontal item: NW samples starting at frame column `fc` of `srow`.  Away
// from the image edges this is a run of 16-byte loads; an item whose window crosses an
// edge reads the mirrored column for every sample outside the image (the frame starts at
// image column f0 and is fw wide; the mirror of every sample a needed output uses lies
// inside it).
template <typename T, int NW>
__device__ __forceinline__ void load_window(T *win, const T *srow, int fc, bool edge, int f0, int fw, int w) {
  using Vt = typename Vec16<T>::type;
  constexpr int VEC = Vec16<T>::n;
  if (!edge) {
#pragma unroll
    for (int i = 0; i < NW / VEC; i++) vec_split<T>(reinterpret_cast<const Vt *>(srow + fc)[i], win + i * VEC);
  } else {
#pragma unroll
    for (int i = 0; i < NW; i++) {
      const int g = f0 + fc + i;
      const int src = g < 0 ? -1 - g : (g >= w ? 2 * w - 1 - g : g);
      win[i] = srow[min(max(src - f0, 0), fw - 1)];
    }
  }
}

// Vertical pass over a column pair: VC outputs from VC + 2HW consecutive rows at `src` (pitch).
template <typename T, int HW, int VC, int PITCH>
__device__ __forceinline__ void vpass(const T *src, const BlurStreamParams<T, HW> &p, typename Pair<T>::t *acc,
                                      const typename Pair<T>::t *init = nullptr) {
  using P = typename Pair<T>::t;
  P win[VC + 2 * HW];
#pragma unroll
  for (int i = 0; i < VC + 2 * HW; i++) win[i] = *reinterpret_cast<const P *>(src + i * PITCH);
  // tap-outer, two independent chains (even / odd taps) per output; the even chain starts
  // at `init` (the residual's -b) when given
  P a[VC], b[VC];
#pragma unroll
  for (int v = 0; v < VC; v++) {
    a[v] = init ? init[v] : zero2<P>();
    b[v] = zero2<P>();
  }
#pragma unroll
  for (int d = 0; d < 2 * HW + 1; d++) {
    const P c = p.cc[d];
#pragma unroll
    for (int v = 0; v < VC; v++) {
      if (d % 2 == 0) a[v] = fma2(c, win[v + d], a[v]);
      else b[v] = fma2(c, win[v + d], b[v]);
    }
  }
#pragma unroll
  for (int v = 0; v < VC; v++) acc[v] = add2(a[v], b[v]);
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

#ifndef WL_BLUR_MINB
#define WL_BLUR_MINB 3  // fp32 CTAs per SM the register budget is sized for
#endif

template <typename T, int HW, bool RESID>
__global__ void __launch_bounds__(BCfg<T, HW, RESID>::NT, sizeof(T) == 4 ? (BCfg<T, HW, RESID>::NT <= 256 ? WL_BLUR_MINB : 2) : 1)
    k_blur_stream(const __grid_constant__ BlurStreamParams<T, HW> p) {
  using C = BCfg<T, HW, RESID>;
  using P = typename C::P;
  using Vt = typename Vec16<T>::type;
  constexpr int G = C::G, VC = C::VC, VEC = C::VEC, HA = C::HA;
  // no static shared memory in this kernel: the dynamic window starts at offset 0 (aligned);
  // indexing smem_raw directly keeps every access in the shared state space (LDS/STS)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char *sm = smem_raw;
  T *ubuf = reinterpret_cast<T *>(sm + C::OFF_U);    // [2][G][UP]   u rows e .. e+G-1
  T *bbuf = reinterpret_cast<T *>(sm + C::OFF_B);    // [2][G][BP]   b, then r, rows e-HW ..    (residual)
  T *h1 = reinterpret_cast<T *>(sm + C::OFF_H1);     // [HR][H1P]    h1 rows e-2HW .. e+G-1
  T *h2 = reinterpret_cast<T *>(sm + C::OFF_H2);     // [HR][H2P]    h2 rows e-3HW .. e-HW+G-1  (residual)
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);  // [2] batch barriers
  double *red = reinterpret_cast<double *>(sm + C::OFF_RED);

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our inputs
  unsigned phase = 0;  // parity of the completed phases of bar[0] (bit 0) and bar[1] (bit 1)

  // per-thread work items of every stage (fixed for the whole kernel)
  const bool actB0 = tid < C::ITEMS_B;
  const int segB = tid % C::SEG1, rowB = tid / C::SEG1;
  constexpr int NPC = RESID ? C::NH1 / 2 : C::TW / 2;
  const bool actC0 = tid < C::ITEMS_C;
  const int mC = tid % NPC, grpC = tid / NPC;
  const bool actH0 = RESID && tid < C::ITEMS_H2;
  const int segH = tid % C::SEG2, rowH = tid / C::SEG2;
  const bool actD0 = RESID && tid < C::ITEMS_D;
  const int mD = tid % (C::TW / 2), grpD = tid / (C::TW / 2);

  const int nruns = p.runs.nruns();
  for (int run = blockIdx.x; run < nruns; run += gridDim.x) {
    int col, r0, r1;
    p.runs.get(run, col, r0, r1);
    const int img = col / p.nstrips, strip = col - img * p.nstrips;
    if (r0 >= r1) continue;  // (uniform) empty trailing band
    const int c0 = strip * C::TW;
    // interior strips (the u window and every output inside the image, 16-byte rows) run a copy
    // of the body without the per-item edge and column guards
    const bool interior = p.fast && c0 - C::A >= 0 && c0 + C::TW + C::A <= p.w;
    auto run_body = [&](auto edge_tag) {
    constexpr bool EDGE = decltype(edge_tag)::value;
    const T *u = p.u + (long long)img * p.h * p.w;
    const T *bimg = RESID ? p.b + (long long)img * p.h * p.w : nullptr;
    T *out = p.out + (long long)img * p.h * p.w;
    const int e_begin = r0 - HA;
    // output row = loaded row - 2*HA (first valid output r0): n_it iterations cover [r0, r1)
    const int n_it = (r1 - r0 + 2 * HA + G - 1) / G;

    // per-run item facts: skip items whose outputs are all outside the image (never read)
    const int oB = c0 - C::HB + C::V * segB;  // image column of B's first output
    const bool actB = actB0 && (!EDGE || (oB < p.w && oB + C::V > 0));
    const int gB = c0 - C::A + C::V * segB;   // image column of B's window start
    const bool edgeB = EDGE && (gB < 0 || gB + C::NW1 > p.w);
    const int colC = RESID ? c0 - C::HB + 2 * mC : c0 + 2 * mC;  // image column of C's pair
    const bool actC = actC0 && (!EDGE || (colC < p.w && colC + 2 > 0));
    const bool ovecC = !EDGE || (p.fast && colC + 1 < p.w);
    P fmask;  // f counts each in-image pixel of the tile once
    fmask.x = (colC >= c0 && colC < c0 + C::TW && colC < p.w) ? T(1) : T(0);
    fmask.y = (colC + 1 >= c0 && colC + 1 < c0 + C::TW && colC + 1 < p.w) ? T(1) : T(0);
    const int oH = c0 + C::V * segH;
    const bool actH = actH0 && (!EDGE || oH < p.w);
    const int gH = c0 - C::HB + C::V * segH;  // image column of H2's window start
    const bool edgeH = EDGE && (gH < 0 || gH + C::NW2 > p.w);
    const int colD = c0 + 2 * mD;
    const bool actD = actD0 && (!EDGE || colD < p.w);
    const bool ovecD = !EDGE || (p.fast && colD + 1 < p.w);
    double fsx = 0.0, fsy = 0.0;  // per-column sums of r^2 (masked to the tile at the end)

    // batch k: u rows e_begin + kG .. and (residual) b rows e_begin + kG - HW .. -> slot k & 1.
    // Returns whether the batch armed its barrier.
    auto load_batch = [&](int k) -> bool {
      const int eu = e_begin + k * G, eb = eu - HW;
      const bool tma_u = p.tma && eu >= 0 && eu + G <= p.h;
      const bool tma_b = RESID && p.tma && eb >= 0 && eb + G <= p.h;
      T *ud = ubuf + (k & 1) * G * C::UP;
      T *bd = bbuf + (k & 1) * G * C::BP;
      const unsigned bytes = (tma_u ? G * C::UW * sizeof(T) : 0) + (tma_b ? G * C::NH1 * sizeof(T) : 0);
      if (tid == 0 && bytes) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar + (k & 1), bytes);
        if (tma_u) tma_load_3d(ud, &p.tmap_u, bar + (k & 1), c0 - C::A, eu, img);
        if (tma_b) tma_load_3d(bd, &p.tmap_b, bar + (k & 1), c0 - C::HB, eb, img);
      }
      const int lo = tma_u ? G * C::NV : 0;
      const int hi = (RESID && !tma_b) ? C::NCHUNK : G * C::NV;
      for (int idx = lo + tid; idx < hi; idx += C::NT) {
        const bool sb = idx >= G * C::NV;
        const int j = sb ? idx - G * C::NV : idx;
        const int per = sb ? (C::NVB > 0 ? C::NVB : 1) : C::NV;
        const int r = j / per, v = j - r * per;
        const int sr = refl_inf((sb ? eb : eu) + r, p.h);
        const int cg = (sb ? c0 - C::HB : c0 - C::A) + v * VEC;
        T *dst = sb ? bd + r * C::BP + v * VEC : ud + r * C::UP + v * VEC;
        const T *row = (sb ? bimg : u) + (long long)sr * p.w;
        if (p.fast && cg >= 0 && cg + VEC <= p.w) {
          cp_async16(dst, row + cg);
        } else {
          T z[VEC];
#pragma unroll
          for (int i = 0; i < VEC; i++) z[i] = row[refl_inf(cg + i, p.w)];
          *reinterpret_cast<Vt *>(dst) = vec_make<T>(z);
        }
      }
      return bytes != 0;
    };

    __syncthreads();  // the previous run's readers of every buffer are done
    bool armed = load_batch(0);
    cp_async_commit();
    for (int it = 0; it < n_it; it++) {
      const int e = e_begin + it * G;
      cp_async_wait_all();
      if (armed) {
        mbar_wait(bar + (it & 1), (phase >> (it & 1)) & 1);
        phase ^= 1u << (it & 1);
      }
      __syncthreads();  // (1) batch it landed; every stage of it-1 finished
      armed = (it + 1 < n_it) ? load_batch(it + 1) : false;
      cp_async_commit();
      if (RESID) {
        // carry the last 2HW h2 rows to the head of the h2 history (D of it-1 has finished)
#pragma unroll
        for (int k = 0; k < C::NM2; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV2) {
            const int r = idx / (C::TW / VEC), c = idx - r * (C::TW / VEC);
            *reinterpret_cast<Vt *>(h2 + r * C::H2P + c * VEC) =
                *reinterpret_cast<const Vt *>(h2 + (r + G) * C::H2P + c * VEC);
          }
        }
      } else if (it > 0) {
        // R: carry the h1 history now (stage C of it-1 finished at barrier (1))
#pragma unroll
        for (int k = 0; k < C::NM1; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV1) {
            const int r = idx / (C::NH1 / VEC), c = idx - r * (C::NH1 / VEC);
            *reinterpret_cast<Vt *>(h1 + r * C::H1P + c * VEC) =
                *reinterpret_cast<const Vt *>(h1 + (r + G) * C::H1P + c * VEC);
          }
        }
        __syncthreads();
      }
      // B: horizontal pass of u rows e .. e+G-1 -> h1 rows 2HW .. 2HW+G-1
      if (actB) {
        T win[C::NW1], hv[C::V];
        load_window<T, C::NW1>(win, ubuf + ((it & 1) * G + rowB) * C::UP, C::V * segB, edgeB, c0 - C::A, C::UW,
                               p.w);
        hpass_win<T, HW, C::V, C::OFF1, C::NW1>(win, p, hv);
        Vt *dst = reinterpret_cast<Vt *>(h1 + (2 * HW + rowB) * C::H1P + C::V * segB);
#pragma unroll
        for (int i = 0; i < C::V / VEC; i++) dst[i] = vec_make<T>(hv + i * VEC);
      }
      __syncthreads();  // (2)
      // C: vertical pass -> rows x = e - HW + grpC*VC + v  (h1 index of x - HW is grpC*VC + v)
      if (actC) {
        const int xb = e - HW + grpC * VC;
        P acc[VC];
        if (RESID) {
          // r = V h1 - b (the chain starts at -b); f sums r^2 over the item's valid rows per
          // column, the tile column mask is applied once per run
          P *rb = reinterpret_cast<P *>(bbuf + ((it & 1) * G + grpC * VC) * C::BP + 2 * mC);
          P nb[VC];
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const P bv = rb[v * (C::BP / 2)];
            nb[v].x = -bv.x;
            nb[v].y = -bv.y;
          }
          vpass<T, HW, VC, C::H1P>(h1 + grpC * VC * C::H1P + 2 * mC, p, acc, nb);
          P fa = zero2<P>();
          const bool rows_in = xb >= r0 && xb + VC <= r1;
#pragma unroll
          for (int v = 0; v < VC; v++) {
            rb[v * (C::BP / 2)] = acc[v];
            if (rows_in || (xb + v >= r0 && xb + v < r1)) fa = fma2(acc[v], acc[v], fa);
          }
          fsx += (double)fa.x;
          fsy += (double)fa.y;
        } else {
          vpass<T, HW, VC, C::H1P>(h1 + grpC * VC * C::H1P + 2 * mC, p, acc);
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const int x = xb + v;
            if (x >= r0 && x < r1) store_pair<T>(out + (long long)x * p.w, colC, acc[v], ovecC, p.w);
          }
        }
      }
      if (RESID) {
        __syncthreads();  // (3) r rows complete; h1 readers done
        // H2: horizontal pass of r rows -> h2 rows 2HW .. 2HW+G-1 (rows x = e - HW + row)
        if (actH) {
          T win[C::NW2], hv[C::V];
          load_window<T, C::NW2>(win, bbuf + ((it & 1) * G + rowH) * C::BP, C::V * segH, edgeH, c0 - C::HB, C::NH1,
                                 p.w);
          hpass_win<T, HW, C::V, C::OFF2, C::NW2>(win, p, hv);
          Vt *dst = reinterpret_cast<Vt *>(h2 + (2 * HW + rowH) * C::H2P + C::V * segH);
#pragma unroll
          for (int i = 0; i < C::V / VEC; i++) dst[i] = vec_make<T>(hv + i * VEC);
        }
        // carry the last 2HW h1 rows to the head of the h1 history
#pragma unroll
        for (int k = 0; k < C::NM1; k++) {
          const int idx = tid + k * C::NT;
          if (idx < C::MV1) {
            const int r = idx / (C::NH1 / VEC), c = idx - r * (C::NH1 / VEC);
            *reinterpret_cast<Vt *>(h1 + r * C::H1P + c * VEC) =
                *reinterpret_cast<const Vt *>(h1 + (r + G) * C::H1P + c * VEC);
          }
        }
        __syncthreads();  // (4)
        // D: vertical pass -> s rows y = e - 2HW + grpD*VC + v (h2 index of y - HW is grpD*VC + v)
        const int yb = e - 2 * HW + grpD * VC;
        if (actD && yb + VC > r0 && yb < r1) {
          P acc[VC];
          vpass<T, HW, VC, C::H2P>(h2 + grpD * VC * C::H2P + 2 * mD, p, acc);
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const int y = yb + v;
            if (y >= r0 && y < r1) store_pair<T>(out + (long long)y * p.w, colD, acc[v], ovecD, p.w);
          }
        }
      }
    }
    cp_async_wait_all();
    if (RESID && p.f) {
      double fsum = fsx * (double)fmask.x + fsy * (double)fmask.y;
      for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
      if ((tid & 31) == 0) red[tid >> 5] = fsum;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < C::NT / 32; i++) s += red[i];
        atomicAdd(p.f + img, 0.5 * s);
      }
    }
    };
    if (interior) run_body(std::false_type{});
    else run_body(std::true_type{});
  }
}

template <typename T, int HW, bool RESID>
cudaError_t launch_stream(const BlurArgs &a, cudaStream_t s) {
  using C = BCfg<T, HW, RESID>;
  BlurStreamParams<T, HW> p;
  memset(&p, 0, sizeof p);
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
  bool tma = fast && a.h >= C::G && tma_enabled();  // WL_NO_TMA: debugging / A-B switch
  const uint64_t rs = (uint64_t)p.w * sizeof(T), is = rs * (uint64_t)p.h;
  if (tma) tma = encode_tmap_3d(&p.tmap_u, sizeof(T), a.in, p.w, p.h, a.batch, rs, is, C::UW, C::G);
  if (tma && RESID) tma = encode_tmap_3d(&p.tmap_b, sizeof(T), a.b, p.w, p.h, a.batch, rs, is, C::NH1, C::G);
  p.tma = tma;
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
  const size_t smem = C::smem_bytes();
  auto kern = k_blur_stream<T, HW, RESID>;
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(kern), C::NT, smem, &resident);
  if (e != cudaSuccess) return e;
  // one run per resident CTA when the columns allow it; bands of >= G rows (small images need the CTAs)
#ifndef WL_BLUR_MINROWS
#define WL_BLUR_MINROWS 1  // in units of G; A/B on B200: 1 beat 4 (cfg2 grad -11 %, cfg1 -15 %, cfg3/5 equal)
#endif
  p.runs = RunMap::make((long long)a.batch * p.nstrips, (int)a.h, resident, WL_BLUR_MINROWS * C::G, 1);
  const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
  if (RESID && a.f && !a.f_zeroed) {
    e = cudaMemsetAsync(a.f, 0, sizeof(double) * (size_t)a.batch, s);
    if (e != cudaSuccess) return e;
  }
  e = launch_pdl(kern, grid, C::NT, smem, s, p, 'b');
  g_launches++;
  if (e != cudaSuccess) return e;
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
  cudaError_t e;
  if (launch_blur_ring(dtype, a, false, s, &e)) return e;
  return dtype == WL_F64 ? dispatch_blur<double>(a, s, false) : dispatch_blur<float>(a, s, false);
}

cudaError_t launch_blur_residual(int dtype, const BlurArgs &a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  cudaError_t e;
  if (launch_blur_ring(dtype, a, true, s, &e)) return e;
  return dtype == WL_F64 ? dispatch_blur<double>(a, s, true) : dispatch_blur<float>(a, s, true);
}

}  // namespace wl
