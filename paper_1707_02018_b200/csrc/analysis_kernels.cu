// W* and W-dagger: one 2-D level of the wavelet analysis (sm_100a), streaming column-strip kernel.
//
// Analysis core (reading R5):  out[k] = sum_{j<L} f[j] * yhat[2k+1-j],
// applied along axis 1 (rows) then axis 0 (columns); yhat = E y with E chosen per operator
// (P:52-98):  W-dagger: E_bc;  W*: E_zpd / periodisation / (E_sym^dagger)* = E_sym diag(1/c)
// (Eq. (4); reading R1).  Subband XY = axis-0 filter X, axis-1 filter Y.
//
// A CTA owns TQ coefficient columns of one image and a band of coefficient rows; it walks
// down the input rows 2G at a time (G coefficient rows out per iteration):
//   A  the 2G input rows of the strip's window (2TQ + L - 2 columns) land in a double
//      buffer: one TMA box issued by one thread and completed on an mbarrier when the
//      extension is the zero extension (TMA's zero fill) or the block lies inside the image;
//      otherwise (symmetric / periodic / EDAG-weighted edges) they are gathered with the
//      extension map by cp.async / per-element loads;
//   B  axis-1 pass: every input row -> (lo, hi) coefficient pairs with FFMA2 on the tap pair
//      (f_lo[j], f_hi[j]) against a broadcast sample, into the lo / hi row histories
//      (L-2 carried rows + 2G new);
//   C  axis-0 pass: each thread owns a column pair of one history and produces VC coefficient
//      rows of two subbands (X = lo, hi) from a register window, stored as float2 pairs
//      (padding columns of the pitched rows written as 0).  With the FISTA epilogue (FU) the
//      coefficient pair is not stored: it is g of grad f(y), and the store becomes the prox +
//      momentum update of (x, y) in place (prox fused into W*'s store).
// Loops run tap-outer so only one tap pair is live at a time (no register spills).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

#ifdef WL_ANA_PROFILE  // debug builds only: per-run start / end times and SM id (tools/anaprof.py)
__device__ unsigned long long g_ana_prof[8192][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#endif

// Source index of extended position t (or -1 for a zero) and its weight.
template <typename T>
__device__ __forceinline__ int ext_src(int t, int n, int ext, int Lp, T &w) {
  w = T(1);
  if (ext == EXT_ZERO) return (t >= 0 && t < n) ? t : -1;
  if (ext == EXT_PER) {
    if (t >= 0 && t < n) return t;  // the common case: no integer division
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

#ifndef WL_L2HINT
#define WL_L2HINT 1  // 0: plain stores; 1: LL of a non-last level evict_last; 2: + other subbands evict_first
#endif
#ifndef WL_ANA_NS
#define WL_ANA_NS 2  // A/B on B200: 3 or 4 stages did not beat 2
#endif
template <typename T, int L, int NS_ = 0, bool FU_ = false>
struct ACfg {
  using P = typename Pair<T>::t;
  static constexpr int VEC = Vec16<T>::n;
  // fp32 tile (A/B on B200): 16 coefficient outputs per B item, 8 rows per C item, 16 rows per
  // iteration beat (8, 4, 8) by 6 % at cfg5 and 5 % at cfg4 (less shared-memory traffic per FFMA2:
  // fewer window re-reads).  The fused FISTA variant keeps (8, 4, 8): its (y, x) tiles scale with G.
#ifndef WL_ANA_TQ
#define WL_ANA_TQ 64
#endif
#ifndef WL_ANA_V
#define WL_ANA_V 16
#endif
#ifndef WL_ANA_VC
#define WL_ANA_VC 8
#endif
#ifndef WL_ANA_G
#define WL_ANA_G 16
#endif
  static constexpr bool F32 = sizeof(T) == 4;
  static constexpr int TQ = F32 ? WL_ANA_TQ : 32;                     // coefficient columns per strip
#ifndef WL_ANA_SHORT_SMALL
#define WL_ANA_SHORT_SMALL 1
#endif
  // the small tile (8 rows per iteration): the fused FISTA variant, and the short-run variant for
  // filters shorter than db8 (A/B on B200: cfg2 W* -18 %, cfg3 -2 %, cfg5 -1 %; db8 +4 %, so not there)
  static constexpr bool SMALL = FU_ || (WL_ANA_SHORT_SMALL && NS_ == 4 && L < 16);
  static constexpr int G = (F32 && !SMALL) ? WL_ANA_G : 8;              // coefficient rows per iteration
  static constexpr int GI = 2 * G;                       // input rows per iteration
  static constexpr int V = (F32 && !SMALL) ? WL_ANA_V : 8;    // coefficient outputs per B item
  // coefficient rows per C item: the 16-tap db8 window (2 VC + 14 history rows) does better with
  // 4 (cfg4 W* -3.6 %), the shorter filters with 8
  static constexpr int VC = (F32 && !SMALL) ? (L >= 16 ? 4 : WL_ANA_VC) : 4;
  static constexpr int SHIFT = ((2 - L) % VEC + VEC) % VEC;  // box column of input column 2q0+2-L
  // input box width.  Padded so that a row is 4 mod 8 words (the B-stage 16-byte window loads of 8
  // consecutive rows then fall in 8 distinct 4-bank groups: row-fastest items, no bank conflicts)
  // unless the padding would cost a resident CTA per SM (B200: CDF 9/7 keeps 4 CTAs with dense
  // rows and 2-way conflicts, measured 1 % faster; db8 has 3 CTAs either way and pads)
  static constexpr int UW0 = round_up_c(SHIFT + 2 * TQ + L - 2, VEC);
  static constexpr int UWP = bank_pad<T>(UW0);
  static constexpr int HR_ = L - 2 + 2 * G;
  static constexpr int NS0 = NS_ > 0 ? NS_ : WL_ANA_NS;
  static constexpr int ctas_for(int uw) {
    return (228 * 1024) / (round_up_c(NS0 * 2 * G * uw * (int)sizeof(T), 128) +
                           2 * HR_ * conflict_free_pitch<T>(TQ) * (int)sizeof(T) + 16 + 1024);
  }
#ifdef WL_ANA_NOPAD  // A/B: dense box rows always
  static constexpr int UW = UW0;
#else
  static constexpr int UW = ctas_for(UWP) >= ctas_for(UW0) ? UWP : UW0;
#endif
  static constexpr int UP = UW;                          // dense TMA box rows
  static constexpr int NV = UW / VEC;
  static constexpr int NWB = round_up_c(SHIFT + 2 * V + L - 2, VEC);  // B window
  static constexpr int SEGB = TQ / V;
  static constexpr int HR = L - 2 + GI;                  // history rows (L-2 carried + 2G new)
  static constexpr int HP = conflict_free_pitch<T>(TQ);
  static_assert(2 * V * (SEGB - 1) + NWB <= UW, "B window overruns the input row");
  static_assert(GI >= L - 2, "history move must not overlap");
  static constexpr int ITEMS_B = SEGB * GI;
  static constexpr int ITEMS_C = 2 * (TQ / 2) * (G / VC);
  static constexpr int NT = round_up_c(std::max(ITEMS_B, ITEMS_C), 32);
  // input stages (prefetch depth NS-1); short runs (coarse levels) use 4 so every block of the
  // run is in flight at once instead of one TMA round trip per block
  static constexpr int NS = NS_ > 0 ? NS_ : WL_ANA_NS;
  static constexpr size_t OFF_U = 0;  // [NS][GI][UP]
  static constexpr size_t OFF_H = OFF_U + round_up_c(NS * GI * UP * (int)sizeof(T), 128);  // [2 sets][HR][HP]
  static constexpr size_t OFF_BAR = OFF_H + 2 * (size_t)HR * HP * sizeof(T);
  // FISTA epilogue (FU): per stage, the (y, x) tiles of the block's G coefficient rows x TQ
  // columns for the 4 subbands, prefetched by cp.async with the input rows (no load latency
  // in the store stage)
  static constexpr int FT = G * TQ;                      // elements per (subband, array) tile
  static constexpr size_t OFF_F = round_up_c(OFF_BAR + NS * sizeof(uint64_t), 128);  // [NS][4][2][G][TQ]
  static constexpr size_t smem_bytes(bool fu = false) {
    return fu ? OFF_F + (size_t)NS * 8 * FT * sizeof(T) : OFF_BAR + NS * sizeof(uint64_t);
  }
};

template <typename T, int L>
struct AnaStreamParams {
  using P = typename Pair<T>::t;
  CUtensorMap tmap;          // input: box (UW, GI, 1)   (valid if tma)
  const T *in;
  long long in_pitch, in_bstride;
  int n0, n1;
  T *out[4];                 // LL, LH, HL, HH
  long long out_pitch[4], out_bstride[4];
  int m0, m1, ext, tma, tma_any_block, fast;
  int nstrips;
  RunMap runs;               // (image, strip) columns x bands of coefficient rows
  T flo[L], fhi[L];          // raw taps (gather weights)
  P fb[L];                   // B tap pairs (f_lo[j], f_hi[j])
  P slo[L], shi[L];          // C broadcast taps (f[j], f[j])
  // fused FISTA epilogue (FU): for subbands in fmask the output pointer is y; x = y + xdelta.
  // The W* value g never reaches HBM:  x+ = soft(y - g/L, lambda/L), y+ = x+ + mom (x+ - x)
  int ll_keep;               // LL feeds the next level: stored evict_last (WL_L2HINT)
  int fmask;
  long long xdelta;
  T inv_lip, tau, mom;
  const double *tdev;  // non-null: mom = (t - 1) / t+ from the device-resident t (graph-replayable)
};

template <typename T>
__device__ __forceinline__ T soft_thr(T v, T tau) {
  const T a = v > T(0) ? v : -v;
  const T m = a - tau;
  return m > T(0) ? (v > T(0) ? m : -m) : T(0);
}

// fused FISTA update of one coefficient pair: g of grad f(y); (y, x) old values from the
// prefetched tile; writes x+ and y+ at yp and yp + xdelta
template <typename T, int L>
__device__ __forceinline__ void fista_pair(const AnaStreamParams<T, L> &p, T mom, T *yp, typename Pair<T>::t g,
                                           const T *tile_y, const T *tile_x) {
  using P = typename Pair<T>::t;
  const P yv = *reinterpret_cast<const P *>(tile_y), xv = *reinterpret_cast<const P *>(tile_x);
  P xn, yn;
  xn.x = soft_thr<T>(yv.x - g.x * p.inv_lip, p.tau);
  xn.y = soft_thr<T>(yv.y - g.y * p.inv_lip, p.tau);
  yn.x = xn.x + mom * (xn.x - xv.x);
  yn.y = xn.y + mom * (xn.y - xv.y);
  *reinterpret_cast<P *>(yp + p.xdelta) = xn;
  *reinterpret_cast<P *>(yp) = yn;
}

// The element-gather load of one input block (any extension, any alignment): the fallback of the block loader,
// kept out of line so the kernel's hot paths stay compact (instruction-cache footprint).
template <typename T, int L, typename C>
__device__ __noinline__ void gather_block(const AnaStreamParams<T, L> &p, const T *in, T *dst0, int r_in, int cbox,
                                          int tid, int ext) {
  using Vt = typename Vec16<T>::type;
  constexpr int GI = C::GI, VEC = C::VEC;
  for (int idx = tid; idx < GI * C::NV; idx += C::NT) {
    const int r = idx / C::NV, v = idx - r * C::NV;
    T wr;
    const int sr = ext_src<T>(r_in + r, p.n0, ext, L - 1, wr);
    T *dst = dst0 + r * C::UP + v * VEC;
    const int cg = cbox + v * VEC;
    // extended positions t >= 2m feed no stored output (out[k] reads t = 2k+1-j <= 2m-1): the
    // window of a partial last strip / band is zero-filled there instead of gathered
    if (sr < 0 || cg >= 2 * p.m1 || r_in + r >= 2 * p.m0) {
      T z[VEC];
#pragma unroll
      for (int u = 0; u < VEC; u++) z[u] = T(0);
      *reinterpret_cast<Vt *>(dst) = vec_make<T>(z);
    } else if (p.fast && cg >= 0 && cg + VEC <= p.n1 &&
               (ext != EXT_SYM_PADJ || (wr == T(1) && cg >= L - 1 && cg + VEC <= p.n1 - (L - 1)))) {
      // a plain 16-byte copy (for the weighted (E_sym^dagger)* extension only where every weight is 1)
      cp_async16(dst, in + (long long)sr * p.in_pitch + cg);
    } else if (p.fast && ext == EXT_PER && p.n1 % VEC == 0 && ((cg % p.n1) + p.n1) % p.n1 + VEC <= p.n1) {
      // periodic wrap of a whole aligned chunk (n1 is a multiple of VEC when p.fast)
      cp_async16(dst, in + (long long)sr * p.in_pitch + ((cg % p.n1) + p.n1) % p.n1);
    } else {
      T z[VEC];
#pragma unroll
      for (int u = 0; u < VEC; u++) {
        T wc;
        const int sc = ext_src<T>(cg + u, p.n1, ext, L - 1, wc);
        z[u] = sc >= 0 ? in[(long long)sr * p.in_pitch + sc] * (wr * wc) : T(0);
      }
      *reinterpret_cast<Vt *>(dst) = vec_make<T>(z);
    }
  }
}

// One level's runs, handed to the CTAs of the grid (the body of k_ana_stream; k_ana_multi calls it
// once per level of the coarse tail).  `phase` carries the stage barriers' parities across calls.
// KIND 1 (PLAIN): zero extension with every block by TMA (W* under zero / symmetric BC on 16-byte aligned input): the
// gather, bulk-row, wrap and mirror paths are compiled out (a compact hot path: the coarse levels start with a cold
// instruction cache).  KIND 2 / 3: the extension is E_sym / (E_sym^dagger)* at compile time (W-dagger under symmetric
// BC, the paper-literal W*): the wrap path and the other extension's branches are compiled out.  KIND 0: p.ext.
template <typename T, int L, bool FU, int NS, int ZV = 0, int KIND = 0>
__device__ __forceinline__ void ana_level_runs(const AnaStreamParams<T, L> &p, unsigned char *smem_raw,
                                               unsigned &phase) {
  constexpr bool PLAIN = KIND == 1;
  const int ext = KIND == 1 ? EXT_ZERO : (KIND == 2 ? EXT_SYM : (KIND == 3 ? EXT_SYM_PADJ : p.ext));
  using C = ACfg<T, L, NS, FU>;
  using P = typename C::P;
  using Vt = typename Vec16<T>::type;
  constexpr int G = C::G, GI = C::GI, VEC = C::VEC, V = C::V, VC = C::VC, TQ = C::TQ;
  T *ubuf = reinterpret_cast<T *>(smem_raw + C::OFF_U);  // [NS][GI][UP] input rows
  T *hist = reinterpret_cast<T *>(smem_raw + C::OFF_H);  // [2][HR][HP] lo / hi coefficient columns
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::OFF_BAR);
  T *ftile = reinterpret_cast<T *>(smem_raw + C::OFF_F);  // FU only: [NS][4][2 (y, x)][G][TQ]
  const int tid = threadIdx.x;
  T mom = p.mom;
  if (FU && p.tdev) {
    const double t = *p.tdev, t_new = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
    mom = T((t - 1.0) / t_new);
  }
  // B item: input row fastest; C item: column pair fastest, then set (lo / hi), then group
  const bool actB = tid < C::ITEMS_B;
  const int rowB = tid % C::GI, segB = tid / C::GI;  // row fastest: a warp's loads hit distinct banks
  const bool actC = tid < C::ITEMS_C;
  const int mC = tid % (TQ / 2), setC = (tid / (TQ / 2)) & 1, grpC = tid / TQ;

  int col, kr0, kr1;
  for (RunIter itr(p.runs); itr.next(col, kr0, kr1);) {
    if (kr0 >= kr1) continue;  // (uniform) empty trailing band
#ifdef WL_ANA_PROFILE
    const unsigned long long t_start = gtimer();
#endif
    const int img = col / p.nstrips, strip = col - img * p.nstrips;
    const int q0 = strip * TQ;
    const int cbox = 2 * q0 + 2 - L - C::SHIFT;  // input column of box column 0 (VEC aligned)
    const T *in = p.in + (long long)img * p.in_bstride;
    const int wpc = ext == EXT_SYM_PADJ ? L - 1 : 0;  // weighted edge columns (E_sym^dagger)*
    const bool cols_in = cbox >= wpc && cbox + C::UW <= p.n1 - wpc;
    // outside columns a stored output reads: [cbox, 0) and [n1, min(cbox + UW, 2 m1)); sym_fix needs
    // their mirror images inside the box
    const int fix_lim = min(cbox + C::UW, 2 * p.m1);
    const int fix_nl = max(0, min(-cbox, C::UW)), fix_r0 = max(p.n1, cbox), fix_nr = max(0, fix_lim - fix_r0);
    const bool sym_fix = !PLAIN && (ext == EXT_SYM || ext == EXT_SYM_PADJ) && !cols_in &&
                         (cbox >= 0 || -2 * cbox - 1 < C::UW) && (fix_nr == 0 || 2 * p.n1 - fix_lim >= cbox);
    const int nblk = (kr1 - kr0 + G - 1) / G;
    // C output columns q = q0 + 2 mC (+1) of subbands (setC: LL/HL from lo, LH/HH from hi)
    const int qc = q0 + 2 * mC;
    T *oX0 = p.out[setC] + (long long)img * p.out_bstride[setC];          // X = lo: LL or LH
    T *oX1 = p.out[setC + 2] + (long long)img * p.out_bstride[setC + 2];  // X = hi: HL or HH
    const long long pX0 = p.out_pitch[setC], pX1 = p.out_pitch[setC + 2];
    const bool fu0 = FU && ((p.fmask >> setC) & 1), fu1 = FU && ((p.fmask >> (setC + 2)) & 1);

    // input block b (b = -1 .. nblk-1): rows 2(kr0 + bG) .. +2G -> ubuf[(b + 1) % NS]
    auto load_block = [&](int b) -> bool {
      const int r_in = 2 * (kr0 + b * G);
      const int sl = (b + 1) % C::NS;
      T *dst0 = ubuf + sl * GI * C::UP;
      if (FU && b >= 0) {  // (y, x) tiles of coefficient rows kr0 + bG .. for the fused update
        constexpr int CPR = TQ / VEC;
        T *fdst = ftile + sl * 8 * C::FT;
        for (int idx = tid; idx < 8 * G * CPR; idx += C::NT) {
          const int c = idx % CPR, r = (idx / CPR) % G, arr = (idx / (CPR * G)) & 1, band = idx / (2 * CPR * G);
          const int kr = kr0 + b * G + r, col = q0 + c * VEC;
          if (!((p.fmask >> band) & 1) || kr >= kr1 || col >= p.out_pitch[band]) continue;
          const T *src = p.out[band] + (long long)img * p.out_bstride[band] + (long long)kr * p.out_pitch[band] + col +
                         (arr ? p.xdelta : 0);
          cp_async16(fdst + ((band * 2 + arr) * G + r) * TQ + c * VEC, src);
        }
      }
      if (PLAIN) {  // TMA's zero fill is the zero extension
        if (tid == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(bar + sl, GI * C::UW * sizeof(T));
          tma_load_3d(dst0, &p.tmap, bar + sl, cbox, r_in, img);
        }
        return true;
      }
      // (E_sym^dagger)*: TMA only where every row and column weight is 1 (L-1 inside the edges)
      const int wpad = ext == EXT_SYM_PADJ ? L - 1 : 0;
      const bool rows_in = r_in >= wpad && r_in + GI <= p.n0 - wpad;
      // symmetric edge strips: the box still comes by TMA (zero fill outside) and the outside
      // columns are mirrored inside shared memory after it lands (sym_fix)
      if (p.tma && (p.tma_any_block || (rows_in && (cols_in || sym_fix)))) {
        if (tid == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(bar + sl, GI * C::UW * sizeof(T));
          tma_load_3d(dst0, &p.tmap, bar + sl, cbox, r_in, img);
        }
        return true;
      }
      // symmetric extensions, blocks reaching past the top / bottom or into the weighted rows: one
      // bulk copy per row from its reflected source row (P:82 applied to rows), columns clipped to
      // the image (a row end that is not 16-byte aligned copied by the lane); the outside columns
      // are mirrored and the (E_sym^dagger)* column weights applied in shared memory after it
      // lands, the row weights to the B-stage output.  (TMA row boxes would need 128-byte aligned
      // shared rows.)
      if (p.tma && (ext == EXT_SYM || ext == EXT_SYM_PADJ) && (cols_in || sym_fix)) {
        if (tid < 32) {  // warp 0: lane r copies rows r, r + 32, ...
          const int a0 = max(cbox, 0), e = min(cbox + C::UW, p.n1), e4 = max(a0, e / VEC * VEC);
          if (tid == 0) mbar_arrive_expect_tx(bar + sl, (unsigned)(GI * (e4 - a0) * sizeof(T)));
          __syncwarp();
          fence_proxy_async();
          for (int r = tid; r < GI; r += 32) {
            const T *srow = in + (long long)refl_inf(r_in + r, p.n0) * p.in_pitch;
            T *drow = dst0 + r * C::UP - cbox;
            if (e4 > a0) bulk_load(drow + a0, srow + a0, (unsigned)((e4 - a0) * sizeof(T)), bar + sl);
            for (int c = e4; c < e; c++) drow[c] = srow[c];  // a row end that is not 16-byte aligned
          }
        }
        return true;
      }
      // periodic extension, blocks that wrap (edge strips, top / bottom): per row one bulk copy of the
      // in-image columns (warp 0's lanes) and cp.async of the wrapped 16-byte chunks at either end (all
      // threads), from the wrapped source row (reading R2: indices mod n) -- every box column
      // filled, no shared-memory fix
      if (p.tma && ext == EXT_PER && p.n1 % VEC == 0 && -cbox <= p.n1 && cbox + C::UW - p.n1 <= p.n1) {
        const int a0 = max(cbox, 0), e = min(cbox + C::UW, p.n1);
        const int nl = max(0, -cbox) / VEC, nr = max(0, cbox + C::UW - p.n1) / VEC;  // wrapped chunks
        auto row_of = [&](int r) {
          int sr = (r_in + r) % p.n0;
          if (sr < 0) sr += p.n0;
          return in + (long long)sr * p.in_pitch;
        };
        if (tid < 32) {
          if (tid == 0) mbar_arrive_expect_tx(bar + sl, (unsigned)(GI * (e - a0) * sizeof(T)));
          __syncwarp();
          fence_proxy_async();
          for (int r = tid; r < GI; r += 32)
            bulk_load(dst0 + r * C::UP + (a0 - cbox), row_of(r) + a0, (unsigned)((e - a0) * sizeof(T)), bar + sl);
        }
        for (int idx = tid; idx < GI * (nl + nr); idx += C::NT) {
          const int r = idx / (nl + nr), c = idx - r * (nl + nr);
          const int col = c < nl ? cbox + VEC * c : p.n1 + VEC * (c - nl);  // box column of the chunk
          const int srcc = c < nl ? col + p.n1 : col - p.n1;
          cp_async16(dst0 + r * C::UP + (col - cbox), row_of(r) + srcc);
        }
        return true;
      }
      gather_block<T, L, C>(p, in, dst0, r_in, cbox, tid, ext);
      return false;
    };

    __syncthreads();  // previous run's readers are done
    unsigned armed = 0;  // bit s: the batch in slot s armed its barrier
    // (a loop, not NS-1 inlined copies of the block loader: the short-run variant's code 98 -> 59 KB and the coarse
    // levels, which start with a cold instruction cache, run faster: cfg5 W* 156.6 -> 153.0 us, cfg3 92.2 -> 88.7 us)
#pragma unroll 1
    for (int b = -1; b < C::NS - 2; b++) {
      if (b < nblk && load_block(b)) armed |= 1u << ((b + 1) % C::NS);
      cp_async_commit();
    }
    for (int it = -1; it < nblk; it++) {
      const int slot = (it + 1) % C::NS;
      cp_async_wait_group<C::NS - 2>();  // this thread's gathers of block it are done
      const bool async_blk = PLAIN || ((armed >> slot) & 1);  // block it came by TMA / bulk copies
      if (async_blk) {
        mbar_wait(bar + slot, (phase >> slot) & 1);
        phase ^= 1u << slot;
      }
      __syncthreads();  // (1) block it landed; the history move of it-1 is done
      bool padj_rows = false;  // async (E_sym^dagger)* block with weighted rows
      const int r_blk = 2 * (kr0 + it * G);
      if (!PLAIN && async_blk && (ext == EXT_SYM || ext == EXT_SYM_PADJ)) {
        const int wpad = ext == EXT_SYM_PADJ ? L - 1 : 0;
        const bool blk_rows_in = r_blk >= wpad && r_blk + GI <= p.n0 - wpad;
        T *ub = ubuf + slot * GI * C::UP;
        if (sym_fix) {
          // one pass: thread -> one source column s near an edge (every rstep-th row); it writes its
          // mirror images [cbox, 0) / [n1, fix_lim) (half-point reflection) and, for
          // (E_sym^dagger)* = E_sym diag(1/c), scales s and its images by 1/c_s
          // (c = 1 + [s < L-1] + [s >= n-L+1]).  Reading each source once keeps it race-free.
          const int Lw = ext == EXT_SYM_PADJ ? L - 1 : 0;
          const int a = min(max(Lw, fix_nl), p.n1);              // left sources [0, a)
          const int b0 = max(a, p.n1 - max(Lw, fix_nr));          // right sources [b0, n1)
          const int la0 = max(0, cbox), la1 = min(a, cbox + C::UW);
          const int ra0 = max(b0, cbox), ra1 = min(p.n1, cbox + C::UW);
          const int nl = max(0, la1 - la0), nr = max(0, ra1 - ra0), per = nl + nr;
          if (per > 0) {
            const int rstep = C::NT / per > 0 ? C::NT / per : 1, k = tid % per;
            const int sc = k < nl ? la0 + k : ra0 + (k - nl);
            const int gl = -1 - sc, gr = 2 * p.n1 - 1 - sc;
            const bool wl = gl >= cbox, wr = gr < fix_lim && gr < cbox + C::UW;
            const int c = Lw ? 1 + (sc < Lw ? 1 : 0) + (sc >= p.n1 - Lw ? 1 : 0) : 1;
            const T wgt = T(1) / T(c);
            for (int r = tid / per; r < GI && tid < rstep * per; r += rstep) {
              T *row = ub + r * C::UP - cbox;
              const T v = row[sc] * wgt;
              if (c > 1) row[sc] = v;
              if (wl) row[gl] = v;
              if (wr) row[gr] = v;
            }
          }
          __syncthreads();
        }
        // rows of (E_sym^dagger)*: applied to the B-stage output of the row (row_w below)
        padj_rows = ext == EXT_SYM_PADJ && !blk_rows_in;
      }
      {
        const int nb = it + C::NS - 1;  // its slot held block it-1, consumed before (1)
        armed &= ~(1u << (nb + 1) % C::NS);
        if (nb < nblk && load_block(nb)) armed |= 1u << ((nb + 1) % C::NS);
      }
      cp_async_commit();
      // B: input row rowB of the block -> lo/hi history row L-2+rowB, coefficient columns V*segB ..
      if (actB) {
        const T *src = ubuf + (slot * GI + rowB) * C::UP + 2 * V * segB;
        T win[C::NWB];
#pragma unroll
        for (int i = 0; i < C::NWB / VEC; i++) vec_split<T>(reinterpret_cast<const Vt *>(src)[i], win + i * VEC);
        P acc[V];
#pragma unroll
        for (int k = 0; k < V; k++) acc[k] = zero2<P>();
        using TR = TapRange<L, ZV>;
#pragma unroll
        for (int j = L - 1; j >= 0; j--) {  // tap-outer, lowest window samples first (earliest loads)
          if (j < (TR::l0 < TR::h0 ? TR::l0 : TR::h0) || j >= (TR::l1 > TR::h1 ? TR::l1 : TR::h1)) continue;
          const P f = p.fb[j];
#pragma unroll
          for (int k = 0; k < V; k++) acc[k] = fma2(f, splat2<P>(win[C::SHIFT + 2 * k + L - 1 - j]), acc[k]);
        }
        if (!PLAIN && padj_rows) {  // (E_sym^dagger)* row weight 1/c of the row's source (linear: scale the output)
          const int sr = refl_inf(r_blk + rowB, p.n0), Lp = L - 1;
          const int c = 1 + (sr < Lp ? 1 : 0) + (sr >= p.n0 - Lp ? 1 : 0);
          if (c > 1) {
            const P wv = splat2<P>(T(1) / T(c));
#pragma unroll
            for (int k = 0; k < V; k++) acc[k] = mul2(acc[k], wv);
          }
        }
        T lo[V], hi[V];
#pragma unroll
        for (int k = 0; k < V; k++) {
          lo[k] = acc[k].x;
          hi[k] = acc[k].y;
        }
        Vt *dl = reinterpret_cast<Vt *>(hist + (L - 2 + rowB) * C::HP + V * segB);
        Vt *dh = reinterpret_cast<Vt *>(hist + (C::HR + L - 2 + rowB) * C::HP + V * segB);
#pragma unroll
        for (int i = 0; i < V / VEC; i++) {
          dl[i] = vec_make<T>(lo + i * VEC);
          dh[i] = vec_make<T>(hi + i * VEC);
        }
      }
      __syncthreads();  // (2)
      // C: coefficient rows kr = kr0 + it*G + grpC*VC + v (history rows 2(grpC*VC+v) + L-1-j)
      if (actC && it >= 0) {
        const int krb = kr0 + it * G + grpC * VC;
        const T *hs = hist + setC * C::HR * C::HP + (2 * grpC * VC) * C::HP + 2 * mC;
        P win[2 * VC + L - 2];
#pragma unroll
        for (int i = 0; i < 2 * VC + L - 2; i++) win[i] = *reinterpret_cast<const P *>(hs + i * C::HP);
        P a0[VC], a1[VC];
#pragma unroll
        for (int v = 0; v < VC; v++) a0[v] = a1[v] = zero2<P>();
        using TRC = TapRange<L, ZV>;
#pragma unroll
        for (int j = L - 1; j >= 0; j--) {
          const P fl = p.slo[j], fh = p.shi[j];
#pragma unroll
          for (int v = 0; v < VC; v++) {
            if (j >= TRC::l0 && j < TRC::l1) a0[v] = fma2(fl, win[2 * v + L - 1 - j], a0[v]);
            if (j >= TRC::h0 && j < TRC::h1) a1[v] = fma2(fh, win[2 * v + L - 1 - j], a1[v]);
          }
        }
        // pitched rows: columns [m1, pitch) are padding written as 0; qc is even and so is
        // every pitch, so a pair never straddles the pitch
        // FU: this item's (y, x) tile entries: subband setC / setC + 2, row grpC*VC + v, column 2 mC
        const T *ft0 = ftile + (slot * 8 + setC * 2) * C::FT + (grpC * VC) * TQ + 2 * mC;
        const T *ft1 = ftile + (slot * 8 + (setC + 2) * 2) * C::FT + (grpC * VC) * TQ + 2 * mC;
        const bool in0 = qc < p.m1, in1 = qc + 1 < p.m1;
        const bool st0 = qc < pX0;
        if (in1 && krb + VC <= kr1) {  // fast path: whole item inside the band and the image
          T *d0 = oX0 + (long long)krb * pX0 + qc;
          T *d1 = oX1 + (long long)krb * pX1 + qc;
          if (FU && (fu0 || fu1)) {
#pragma unroll
            for (int v = 0; v < VC; v++) {
              if (fu0) fista_pair<T, L>(p, mom, d0 + v * pX0, a0[v], ft0 + v * TQ, ft0 + C::FT + v * TQ);
              else *reinterpret_cast<P *>(d0 + v * pX0) = a0[v];
              if (fu1) fista_pair<T, L>(p, mom, d1 + v * pX1, a1[v], ft1 + v * TQ, ft1 + C::FT + v * TQ);
              else *reinterpret_cast<P *>(d1 + v * pX1) = a1[v];
            }
          } else if (WL_L2HINT && p.ll_keep) {  // LL (setC 0, X = lo) evict_last; the other subbands
            const uint64_t pol0 = setC == 0 ? l2_evict_last() : l2_evict_first(), pol1 = l2_evict_first();
#pragma unroll
            for (int v = 0; v < VC; v++) {
              if (WL_L2HINT >= 2 || setC == 0) st_hint(reinterpret_cast<P *>(d0 + v * pX0), a0[v], pol0);
              else *reinterpret_cast<P *>(d0 + v * pX0) = a0[v];
              if (WL_L2HINT >= 2) st_hint(reinterpret_cast<P *>(d1 + v * pX1), a1[v], pol1);
              else *reinterpret_cast<P *>(d1 + v * pX1) = a1[v];
            }
          } else
#pragma unroll
          for (int v = 0; v < VC; v++) {
            *reinterpret_cast<P *>(d0 + v * pX0) = a0[v];
            *reinterpret_cast<P *>(d1 + v * pX1) = a1[v];
          }
        } else
#pragma unroll
        for (int v = 0; v < VC; v++) {
          const int kr = krb + v;
          if (kr >= kr1 || !st0) continue;
          P z0 = a0[v], z1 = a1[v];
          if (!in0) z0.x = z1.x = T(0);
          if (!in1) z0.y = z1.y = T(0);
          T *e0 = oX0 + (long long)kr * pX0 + qc, *e1 = oX1 + (long long)kr * pX1 + qc;
          if (FU && fu0) {  // padding entries of x and y stay 0
            fista_pair<T, L>(p, mom, e0, z0, ft0 + v * TQ, ft0 + C::FT + v * TQ);
            if (!in0) e0[0] = e0[p.xdelta] = T(0);
            if (!in1) e0[1] = e0[p.xdelta + 1] = T(0);
          } else {
            *reinterpret_cast<P *>(e0) = z0;
          }
          if (FU && fu1) {
            fista_pair<T, L>(p, mom, e1, z1, ft1 + v * TQ, ft1 + C::FT + v * TQ);
            if (!in0) e1[0] = e1[p.xdelta] = T(0);
            if (!in1) e1[1] = e1[p.xdelta + 1] = T(0);
          } else {
            *reinterpret_cast<P *>(e1) = z1;
          }
        }
      }
      __syncthreads();  // (3) history readers done
      // carry history rows [GI, GI+L-2) to [0, L-2) in both sets
      constexpr int CPR = TQ / VEC;
      constexpr int HC = (L - 2) * CPR > 0 ? (L - 2) * CPR : 1;  // (Haar carries nothing)
      for (int idx = tid; idx < 2 * (L - 2) * CPR; idx += C::NT) {
        const int set = idx / HC, rem = idx - set * HC;
        const int r = rem / CPR, c = rem - r * CPR;
        T *hb = hist + set * C::HR * C::HP;
        *reinterpret_cast<Vt *>(hb + r * C::HP + c * VEC) = *reinterpret_cast<const Vt *>(hb + (r + GI) * C::HP + c * VEC);
      }
    }
    cp_async_wait_all();
#ifdef WL_ANA_PROFILE
    __syncthreads();
    if (tid == 0 && blockIdx.x < 8192) {
      g_ana_prof[blockIdx.x][0] = t_start;
      g_ana_prof[blockIdx.x][1] = gtimer();
      g_ana_prof[blockIdx.x][2] = smid();
      g_ana_prof[blockIdx.x][3] = ((unsigned long long)col << 32) | (unsigned)(kr1 - kr0);
    }
#endif
  }
}

#ifndef WL_ANA_REGCAP
// threads per SM the register allocation must allow (fp32).  Shared memory holds 4 CTAs of 128 threads (a
// 128-register budget); asked for 6 CTAs (768) ptxas stops at 80 registers, for 4 (512) at 93-98, for 3 (384) at
// 116-124 -- still 4 CTAs per SM, with more loads in flight.  A/B on B200, 768 / 512 / 384: cfg5 W* 167.3 / 163.4 /
// 161.4 us, cfg3 W* 101.7 / 97.1 / 96.0 us, cfg5 grad 558.9 / 555.1 / 549.2 us (with the ring blur's cap)
#define WL_ANA_REGCAP 384
#endif
template <typename T, int L, bool FU, int NS, int ZV = 0, int KIND = 0>
__global__ void __launch_bounds__(ACfg<T, L, NS, FU>::NT, sizeof(T) == 4 ? WL_ANA_REGCAP / ACfg<T, L, NS, FU>::NT : 1)
    k_ana_stream(const __grid_constant__ AnaStreamParams<T, L> p) {
  using C = ACfg<T, L, NS, FU>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::OFF_BAR);
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; i++) mbar_init(bar + i, 1);
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our inputs
  unsigned phase = 0;
  ana_level_runs<T, L, FU, NS, ZV, KIND>(p, smem_raw, phase);
}

// The coarse tail of a W* / W-dagger chain in one persistent launch: levels
// j0 .. J one after another, separated by grid-wide barriers (cooperative launch: every CTA is
// resident), so the short, latency-bound levels pay no kernel boundary each.
constexpr int kMaxMulti = 12;
template <typename T, int L>
struct AnaMultiParams {
  AnaStreamParams<T, L> lev[kMaxMulti];
  int nlev;
};

template <typename T, int L>
__global__ void __launch_bounds__(ACfg<T, L, 4, false>::NT, sizeof(T) == 4 ? 768 / ACfg<T, L, 4, false>::NT : 1)
    k_ana_multi(const __grid_constant__ AnaMultiParams<T, L> mp) {
  using C = ACfg<T, L, 4, false>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::OFF_BAR);
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; i++) mbar_init(bar + i, 1);
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  unsigned phase = 0;
  for (int l = 0; l < mp.nlev; l++) {
    if (l > 0) {
      // level l-1 wrote LL_{l-1} with generic stores; level l reads it by TMA (async proxy)
      grid_sync_all();
      fence_proxy_async_all();
    }
    ana_level_runs<T, L, false, 4>(mp.lev[l], smem_raw, phase);
  }
}

#ifndef WL_ANA_MINROWS
#define WL_ANA_MINROWS 1  // minimum band height in units of G/2 coefficient rows (A/B on B200: 1 beat 2, cfg4 W* -7 %)
#endif

// Fill the launch parameters of one level.  short_run (out): the level's bands are at most
// short_run_max(3) blocks, so it runs the 4-stage variant (NS = 4); force_short: build the NS = 4
// configuration regardless (levels of k_ana_multi), with `resident4` CTAs sharing the runs.
template <typename T, int L, bool FU>
cudaError_t make_ana_params(const AnalysisArgs &a, AnaStreamParams<T, L> &p, bool &short_run, bool force_short,
                            long long resident4 = 0) {
  using C = ACfg<T, L, 0, FU>;
  using C4 = ACfg<T, L, 4, FU>;
  memset(&p, 0, sizeof p);
  p.in = static_cast<const T *>(a.in);
  p.in_pitch = a.in_pitch;
  p.in_bstride = a.in_bstride;
  p.n0 = a.n0;
  p.n1 = a.n1;
  for (int i = 0; i < 4; i++) {
    p.out[i] = static_cast<T *>(a.out[i]);
    p.out_pitch[i] = a.out_pitch[i];
    p.out_bstride[i] = a.out_bstride[i];
  }
  p.m0 = a.m0;
  p.m1 = a.m1;
  p.ext = a.ext;
  p.fast = (a.in_pitch % C::VEC == 0) && (a.in_bstride % C::VEC == 0) && (reinterpret_cast<uintptr_t>(a.in) % 16 == 0);
  const bool tma_ok = p.fast && tma_enabled();
  // the tensor map's box is the launched configuration's input block (UW columns x GI rows)
  auto encode = [&](int uw, int gi) {
    p.tma = tma_ok && encode_tmap_3d(&p.tmap, sizeof(T), a.in, (uint64_t)a.n1, (uint64_t)a.n0, (uint64_t)a.batch,
                                     (uint64_t)a.in_pitch * sizeof(T), (uint64_t)a.in_bstride * sizeof(T), uw, gi);
  };
  p.tma_any_block = a.ext == EXT_ZERO;  // TMA's zero fill is the zero extension
  for (int j = 0; j < L; j++) {
    p.flo[j] = T(a.lo[j]);
    p.fhi[j] = T(a.hi[j]);
    p.fb[j].x = T(a.lo[j]);
    p.fb[j].y = T(a.hi[j]);
    p.slo[j].x = p.slo[j].y = T(a.lo[j]);
    p.shi[j].x = p.shi[j].y = T(a.hi[j]);
  }
  p.ll_keep = a.ll_keep;
  p.fmask = a.fista_mask;
  p.xdelta = a.fista_xdelta;
  p.inv_lip = T(a.fista_inv_lip);
  p.tau = T(a.fista_tau);
  p.mom = T(a.fista_mom);
  p.tdev = a.fista_tdev;
  p.nstrips = (a.m1 + C::TQ - 1) / C::TQ;
  long long resident = 0;
  cudaError_t e;
  if (force_short) {
    short_run = true;
  } else {
    // runs of at most 3 blocks (coarse levels) prefetch all their blocks at once (NS = 4)
    e = kernel_resident(reinterpret_cast<const void *>(k_ana_stream<T, L, FU, 0>), C::NT, C::smem_bytes(FU),
                        &resident);
    if (e != cudaSuccess) return e;
    p.runs = RunMap::make((long long)a.batch * p.nstrips, a.m0, resident, std::max(1, C::G * WL_ANA_MINROWS / 2), 1,
                          balanced_runs());
    const int band = p.runs.mean_rows();
    short_run = (band + C::G - 1) / C::G <= short_run_max(3, 'a');
  }
  if (short_run) {
    if (!force_short) {
      e = kernel_resident(reinterpret_cast<const void *>(k_ana_stream<T, L, FU, 4>), C4::NT, C4::smem_bytes(FU),
                          &resident4);
      if (e != cudaSuccess) return e;
    }
    p.runs = RunMap::make((long long)a.batch * p.nstrips, a.m0, resident4, std::max(1, C4::G * WL_ANA_MINROWS / 2), 1,
                          balanced_runs());
    encode(C4::UW, C4::GI);
  } else {
    encode(C::UW, C::GI);
  }
  return cudaSuccess;
}

template <typename T, int L, bool FU, int ZV = 0>
cudaError_t launch_ana_stream_t(const AnalysisArgs &a, cudaStream_t s) {
  if (!FU && sizeof(T) == 4) {  // zero-extension levels: the register-ring kernel
    cudaError_t e = cudaSuccess;
    if (launch_analysis_ring(WL_F32, a, s, &e)) return e;
  }
  using C = ACfg<T, L, 0, FU>;
  using C4 = ACfg<T, L, 4, FU>;
  AnaStreamParams<T, L> p;
  bool short_run = false;
  cudaError_t e = make_ana_params<T, L, FU>(a, p, short_run, false);
  if (e != cudaSuccess) return e;
  long long resident = 0;
  // the compact zero-extension instantiation (fp32, plain stores) when every block comes by TMA
  constexpr bool F32 = sizeof(T) == 4;
  constexpr int K1 = F32 ? 1 : 0, K2 = (F32 && !FU) ? 2 : 0, K3 = (F32 && !FU) ? 3 : 0;  // instantiated kinds
  int kind = 0;
  if (p.tma && plain_enabled()) kind = p.tma_any_block ? K1 : (a.ext == EXT_SYM ? K2 : (a.ext == EXT_SYM_PADJ ? K3 : 0));
  auto kshort = kind == 1 ? k_ana_stream<T, L, FU, 4, ZV, K1>
                          : (kind == 2 ? k_ana_stream<T, L, FU, 4, ZV, K2>
                                       : (kind == 3 ? k_ana_stream<T, L, FU, 4, ZV, K3> : k_ana_stream<T, L, FU, 4, ZV, 0>));
  auto klong = kind == 1 ? k_ana_stream<T, L, FU, 0, ZV, K1>
                         : (kind == 2 ? k_ana_stream<T, L, FU, 0, ZV, K2>
                                      : (kind == 3 ? k_ana_stream<T, L, FU, 0, ZV, K3> : k_ana_stream<T, L, FU, 0, ZV, 0>));
  if (short_run) {
    e = kernel_resident(reinterpret_cast<const void *>(kshort), C4::NT, C4::smem_bytes(FU), &resident);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
    e = launch_pdl(kshort, grid, C4::NT, C4::smem_bytes(FU), s, p, 'a');
  } else {
    e = kernel_resident(reinterpret_cast<const void *>(klong), C::NT, C::smem_bytes(FU), &resident);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
    e = launch_pdl(klong, grid, C::NT, C::smem_bytes(FU), s, p, 'A');
  }
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// A whole W* / W-dagger chain: the long levels one launch each, the short coarse tail (>= 2
// levels) as one cooperative k_ana_multi launch (only with WL_MULTI: per-level PDL launches measured faster).
template <typename T, int L, int ZV = 0>
cudaError_t launch_ana_chain_t(const AnalysisArgs *a, int n, cudaStream_t s) {
  using C4 = ACfg<T, L, 4, false>;
  {  // the coarse levels that fit in one CTA's shared memory: one launch, one CTA per image
    const int dtype = sizeof(T) == 8 ? WL_F64 : WL_F32;
    const int i0 = small_analysis_start(dtype, a, n);
    if (i0 < n) {
      for (int i = 0; i < i0; i++) {
        cudaError_t e = launch_ana_stream_t<T, L, false, ZV>(a[i], s);
        if (e != cudaSuccess) return e;
      }
      return launch_analysis_small(dtype, a + i0, n - i0, s);
    }
  }
  int first_short = n;
  for (int i = 0; i < n && first_short == n; i++) {
    AnaStreamParams<T, L> p;
    bool sr = false;
    cudaError_t e = make_ana_params<T, L, false>(a[i], p, sr, false);
    if (e != cudaSuccess) return e;
    if (sr) first_short = i;
  }
  const int nmulti = multi_enabled() ? std::min(n - first_short, kMaxMulti) : 0;
  const int nsingle = nmulti >= 2 ? n - nmulti : n;
  for (int i = 0; i < nsingle; i++) {
    cudaError_t e = launch_ana_stream_t<T, L, false, ZV>(a[i], s);
    if (e != cudaSuccess) return e;
  }
  if (nsingle == n) return cudaSuccess;
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(k_ana_multi<T, L>), C4::NT, C4::smem_bytes(false),
                                  &resident);
  if (e != cudaSuccess) return e;
  static AnaMultiParams<T, L> mp;  // large: not on the host stack; launches copy it
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  memset(&mp, 0, sizeof mp);
  mp.nlev = n - nsingle;
  long long maxruns = 0;
  for (int l = 0; l < mp.nlev; l++) {
    bool sr = true;
    e = make_ana_params<T, L, false>(a[nsingle + l], mp.lev[l], sr, true, resident);
    if (e != cudaSuccess) return e;
    maxruns = std::max<long long>(maxruns, mp.lev[l].runs.nruns());
  }
  const int grid = (int)std::min<long long>(maxruns, resident);
  e = launch_coop(k_ana_multi<T, L>, grid, C4::NT, C4::smem_bytes(false), s, mp);
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Which TapRange matches the level's filter pair exactly (0: none, use every tap).
int zero_variant(const AnalysisArgs &a) {
  if (!zero_taps_enabled()) return 0;
  return match_tap_range(a.lo, a.hi, a.L);
}

template <typename T>
cudaError_t dispatch(const AnalysisArgs &a, cudaStream_t s) {
  if (a.fista_mask) switch (a.L) {
      case 2: return launch_ana_stream_t<T, 2, true>(a, s);
      case 4: return launch_ana_stream_t<T, 4, true>(a, s);
      case 8: return launch_ana_stream_t<T, 8, true>(a, s);
      case 10:
        switch (zero_variant(a)) {
          case 1: return launch_ana_stream_t<T, 10, true, 1>(a, s);
          case 2: return launch_ana_stream_t<T, 10, true, 2>(a, s);
          default: return launch_ana_stream_t<T, 10, true>(a, s);
        }
      case 16: return launch_ana_stream_t<T, 16, true>(a, s);
    }
  else switch (a.L) {
      case 2: return launch_ana_stream_t<T, 2, false>(a, s);
      case 4: return launch_ana_stream_t<T, 4, false>(a, s);
      case 8: return launch_ana_stream_t<T, 8, false>(a, s);
      case 10:
        switch (zero_variant(a)) {
          case 1: return launch_ana_stream_t<T, 10, false, 1>(a, s);
          case 2: return launch_ana_stream_t<T, 10, false, 2>(a, s);
          default: return launch_ana_stream_t<T, 10, false>(a, s);
        }
      case 16: return launch_ana_stream_t<T, 16, false>(a, s);
    }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t dispatch_chain(const AnalysisArgs *a, int n, cudaStream_t s) {
  switch (a[0].L) {
    case 2: return launch_ana_chain_t<T, 2>(a, n, s);
    case 4: return launch_ana_chain_t<T, 4>(a, n, s);
    case 8: return launch_ana_chain_t<T, 8>(a, n, s);
    case 10:
      switch (zero_variant(a[0])) {
        case 1: return launch_ana_chain_t<T, 10, 1>(a, n, s);
        case 2: return launch_ana_chain_t<T, 10, 2>(a, n, s);
        default: return launch_ana_chain_t<T, 10>(a, n, s);
      }
    case 16: return launch_ana_chain_t<T, 16>(a, n, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

#ifdef WL_ANA_PROFILE
extern "C" __attribute__((visibility("default"))) int wl_debug_ana_prof(void *host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_ana_prof, sizeof(unsigned long long) * 4 * (size_t)n);
}
#endif

cudaError_t launch_analysis_chain(int dtype, const AnalysisArgs *a, int n, cudaStream_t s) {
  if (n <= 0 || a[0].batch == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_chain<double>(a, n, s) : dispatch_chain<float>(a, n, s);
}

cudaError_t launch_analysis(int dtype, const AnalysisArgs &a, cudaStream_t s) {
  if (a.batch == 0 || a.m0 == 0 || a.m1 == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch<double>(a, s) : dispatch<float>(a, s);
}

}  // namespace wl
