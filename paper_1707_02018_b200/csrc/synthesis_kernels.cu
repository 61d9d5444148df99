// W: one 2-D level of the wavelet reconstruction (sm_100a), streaming column-strip kernel.
//
// Per axis the level is the exact transpose of the analysis core out[k] = sum_j f[j] yhat[2k+1-j]
// (readings R1, R5), written in gather form over extended positions t:
//     y[t] = sum_{q < H} g[2q + 1 - (t & 1)] * c[floor(t/2) + q],      H = L/2,
// with g = d_lo for the lowpass and d_hi for the highpass coefficients, c taken as zero outside
// [0, m) (zero / symmetric BC: W crops) or modulo m (periodisation: W wraps).  Output index
// i <-> extended position t = i + o (o = 0, or -(L-1) for the SYMMETRIC_EDAG variant, whose
// weighted fold runs afterwards).
//
// A CTA owns TW extended output columns of one image and a band of output rows; it walks
// down the coefficient rows G at a time:
//   A   the 4 subband windows (G rows x KCW coefficient columns) land in a double buffer:
//       one TMA box per subband (zero fill = the crop's zero coefficients), issued by one
//       thread, completed on an mbarrier; periodic plans gather with cp.async instead;
//   S1  axis-1 synthesis of each coefficient row: (LL, LH) -> VL row, (HL, HH) -> VH row
//       (FFMA2 with the tap pair (g[2q+1], g[2q]) against a broadcast coefficient) into a
//       history of H-1 carried + G new V rows;
//   S0  axis-0 synthesis: output rows 2s and 2s+1 from V rows s .. s+H-1 (FFMA2 over
//       adjacent output columns), stored as float2 pairs.
// Runs are ordered (image, band, strip) and handed to persistent CTAs so neighbouring strips
// share their coefficient halo through L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

constexpr int H_MAX = kMaxL / 2;

#ifndef WL_SYN_L2HINT
#define WL_SYN_L2HINT 1  // the LL outputs of the coarse levels stored evict_last
#endif
template <typename T, int L, int NS_ = 0>
struct SCfg {
  using P = typename Pair<T>::t;
  static constexpr int VEC = Vec16<T>::n;
  static constexpr int H = L / 2;
  static constexpr int TW = sizeof(T) == 4 ? 128 : 64;  // extended output columns per strip (even)
#ifndef WL_SYN_G
#define WL_SYN_G 16
#endif
#ifndef WL_SYN_SHORT_G
#define WL_SYN_SHORT_G 0
#endif
  // coefficient rows per iteration (short runs: WL_SYN_SHORT_G if set, A/B)
  static constexpr int G = (NS_ == 4 && WL_SYN_SHORT_G > 0) ? WL_SYN_SHORT_G : WL_SYN_G;
#ifndef WL_SYN_SP
#define WL_SYN_SP 4  // A/B on B200: 4 output column pairs per S1 item (S1 then uses all 256 threads) beat 8
#endif                // by 11 % at cfg5 and 8 % at cfg4
#ifndef WL_SYN_VC
#define WL_SYN_VC 4
#endif
  static constexpr int SP = sizeof(T) == 4 ? WL_SYN_SP : 8;   // output column pairs per S1 item
  static constexpr int VC = sizeof(T) == 4 ? WL_SYN_VC : 4;   // s-values (output row pairs) per S0 item
  static constexpr int KCW = bank_pad<T>(TW / 2 + H - 1);  // coefficient columns loaded (rows 4 mod 8 words)
  static constexpr int KCP = KCW;                        // dense TMA box rows
  static constexpr int NWC = round_up_c(SP + H - 1, VEC);  // S1 window per subband
  static constexpr int NSEG = TW / (2 * SP);
  static constexpr int TWP = conflict_free_pitch<T>(TW);
  static constexpr int HR = H - 1 + G;                   // V history rows
  static_assert(2 * SP * (NSEG - 1) / 2 + NWC <= KCW, "S1 window overruns the coefficient row");
  static_assert(G >= H - 1, "history move must not overlap");
  static constexpr int ITEMS1 = NSEG * G;
  static constexpr int ITEMS0 = (TW / 2) * (G / VC);
  static constexpr int NT = round_up_c(std::max(ITEMS1, ITEMS0), 32);
  static constexpr int NCH = KCW / VEC;                  // 16-byte chunks per coefficient row
  static constexpr size_t BAND_ELEMS = (size_t)G * KCP;  // one subband window
#ifndef WL_SYN_NS
#define WL_SYN_NS 2  // A/B on B200: 3 or 4 stages did not beat 2
#endif
  // coefficient stages (prefetch depth NS-1); short runs (coarse levels) use 4
  static constexpr int NS = NS_ > 0 ? NS_ : WL_SYN_NS;
  static constexpr size_t OFF_C = 0;                     // [NS][4][G][KCP]
  static constexpr size_t OFF_V = OFF_C + round_up_c(NS * 4 * G * KCP * (int)sizeof(T), 128);
  static constexpr size_t OFF_BAR = OFF_V + 2 * (size_t)HR * TWP * sizeof(T);  // VL, VH histories
  static constexpr size_t smem_bytes() { return OFF_BAR + NS * sizeof(uint64_t); }
};

// Structural zeros of the filter pair: nonzero tap ranges [l0, l1) (lowpass) and
// [h0, h1) (highpass) of the L-tap frame; ZV = 0: every tap (see analysis_kernels.cu TapRange).
template <int L, int ZV>
struct SynTaps {
  static constexpr int l0 = 0, l1 = L, h0 = 0, h1 = L;
};
template <>
struct SynTaps<10, 1> {  // CDF 9/7 dual filters (d_lo, d_hi): W
  static constexpr int l0 = 2, l1 = 9, h0 = 0, h1 = 9;
};
template <>
struct SynTaps<10, 2> {  // CDF 9/7 analysis filters (a_lo, a_hi): (W-dagger)*
  static constexpr int l0 = 1, l1 = 10, h0 = 1, h1 = 8;
};
template <int A0, int A1>
__host__ __device__ constexpr bool tap_in(int j) { return j >= A0 && j < A1; }

template <typename T, int L>
struct SynStreamParams {
  using P = typename Pair<T>::t;
  CUtensorMap tmap[4];       // LL, LH, HL, HH windows: box (KCW, G, 1)   (valid if tma)
  const T *in[4];
  long long in_pitch[4], in_bstride[4];
  T *out;
  long long out_pitch, out_bstride;
  int m0, m1, coef_mod, N0, N1, o0, o1;
  int t00, t01;              // first extended row / column of the output span (even)
  int nstrips;
  RunMap runs;               // (image, strip) columns x bands of extended output rows
  int tma, vec_store;
  T *y;                      // split output (symmetric folds): in-image positions go to y
  long long y_pitch, y_bstride;
  int split, yn0, yn1, y_vec;
  int out_keep;              // the output is the next level's LL: stored evict_last (WL_L2HINT)
  P g1lo[H_MAX], g1hi[H_MAX];  // S1 tap pairs (g[2q+1], g[2q])
  P e_lo[H_MAX], o_lo[H_MAX];  // S0 broadcast taps (g[2q+1], g[2q+1]) and (g[2q], g[2q])
  P e_hi[H_MAX], o_hi[H_MAX];
};

// One level's runs (the body of k_synth_stream; k_synth_multi calls it once per level of the
// coarse head of a W chain).  `phase` carries the stage barriers' parities across calls.
// PLAIN: crop (zero coefficients outside) with every window by TMA: the gather path is compiled out (a compact hot
// path for the coarse levels, which start with a cold instruction cache; see the analysis kernel).
template <typename T, int L, int NS, int ZV = 0, bool SPLIT = false, bool PLAIN = false>
__device__ __forceinline__ void syn_level_runs(const SynStreamParams<T, L> &p, unsigned char *smem_raw,
                                               unsigned &phase) {
  using C = SCfg<T, L, NS>;
  using P = typename C::P;
  using Vt = typename Vec16<T>::type;
  constexpr int G = C::G, H = C::H, VEC = C::VEC, VC = C::VC, SP = C::SP;
  T *cbuf = reinterpret_cast<T *>(smem_raw + C::OFF_C);  // [NS][4][G][KCP] coefficient windows
  T *vl = reinterpret_cast<T *>(smem_raw + C::OFF_V);    // [HR][TWP] VL history (rows s)
  T *vh = vl + C::HR * C::TWP;                           // [HR][TWP] VH history
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::OFF_BAR);
  const int tid = threadIdx.x;
  // S1 item: coefficient row fastest; S0 item: column pair fastest
  const bool act1 = tid < C::ITEMS1;
  // row fastest: the 16-byte V-history stores of 8 consecutive rows (pitch 4 mod 8 words) and the
  // coefficient window loads (box rows 4 mod 8 words) hit 8 distinct 4-bank groups
  const int row1 = tid % G, seg1 = tid / G;
  const bool act0 = tid < C::ITEMS0;
  const int m0c = tid % (C::TW / 2), grp0 = tid / (C::TW / 2);

  int col, b0, b1;
  for (RunIter itr(p.runs); itr.next(col, b0, b1);) {
    const int img = col / p.nstrips, strip = col - img * p.nstrips;
    if (b0 >= b1) continue;  // (uniform) empty trailing band
    const int tr0 = p.t00 + b0;  // even (bands are even)
    const int tr1 = p.t00 + b1;
    const int tc0 = p.t01 + strip * C::TW;                            // even
    const int kc0 = tc0 / 2;                                          // first coefficient column
    const int s_first = tr0 / 2, s_last = (tr1 - 1) >> 1;
    const int n_it = (s_last - s_first + H - 1) / G + 1;
    T *out = p.out + (long long)img * p.out_bstride;
    // S0 output column pair (extended t = tc0 + 2 m0c, +1) -> output index
    const int oc = tc0 + 2 * m0c - p.o1;
    const bool col_in = oc + 1 >= 0 && oc < p.N1;
    const bool vec_ok = p.vec_store && oc >= 0 && oc + 1 < p.N1;

    // batch k: coefficient rows s_first + kG .. of the 4 subbands -> cbuf[k % NS]
    auto load_batch = [&](int k) -> bool {
      const int kr = s_first + k * G;
      const int sl = k % C::NS;
      T *dst0 = cbuf + sl * 4 * C::BAND_ELEMS;
      // periodic plans: TMA only for windows that need no wrap (the zero fill is the crop otherwise)
      if (PLAIN || (p.tma && (!p.coef_mod || (kr >= 0 && kr + G <= p.m0 && kc0 >= 0 && kc0 + C::KCW <= p.m1)))) {
        if (tid == 0) {
          fence_proxy_async();
          mbar_arrive_expect_tx(bar + sl, 4 * C::BAND_ELEMS * sizeof(T));
#pragma unroll
          for (int bnd = 0; bnd < 4; bnd++) tma_load_3d(dst0 + bnd * C::BAND_ELEMS, &p.tmap[bnd], bar + sl, kc0, kr, img);
        }
        return true;
      }
      if (PLAIN) return true;  // (unreachable: the branch above is taken)
      for (int idx = tid; idx < 4 * G * C::NCH; idx += C::NT) {
        const int bnd = idx / (G * C::NCH), rem = idx - bnd * G * C::NCH;
        const int r = rem / C::NCH, v = rem - r * C::NCH;
        int krr = kr + r;
        const int cg = kc0 + v * VEC;
        T *dst = dst0 + bnd * C::BAND_ELEMS + r * C::KCP + v * VEC;
        bool row_ok = true;
        if (p.coef_mod) {
          if (krr < 0 || krr >= p.m0) {  // wrap (integer division only off the common path)
            krr %= p.m0;
            if (krr < 0) krr += p.m0;
          }
        } else {
          row_ok = krr >= 0 && krr < p.m0;
        }
        const T *row = p.in[bnd] + (long long)img * p.in_bstride[bnd] + (long long)krr * p.in_pitch[bnd];
        if (row_ok && cg >= 0 && cg + VEC <= p.m1 && ((cg & (VEC - 1)) == 0)) {
          cp_async16(dst, row + cg);
        } else if (p.coef_mod && p.m1 % VEC == 0 && (cg & (VEC - 1)) == 0 && (cg >= -p.m1 && cg < 2 * p.m1) &&
                   (cg < 0 ? cg + p.m1 : (cg >= p.m1 ? cg - p.m1 : cg)) + VEC <= p.m1) {
          cp_async16(dst, row + (cg < 0 ? cg + p.m1 : (cg >= p.m1 ? cg - p.m1 : cg)));  // whole aligned wrapped chunk
        } else {
          T z[VEC];
#pragma unroll
          for (int i = 0; i < VEC; i++) {
            int c = cg + i;
            bool ok = row_ok;
            if (p.coef_mod) {
              if (c < 0 || c >= p.m1) {
                c %= p.m1;
                if (c < 0) c += p.m1;
              }
            } else {
              ok = ok && c >= 0 && c < p.m1;
            }
            z[i] = ok ? row[c] : T(0);
          }
          *reinterpret_cast<Vt *>(dst) = vec_make<T>(z);
        }
      }
      return false;
    };

    __syncthreads();  // previous run's readers are done
    unsigned armed = 0;  // bit s: the batch in slot s armed its barrier
#pragma unroll 1  // one copy of the batch loader (code size; see the analysis kernel)
    for (int k = 0; k < C::NS - 1; k++) {
      if (k < n_it && load_batch(k)) armed |= 1u << (k % C::NS);
      cp_async_commit();
    }
    for (int it = 0; it < n_it; it++) {
      const int slot = it % C::NS;
      cp_async_wait_group<C::NS - 2>();  // this thread's gathers of batch it are done
      if ((armed >> slot) & 1) {
        mbar_wait(bar + slot, (phase >> slot) & 1);
        phase ^= 1u << slot;
      }
      __syncthreads();  // (1) batch it landed; the history move of it-1 is done
      {
        const int nb = it + C::NS - 1;  // its slot held batch it-1, consumed before (1)
        armed &= ~(1u << (nb % C::NS));
        if (nb < n_it && load_batch(nb)) armed |= 1u << (nb % C::NS);
      }
      cp_async_commit();
      // S1: coefficient row r of the batch -> V rows (history index H-1+r), output pairs SP*seg1 ..
      if (act1) {
        const T *cb = cbuf + (it % C::NS) * 4 * C::BAND_ELEMS + row1 * C::KCP + SP * seg1;
#pragma unroll 1
        for (int pr = 0; pr < 2; pr++) {  // pr 0: (LL, LH) -> VL; 1: (HL, HH) -> VH
          T a[C::NWC], d[C::NWC];
          const Vt *sa = reinterpret_cast<const Vt *>(cb + (2 * pr) * C::BAND_ELEMS);
          const Vt *sd = reinterpret_cast<const Vt *>(cb + (2 * pr + 1) * C::BAND_ELEMS);
#pragma unroll
          for (int i = 0; i < C::NWC / VEC; i++) {
            vec_split<T>(sa[i], a + i * VEC);
            vec_split<T>(sd[i], d + i * VEC);
          }
          P ov[SP];
#pragma unroll
          for (int j = 0; j < SP; j++) ov[j] = zero2<P>();
          using TS = SynTaps<L, ZV>;
#pragma unroll
          for (int q = 0; q < H; q++) {  // tap-outer: two tap pairs live at a time
            const P gl = p.g1lo[q], gh = p.g1hi[q];
            // pair q = (g[2q+1], g[2q]): skipped when both taps are structural zeros
#pragma unroll
            for (int j = 0; j < SP; j++) {
              if (2 * q + 2 > TS::l0 && 2 * q < TS::l1) ov[j] = fma2(gl, splat2<P>(a[j + q]), ov[j]);
              if (2 * q + 2 > TS::h0 && 2 * q < TS::h1) ov[j] = fma2(gh, splat2<P>(d[j + q]), ov[j]);
            }
          }
          T *vrow = (pr == 0 ? vl : vh) + (H - 1 + row1) * C::TWP + 2 * SP * seg1;
#pragma unroll
          for (int i = 0; i < 2 * SP / VEC; i++) {
            T tmp[VEC];
#pragma unroll
            for (int u = 0; u < VEC; u += 2) {
              tmp[u] = ov[(i * VEC + u) / 2].x;
              tmp[u + 1] = ov[(i * VEC + u) / 2].y;
            }
            reinterpret_cast<Vt *>(vrow)[i] = vec_make<T>(tmp);
          }
        }
      }
      __syncthreads();  // (2)
      // S0: s = s_first + it*G - (H-1) + grp0*VC + v  (history index grp0*VC + v)
      if (act0 && col_in) {
        const int sb = s_first + it * G - (H - 1) + grp0 * VC;
        P wl[VC + H - 1], wh[VC + H - 1];
#pragma unroll
        for (int i = 0; i < VC + H - 1; i++) {
          wl[i] = *reinterpret_cast<const P *>(vl + (grp0 * VC + i) * C::TWP + 2 * m0c);
          wh[i] = *reinterpret_cast<const P *>(vh + (grp0 * VC + i) * C::TWP + 2 * m0c);
        }
        // tap-outer order: only the 4 broadcast tap pairs of one q are live at a time
        P e[VC], o[VC];
#pragma unroll
        for (int v = 0; v < VC; v++) e[v] = o[v] = zero2<P>();
        using TS0 = SynTaps<L, ZV>;
#pragma unroll
        for (int q = 0; q < H; q++) {
          const P el = p.e_lo[q], ol = p.o_lo[q], eh = p.e_hi[q], oh = p.o_hi[q];
#pragma unroll
          for (int v = 0; v < VC; v++) {  // e: g[2q+1], o: g[2q]; structural zeros skipped
            if (tap_in<TS0::l0, TS0::l1>(2 * q + 1)) e[v] = fma2(el, wl[v + q], e[v]);
            if (tap_in<TS0::l0, TS0::l1>(2 * q)) o[v] = fma2(ol, wl[v + q], o[v]);
            if (tap_in<TS0::h0, TS0::h1>(2 * q + 1)) e[v] = fma2(eh, wh[v + q], e[v]);
            if (tap_in<TS0::h0, TS0::h1>(2 * q)) o[v] = fma2(oh, wh[v + q], o[v]);
          }
        }
        // fast path: every output row of the item lies in the run and the image, pair stores
        const int t_lo = 2 * sb, t_hi = 2 * (sb + VC);  // [t_lo, t_hi)
        const bool run_in = sb >= s_first && sb + VC - 1 <= s_last && t_lo >= tr0 && t_hi <= tr1;
        // split output: pairs inside the image go to y, the rest to out (U's border frame)
        const int t1 = oc + p.o1;  // extended column of the pair (even)
        const bool pair_y = SPLIT && t1 >= 0 && t1 + 1 < p.yn1;
        const bool pair_u = !SPLIT || t1 + 1 < 0 || t1 >= p.yn1;
        if (SPLIT && pair_y && p.y_vec && run_in && t_lo >= 0 && t_hi <= p.yn0) {
          T *op = p.y + (long long)img * p.y_bstride + (long long)t_lo * p.y_pitch + t1;
#pragma unroll
          for (int v = 0; v < VC; v++) {
            *reinterpret_cast<P *>(op + (2 * v) * p.y_pitch) = e[v];
            *reinterpret_cast<P *>(op + (2 * v + 1) * p.y_pitch) = o[v];
          }
        } else if ((pair_u || t_hi <= 0 || t_lo >= p.yn0) && vec_ok && run_in && t_lo - p.o0 >= 0 &&
                   t_hi - p.o0 <= p.N0) {
          T *op = out + (long long)(t_lo - p.o0) * p.out_pitch + oc;
          if (WL_SYN_L2HINT && p.out_keep) {
            const uint64_t pol = l2_evict_last();
#pragma unroll
            for (int v = 0; v < VC; v++) {
              st_hint(reinterpret_cast<P *>(op + (2 * v) * p.out_pitch), e[v], pol);
              st_hint(reinterpret_cast<P *>(op + (2 * v + 1) * p.out_pitch), o[v], pol);
            }
          } else
#pragma unroll
          for (int v = 0; v < VC; v++) {
            *reinterpret_cast<P *>(op + (2 * v) * p.out_pitch) = e[v];
            *reinterpret_cast<P *>(op + (2 * v + 1) * p.out_pitch) = o[v];
          }
        } else if (SPLIT) {  // split output, item at a band end or the image border: route per row
#pragma unroll
          for (int v = 0; v < VC; v++) {
            const int s = sb + v;
            if (s < s_first || s > s_last) continue;
#pragma unroll
            for (int par = 0; par < 2; par++) {
              const int t = 2 * s + par;
              const int orow = t - p.o0;
              if (t < tr0 || t >= tr1 || orow < 0 || orow >= p.N0) continue;
              const P val = par ? o[v] : e[v];
              const bool row_y = t >= 0 && t < p.yn0;
              T *yp = p.y + (long long)img * p.y_bstride + (long long)t * p.y_pitch + t1;
              T *op = out + (long long)orow * p.out_pitch + oc;
              if (row_y && pair_y && p.y_vec) {
                *reinterpret_cast<P *>(yp) = val;
              } else if ((!row_y || pair_u) && vec_ok) {
                *reinterpret_cast<P *>(op) = val;
              } else {  // a pair straddling the image's right edge (odd n1)
                if (row_y && t1 >= 0 && t1 < p.yn1) yp[0] = val.x;
                else if (oc >= 0 && oc < p.N1) op[0] = val.x;
                if (row_y && t1 + 1 >= 0 && t1 + 1 < p.yn1) yp[1] = val.y;
                else if (oc + 1 >= 0 && oc + 1 < p.N1) op[1] = val.y;
              }
            }
          }
        } else {
#pragma unroll
        for (int v = 0; v < VC; v++) {
          const int s = sb + v;
          if (s < s_first || s > s_last) continue;
#pragma unroll
          for (int par = 0; par < 2; par++) {
            const int t = 2 * s + par;
            const int orow = t - p.o0;
            if (t < tr0 || t >= tr1 || orow < 0 || orow >= p.N0) continue;
            const P val = par ? o[v] : e[v];
            T *op = out + (long long)orow * p.out_pitch + oc;
            if (vec_ok) {
              *reinterpret_cast<P *>(op) = val;
            } else {
              if (oc >= 0 && oc < p.N1) op[0] = val.x;
              if (oc + 1 >= 0 && oc + 1 < p.N1) op[1] = val.y;
            }
          }
        }
        }
      }
      __syncthreads();  // (3) V history readers done
      // carry V rows [G, G+H-1) to the head of the history
      constexpr int HC = (H - 1) * (C::TW / VEC) > 0 ? (H - 1) * (C::TW / VEC) : 1;  // (Haar carries nothing)
      for (int idx = tid; idx < 2 * (H - 1) * (C::TW / VEC); idx += C::NT) {
        const int half = idx / HC;
        const int rem = idx - half * HC;
        const int r = rem / (C::TW / VEC), c = rem - r * (C::TW / VEC);
        T *hb = half ? vh : vl;
        *reinterpret_cast<Vt *>(hb + r * C::TWP + c * VEC) = *reinterpret_cast<const Vt *>(hb + (r + G) * C::TWP + c * VEC);
      }
    }
    cp_async_wait_all();
  }
}

// (the split variant is capped at the plain kernel's register count so it keeps its CTAs per SM)
#ifndef WL_SYN_REGCAP
#define WL_SYN_REGCAP 768  // threads per SM the register allocation must allow (fp32)
#endif
template <typename T, int L, int NS, int ZV = 0, bool SPLIT = false, bool PLAIN = false>
__global__ void __launch_bounds__(SCfg<T, L>::NT, sizeof(T) == 4 ? (SPLIT ? 1024 : WL_SYN_REGCAP) / SCfg<T, L>::NT : 1)
    k_synth_stream(const __grid_constant__ SynStreamParams<T, L> p) {
  using C = SCfg<T, L, NS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::OFF_BAR);
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; i++) mbar_init(bar + i, 1);
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our inputs
  unsigned phase = 0;
  syn_level_runs<T, L, NS, ZV, SPLIT, PLAIN>(p, smem_raw, phase);
}

// The coarse head of a W chain (levels J .. j0, coarse -> fine) in one persistent cooperative
// launch with grid-wide barriers between the levels.
constexpr int kMaxMulti = 12;
template <typename T, int L>
struct SynMultiParams {
  SynStreamParams<T, L> lev[kMaxMulti];
  int nlev;
};

template <typename T, int L>
__global__ void __launch_bounds__(SCfg<T, L>::NT, sizeof(T) == 4 ? 768 / SCfg<T, L>::NT : 1)
    k_synth_multi(const __grid_constant__ SynMultiParams<T, L> mp) {
  using C = SCfg<T, L, 4>;
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
      grid_sync_all();          // level l-1 stored LL with generic stores ...
      fence_proxy_async_all();  // ... level l reads it by TMA (async proxy)
    }
    syn_level_runs<T, L, 4>(mp.lev[l], smem_raw, phase);
  }
}

#ifndef WL_SYN_MINROWS
#define WL_SYN_MINROWS 1  // minimum band height in units of G output rows (A/B on B200: 1 beat 2 on every small config)
#endif

// Fill the launch parameters of one level; short_run (out): bands of at most short_run_max(2)
// batches run the 4-stage variant; force_short: NS = 4 with `resident4` CTAs (k_synth_multi levels).
template <typename T, int L>
cudaError_t make_syn_params(const SynthesisArgs &a, SynStreamParams<T, L> &p, bool &short_run, bool force_short,
                            long long resident4 = 0) {
  using C = SCfg<T, L>;
  using C4 = SCfg<T, L, 4>;
  static_assert(C::H <= H_MAX, "H_MAX");
  memset(&p, 0, sizeof p);
  const bool tma_ok = tma_enabled();  // WL_NO_TMA: debugging / A-B switch
  for (int i = 0; i < 4; i++) {
    p.in[i] = static_cast<const T *>(a.in[i]);
    p.in_pitch[i] = a.in_pitch[i];
    p.in_bstride[i] = a.in_bstride[i];
  }
  // the tensor maps' box is the launched configuration's coefficient window (KCW x G)
  auto encode = [&](int kcw, int g) {
    bool tma = tma_ok;
    for (int i = 0; i < 4 && tma; i++)
      tma = encode_tmap_3d(&p.tmap[i], sizeof(T), a.in[i], (uint64_t)a.m1, (uint64_t)a.m0, (uint64_t)a.batch,
                           (uint64_t)a.in_pitch[i] * sizeof(T), (uint64_t)a.in_bstride[i] * sizeof(T), kcw, g);
    p.tma = tma;
  };
  p.out = static_cast<T *>(a.out);
  p.out_pitch = a.out_pitch;
  p.out_bstride = a.out_bstride;
  p.m0 = a.m0; p.m1 = a.m1; p.coef_mod = a.coef_mod;
  p.N0 = a.N0; p.N1 = a.N1; p.o0 = a.o0; p.o1 = a.o1;
  p.t00 = 2 * (a.o0 >> 1);
  // strips start at a column whose coefficient column kc0 = t01/2 is 16-byte aligned: TMA box
  // coordinates must address 16-byte aligned global columns (odd EDAG offsets would not)
  p.t01 = 2 * C::VEC * (int)std::floor((double)a.o1 / (2.0 * C::VEC));
  p.vec_store = (a.o1 % 2 == 0) && (a.out_pitch % 2 == 0) && (a.out_bstride % 2 == 0) &&
                (reinterpret_cast<uintptr_t>(a.out) % (2 * sizeof(T)) == 0);
  p.out_keep = a.out_keep;
  p.y = static_cast<T *>(a.y);
  p.split = a.y != nullptr;
  p.y_pitch = a.y_pitch;
  p.y_bstride = a.y_bstride;
  p.yn0 = a.yn0;
  p.yn1 = a.yn1;
  // pairs start at even extended columns t1: 8-byte aligned in y when its pitch is even
  p.y_vec = p.split && (a.y_pitch % 2 == 0) && (a.y_bstride % 2 == 0) &&
            (reinterpret_cast<uintptr_t>(a.y) % (2 * sizeof(T)) == 0);
  for (int q = 0; q < C::H; q++) {
    p.g1lo[q].x = T(a.lo[2 * q + 1]); p.g1lo[q].y = T(a.lo[2 * q]);
    p.g1hi[q].x = T(a.hi[2 * q + 1]); p.g1hi[q].y = T(a.hi[2 * q]);
    p.e_lo[q].x = p.e_lo[q].y = T(a.lo[2 * q + 1]);
    p.o_lo[q].x = p.o_lo[q].y = T(a.lo[2 * q]);
    p.e_hi[q].x = p.e_hi[q].y = T(a.hi[2 * q + 1]);
    p.o_hi[q].x = p.o_hi[q].y = T(a.hi[2 * q]);
  }
  const int span0 = a.o0 + a.N0 - p.t00, span1 = a.o1 + a.N1 - p.t01;
  p.nstrips = (span1 + C::TW - 1) / C::TW;
  long long resident = 0;
  cudaError_t e;
  if (force_short) {
    short_run = true;
  } else {
    e = kernel_resident(reinterpret_cast<const void *>(k_synth_stream<T, L, 0>), C::NT, C::smem_bytes(), &resident);
    if (e != cudaSuccess) return e;
    // one run per resident CTA when the columns allow it; even bands of >= 4 iterations
    p.runs = RunMap::make((long long)a.batch * p.nstrips, span0, resident, WL_SYN_MINROWS * C::G, 2, balanced_runs());
    const int band = p.runs.mean_rows();
    short_run = (band / 2 + C::H - 1) / C::G + 1 <= short_run_max(2, 's');
  }
  if (short_run) {
    // short runs (coarse levels): every batch of the run in flight at once
    if (!force_short) {
      e = kernel_resident(reinterpret_cast<const void *>(k_synth_stream<T, L, 4>), C4::NT, C4::smem_bytes(),
                          &resident4);
      if (e != cudaSuccess) return e;
    }
    p.runs = RunMap::make((long long)a.batch * p.nstrips, span0, resident4, WL_SYN_MINROWS * C4::G, 2,
                          balanced_runs());
    encode(C4::KCW, C4::G);
  } else {
    encode(C::KCW, C::G);
  }
  return cudaSuccess;
}

template <typename T, int L, int ZV = 0>
cudaError_t launch_synth_stream_t(const SynthesisArgs &a, cudaStream_t s) {
  using C = SCfg<T, L>;
  using C4 = SCfg<T, L, 4>;
  SynStreamParams<T, L> p;
  bool short_run = false;
  cudaError_t e = make_syn_params<T, L>(a, p, short_run, false);
  if (e != cudaSuccess) return e;
  long long resident = 0;
  // split outputs (symmetric folds) take their own instantiation: the routing costs registers
  // the compact crop instantiation (fp32) when every window comes by TMA
  constexpr bool HAS_PLAIN = sizeof(T) == 4;
  const bool plain = HAS_PLAIN && !p.split && p.tma && !p.coef_mod && plain_enabled();
  auto kshort = p.split ? k_synth_stream<T, L, 4, ZV, true>
                        : (plain ? k_synth_stream<T, L, 4, ZV, false, HAS_PLAIN> : k_synth_stream<T, L, 4, ZV, false>);
  auto klong = p.split ? k_synth_stream<T, L, 0, ZV, true>
                       : (plain ? k_synth_stream<T, L, 0, ZV, false, HAS_PLAIN> : k_synth_stream<T, L, 0, ZV, false>);
  if (short_run) {
    e = kernel_resident(reinterpret_cast<const void *>(kshort), C4::NT, C4::smem_bytes(), &resident);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
    e = launch_pdl(kshort, grid, C4::NT, C4::smem_bytes(), s, p, 's');
  } else {
    e = kernel_resident(reinterpret_cast<const void *>(klong), C::NT, C::smem_bytes(), &resident);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
    e = launch_pdl(klong, grid, C::NT, C::smem_bytes(), s, p, 'S');
  }
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// A whole W chain given coarse -> fine (a[0] = level J): its short head (>= 2 levels) as one
// cooperative k_synth_multi launch, then the long levels one launch each (only with WL_MULTI: per-level PDL launches measured faster).
template <typename T, int L, int ZV = 0>
cudaError_t launch_syn_chain_t(const SynthesisArgs *a, int n, cudaStream_t s) {
  using C4 = SCfg<T, L, 4>;
  {  // the coarse levels that fit in one CTA's shared memory: one launch, one CTA per image
    const int dtype = sizeof(T) == 8 ? WL_F64 : WL_F32;
    const int i1 = small_synthesis_end(dtype, a, n);
    if (i1 > 0) {
      cudaError_t e = launch_synthesis_small(dtype, a, i1, s);
      if (e != cudaSuccess) return e;
      for (int i = i1; i < n; i++) {
        e = launch_synth_stream_t<T, L, ZV>(a[i], s);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
  }
  int nshort = 0;  // coarse levels are short first: count the leading short ones
  for (int i = 0; i < n; i++) {
    SynStreamParams<T, L> p;
    bool sr = false;
    cudaError_t e = make_syn_params<T, L>(a[i], p, sr, false);
    if (e != cudaSuccess) return e;
    if (!sr) break;
    nshort++;
  }
  const int nmulti = (multi_enabled() && nshort >= 2) ? std::min(nshort, kMaxMulti) : 0;
  if (nmulti) {
    long long resident = 0;
    cudaError_t e = kernel_resident(reinterpret_cast<const void *>(k_synth_multi<T, L>), C4::NT, C4::smem_bytes(),
                                    &resident);
    if (e != cudaSuccess) return e;
    static SynMultiParams<T, L> mp;  // large: not on the host stack; launches copy it
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    memset(&mp, 0, sizeof mp);
    mp.nlev = nmulti;
    long long maxruns = 0;
    for (int l = 0; l < nmulti; l++) {
      bool sr = true;
      e = make_syn_params<T, L>(a[l], mp.lev[l], sr, true, resident);
      if (e != cudaSuccess) return e;
      maxruns = std::max<long long>(maxruns, mp.lev[l].runs.nruns());
    }
    const int grid = (int)std::min<long long>(maxruns, resident);
    e = launch_coop(k_synth_multi<T, L>, grid, C4::NT, C4::smem_bytes(), s, mp);
    g_launches++;
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  for (int i = nmulti; i < n; i++) {
    cudaError_t e = launch_synth_stream_t<T, L, ZV>(a[i], s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t dispatch(const SynthesisArgs &a, cudaStream_t s) {
  switch (a.L) {
    case 2: return launch_synth_stream_t<T, 2>(a, s);
    case 4: return launch_synth_stream_t<T, 4>(a, s);
    case 8: return launch_synth_stream_t<T, 8>(a, s);
    case 10:
      switch (zero_taps_enabled() ? match_tap_range(a.lo, a.hi, 10) : 0) {
        case 1: return launch_synth_stream_t<T, 10, 1>(a, s);
        case 2: return launch_synth_stream_t<T, 10, 2>(a, s);
        default: return launch_synth_stream_t<T, 10>(a, s);
      }
    case 16: return launch_synth_stream_t<T, 16>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t dispatch_chain(const SynthesisArgs *a, int n, cudaStream_t s) {
  switch (a[0].L) {
    case 2: return launch_syn_chain_t<T, 2>(a, n, s);
    case 4: return launch_syn_chain_t<T, 4>(a, n, s);
    case 8: return launch_syn_chain_t<T, 8>(a, n, s);
    case 10:
      switch (zero_taps_enabled() ? match_tap_range(a[0].lo, a[0].hi, 10) : 0) {
        case 1: return launch_syn_chain_t<T, 10, 1>(a, n, s);
        case 2: return launch_syn_chain_t<T, 10, 2>(a, n, s);
        default: return launch_syn_chain_t<T, 10>(a, n, s);
      }
    case 16: return launch_syn_chain_t<T, 16>(a, n, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_synthesis_chain(int dtype, const SynthesisArgs *a, int n, cudaStream_t s) {
  if (n <= 0 || a[0].batch == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch_chain<double>(a, n, s) : dispatch_chain<float>(a, n, s);
}

cudaError_t launch_synthesis(int dtype, const SynthesisArgs &a, cudaStream_t s) {
  if (a.batch == 0 || a.N0 == 0 || a.N1 == 0) return cudaSuccess;
  return dtype == WL_F64 ? dispatch<double>(a, s) : dispatch<float>(a, s);
}

}  // namespace wl
