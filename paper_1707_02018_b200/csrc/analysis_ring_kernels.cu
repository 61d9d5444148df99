// Register-ring analysis level (sm_100a, fp32): one 2-D level of W* (and of W-dagger under the
// zero extension), for every level whose extension is the zero extension -- W* under zero and
// symmetric BC (Eq. (4) with E = E_zpd, reading R1), W-dagger under zero BC.
//
// Analysis core (reading R5):  out[k] = sum_{j<L} f[j] * yhat[2k+1-j], along
// axis 1 then axis 0; subband XY = axis-0 filter X, axis-1 filter Y.
//
// Design (DESIGN.md §6 "k_ana_ring").  A CTA of 128 threads owns 128 coefficient columns of one
// image and walks down a band of coefficient rows, one row (two input rows) per step.  Thread q
// owns coefficient column k = q0 + q in every stage, so no value crosses threads:
//   * axis-1 pass: the window yhat[2k+2-L .. 2k+1] of each new input row (L/2 aligned 8-byte
//     loads from shared memory) gives the pair (lo[k], hi[k]) with one FFMA2 per tap (tap pair
//     (f_lo[j], f_hi[j]) against the broadcast sample);
//   * axis-0 pass: the thread keeps the last L (lo, hi) rows in a register ring and emits
//     (LL, LH) = sum_j f_lo[j] ring[2kr+1-j] and (HL, HH) = sum_j f_hi[j] ring[2kr+1-j] with one
//     FFMA2 per tap and subband pair.  A group of input rows is a whole number of ring periods,
//     so every ring index is a compile-time register; the vertical halo costs no shared memory
//     and no barrier.
// Input rows arrive G per group (two TMA boxes: threads 0-63 read box 0, 64-127 box 1) into a
// 3-stage ring completed on mbarriers; TMA's zero fill outside the image *is* the zero extension,
// so edge strips and the top / bottom of a band need no special case.  One __syncthreads per group
// frees its stage.  Stores: four coalesced 4-byte rows per step (one per subband); the columns in
// [m1, pitch) read only zero-filled samples, so the pitch padding is written as 0 by the same
// stores.  Bytes: es (N + p) per image and level; FLOPs: 2L FFMA2 lane pairs per coefficient.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

template <int L>
struct ARingCfg {
  static constexpr int NT = 128;                        // threads = coefficient columns per strip
  static constexpr int TQ = NT;
  static constexpr int HALF = NT / 2;                   // threads per TMA box
  static constexpr int SHIFT = ((2 - L) % 4 + 4) % 4;   // box column of input column 2 q0 + 2 - L
  // thread q' of a box reads box columns [2q' + SHIFT, 2q' + SHIFT + L)
  static constexpr int UBX = round_up_c(2 * HALF - 2 + SHIFT + L, 4);
  static constexpr int P = (L - 2) / 2;                 // priming steps of a band (ring fill)
  static constexpr int NSG = (L / 2 >= 4) ? L / 2 : 4;  // steps per group: whole ring periods (L/2)
  static constexpr int G = 2 * NSG;                     // input rows per group
#ifndef WL_ARING_S
#define WL_ARING_S 2  // A/B on B200: 2 stages (5 CTAs per SM, register-bound) beat 3 (4 CTAs): cfg4 W* level 1 38.9 -> 36.9 us cold
#endif
  static constexpr int S = WL_ARING_S;                  // shared-memory stages
  static constexpr int REG = round_up_c(G * UBX * 4, 128) / 4;  // floats per (stage, box)
  static constexpr size_t OFF_BAR = (size_t)S * 2 * REG * 4;
  static constexpr size_t SMEM = OFF_BAR + S * sizeof(uint64_t);
  static_assert(NSG % (L / 2 > 0 ? L / 2 : 1) == 0, "a group must be whole ring periods");
};

template <int L>
struct ARingParams {
  CUtensorMap tmap;  // input: box (UBX, G, 1)
  float *out[4];     // LL, LH, HL, HH
  long long out_bstride[4];
  long long pitch;   // common row pitch of the four subbands
  int nstrips;
  RunMap runs;       // (image, strip) columns x bands of coefficient rows
  float2 tp[L];      // tap pairs (f_lo[j], f_hi[j]): axis 1 as pairs, axis 0 broadcast per half
};

#ifndef WL_ARING_MINB
#define WL_ARING_MINB 4
#endif
template <int L, int ZV>
__global__ void __launch_bounds__(128, WL_ARING_MINB) k_ana_ring(const __grid_constant__ ARingParams<L> p) {
  using C = ARingCfg<L>;
  using TR = TapRange<L, ZV>;
  constexpr int G = C::G, S = C::S, NSG = C::NSG, P = C::P;
  constexpr int JH0 = TR::l0 < TR::h0 ? TR::l0 : TR::h0, JH1 = TR::l1 > TR::h1 ? TR::l1 : TR::h1;
  extern __shared__ __align__(128) unsigned char sm[];
  float *ubase = reinterpret_cast<float *>(sm);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int s = 0; s < S; s++) mbar_init(full + s, 1);
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our input
  float2 ring[L];
#pragma unroll
  for (int i = 0; i < L; i++) ring[i] = make_float2(0.f, 0.f);
  const int box = tid / C::HALF, qq = tid - box * C::HALF;
  const long long pitch = p.pitch;

  unsigned gbase = 0;  // groups of earlier runs: global group g = gbase + k fixes stages and parities
  int col, kr0, kr1;
  for (RunIter itr(p.runs); itr.next(col, kr0, kr1);) {
    if (kr0 >= kr1) continue;  // (uniform) empty trailing band
    const int img = col / p.nstrips, strip = col - img * p.nstrips;
    const int q0 = strip * C::TQ, k = q0 + tid;
    const int cbox = 2 * q0 + 2 - L - C::SHIFT;  // input column of box 0's column 0 (16-byte aligned)
    const int nsteps = kr1 - kr0 + P;
    const int ngroups = (nsteps + NSG - 1) / NSG;
    const int row0 = 2 * (kr0 - P);              // input row of step 0
    const bool kst = k < pitch;                  // columns [m1, pitch) are padding (stored 0)
    // this thread's output column of coefficient row kr0 (step P)
    float *o0 = p.out[0] + img * p.out_bstride[0] + (long long)kr0 * pitch + k;
    float *o1 = p.out[1] + img * p.out_bstride[1] + (long long)kr0 * pitch + k;
    float *o2 = p.out[2] + img * p.out_bstride[2] + (long long)kr0 * pitch + k;
    float *o3 = p.out[3] + img * p.out_bstride[3] + (long long)kr0 * pitch + k;
    long long roff = 0;

    __syncthreads();  // the previous run's readers of every stage are done
    auto issue = [&](int g) {
      const int st = (gbase + g) % S;
      float *dst = ubase + st * 2 * C::REG;
      fence_proxy_async();
      mbar_arrive_expect_tx(full + st, 2u * G * C::UBX * 4u);
      tma_load_3d(dst, &p.tmap, full + st, cbox, row0 + g * G, img);
      tma_load_3d(dst + C::REG, &p.tmap, full + st, cbox + 2 * C::HALF, row0 + g * G, img);
    };
    if (tid == 0)
      for (int g = 0; g < S && g < ngroups; g++) issue(g);

    for (int g = 0; g < ngroups; g++) {
      const unsigned gg = gbase + g;
      const int st = gg % S;
      mbar_wait(full + st, (gg / S) & 1);
      const float *src = ubase + st * 2 * C::REG + box * C::REG + 2 * qq + C::SHIFT;
      // steps t of this group with an output row: vlo <= t < vhi
      const int vlo = P - g * NSG, vhi = P + (kr1 - kr0) - g * NSG;
#pragma unroll
      for (int t = 0; t < NSG; t++) {
        // axis-1 pass of input rows 2t, 2t+1 of the group -> ring slots (2t) % L, (2t+1) % L
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const float2 *w2 = reinterpret_cast<const float2 *>(src + (2 * t + e) * C::UBX);
          float win[L];
#pragma unroll
          for (int j = 0; j < L / 2; j++) {
            const float2 v = w2[j];
            win[2 * j] = v.x;
            win[2 * j + 1] = v.y;
          }
          // two accumulator chains (even / odd taps): half the dependent-FFMA2 latency
          float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = JH0; j < JH1; j++) {
            if ((j - JH0) % 2 == 0) acc0 = fma2(p.tp[j], splat2<float2>(win[L - 1 - j]), acc0);
            else acc1 = fma2(p.tp[j], splat2<float2>(win[L - 1 - j]), acc1);
          }
          ring[(2 * t + e) % L] = JH1 - JH0 > 1 ? add2(acc0, acc1) : acc0;
        }
        // axis-0 pass: coefficient row kr0 - P + (g NSG + t) from ring rows 2kr+1-j
        if (t >= vlo && t < vhi) {
          float2 al = make_float2(0.f, 0.f), ah = make_float2(0.f, 0.f);
          float2 al1 = make_float2(0.f, 0.f), ah1 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < L; j++) {
            const float2 hv = ring[(2 * t + 1 - j + 2 * L) % L];
            if (j >= TR::l0 && j < TR::l1) {
              if (j % 2 == 0) al = fma2(splat2<float2>(p.tp[j].x), hv, al);
              else al1 = fma2(splat2<float2>(p.tp[j].x), hv, al1);
            }
            if (j >= TR::h0 && j < TR::h1) {
              if (j % 2 == 0) ah = fma2(splat2<float2>(p.tp[j].y), hv, ah);
              else ah1 = fma2(splat2<float2>(p.tp[j].y), hv, ah1);
            }
          }
          al = add2(al, al1);
          ah = add2(ah, ah1);
          if (kst) {
            o0[roff] = al.x;
            o1[roff] = al.y;
            o2[roff] = ah.x;
            o3[roff] = ah.y;
          }
          roff += pitch;
        }
      }
      __syncthreads();  // every thread has read stage st
      if (tid == 0 && g + S < ngroups) issue(g + S);
    }
    gbase += ngroups;
  }
}

template <int L, int ZV>
cudaError_t launch_ring_t(const AnalysisArgs &a, cudaStream_t s) {
  using C = ARingCfg<L>;
  ARingParams<L> p;
  memset(&p, 0, sizeof p);
  for (int i = 0; i < 4; i++) {
    p.out[i] = static_cast<float *>(a.out[i]);
    p.out_bstride[i] = a.out_bstride[i];
  }
  p.pitch = a.out_pitch[0];
  for (int j = 0; j < L; j++) {
    p.tp[j] = make_float2((float)a.lo[j], (float)a.hi[j]);
  }
  if (!encode_tmap_3d(&p.tmap, 4, a.in, (uint64_t)a.n1, (uint64_t)a.n0, (uint64_t)a.batch,
                      (uint64_t)a.in_pitch * 4, (uint64_t)a.in_bstride * 4, C::UBX, C::G))
    return cudaErrorNotSupported;
  p.nstrips = (int)((p.pitch + C::TQ - 1) / C::TQ);
  auto kern = k_ana_ring<L, ZV>;
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(kern), C::NT, C::SMEM, &resident);
  if (e != cudaSuccess) return e;
  // one run per resident CTA when the columns allow it; bands of >= 2 groups
  p.runs = RunMap::make((long long)a.batch * p.nstrips, a.m0, resident, 2 * C::NSG, 1);
  const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
  e = launch_pdl(kern, grid, C::NT, C::SMEM, s, p, 'A');
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int L>
cudaError_t launch_ring_l(const AnalysisArgs &a, cudaStream_t s) {
  if (L == 10 && zero_taps_enabled()) {
    switch (match_tap_range(a.lo, a.hi, a.L)) {
      case 1: return launch_ring_t<L, 1>(a, s);
      case 2: return launch_ring_t<L, 2>(a, s);
      default: break;
    }
  }
  return launch_ring_t<L, 0>(a, s);
}

bool aring_disabled() {
  static const bool v = getenv("WL_NO_ARING") != nullptr;  // A/B switch: force k_ana_stream
  return v;
}

}  // namespace

bool launch_analysis_ring(int dtype, const AnalysisArgs &a, cudaStream_t s, cudaError_t *err) {
  if (dtype != WL_F32 || a.ext != EXT_ZERO || a.fista_mask || aring_disabled() || !tma_enabled()) return false;
  if (a.batch == 0 || a.m0 == 0 || a.m1 == 0) return false;
  // measured on B200 (graph replay, cold L2): the ring wins for the 16-tap db8 frame on large levels
  // (cfg4 W* level 1 37.6 vs 41.6 us, level 2 14.0 vs 14.6 us) and loses for shorter frames (CDF 9/7
  // cfg5 level 1 119 vs 109 us: the streaming kernel's wider reuse wins when the FMA work is light)
  // and on small levels (short bands: the L - 2 priming rows per band dominate).  WL_ARING=1 forces
  // it for every zero-extension level (A/B).
  static const bool force = getenv("WL_ARING") != nullptr;
  static const int min_log2 = [] {
    const char *e = getenv("WL_ARING_MIN");  // A/B: log2 of the smallest level (in coefficients) the ring takes
    return e ? atoi(e) : 20;
  }();
  if (!force && (a.L < 16 || (long long)a.batch * a.m0 * a.m1 < (1LL << min_log2))) return false;
  // one pitch for the four subbands, 16-byte aligned rows and images (TMA strides), aligned base
  for (int i = 1; i < 4; i++)
    if (a.out_pitch[i] != a.out_pitch[0]) return false;
  if (a.in_pitch % 4 || a.in_bstride % 4 || (reinterpret_cast<uintptr_t>(a.in) & 15)) return false;
  if (a.n0 > (1 << 30) || a.n1 > (1 << 30)) return false;
  cudaError_t e = cudaErrorNotSupported;
  switch (a.L) {
    case 2: e = launch_ring_l<2>(a, s); break;
    case 4: e = launch_ring_l<4>(a, s); break;
    case 8: e = launch_ring_l<8>(a, s); break;
    case 10: e = launch_ring_l<10>(a, s); break;
    case 16: e = launch_ring_l<16>(a, s); break;
    default: return false;
  }
  if (e == cudaErrorNotSupported) return false;  // no TMA descriptor: the streaming kernel takes it
  *err = e;
  return true;
}

}  // namespace wl
