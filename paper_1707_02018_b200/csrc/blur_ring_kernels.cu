// Register-ring blur kernels (sm_100a, fp32, PSFs of up to 15 taps): R, and the fused middle
// stage of grad f, s = R*(R u - b) (= R (R u - b) for the symmetric PSFs the plan accepts),
// optionally with f = 1/2 ||R u - b||^2.
//
// Per axis (reading R12):  (R_a y)[i] = sum_{t=-h..h} k[t] yhat[i - t],
// yhat = half-point symmetric extension of y.  R = R_v R_h, and R_v, R_h commute, so
//     s = R_v R_h (R_v R_h u - b):   h1 = R_h u,  r = R_v h1 - b,  h2 = R_h r,  s = R_v h2.
//
// Design (DESIGN.md §6 "k_blur_ring").  A CTA of 128 threads owns one strip of 2*128 stage-1
// columns of one image (h1 / r columns for the residual, output columns for R) and walks down a
// band of rows, one row per step.  Thread q owns the column pair (2q, 2q+1) of every stage:
//   * H passes read a 16-sample window of one shared-memory row (8 aligned 8-byte loads) and
//     produce the pair with FFMA2 on (even, odd) tap pairs;
//   * V passes are register rings: the thread keeps the last 15 rows of its pair in registers
//     and emits one output row per step (15 FFMA2, two chains), so a vertical halo costs no
//     shared memory and no barrier.  The step loop is unrolled over the 15-slot ring period, so
//     every ring index is a compile-time register.
// Rows arrive G = 5 per group into a 3-stage shared-memory ring: TMA boxes (two per operand,
// one per warp pair, so that a thread's window never straddles a box), completion on an
// mbarrier; groups touching the top or bottom edge gather their row-reflected rows with
// cp.async instead.  The residual exchanges r between threads through a double-buffered
// shared row block: one __syncthreads per group, which also frees the group's TMA slot.
//
// Boundary handling: rows are reflected when loaded; in strips that reach past an image edge the
// HW columns beyond it are overwritten in shared memory with their mirror images (u and r are
// both symmetric about the edges for a symmetric PSF) before the H pass reads them, so the hot
// loop has no edge branches; outputs outside the image are skipped.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "wl_internal.h"

namespace wl {
namespace {

constexpr int kRing = 15;  // register-ring slots: the vertical window of the largest PSF taken here

#ifdef WL_RING_PROFILE  // debug builds only: per-run start / end times and SM id (tools/ringprof.py)
__device__ unsigned long long g_ring_prof[8192][4];
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

template <int HW, bool RESID>
struct RingCfg {
  static_assert(2 * HW + 1 <= kRing, "ring too short for this PSF");
#ifndef WL_RING_NB
#define WL_RING_NB 2
#endif
  // TMA boxes per operand, 64 column pairs (2 warps) each.  A/B on B200 (cfg5 residual): 2 boxes
  // (128 threads, 4 CTAs per SM) 251 us; 4 boxes (256 threads, 2 CTAs, half the strip halo) 258 us
  static constexpr int NB = WL_RING_NB;
  static constexpr int NP = 64 * NB;      // column pairs per strip
  static constexpr int NT = NP;           // one thread per pair; it runs both stages
  static constexpr int G = 5;             // rows per group (divides kRing)
#ifndef WL_RING_S
#define WL_RING_S 3
#endif
  static constexpr int S = WL_RING_S;     // shared-memory stages
  static constexpr int NG = kRing / G;    // groups per unrolled body
  static constexpr int NC = 2 * NP;       // stage-1 columns
  static constexpr int T = RESID ? NC - 2 * HW : NC;  // output columns per strip
  static constexpr int UH = RESID ? 2 * HW : HW;      // u halo (rows and columns)
  // pair windows start at an even shared index; an odd first tap sample (R with odd HW) shifts
  // the first output to window position 1
  static constexpr int S0 = RESID ? 0 : (HW & 1);
  static constexpr int NWIN = 2 * HW + 2 + 2 * S0;
  static constexpr int UBOX = round_up_c(130 + NWIN, 4);  // box b: [128 b, 128 b + UBOX)
  static constexpr int BBOX = 132;
  // one (stage, box) region holds G dense rows (a G-row TMA box), 128-byte aligned
  static constexpr int UREG = round_up_c(G * UBOX * 4, 128) / 4;
  static constexpr int BREG = round_up_c(G * BBOX * 4, 128) / 4;
  static constexpr size_t OFF_U = 0;  // [S][NB boxes][UREG]
  static constexpr size_t OFF_B = OFF_U + (size_t)S * NB * UREG * 4;  // [S][NB][BREG]
  static constexpr int NR = 2;            // r row blocks (double buffer: one barrier per group)
  static constexpr size_t OFF_R = OFF_B + (RESID ? (size_t)S * NB * BREG * 4 : 0);  // [NR][G][NC]
  static constexpr size_t OFF_BAR = OFF_R + (RESID ? (size_t)NR * G * NC * 4 : 0);
  static constexpr size_t SMEM = OFF_BAR + S * sizeof(uint64_t);  // mbarriers full[S] (TMA landed)
  static constexpr unsigned TX = (unsigned)NB * G * (UBOX + (RESID ? BBOX : 0)) * 4u;  // bytes per group
};

template <int HW>
struct RingParams {
  CUtensorMap tmap_u;  // u: box (UBOX columns, G rows, 1 image)
  CUtensorMap tmap_b;  // b: box (BBOX columns, G rows, 1 image)   (residual)
  const float *u;
  const float *b;
  float *out;
  double *f;  // residual only (nullable)
  int h, w, nstrips, batch;
  RunMap runs;
  float cv[HW + 1];               // c[d] = k[HW - d] for d <= HW (symmetric PSF: c[2HW - d] = c[d])
  float2 cs[2 * HW + 1];          // (c[d], c[d]): FFMA2 taps of the aligned window pairs
};

__device__ __forceinline__ int ocol_of(int c0, int tid) { return c0 + 2 * tid; }
__device__ __forceinline__ int floor4(int v) { return v >= 0 ? (v & ~3) : -(((-v) + 3) & ~3); }

// Pair (out[s0], out[s0+1]) of a 2HW+1-tap correlation over the window w (s0 = S0):
// out[s] = sum_d c[d] w[s + d].  Taps d whose sample pair (w[s0+d], w[s0+d+1]) is an aligned
// register pair of the window (s0 + d even) take one FFMA2 with the splat tap (c[d], c[d]); the
// others are two scalar FFMAs into a second accumulator pair (their samples straddle two pairs).
// 2HW+1 lane-FMAs per output and no cross-lane reduction: the FMA pipe does the minimum work.
template <int HW, int S0>
__device__ __forceinline__ float2 hpair(const float *w, const RingParams<HW> &p) {
  float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
#pragma unroll
  for (int d = 0; d <= 2 * HW; d++) {
    const int s = S0 + d;
    if (s % 2 == 0) {
      a = fma2(p.cs[d], make_float2(w[s], w[s + 1]), a);
    } else {
      const float c = p.cs[d].x;
      b.x = fmaf(c, w[s], b.x);
      b.y = fmaf(c, w[s + 1], b.y);
    }
  }
  return add2(a, b);
}

// Row-wise loads of one operand box of a group that reaches past the top or bottom of the image:
// one bulk copy per row with the row reflected (P:82 applied to rows), clipped to the image
// columns (the kernel mirrors the edge columns afterwards).  Out of line: rare.
__device__ __noinline__ void ring_rows_edge(float *dst, int pitch, const float *img, int y0, int G, int h, int w,
                                           int c_start, int c_width, uint64_t *bar) {
  const int a0 = max(c_start, 0), n = max(min(c_start + c_width, w) - a0, 0);
  if (n == 0) return;
  for (int r = 0; r < G; r++)
    bulk_load(dst + r * pitch + a0 - c_start, img + (long long)refl_inf(y0 + r, h) * w + a0, n * 4, bar);
}

// Bytes one operand box of a group delivers: a full TMA box, or its in-image columns per row.
__device__ __forceinline__ unsigned ring_box_bytes(bool inside, int G, int c_start, int c_width, int w) {
  const int a0 = max(c_start, 0), n = max(min(c_start + c_width, w) - a0, 0);
  return (unsigned)(G * (inside ? c_width : n) * 4);
}

__device__ __forceinline__ void st_pair_if(float *ptr, float2 v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n @p st.global.v2.f32 [%0], {%1, %2};\n}\n" ::"l"(ptr),
               "f"(v.x), "f"(v.y), "r"((int)pred)
               : "memory");
}

// Vertical output from a ring whose newest row sits in slot `nw`: sum_d c[d] ring[nw - 2HW + d],
// folded on the PSF symmetry: c[HW] ring[mid] + sum_{d<HW} c[d] (ring[lo + d] + ring[hi - d]).
// Called from fully unrolled loops only, so every ring index folds to a register.
template <int HW>
__device__ __forceinline__ float2 vring(const float2 (&ring)[kRing], int nw, const RingParams<HW> &p, float2 init) {
  const int lo = nw - 2 * HW + kRing;
  // one accumulator chain (HW + 1 FFMA2; the HW pre-adds are independent): no final add
  float2 a = fma2(splat2<float2>(p.cv[HW]), ring[(lo + HW) % kRing], init);
#pragma unroll
  for (int d = 0; d < HW; d++) {
    const float2 sp = add2(ring[(lo + d) % kRing], ring[(lo + 2 * HW - d) % kRing]);
    a = fma2(splat2<float2>(p.cv[d]), sp, a);
  }
  return a;
}

// Register cap: shared memory holds 4 CTAs of 128 threads, i.e. 128 registers.  Asking ptxas for 4 CTAs makes it
// stop at 106 registers; asking for 3 lets the long PSFs (half-width >= 5) take 121-126, still 4 CTAs per SM:
// cfg5 residual 251.6 -> 247.4 us, grad 555.9 -> 551.3 us.  The shorter PSFs would pass 128 (3 CTAs) and keep 4.
#ifndef WL_RING_MINB
#define WL_RING_MINB(HW) ((HW) >= 5 ? 6 / WL_RING_NB : 8 / WL_RING_NB)
#endif
template <int HW, bool RESID>
__global__ void __launch_bounds__(64 * WL_RING_NB, WL_RING_MINB(HW)) k_blur_ring(const __grid_constant__ RingParams<HW> p) {
  using C = RingCfg<HW, RESID>;
  constexpr int G = C::G, S = C::S, NWIN = C::NWIN, S0 = C::S0;
  extern __shared__ __align__(128) unsigned char sm[];
  float *ubase = reinterpret_cast<float *>(sm + C::OFF_U);
  float *bbase = reinterpret_cast<float *>(sm + C::OFF_B);
  float *rbuf = reinterpret_cast<float *>(sm + C::OFF_R);  // [2][G][NC]   r rows (residual)
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);
  const int tid = threadIdx.x;
  const int box = tid >> 6;  // warps 2b, 2b+1 read box b
  // stage regions start finite: edge-group copies leave the out-of-image columns untouched
  for (int i = tid; i < (int)(C::OFF_BAR / 16); i += C::NT)
    reinterpret_cast<float4 *>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid == 0)
    for (int s = 0; s < S; s++) mbar_init(full + s, 1);
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel of the stream wrote our inputs
  // rings start finite: the first 2HW outputs of every run are computed from stale slots and dropped
  float2 ring1[kRing], ring2[kRing];
#pragma unroll
  for (int i = 0; i < kRing; i++) ring1[i] = ring2[i] = make_float2(0.f, 0.f);

  const int h = p.h, w = p.w;
  const int nruns = p.runs.nruns();
  unsigned gbase = 0;  // groups of earlier runs: global group g = gbase + k fixes stages and parities
  for (int run = blockIdx.x; run < nruns; run += gridDim.x) {
    int col, r0, r1;
    p.runs.get(run, col, r0, r1);
    if (r0 >= r1) continue;  // (uniform) empty trailing band
#ifdef WL_RING_PROFILE
    const unsigned long long t_start = gtimer();
#endif
    // column order: the edge strips of every image first (they cost more per row: mirror fixes),
    // so RunMap's first columns -- the ones cut into one band more -- carry them (SM balance).
    // (A split into equal-cost parts that continue across columns measured slower: the SMs'
    // speeds differ by up to 20 % on identical parts, and the neighbouring strips' halo columns
    // no longer meet in L2.)
    int img, strip;
    if (p.nstrips >= 3 && col < 2 * p.batch) {
      img = col >> 1;
      strip = (col & 1) ? p.nstrips - 1 : 0;
    } else if (p.nstrips >= 3) {
      const int k = col - 2 * p.batch;
      img = k / (p.nstrips - 2);
      strip = 1 + k - img * (p.nstrips - 2);
    } else {
      img = col / p.nstrips;
      strip = col - img * p.nstrips;
    }
    const int c0 = strip * C::T;
    const int col1 = RESID ? c0 - HW : c0;  // image column of stage-1 pair 0
    const int ustart = floor4(col1 - HW);    // u box 0 origin (16-byte aligned)
    const int bstart = floor4(col1);
    const int n_steps = r1 - r0 + 2 * C::UH;
    const int n_groups = (n_steps + G - 1) / G;
    const int urow0 = r0 - C::UH;            // u row of step 0
    const int brow0 = urow0 - HW;            // b / r row of step 0 (residual)
    // strips whose u / r rows reach past an image edge mirror the HW columns beyond it in shared
    // memory (u and r are symmetric about the edges for a symmetric PSF), once per group
    // Edge strips: the HW image columns beyond an edge, [-HW, 0) and [w, w + HW), are overwritten
    // in shared memory with their mirror images (u and r are symmetric about the edges for a
    // symmetric PSF) before a horizontal pass reads them.  Lane j < 2HW of each warp owns edge
    // column j: when it lies in the warp's read range, the lane copies its source column row by
    // row (offsets fixed per run) and the warp syncs itself; overlapping warps write equal values.
    const int lane = tid & 31, wq = (tid >> 5) * 64;
    int ufix_t = -1, ufix_s = 0, rfix_t = -1, rfix_s = 0;
    if (lane < 2 * HW) {
      const int c = lane < HW ? lane - HW : w + lane - HW;  // the edge column of this lane
      const int x = c - ustart;                              // its u index over [0, 128 + UBOX)
      const int ulo = wq + (col1 - HW - ustart) - S0;        // this warp's u read range
      if (x >= ulo && x < ulo + 62 + NWIN && x >= box * 128 && x < box * 128 + C::UBOX) {
        const int sx = refl_inf(c, w) - ustart;
        ufix_t = box * C::UREG + x - box * 128;
        const int sbx = min(C::NB - 1, sx / 128);  // a box holding the source column
        ufix_s = sbx * C::UREG + sx - sbx * 128;
      }
      const int xr = c - col1;                               // its r index over [0, NC)
      if (RESID && xr >= wq && xr < wq + 62 + NWIN && xr < C::NC) {
        rfix_t = xr;
        rfix_s = refl_inf(c, w) - col1;
      }
    }
    const bool uedge = __any_sync(0xffffffffu, ufix_t >= 0);
    const bool redge = RESID && __any_sync(0xffffffffu, rfix_t >= 0);
    const int widx = box * C::UREG + 2 * tid + (col1 - HW - ustart) - S0 - box * 128;  // even
    const int bidx = box * C::BREG + 2 * tid + (col1 - bstart) - box * 128;
    // output pair columns (c0 + 2 tid, +1)
    const int ocol = c0 + 2 * tid;
    const bool act = (!RESID || 2 * tid < C::T) && ocol < w;
    float *obase = p.out + (long long)img * h * w + ocol;
    // f: r pair columns (col1 + 2 tid, +1) counted once per image
    const int rc = col1 + 2 * tid;
    const float mx = (rc >= c0 && rc < c0 + C::T && rc >= 0 && rc < w) ? 1.f : 0.f;
    const float my = (rc + 1 >= c0 && rc + 1 < c0 + C::T && rc + 1 >= 0 && rc + 1 < w) ? 1.f : 0.f;
    double fsum = 0.0;

    __syncthreads();  // the previous run's readers of every buffer are done
    // group kk -> stage (gbase + kk) % S: lane 0 of warp `part` loads operand box `part` (u boxes 0 .. NB-1,
    // then b boxes 0 .. NB-1); groups inside the image take one G-row TMA box, edge groups
    // row-wise bulk copies; part 0 also arms the stage's barrier with the group's bytes
    auto issue_part = [&](int kk, int part) {
      const int st = (gbase + kk) % S;
      const int yu = urow0 + kk * G, yb = brow0 + kk * G;
      const bool tu = yu >= 0 && yu + G <= h, tb = yb >= 0 && yb + G <= h;
      if (part == 0) {
        unsigned bytes = 0;
        for (int bx = 0; bx < C::NB; bx++) {
          bytes += ring_box_bytes(tu, G, ustart + 128 * bx, C::UBOX, w);
          if (RESID) bytes += ring_box_bytes(tb, G, bstart + 128 * bx, C::BBOX, w);
        }
        mbar_arrive_expect_tx(full + st, bytes);
      }
      if (part >= C::NB && !RESID) return;
      const bool isu = part < C::NB, inside = isu ? tu : tb;
      const int bx = isu ? part : part - C::NB;
      float *dst = isu ? ubase + (st * C::NB + bx) * C::UREG : bbase + (st * C::NB + bx) * C::BREG;
      const int cs = (isu ? ustart : bstart) + 128 * bx;
      fence_proxy_async();
      if (inside)
        tma_load_3d(dst, isu ? &p.tmap_u : &p.tmap_b, full + st, cs, isu ? yu : yb, img);
      else
        ring_rows_edge(dst, isu ? C::UBOX : C::BBOX, (isu ? p.u : p.b) + (long long)img * h * w, isu ? yu : yb, G, h,
                       w, cs, isu ? C::UBOX : C::BBOX, full + st);
    };
    if ((tid & 31) == 0)
      for (int kk = 0; kk < S && kk < n_groups; kk++) issue_part(kk, tid >> 5);

    for (int kb = 0; kb < n_groups; kb += C::NG) {
#pragma unroll
      for (int gg = 0; gg < C::NG; gg++) {
        const int k = kb + gg;
        if (k >= n_groups) break;
        const unsigned g = gbase + k;
        const int st = g % S;
        mbar_wait(full + st, (g / S) & 1);
        float *ust = ubase + st * C::NB * C::UREG;
        if (uedge) {
          if (ufix_t >= 0) {  // all G loads first, then the stores: one shared-memory latency
            float v[G];
#pragma unroll
            for (int r = 0; r < G; r++) v[r] = ust[r * C::UBOX + ufix_s];
#pragma unroll
            for (int r = 0; r < G; r++) ust[r * C::UBOX + ufix_t] = v[r];
          }
          __syncwarp();
        }
        const float *ub = ust + widx;
        const float *bb = bbase + st * C::NB * C::BREG + bidx;
        float *rw = rbuf + (k & 1) * G * C::NC;
        float2 fa = make_float2(0.f, 0.f);
        // output row of step 0 of this group (stage 1 for R, stage 2 for the residual)
        float *orow = obase + (long long)((RESID ? brow0 : urow0) + k * G - HW) * w;
        // rows r of this group with a stored output: olo <= r < ohi (the first 2HW (R) / 4HW
        // (residual) steps of a run only prime the rings); f counts rows flo <= r < fhi
        const int olo = (RESID ? 4 * HW : 2 * HW) - k * G;
        const int ohi = act ? r1 + HW - (RESID ? brow0 : urow0) - k * G : 0;
        const int flo = r0 - brow0 - k * G, fhi = r1 - brow0 - k * G;
        // ---------------- stage 1: h1 = R_h u -> ring1; r = R_v h1 - b (residual) or out = R_v h1
        // (the window of step r + 1 is loaded before step r computes: WL_RING_PF)
        float2 wb[2][NWIN / 2];
#pragma unroll
        for (int j = 0; j < NWIN / 2; j++) wb[0][j] = reinterpret_cast<const float2 *>(ub)[j];
#pragma unroll
        for (int r = 0; r < G; r++) {
          const int slot = gg * G + r;  // == step % kRing (kb G is a multiple of kRing)
          if (r + 1 < G) {
            const float2 *src = reinterpret_cast<const float2 *>(ub + (r + 1) * C::UBOX);
#pragma unroll
            for (int j = 0; j < NWIN / 2; j++) wb[(r + 1) & 1][j] = src[j];
          }
          float win[NWIN];
#pragma unroll
          for (int j = 0; j < NWIN / 2; j++) {
            win[2 * j] = wb[r & 1][j].x;
            win[2 * j + 1] = wb[r & 1][j].y;
          }
          ring1[slot] = hpair<HW, S0>(win, p);
          if (RESID) {
            const float *bp = bb + r * C::BBOX;
            const float2 rv = vring<HW>(ring1, slot, p, make_float2(-bp[0], -bp[1]));
            *reinterpret_cast<float2 *>(rw + r * C::NC + 2 * tid) = rv;
            if (r >= flo && r < fhi) fa = fma2(rv, rv, fa);
          } else {
            const float2 o = vring<HW>(ring1, slot, p, make_float2(0.f, 0.f));
            st_pair_if(orow, o, r >= olo && r < ohi);
            orow += w;
          }
        }
        if (RESID) fsum += (double)fa.x * mx + (double)fa.y * my;
        __syncthreads();  // r rows of group k complete; stage st free
        if ((tid & 31) == 0 && k + S < n_groups) issue_part(k + S, tid >> 5);
        // groups whose steps all precede 2HW only prime ring1 (their r rows feed no output)
        if (RESID && (k + 1) * G > 2 * HW) {
          if (redge) {
            if (rfix_t >= 0) {
              float v[G];
#pragma unroll
              for (int r = 0; r < G; r++) v[r] = rw[r * C::NC + rfix_s];
#pragma unroll
              for (int r = 0; r < G; r++) rw[r * C::NC + rfix_t] = v[r];
            }
            __syncwarp();
          }
          // ---------------- stage 2: h2 = R_h r -> ring2; s = R_v h2
          const float2 *rsrc = reinterpret_cast<const float2 *>(rw + 2 * tid);
          float2 vb[2][NWIN / 2];
#pragma unroll
          for (int j = 0; j < NWIN / 2; j++) vb[0][j] = rsrc[j];
#pragma unroll
          for (int r = 0; r < G; r++) {
            const int slot = gg * G + r;
            if (r + 1 < G) {
#pragma unroll
              for (int j = 0; j < NWIN / 2; j++) vb[(r + 1) & 1][j] = rsrc[(r + 1) * (C::NC / 2) + j];
            }
            float win[NWIN];
#pragma unroll
            for (int j = 0; j < NWIN / 2; j++) {
              win[2 * j] = vb[r & 1][j].x;
              win[2 * j + 1] = vb[r & 1][j].y;
            }
            ring2[slot] = hpair<HW, 0>(win, p);
            const float2 o = vring<HW>(ring2, slot, p, make_float2(0.f, 0.f));
            st_pair_if(orow, o, r >= olo && r < ohi);
            orow += w;
          }
        }
      }
    }
    gbase += n_groups;
#ifdef WL_RING_PROFILE
    __syncthreads();
    if (tid == 0 && run < 8192) {
      g_ring_prof[run][0] = t_start;
      g_ring_prof[run][1] = gtimer();
      g_ring_prof[run][2] = smid();
      g_ring_prof[run][3] = ((unsigned long long)col << 32) | (unsigned)(r1 - r0);
    }
#endif
    if (RESID && p.f) {
      for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
      if ((tid & 31) == 0) atomicAdd(p.f + img, 0.5 * fsum);
    }
  }
}

template <int HW, bool RESID>
cudaError_t launch_ring(const BlurArgs &a, cudaStream_t s) {
  using C = RingCfg<HW, RESID>;
  RingParams<HW> p;
  memset(&p, 0, sizeof p);
  p.u = static_cast<const float *>(a.in);
  p.b = static_cast<const float *>(a.b);
  p.out = static_cast<float *>(a.out);
  p.f = RESID ? a.f : nullptr;
  p.h = (int)a.h;
  p.w = (int)a.w;
  p.nstrips = (int)((a.w + C::T - 1) / C::T);
  p.batch = a.batch;
  const uint64_t rs = (uint64_t)p.w * 4, is = rs * (uint64_t)p.h;
  if (!encode_tmap_3d(&p.tmap_u, 4, a.in, p.w, p.h, a.batch, rs, is, C::UBOX, C::G)) return cudaErrorNotSupported;
  if (RESID && !encode_tmap_3d(&p.tmap_b, 4, a.b, p.w, p.h, a.batch, rs, is, C::BBOX, C::G))
    return cudaErrorNotSupported;
  double c[2 * HW + 1];
  for (int d = 0; d <= 2 * HW; d++) c[d] = a.taps[2 * HW - d];
  for (int d = 0; d <= HW; d++) p.cv[d] = (float)c[d];
  for (int d = 0; d <= 2 * HW; d++) p.cs[d] = make_float2((float)c[d], (float)c[d]);
  auto kern = k_blur_ring<HW, RESID>;
  long long resident = 0;
  cudaError_t e = kernel_resident(reinterpret_cast<const void *>(kern), C::NT, C::SMEM, &resident);
  if (e != cudaSuccess) return e;
  // one run per resident CTA when the columns allow it; bands of >= 2 groups
  p.runs = RunMap::make((long long)a.batch * p.nstrips, (int)a.h, resident, 2 * C::G, 1);
  const int grid = (int)std::min<long long>(p.runs.nruns(), resident);
  if (RESID && a.f && !a.f_zeroed) {
    e = cudaMemsetAsync(a.f, 0, sizeof(double) * (size_t)a.batch, s);
    if (e != cudaSuccess) return e;
  }
  e = launch_pdl(kern, grid, C::NT, C::SMEM, s, p, 'b');
  g_launches++;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool ring_disabled() {
  static const bool v = getenv("WL_BLUR_STREAM") != nullptr;  // A/B switch: force k_blur_stream
  return v;
}

}  // namespace

#ifdef WL_RING_PROFILE
extern "C" __attribute__((visibility("default"))) int wl_debug_ring_prof(void *host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_ring_prof, sizeof(unsigned long long) * 4 * (size_t)n);
}
#endif

bool launch_blur_ring(int dtype, const BlurArgs &a, bool residual, cudaStream_t s, cudaError_t *err) {
  if (dtype != WL_F32 || ring_disabled() || !tma_enabled()) return false;
  if (a.w % 4 || (reinterpret_cast<uintptr_t>(a.in) & 15) || (reinterpret_cast<uintptr_t>(a.out) & 15)) return false;
  if (residual && (reinterpret_cast<uintptr_t>(a.b) & 15)) return false;
  if (a.h > (1 << 30) || a.w > (1 << 30)) return false;
  switch (a.ntaps / 2) {
#define WL_RING_CASE(H)                                                               \
  case H:                                                                             \
    *err = residual ? launch_ring<H, true>(a, s) : launch_ring<H, false>(a, s);       \
    return *err != cudaErrorNotSupported; /* no TMA descriptor: the streaming kernel takes it */
    WL_RING_CASE(1) WL_RING_CASE(2) WL_RING_CASE(3) WL_RING_CASE(4) WL_RING_CASE(5) WL_RING_CASE(6)
    WL_RING_CASE(7)
#undef WL_RING_CASE
  }
  return false;
}

}  // namespace wl
