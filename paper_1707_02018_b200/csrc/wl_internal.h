// Internal declarations shared by the host plan code and the CUDA kernels of libwl.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/wl.h"

namespace wl {

constexpr int kMaxL = 16;     // longest filter frame (db8)
constexpr int kMaxTaps = 31;  // longest blur PSF per axis

struct FilterBank {
  int L = 0;
  double a_lo[kMaxL] = {}, a_hi[kMaxL] = {}, d_lo[kMaxL] = {}, d_hi[kMaxL] = {};
};
bool build_filter_bank(int filter, FilterBank &fb);

// Extension applied before an analysis pass.
enum Ext : int { EXT_ZERO = 0, EXT_PER = 1, EXT_SYM = 2, EXT_SYM_PADJ = 3 };

extern std::atomic<int64_t> g_launches;

// ------------------------------------------------------------ launch args
// All strides/pitches in elements.  Subband order in arrays: LL, LH, HL, HH.
struct AnalysisArgs {
  const void *in;
  int64_t in_pitch, in_bstride;
  int n0, n1;
  void *out[4];
  int64_t out_pitch[4], out_bstride[4];
  int m0, m1;
  int ext;
  const double *lo, *hi;
  int L;
  int batch;
  // fused FISTA epilogue (0 = plain store): bit i set -> out[i] is y and x = y + fista_xdelta
  int fista_mask = 0;
  int64_t fista_xdelta = 0;
  double fista_inv_lip = 0, fista_tau = 0, fista_mom = 0;
  const double *fista_tdev = nullptr;  // non-null: the momentum comes from the device-resident t
  int ll_keep = 0;  // 1: out[0] (LL) is the next level's input: stored with the L2 evict_last policy
};

struct SynthesisArgs {
  const void *in[4];
  int64_t in_pitch[4], in_bstride[4];
  int m0, m1;
  int coef_mod;  // 1: coefficient index taken mod m (periodisation); 0: zero outside [0, m)
  void *out;
  int64_t out_pitch, out_bstride;
  int N0, N1;  // output extent
  int o0, o1;  // output index i <-> extended position t = i + o
  const double *lo, *hi;
  int L;
  int batch;
  int out_keep = 0;  // 1: out is the next level's LL input: stored with the L2 evict_last policy
  // split output (symmetric folds): extended positions inside the image, t in [0, yn0) x [0, yn1),
  // go to y (the fold's output, written in place of its interior) and only the rest to out
  void *y = nullptr;
  int64_t y_pitch = 0, y_bstride = 0;
  int yn0 = 0, yn1 = 0;
};

struct FoldArgs {  // y = diag(1/c) E_sym^T U per axis (weighted: W of SYMMETRIC_EDAG) or E_sym^T U
  const void *in;
  int64_t in_pitch, in_bstride;  // U over [-Lp, n+Lp) per axis
  void *out;
  int64_t out_pitch, out_bstride;
  int n0, n1, Lp;
  int weighted;                  // 1: E_sym^dagger = diag(1/c) E_sym^T; 0: E_sym^T ((W-dagger)*)
  int batch;
  int col_off = 0;               // U column of extended position t is t + Lp + col_off
  int border_only = 0;           // 1: y already holds U's in-image part (split synthesis); fold the
                                 //    L'-wide border only, reading the outside positions from U
};



struct BlurArgs {
  const void *in;
  const void *b;  // residual mode only
  void *out;
  double *f;      // residual mode only (nullable)
  int64_t h, w;
  int ntaps;
  const double *taps;
  int batch;
  int f_zeroed = 0;  // residual mode: the caller zeroed f earlier in the stream (no memset between its kernels)
};

cudaError_t launch_analysis(int dtype, const AnalysisArgs &a, cudaStream_t s);
// A full chain of n analysis levels (fine -> coarse): the short coarse tail runs as one persistent
// cooperative launch (k_ana_multi) with grid-wide barriers between its levels.
cudaError_t launch_analysis_chain(int dtype, const AnalysisArgs *a, int n, cudaStream_t s);
cudaError_t launch_synthesis(int dtype, const SynthesisArgs &a, cudaStream_t s);
// A full chain of n synthesis levels given coarse -> fine: the short coarse head runs as one
// persistent cooperative launch (k_synth_multi).
cudaError_t launch_synthesis_chain(int dtype, const SynthesisArgs *a, int n, cudaStream_t s);
cudaError_t launch_fold(int dtype, const FoldArgs &a, cudaStream_t s);
cudaError_t launch_blur(int dtype, const BlurArgs &a, cudaStream_t s);
cudaError_t launch_blur_residual(int dtype, const BlurArgs &a, cudaStream_t s);
// Register-ring kernels (blur_ring_kernels.cu): fp32, PSFs of <= 15 taps, width % 4 == 0, 16-byte
// aligned buffers.  Returns false (nothing launched) when the arguments are outside that domain;
// otherwise launches and stores the launch status in *err.
bool launch_blur_ring(int dtype, const BlurArgs &a, bool residual, cudaStream_t s, cudaError_t *err);
// Register-ring analysis level (analysis_ring_kernels.cu): fp32, zero extension (W* under zero /
// symmetric BC, W-dagger under zero BC), no FISTA epilogue.  Returns false (nothing launched)
// outside that domain; otherwise launches and stores the launch status in *err.
bool launch_analysis_ring(int dtype, const AnalysisArgs &a, cudaStream_t s, cudaError_t *err);
// Small-level kernels (small_kernels.cu): the coarse levels whose input fits in one CTA's shared
// memory run as one launch with one CTA per image.  small_analysis_start returns the first index
// of a (fine -> coarse) chain that the small kernel takes (n: none); small_synthesis_end the end of
// the (coarse -> fine) prefix it takes (0: none).  WL_NO_SMALL disables both (A/B).
int small_analysis_start(int dtype, const AnalysisArgs *a, int n);
cudaError_t launch_analysis_small(int dtype, const AnalysisArgs *a, int n, cudaStream_t s);
int small_synthesis_end(int dtype, const SynthesisArgs *a, int n);
cudaError_t launch_synthesis_small(int dtype, const SynthesisArgs *a, int n, cudaStream_t s);
cudaError_t launch_zero(void *ptr, size_t bytes, cudaStream_t s);
// FISTA pieces (fista_kernels.cu); n = elements per call (batch * p_alloc for the update)
// Example 2: batched valid cross-correlation out_b[i] = sum_{j<ta} a_b[j] b_b[i+j]
// with a_b[j] = a[ta-1-j] if a_rev, and b_b[i] = b[i - b_off] on [b_off, b_off + lb), else 0.
struct XcorrArgs {
  const void *a;
  int64_t a_bstride;
  int ta, a_rev;
  const void *b;
  int64_t b_bstride;
  int lb, b_off;
  void *out;
  int64_t out_bstride;
  int n_out;
  int64_t batch;
};
// Fused gradient of Eq. (6) for `problems` independent (h [C][K], s [N]) pairs.
struct BceArgs {
  const void *h, *s, *x;
  int x_shared;
  void *gh, *gs;
  double *f;
  int C, K, N;
  int64_t problems;
  double lam_tv, delta;
};
size_t xcorr_smem_bytes(int dtype, int ta, int n_out);
size_t bce_smem_bytes(int dtype, const BceArgs &a);
cudaError_t launch_xcorr(int dtype, const XcorrArgs &x, cudaStream_t s);
cudaError_t launch_bce_grad(int dtype, const BceArgs &a, cudaStream_t s);

// t <- (1 + sqrt(1 + 4 t^2)) / 2 on the device (one thread; FISTA with device-resident t)
cudaError_t launch_fista_advance_t(double *t_dev, cudaStream_t s);
cudaError_t launch_fista_update(int dtype, const void *g, void *x, void *y, long long n, double t, double lambda,
                                double lip, cudaStream_t s);
cudaError_t launch_dot(int dtype, const void *a, const void *b, long long n, int batch, double *out, cudaStream_t s);
cudaError_t launch_scale(int dtype, void *v, long long n, double alpha, cudaStream_t s);
cudaError_t launch_fill_seeded(int dtype, void *v, long long n, unsigned long long seed, cudaStream_t s);

// Encode a 3-D tiled TMA descriptor (CUtensorMap, 128 bytes at `map`) over a tensor of
// d0 x d1 x d2 elements of `elem_bytes` (4: fp32, 8: fp64) with byte strides s1 (dim 1) and
// s2 (dim 2), box (box0, box1, 1), no swizzle, zero out-of-bounds fill.  Returns false if
// the driver entry point is unavailable or the layout is not TMA-legal (16-byte strides...).
bool encode_tmap_3d(void *map, int elem_bytes, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                    uint64_t s2, uint32_t box0, uint32_t box1);

// Opt `kern` into `smem` bytes of dynamic shared memory and return the number of CTAs of
// `nt` threads the current device keeps resident (SMs x CTAs per SM).  Cached per (kernel,
// device), so a launch pays the attribute / occupancy queries once.
cudaError_t kernel_resident(const void *kern, int nt, size_t smem, long long *resident);

// Longest run (in blocks / batches) that the streaming kernels treat as short and launch with
// every block in flight at once (4 stages): `dflt` is the kernel's measured best (analysis 3,
// synthesis 2 on B200); WL_SHORT_MAX overrides both (0 disables; A/B switch).
int short_run_max(int dflt, char kind = 0);  // kind 'a' / 's': WL_SHORT_MAX_A / WL_SHORT_MAX_S override one family

// TMA loads unless WL_NO_TMA is set (debugging / A-B switch); read once per process
bool tma_enabled();
// Structural-zero tap variants: 1 if (lo, hi) are the CDF 9/7 dual filters of the
// L = 10 frame (d_lo nonzero on [2, 9), d_hi on [0, 9)), 2 if the analysis filters (a_lo on
// [1, 10), a_hi on [1, 8)), 0 otherwise.  The kernels then skip the zero taps at compile time.
int match_tap_range(const double *lo, const double *hi, int L);
// zero-tap skipping unless WL_ALL_TAPS is set (A-B switch)
bool zero_taps_enabled();
// multi-level persistent launches for the coarse tails only when WL_MULTI is set (A-B switch)
bool multi_enabled();
// balanced (equal-row, column-spanning) runs for the analysis / synthesis level kernels (A/B: WL_BALANCED=1;
// measured slower, see RunMap)
bool balanced_runs();
// the compact instantiations of the level kernels (analysis: zero extension, synthesis: crop; every block by
// TMA) unless WL_NO_PLAIN is set (A/B switch)
bool plain_enabled();

// PDL per launch site: kind 'A' / 'a' (analysis, long / short runs), 'S' / 's' (synthesis), 'b'
// (blur).  WL_NO_PDL lists the kinds launched without it (an A/B switch; "AasSb" = none).
bool pdl_enabled(char kind);

// Launch with programmatic stream serialization (PDL): the kernel may start while the
// previous kernel of the stream drains; it must call pdl_wait() before its first global
// memory access (every streaming kernel of libwl does, right after its shared-memory setup).
template <typename Kern, typename Params>
cudaError_t launch_pdl(Kern kern, int grid, int nt, size_t smem, cudaStream_t s, const Params &p, char kind) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(kind) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

// Cooperative launch (every CTA resident; grid-wide barriers allowed), with PDL when enabled for
// kind 'm' (falls back to a plain cooperative launch if the combination is refused).
template <typename Kern, typename Params>
cudaError_t launch_coop(Kern kern, int grid, int nt, size_t smem, cudaStream_t s, const Params &p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled('m') ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess && cfg.numAttrs == 2) {
    cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p);
  }
  return e;
}

}  // namespace wl

struct wl_plan {
  int64_t h = 0, w = 0;
  int J = 0, filter = 0, bc = 0, dtype = 0, es = 4;
  wl::FilterBank fb;
  int64_t n0[WL_MAX_LEVELS + 1] = {}, n1[WL_MAX_LEVELS + 1] = {};
  wl_subband band[1 + 3 * WL_MAX_LEVELS] = {};
  int64_t p_valid = 0, p_alloc = 0;
  int64_t ll_pitch[WL_MAX_LEVELS + 1] = {};  // pitch of LL_j in the workspace
  int64_t ws_a_elems = 0, ws_b_elems = 0;    // per image: ping-pong LL buffers (odd / even j)
  int64_t edag_elems = 0;                    // per image: extended U for the EDAG fold
};

struct wl_blur_plan {
  int64_t h = 0, w = 0;
  int dtype = 0, es = 4, ntaps = 0;
  double taps[wl::kMaxTaps] = {};
};
