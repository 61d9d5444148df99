/*
 * wl.h -- C ABI of the B200-native hot path of arXiv 1707.02018
 *         (Folberth & Becker, "Efficient Adjoint Computation for Wavelet and
 *          Convolution Operators", IEEE SPM Lecture Notes).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (the section is named beside it).
 *
 * The problem the ABI follows (§"Example 1: An Image Deblurring Problem"):
 *     min_x 1/2 ||R W x - b||^2 + lambda ||x||_1,     grad f(x) = W* R* (R W x - b)
 * x = multi-level 2-D wavelet coefficients, b = observed (blurred) image,
 * W = wavelet reconstruction (synthesis), W-dagger = analysis,
 * W* = the TRUE adjoint of W (Eq. (2), Eq. (4); not the
 * "pseudoinverse approximation" W-dagger ~ W* of P:47),
 * R = Gaussian PSF blur under symmetric (reflexive) boundary conditions, R* its adjoint.
 *
 * Conventions common to every entry point
 *   - Every data pointer is a DEVICE pointer (cudaMalloc / torch CUDA memory) unless the
 *     argument is marked "host".  Host pointers passed where device memory is required
 *     are rejected with WL_EINVAL.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 *     compute call is stream-ordered and asynchronous: it validates its arguments on the
 *     host, enqueues kernels on `stream` and returns; no host synchronisation happens
 *     inside a call.  Validation errors return BEFORE anything is enqueued.
 *   - Ownership: the caller owns every buffer (inputs, outputs, workspace).  Plans own
 *     only immutable tables; a plan may be shared by concurrent calls on different
 *     streams iff each call has its own workspace.  Destroying a plan while calls that
 *     use it are in flight is undefined.
 *   - dtype: a plan is created for WL_F32 or WL_F64 and every buffer of a call is of that
 *     type (T below), except f_dev which is always double.
 *   - Alignment: data pointers must be 16-byte aligned, the workspace 256-byte aligned
 *     (WL_EALIGN otherwise).  Inputs and outputs of one call must not overlap (WL_EINVAL).
 *   - batch = 0 is a valid no-op.  batch < 0 is WL_EINVAL.
 *   - Errors: every call returns a wl_status; wl_last_error() returns a thread-local
 *     message naming the offending argument / dimension / level.  CUDA launch errors are
 *     reported as WL_ECUDA with the CUDA error string.
 *
 * Layouts
 *   - Images: [batch, h, w], row-major, contiguous, element type T.
 *   - Coefficients x: [batch, p_alloc] of T.  One image's coefficients are the packed
 *     subbands LL_J, then (LH_j, HL_j, HH_j) for j = J..1 (subband XY = axis-0 filter X,
 *     axis-1 filter Y; axis 0 = rows/height, axis 1 = columns/width).  Each subband is
 *     row-major with a row pitch rounded up to 16 bytes; wl_plan_query() returns offset,
 *     rows, cols and pitch of every subband.  Padding entries are written as 0 by
 *     wl_adjoint / wl_analyze / wl_grad and never read by wl_synthesize.
 */
#ifndef WL_H_
#define WL_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define WL_API __attribute__((visibility("default")))
#else
#define WL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WL_OK = 0,
  WL_EINVAL = 1, /* bad argument: null/host pointer, aliasing, unknown enum, batch < 0   */
  WL_ESIZE = 2,  /* impossible size: a level cannot be formed, too many levels, h,w < 1  */
  WL_EDTYPE = 3, /* plan dtypes of the plans used together differ                        */
  WL_EALIGN = 4, /* pointer misaligned                                                    */
  WL_ENOMEM = 5, /* host/device allocation of plan tables failed                          */
  WL_ECUDA = 6   /* a CUDA call failed; wl_last_error() has the CUDA message              */
} wl_status;

/* Filter banks.  The paper names the families (P:101-102 Haar/Daubechies, P:174 CDF 9/7)
 * but prints no taps; the library derives them from their closed forms (Daubechies'
 * minimum-phase spectral factorisation; CDF 9/7 from the roots of 1+4y+10y^2+20y^3).
 * Frame length L: Haar 2, db2 4, db4 8, db8 16, CDF 9/7 10 (9-tap analysis lowpass and
 * 7-tap synthesis lowpass in a common 10-tap frame, reading R3). */
typedef enum { WL_HAAR = 1, WL_DB2 = 2, WL_DB4 = 4, WL_DB8 = 8, WL_CDF97 = 97 } wl_filter;

/* Boundary conditions (§"A few signal extensions").
 *   WL_BC_ZERO       zero padding E_zpd; coefficient length floor((n+L-1)/2)
 *   WL_BC_PERIODIC   periodisation (reading R2); length n/2, n must be even at every level
 *   WL_BC_SYMMETRIC  half-point symmetric E_sym for W-dagger; W/W* form the
 *                    toolbox-consistent exact pair (crop / zero-extension, reading R1),
 *                    so W W-dagger = I; length floor((n+L-1)/2); needs n >= L-1 per level
 *   WL_BC_SYMMETRIC_EDAG  the paper-literal variant of Eq. (4): W* = W~dagger_zpd (E_sym^dagger)*
 *                    with (E_sym^dagger)* = E_sym diag(1/c), W = its transpose.
 *                    An exact adjoint pair, but W W-dagger = I only away from the edges. */
typedef enum {
  WL_BC_ZERO = 0,
  WL_BC_PERIODIC = 1,
  WL_BC_SYMMETRIC = 2,
  WL_BC_SYMMETRIC_EDAG = 3
} wl_bc;

typedef enum { WL_F32 = 0, WL_F64 = 1 } wl_dtype;

typedef enum {
  WL_OP_SYNTHESIZE = 0,
  WL_OP_ADJOINT = 1,
  WL_OP_ANALYZE = 2,
  WL_OP_GRAD = 3,
  WL_OP_ANALYZE_ADJOINT = 4,
  WL_OP_FISTA = 5,
  WL_OP_LIPSCHITZ = 6,
  WL_OP_GRAD_HOST = 7
} wl_op;

typedef struct wl_plan wl_plan;           /* opaque, immutable after create */
typedef struct wl_blur_plan wl_blur_plan; /* opaque, immutable after create */

#define WL_MAX_LEVELS 32

typedef struct {
  int64_t offset; /* elements from the start of one image's coefficient block */
  int64_t rows, cols;
  int64_t pitch;  /* elements between rows (>= cols, multiple of 16 bytes)   */
} wl_subband;

typedef struct {
  int levels;        /* J */
  int filter_length; /* L */
  int64_t p_valid;   /* number of coefficients per image                  */
  int64_t p_alloc;   /* elements per image in x (with row-pitch padding)   */
  int64_t h[WL_MAX_LEVELS + 1], w[WL_MAX_LEVELS + 1]; /* level chains, h[0] = image height */
  wl_subband band[1 + 3 * WL_MAX_LEVELS]; /* LL_J, then LH_j, HL_j, HH_j for j = J..1 */
} wl_plan_info;

/* ----------------------------------------------------------------- plans */

/* Create a wavelet plan for [h, w] images, `levels` = J >= 1 levels.
 * Level chain per axis: n_j = floor((n_{j-1}+L-1)/2) (zero, symmetric*) or n_{j-1}/2
 * (periodic).  Fails with WL_ESIZE naming the first level that cannot be formed
 * (periodic with odd n_{j-1}; symmetric with n_{j-1} < L-1; J > 32; h, w < 1). */
WL_API wl_status wl_plan_create(wl_plan **out, int64_t h, int64_t w, int levels, wl_filter filter, wl_bc bc,
                         wl_dtype dtype);
WL_API void wl_plan_destroy(wl_plan *plan);
/* Fill *info_host (host pointer) with the level chains and the subband table. */
WL_API wl_status wl_plan_query(const wl_plan *plan, wl_plan_info *info_host);
/* Copy the plan's fp64 filter arrays (L taps each, host pointers, any may be NULL):
 * a_lo/a_hi analysis pair (W-dagger), d_lo/d_hi dual pair (W, W*).  Analysis convention:
 * out[k] = sum_j f[j] * yhat[2k+1-j]. */
WL_API wl_status wl_plan_filters(const wl_plan *plan, double *a_lo, double *a_hi, double *d_lo, double *d_hi);

/* Workspace bytes needed by `op` on `batch` images (blur may be NULL except for
 * WL_OP_GRAD).  0 is a valid answer (then ws may be NULL). */
WL_API size_t wl_workspace_bytes(const wl_plan *plan, const wl_blur_plan *blur, wl_op op, int64_t batch);

/* ------------------------------------------------------- wavelet operators */

/* W: coefficients x [batch, p_alloc] -> images img [batch, h, w].
 * Multi-level 2-D reconstruction, coarse to fine. */
WL_API wl_status wl_synthesize(const wl_plan *plan, int64_t batch, const void *x, void *img, void *ws,
                        void *stream);
/* W* (Eq. (4)): images -> coefficients, the exact transpose of wl_synthesize
 * (<W x, y> = <x, W* y>).  Dual-filter analysis after (E^dagger)*. */
WL_API wl_status wl_adjoint(const wl_plan *plan, int64_t batch, const void *img, void *x, void *ws,
                     void *stream);
/* W-dagger (W-dagger = W-dagger_zpd E): images -> coefficients, analysis
 * filters after the boundary extension E_bc.  W W-dagger = I except for SYMMETRIC_EDAG. */
WL_API wl_status wl_analyze(const wl_plan *plan, int64_t batch, const void *img, void *x, void *ws,
                     void *stream);
/* (W-dagger)* (the adjoint "(and analysis)"): coefficients
 * x [batch, p_alloc] -> images img [batch, h, w], the exact transpose of wl_analyze:
 * upsample-convolve with the ANALYSIS filters, then fold with E_bc^T -- truncate (zero),
 * wrap-add (periodic), unweighted reflect-add (symmetric, symmetric_edag).
 * ws: wl_workspace_bytes(plan, NULL, WL_OP_ANALYZE_ADJOINT, batch). */
WL_API wl_status wl_analyze_adjoint(const wl_plan *plan, int64_t batch, const void *x, void *img, void *ws,
                             void *stream);

/* ------------------------------------------------------------------- blur */

/* Separable blur plan for [h, w] images: per axis (R_a y)[i] = sum_t k[t] yhat[i-t],
 * t = -(ntaps/2)..ntaps/2, yhat the half-point symmetric extension; R = R_0 (x) R_1.
 * taps_host: ntaps (odd, <= 31) host doubles, which must be symmetric (k[t] = k[-t]) so that
 * R* = R (WL_EINVAL otherwise); h, w >= ntaps/2.  bc must be WL_BC_SYMMETRIC. */
WL_API wl_status wl_blur_create(wl_blur_plan **out, int64_t h, int64_t w, const double *taps_host, int ntaps,
                         wl_bc bc, wl_dtype dtype);
/* Gaussian PSF: k[t] = exp(-t^2/(2 sigma^2)) / sum (BASELINE.json config 5: 15 taps, sigma 3). */
WL_API wl_status wl_blur_create_gaussian(wl_blur_plan **out, int64_t h, int64_t w, int ntaps, double sigma,
                                  wl_bc bc, wl_dtype dtype);
WL_API void wl_blur_destroy(wl_blur_plan *blur);
/* Copy the plan's fp64 taps (ntaps entries) to taps_host. */
WL_API wl_status wl_blur_taps(const wl_blur_plan *blur, double *taps_host, int *ntaps_host);

/* R: in [batch, h, w] -> out [batch, h, w]. */
WL_API wl_status wl_blur(const wl_blur_plan *blur, int64_t batch, const void *in, void *out, void *stream);
/* R*: the adjoint E_sym^T o correlation per axis; equal to R for the symmetric PSFs accepted. */
WL_API wl_status wl_blur_adjoint(const wl_blur_plan *blur, int64_t batch, const void *in, void *out,
                          void *stream);
/* The middle stage of grad f, fused: s = R*(R u - b).  If f_dev != NULL it receives
 * f = 1/2 ||R u - b||^2 per image (double[batch], overwritten). */
WL_API wl_status wl_blur_residual_adjoint(const wl_blur_plan *blur, int64_t batch, const void *u, const void *b,
                                   void *s, double *f_dev, void *stream);

/* ------------------------------------------------------------- gradient */

/* grad f(x) = W* R* (R W x - b).  x [batch, p_alloc], b [batch, h, w] ->
 * g [batch, p_alloc]; f_dev (nullable) receives f = 1/2 ||R W x - b||^2 per image.
 * The plans must agree in h, w and dtype.  ws: wl_workspace_bytes(plan, blur, WL_OP_GRAD, batch). */
WL_API wl_status wl_grad(const wl_plan *plan, const wl_blur_plan *blur, int64_t batch, const void *x,
                  const void *b, void *g, double *f_dev, void *ws, void *stream);

/* wl_grad with HOST buffers: x_host [batch, p_alloc], b_host [batch, h, w] -> g_host [batch, p_alloc],
 * f_host (nullable, double[batch]).  The images are pipelined through two device slots inside `ws`
 * (wl_workspace_bytes(plan, blur, WL_OP_GRAD_HOST, batch); independent of batch): image i+1 is copied
 * in on an internal copy stream while image i is differentiated on `stream` and image i-1 copied out
 * on a second copy stream, so the transfers overlap each other and the kernels.  Host buffers should
 * be page-locked (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous; pageable
 * buffers still give correct results.  Stream-ordered: the outputs are complete when `stream` reaches
 * the point after the call; the host buffers must stay untouched until then. */
WL_API wl_status wl_grad_host(const wl_plan *plan, const wl_blur_plan *blur, int64_t batch, const void *x_host,
                       const void *b_host, void *g_host, double *f_host, void *ws, void *stream);

/* Which operator closes the gradient (P:117, P:176-177 compare both under FISTA):
 *   WL_ADJ_TRUE  W*  (the true adjoint, Eq. (4)) -> grad f exactly;
 *   WL_ADJ_PINV  W-dagger in place of W* (the common approximation W* ~ W-dagger);
 *                identical to WL_ADJ_TRUE for orthogonal filters under zero / periodic BC. */
typedef enum { WL_ADJ_TRUE = 0, WL_ADJ_PINV = 1 } wl_adj;

/* wl_grad with the choice of closing operator: g = A R* (R W x - b), A = W* or W-dagger. */
WL_API wl_status wl_grad_adj(const wl_plan *plan, const wl_blur_plan *blur, int64_t batch, const void *x,
                      const void *b, void *g, double *f_dev, wl_adj adj, void *ws, void *stream);

/* ------------------------------------------------------------- FISTA */

/* FISTA (Beck & Teboulle 2009; the solver of P:117 and P:174, 2500 iterations there) for
 *     min_x 1/2 ||R W x - b||^2 + lambda ||x||_1      (Eq. (1)).
 * wl_fista_update: given g = grad f(y) [batch, p_alloc], in place
 *     x <- soft(y - g / lip, lambda / lip),  t+ = (1 + sqrt(1 + 4 t^2)) / 2,
 *     y <- x + ((t - 1) / t+) (x - x_old).
 * t is the host-side momentum scalar of the current step (t_1 = 1); *t_next_host (host pointer,
 * nullable) receives t+ for the next call, so the recursion lives in the library only.  lip > 0 is
 * the Lipschitz constant of grad f (wl_lipschitz), lambda >= 0.  Pitch padding stays 0.  x, y, g
 * must not overlap (WL_EINVAL). */
WL_API wl_status wl_fista_update(const wl_plan *plan, int64_t batch, const void *g, void *x, void *y, double t,
                          double lambda, double lip, double *t_next_host, void *stream);
/* One full FISTA iteration: g = grad f(y) (wl_grad_adj with `adj`; f_dev, nullable, receives
 * f(y)), then the wl_fista_update arithmetic, fused into the stores of the closing analysis
 * chain: g itself is never written.  *t_next_host (nullable) receives t_{k+1}, written before the
 * call returns (the launches stay asynchronous).  ws: wl_workspace_bytes(plan, blur, WL_OP_FISTA,
 * batch). */
WL_API wl_status wl_fista_step(const wl_plan *plan, const wl_blur_plan *blur, int64_t batch, const void *b, void *x,
                        void *y, double t, double lambda, double lip, double *f_dev, wl_adj adj, void *ws,
                        double *t_next_host, void *stream);
/* wl_fista_step with the momentum scalar t resident on the device: t_dev (double, device) holds
 * t_k on entry and t_{k+1} on exit (advanced by a one-thread kernel after the update).  Every
 * argument of the launch sequence is then the same from one iteration to the next, so a CUDA
 * graph of one call replays the whole FISTA loop. */
WL_API wl_status wl_fista_step_dev(const wl_plan *plan, const wl_blur_plan *blur, int64_t batch, const void *b,
                            void *x, void *y, double *t_dev, double lambda, double lip, double *f_dev, wl_adj adj,
                            void *ws, void *stream);
/* Power iteration for lip = lambda_max(W* R* R W): v_0 = a seeded uniform(-1, 1)
 * vector, v <- G v with G v = grad f(v) at b = 0, estimate <v, G v> / <v, v> of the last step
 * (a lower bound that increases to lambda_max).  Blocking: synchronises `stream` every iteration
 * to rescale v.  *lip_host (host pointer) receives the estimate.
 * ws: wl_workspace_bytes(plan, blur, WL_OP_LIPSCHITZ, 1). */
WL_API wl_status wl_lipschitz(const wl_plan *plan, const wl_blur_plan *blur, int iters, uint64_t seed,
                       double *lip_host, void *ws, void *stream);

/* ------------------------------------------------- Example 2: blind channel estimation */

/* PAPER.md §"Example 2: Blind Channel Estimation".  Real signals,
 * zero-padded boundaries.  All arrays are contiguous device arrays of `dtype`, batch-major; the
 * caller owns them; outputs must not overlap inputs (WL_EINVAL).  Sizes are limited by one CTA's
 * shared memory (WL_ESIZE names the need): the paper's K_est = 844, N_est = 1767 with two channels
 * use 49 KB (fp32) / 98 KB (fp64).  Element alignment only.  Stream-ordered, asynchronous. */

/* x_est = h * s, the "full" convolution x[m] = sum_k h[k] s[m-k], m < K+N-1.
 * h [batch, K], s [batch, N] -> x [batch, K+N-1]. */
WL_API wl_status wl_conv_full(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *h, const void *s,
                       void *x, void *stream);
/* S* r: the "valid" cross-correlation gh[n] = sum_{k<N} s[k] r[k+n], n < K (MATLAB
 * conv(r, conj(s(end:-1:1)), 'valid')).  s [batch, N], r [batch, K+N-1] -> gh [batch, K]. */
WL_API wl_status wl_conv_adjoint_h(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *s, const void *r,
                            void *gh, void *stream);
/* H* r: gs[k] = sum_{n<K} h[n] r[k+n], k < N.  h [batch, K], r [batch, K+N-1] -> gs [batch, N]. */
WL_API wl_status wl_conv_adjoint_s(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *h, const void *r,
                            void *gs, void *stream);
/* Gradient of the smooth part of Eq. (6), fused, for `problems` independent problems
 * of `channels` channels sharing one source:
 *     F = sum_i ||h_i * s - x_i||^2 + (lam_tv / delta) sum_i L_delta(D h_i)     (no 1/2: Eq. (6))
 *     gh_i = 2 S* r_i + (lam_tv / delta) D^T L_delta'(D h_i),  gs = 2 sum_i H_i* r_i,  r_i = h_i * s - x_i
 * with (D h)_j = h_{j+1} - h_j and the Huber function L_delta.
 * h [problems, channels, K], s [problems, N], x [problems, channels, K+N-1] (x_shared != 0: one
 * [channels, K+N-1] observation for every problem, e.g. random restarts) -> gh like h, gs like s,
 * f_dev (nullable) double[problems] <- F.  delta > 0, lam_tv >= 0. */
WL_API wl_status wl_bce_grad(wl_dtype dtype, int64_t problems, int channels, int64_t K, int64_t N, const void *h,
                      const void *s, const void *x, int x_shared, double lam_tv, double delta, void *gh,
                      void *gs, double *f_dev, void *stream);

/* ---------------------------------------------------------------- misc */

WL_API const char *wl_last_error(void); /* thread-local; never NULL */
/* Number of kernels this library has launched in this process (monotonic). */
WL_API int64_t wl_launch_count(void);
WL_API const char *wl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WL_H_ */
