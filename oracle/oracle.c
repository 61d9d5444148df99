/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the hot path of arXiv 1707.02018
 * (Folberth & Becker, "Efficient Adjoint Computation for Wavelet and Convolution
 * Operators").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path under
 * paper_1707_02018_b200/ (and includes none of its headers).
 *
 * Every function is a direct transcription of a definition; no blocking, fusion or
 * reordering.  Citations: P:n = PAPER.md line n (section named), SURVEY.md §8(c) C.1
 * for the readings the paper leaves open (listed in DESIGN.md "Readings").
 *
 *   extension E (paper §"A few signal extensions"):
 *       E_zpd, E_sym, E_per;
 *       (E^dagger)* = E diag(1/c), c_i = multiplicity of sample i
 *   analysis core (reading R5): A_f(yhat)[k] = sum_{j<L} f[j] yhat[2k+1-j]
 *   W-dagger = W-dagger_zpd E
 *   W* = W~dagger_zpd (E^dagger)*  (Eq. (4)) with reading R1
 *   W  = (W*)^T, written as the literal scatter transpose of the analysis core
 *   R  = crop o conv o E_sym (reading R12); R* = E_sym^T o correlation
 *   2-D: separable, axis 1 (width) then axis 0 (height) (P:57 footnote; reading R8)
 *
 * Parity unpinned: none.  Pins live in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define WLO_EXT_ZERO 0      /* E_zpd                                  */
#define WLO_EXT_PER 1       /* periodisation: yhat[i] = y[i mod n]    */
#define WLO_EXT_SYM 2       /* half-point symmetric E_sym             */
#define WLO_EXT_SYM_PADJ 3  /* (E_sym^dagger)* = E_sym diag(1/c)      */

#define WLO_FOLD_CROP 0     /* y[i] = u[i], i in [0, n)               */
#define WLO_FOLD_WRAP 1     /* y[i] = sum_{t = i mod n} u[t]          */
#define WLO_FOLD_SYM_PINV 2 /* y = E_sym^dagger u = diag(1/c) E_sym^T u */
#define WLO_FOLD_SYM_T 3    /* y = E_sym^T u  (reflect-add; the adjoint of W-dagger's E_sym) */

/* ---------------------------------------------------------------- extension */

/* Source index of extended position i under E; -1 = zero. */
static long src_index(long i, long n, int kind) {
  if (kind == WLO_EXT_ZERO) return (i >= 0 && i < n) ? i : -1;
  if (kind == WLO_EXT_PER) {
    long r = i % n;
    return r < 0 ? r + n : r;
  }
  /* half-point symmetric: ..., y[1], y[0] | y[0], ..., y[n-1] | y[n-1], y[n-2], ... */
  if (i < 0) return -1 - i;
  if (i >= n) return 2 * n - 1 - i;
  return i;
}

/* c_i = #{t in [-Lp, n+Lp) : src(t) = i} (the column sums of E). */
static void multiplicity(long n, long Lp, int kind, double *c) {
  for (long i = 0; i < n; i++) c[i] = 0.0;
  for (long t = -Lp; t < n + Lp; t++) {
    long s = src_index(t, n, kind);
    if (s >= 0) c[s] += 1.0;
  }
}

/* out[t + Lp] = (E y)[t], t in [-Lp, n+Lp)  (mode 0); (E^dagger)* y (mode 1) */
int wlo_extend1d(const double *y, long n, long Lp, int kind, int pinv_adjoint, double *out) {
  double *c = (double *)malloc(sizeof(double) * (size_t)n);
  if (!c) return 1;
  multiplicity(n, Lp, kind, c);
  for (long t = -Lp; t < n + Lp; t++) {
    long s = src_index(t, n, kind);
    double v = 0.0;
    if (s >= 0) v = pinv_adjoint ? y[s] / c[s] : y[s];
    out[t + Lp] = v;
  }
  free(c);
  return 0;
}

/* y = E^T v (mode 0) or E^dagger v = diag(1/c) E^T v (mode 1); v has n + 2 Lp entries */
int wlo_extend_adjoint1d(const double *v, long n, long Lp, int kind, int pinv, double *y) {
  double *c = (double *)malloc(sizeof(double) * (size_t)n);
  if (!c) return 1;
  multiplicity(n, Lp, kind, c);
  for (long i = 0; i < n; i++) y[i] = 0.0;
  for (long t = -Lp; t < n + Lp; t++) {
    long s = src_index(t, n, kind);
    if (s >= 0) y[s] += v[t + Lp];
  }
  if (pinv)
    for (long i = 0; i < n; i++) y[i] /= c[i];
  free(c);
  return 0;
}

/* ------------------------------------------------------------ level chains */

/* Coefficient count of one level (reading R2/R3, BASELINE.json configs 2 and 4):
 * floor((n+L-1)/2) for zero / symmetric, n/2 for periodisation. */
static long coef_len(long n, int L, int periodic) { return periodic ? n / 2 : (n + L - 1) / 2; }

/* Fill out[0..J] with the chain n_0 = n, n_j = coef_len(n_{j-1}); 0 on success,
 * -(j) if level j cannot be formed (per: odd length; sym: n < L-1; any: n < 1). */
int wlo_chain(long n, int L, int ext_kind, int J, long *out) {
  int periodic = (ext_kind == WLO_EXT_PER);
  int sym = (ext_kind == WLO_EXT_SYM || ext_kind == WLO_EXT_SYM_PADJ);
  out[0] = n;
  for (int j = 1; j <= J; j++) {
    long m = out[j - 1];
    if (m < 1) return -j;
    if (periodic && (m % 2 != 0)) return -j;
    if (sym && m < L - 1) return -j;
    out[j] = coef_len(m, L, periodic);
    if (out[j] < 1) return -j;
  }
  return 0;
}

/* ------------------------------------------------------------- 1-D levels */

/* Analysis core over the extension:  out[k] = sum_j f[j] * yhat[2k+1-j], k < m.
 * Input y is read with stride ys, output written with stride os. */
static void analysis_1d(const double *y, long ys, long n, const double *f, int L, int kind,
                        const double *cinv, double *out, long os, long m) {
  for (long k = 0; k < m; k++) {
    double acc = 0.0;
    for (int j = 0; j < L; j++) {
      long t = 2 * k + 1 - j;
      long s = src_index(t, n, kind == WLO_EXT_SYM_PADJ ? WLO_EXT_SYM : kind);
      if (s < 0) continue;
      double v = y[s * ys];
      if (kind == WLO_EXT_SYM_PADJ) v *= cinv[s];
      acc += f[j] * v;
    }
    out[k * os] = acc;
  }
}

/* Synthesis = transpose of the dual analysis: scatter u[2k+1-j] += g_lo[j] a[k] + g_hi[j] d[k]
 * over t in [-Lp, n+Lp), then fold back onto [0, n). */
static void synthesis_1d(const double *a, const double *d, long cs, long m, const double *glo,
                         const double *ghi, int L, int fold, long n, double *u, const double *cinv,
                         double *y, long ys) {
  long Lp = L - 1;
  long U = n + 2 * Lp;
  for (long t = 0; t < U; t++) u[t] = 0.0;
  for (long k = 0; k < m; k++) {
    for (int j = 0; j < L; j++) {
      long t = 2 * k + 1 - j;
      u[t + Lp] += glo[j] * a[k * cs] + ghi[j] * d[k * cs];
    }
  }
  for (long i = 0; i < n; i++) y[i * ys] = 0.0;
  for (long t = -Lp; t < n + Lp; t++) {
    long s;
    if (fold == WLO_FOLD_CROP)
      s = (t >= 0 && t < n) ? t : -1;
    else if (fold == WLO_FOLD_WRAP)
      s = src_index(t, n, WLO_EXT_PER);
    else
      s = src_index(t, n, WLO_EXT_SYM);
    if (s >= 0) y[s * ys] += u[t + Lp];
  }
  if (fold == WLO_FOLD_SYM_PINV)
    for (long i = 0; i < n; i++) y[i * ys] *= cinv[i];
}

/* ------------------------------------------------------------- 2-D levels */

/* Packed oracle layout (reading R7, without the GPU's row pitch):
 * LL_J, then (LH_j, HL_j, HH_j) for j = J..1, each row-major m0_j x m1_j.
 * Subband XY = axis-0 filter X, axis-1 filter Y. */
static long packed_size(const long *c0, const long *c1, int J) {
  long p = c0[J] * c1[J];
  for (int j = 1; j <= J; j++) p += 3 * c0[j] * c1[j];
  return p;
}
static long detail_offset(const long *c0, const long *c1, int J, int j) {
  long off = c0[J] * c1[J];
  for (int l = J; l > j; l--) off += 3 * c0[l] * c1[l];
  return off;
}

/* 1/c_i for the (E_sym^dagger)* / E_sym^dagger weights, or all ones when unweighted. */
static double *cinv_table(long n, int L, int weighted) {
  double *c = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (weighted) {
    multiplicity(n, L - 1, WLO_EXT_SYM, c);
    for (long i = 0; i < n; i++) c[i] = 1.0 / c[i];
  } else {
    for (long i = 0; i < n; i++) c[i] = 1.0;
  }
  return c;
}

long wlo_num_coeffs(long h, long w, int L, int ext_kind, int J) {
  long c0[40], c1[40];
  if (J < 1 || J > 32) return -1;
  if (wlo_chain(h, L, ext_kind, J, c0) != 0) return -1;
  if (wlo_chain(w, L, ext_kind, J, c1) != 0) return -1;
  return packed_size(c0, c1, J);
}

/* Multi-level 2-D analysis with filters (flo, fhi) and extension ext_kind.
 * img: [B, h, w] row-major; x: [B, p] packed.  W-dagger uses (a_lo, a_hi, E_bc);
 * W* uses (d_lo, d_hi) with E_zpd / E_per / (E_sym^dagger)* (reading R1). */
int wlo_analysis2d(const double *img, long B, long h, long w, int J, const double *flo,
                   const double *fhi, int L, int ext_kind, double *x) {
  long c0[40], c1[40];
  if (J < 1 || J > 32) return 1;
  if (wlo_chain(h, L, ext_kind, J, c0) != 0 || wlo_chain(w, L, ext_kind, J, c1) != 0) return 2;
  long p = packed_size(c0, c1, J);
  for (long b = 0; b < B; b++) {
    const double *src = img + b * h * w;
    double *xb = x + b * p;
    double *cur = (double *)malloc(sizeof(double) * (size_t)(h * w));
    memcpy(cur, src, sizeof(double) * (size_t)(h * w));
    for (int j = 1; j <= J; j++) {
      long n0 = c0[j - 1], n1 = c1[j - 1], m0 = c0[j], m1 = c1[j];
      double *tL = (double *)malloc(sizeof(double) * (size_t)(n0 * m1));
      double *tH = (double *)malloc(sizeof(double) * (size_t)(n0 * m1));
      double *ci1 = cinv_table(n1, L, ext_kind == WLO_EXT_SYM_PADJ);
      double *ci0 = cinv_table(n0, L, ext_kind == WLO_EXT_SYM_PADJ);
      /* axis 1: every row */
#pragma omp parallel for schedule(static)
      for (long r = 0; r < n0; r++) {
        analysis_1d(cur + r * n1, 1, n1, flo, L, ext_kind, ci1, tL + r * m1, 1, m1);
        analysis_1d(cur + r * n1, 1, n1, fhi, L, ext_kind, ci1, tH + r * m1, 1, m1);
      }
      double *LL = (double *)malloc(sizeof(double) * (size_t)(m0 * m1));
      long doff = detail_offset(c0, c1, J, j);
      double *LH = xb + doff, *HL = LH + m0 * m1, *HH = HL + m0 * m1;
      /* axis 0: every column */
#pragma omp parallel for schedule(static)
      for (long c = 0; c < m1; c++) {
        analysis_1d(tL + c, m1, n0, flo, L, ext_kind, ci0, LL + c, m1, m0);
        analysis_1d(tL + c, m1, n0, fhi, L, ext_kind, ci0, HL + c, m1, m0);
        analysis_1d(tH + c, m1, n0, flo, L, ext_kind, ci0, LH + c, m1, m0);
        analysis_1d(tH + c, m1, n0, fhi, L, ext_kind, ci0, HH + c, m1, m0);
      }
      free(tL); free(tH); free(ci0); free(ci1); free(cur);
      cur = LL;
    }
    memcpy(xb, cur, sizeof(double) * (size_t)(c0[J] * c1[J]));
    free(cur);
  }
  return 0;
}

/* Multi-level 2-D synthesis (the transpose of wlo_analysis2d with the same filters
 * and the fold that is the adjoint of its extension: CROP <-> ZERO, WRAP <-> PER,
 * SYM_PINV <-> SYM_PADJ, SYM_T <-> SYM).  x: [B, p] packed; img: [B, h, w]. */
int wlo_synthesis2d(const double *x, long B, long h, long w, int J, const double *glo,
                    const double *ghi, int L, int fold, double *img) {
  long c0[40], c1[40];
  int chain_kind = fold == WLO_FOLD_WRAP       ? WLO_EXT_PER
                   : fold == WLO_FOLD_SYM_PINV ? WLO_EXT_SYM_PADJ
                   : fold == WLO_FOLD_SYM_T    ? WLO_EXT_SYM
                                               : WLO_EXT_ZERO;
  if (J < 1 || J > 32) return 1;
  if (wlo_chain(h, L, chain_kind, J, c0) != 0 || wlo_chain(w, L, chain_kind, J, c1) != 0) return 2;
  long p = packed_size(c0, c1, J);
  long Lp = L - 1;
  for (long b = 0; b < B; b++) {
    const double *xb = x + b * p;
    double *cur = (double *)malloc(sizeof(double) * (size_t)(c0[J] * c1[J]));
    memcpy(cur, xb, sizeof(double) * (size_t)(c0[J] * c1[J]));
    for (int j = J; j >= 1; j--) {
      long n0 = c0[j - 1], n1 = c1[j - 1], m0 = c0[j], m1 = c1[j];
      long doff = detail_offset(c0, c1, J, j);
      const double *LH = xb + doff, *HL = LH + m0 * m1, *HH = HL + m0 * m1;
      const double *LL = cur;
      double *ci0 = cinv_table(n0, L, fold == WLO_FOLD_SYM_PINV);
      double *ci1 = cinv_table(n1, L, fold == WLO_FOLD_SYM_PINV);
      double *tL = (double *)malloc(sizeof(double) * (size_t)(n0 * m1));
      double *tH = (double *)malloc(sizeof(double) * (size_t)(n0 * m1));
      /* axis 0 first (transpose of "axis 1 then axis 0") */
#pragma omp parallel for schedule(static)
      for (long c = 0; c < m1; c++) {
        double *u = (double *)malloc(sizeof(double) * (size_t)(n0 + 2 * Lp));
        synthesis_1d(LL + c, HL + c, m1, m0, glo, ghi, L, fold, n0, u, ci0, tL + c, m1);
        synthesis_1d(LH + c, HH + c, m1, m0, glo, ghi, L, fold, n0, u, ci0, tH + c, m1);
        free(u);
      }
      double *out = (j == 1) ? img + b * h * w : (double *)malloc(sizeof(double) * (size_t)(n0 * n1));
#pragma omp parallel for schedule(static)
      for (long r = 0; r < n0; r++) {
        double *u = (double *)malloc(sizeof(double) * (size_t)(n1 + 2 * Lp));
        synthesis_1d(tL + r * m1, tH + r * m1, 1, m1, glo, ghi, L, fold, n1, u, ci1, out + r * n1, 1);
        free(u);
      }
      free(tL); free(tH); free(ci0); free(ci1); free(cur);
      cur = (j == 1) ? NULL : out;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------- blur */

/* R_a y[i] = sum_{t=-hh..hh} k[t+hh] * yhat[i-t],  yhat = E_sym y (pad hh)         */
static void blur_1d(const double *y, long ys, long n, const double *k, int hh, double *out, long os) {
  for (long i = 0; i < n; i++) {
    double acc = 0.0;
    for (int t = -hh; t <= hh; t++) acc += k[t + hh] * y[src_index(i - t, n, WLO_EXT_SYM) * ys];
    out[i * os] = acc;
  }
}

/* R_a^T v = E_sym^T (full correlation):  u[s] = sum_t k[t+hh] v[s+t], s in [-hh, n+hh),
 * then y[i] = sum_{s : src(s) = i} u[s]  (reflect-add). */
static void blur_adjoint_1d(const double *v, long vs, long n, const double *k, int hh, double *u,
                            double *out, long os) {
  for (long s = -hh; s < n + hh; s++) {
    double acc = 0.0;
    for (int t = -hh; t <= hh; t++) {
      long i = s + t;
      if (i >= 0 && i < n) acc += k[t + hh] * v[i * vs];
    }
    u[s + hh] = acc;
  }
  for (long i = 0; i < n; i++) out[i * os] = 0.0;
  for (long s = -hh; s < n + hh; s++) out[src_index(s, n, WLO_EXT_SYM) * os] += u[s + hh];
}

/* 2-D separable blur R = R_0 (x) R_1 (adjoint = 1): axis 1 then axis 0. Needs h,w >= hh. */
int wlo_blur2d(const double *in, long B, long h, long w, const double *k, int ntaps, int adjoint,
               double *out) {
  int hh = ntaps / 2;
  if (ntaps % 2 != 1 || h < hh || w < hh) return 1;
  double *tmp = (double *)malloc(sizeof(double) * (size_t)(h * w));
  for (long b = 0; b < B; b++) {
    const double *src = in + b * h * w;
    double *dst = out + b * h * w;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < h; r++) {
      if (adjoint) {
        double *u = (double *)malloc(sizeof(double) * (size_t)(w + 2 * hh));
        blur_adjoint_1d(src + r * w, 1, w, k, hh, u, tmp + r * w, 1);
        free(u);
      } else {
        blur_1d(src + r * w, 1, w, k, hh, tmp + r * w, 1);
      }
    }
#pragma omp parallel for schedule(static)
    for (long c = 0; c < w; c++) {
      if (adjoint) {
        double *u = (double *)malloc(sizeof(double) * (size_t)(h + 2 * hh));
        blur_adjoint_1d(tmp + c, w, h, k, hh, u, dst + c, w);
        free(u);
      } else {
        blur_1d(tmp + c, w, h, k, hh, dst + c, w);
      }
    }
  }
  free(tmp);
  return 0;
}
