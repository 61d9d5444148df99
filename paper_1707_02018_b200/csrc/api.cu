// C ABI of libwl (include/wl.h): plan construction, validation and the operator drivers.
// Every operator is a chain of kernel launches on the caller's stream; no host sync.
//
//   wl_synthesize  W            coarse -> fine, one synthesis launch per level
//   wl_adjoint     W*  (Eq. (4))    fine -> coarse, dual filters after (E^dagger)*
//   wl_analyze     W-dagger          fine -> coarse, analysis filters after E_bc
//   wl_blur / wl_blur_adjoint   R / R*
//   wl_blur_residual_adjoint    s = R*(R u - b)   (the middle of P:43-45)
//   wl_grad        grad f = W* R* (R W x - b)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "wl_internal.h"

namespace wl {
std::atomic<int64_t> g_launches{0};

cudaError_t launch_zero(void *ptr, size_t bytes, cudaStream_t s) { return cudaMemsetAsync(ptr, 0, bytes, s); }
}  // namespace wl

using namespace wl;

namespace {

thread_local std::string t_err = "";

wl_status fail(wl_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}

wl_status ok() {
  t_err.clear();
  return WL_OK;
}

wl_status cuda_fail(cudaError_t e, const char *what) {
  return fail(WL_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// FISTA momentum recursion t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2 (Beck & Teboulle, cited at P:117;
// DESIGN.md reading R21); the device-resident variant is k_fista_advance_t.
double fista_next_t(double t) { return (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0; }
size_t align256(size_t v) { return (v + 255) / 256 * 256; }

const char *bc_name(int bc) {
  switch (bc) {
    case WL_BC_ZERO: return "zero";
    case WL_BC_PERIODIC: return "periodic";
    case WL_BC_SYMMETRIC: return "symmetric";
    case WL_BC_SYMMETRIC_EDAG: return "symmetric_edag";
  }
  return "?";
}

// pointer checks ------------------------------------------------------------
wl_status check_dev(const void *p, const char *name, size_t align = 16) {
  if (!p) return fail(WL_EINVAL, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(p) % align)
    return fail(WL_EALIGN, "%s = %p is not %zu-byte aligned", name, p, align);
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(WL_EINVAL, "%s = %p is not a CUDA pointer (%s)", name, p, cudaGetErrorString(e));
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(WL_EINVAL, "%s = %p is not device memory", name, p);
  return WL_OK;
}

constexpr size_t kMaxSmemOptin = 227 * 1024;  // sm_100a opt-in dynamic shared memory per CTA
// the launch structures carry the batch as int (grid dimensions and per-image offsets)
constexpr int kMaxBatch = 0x7fffffff;

bool overlap(const void *a, size_t na, const void *b, size_t nb) {
  auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return na && nb && x < y + nb && y < x + na;
}

// workspace carve-up ---------------------------------------------------------
struct WsLayout {
  size_t a = 0, b = 0, e = 0, u = 0, s = 0, g = 0, v = 0, b0 = 0, d = 0, total = 0;  // byte offsets
  size_t hx = 0, hb = 0, hg = 0, hf = 0;  // WL_OP_GRAD_HOST: two device slots each for x, b, g, f
};

WsLayout ws_layout(const wl_plan *p, const wl_blur_plan *bl, wl_op op, int64_t batch) {
  if (op == WL_OP_GRAD_HOST) {  // the grad workspace of one image + two staging slots
    WsLayout L = ws_layout(p, bl, WL_OP_GRAD, 1);
    const size_t es = (size_t)p->es, xs = (size_t)p->p_alloc * es, is = (size_t)p->h * p->w * es;
    size_t off = L.total;
    L.hx = off; off = align256(off + 2 * xs);
    L.hb = off; off = align256(off + 2 * is);
    L.hg = off; off = align256(off + 2 * xs);
    L.hf = off; off = align256(off + 2 * sizeof(double));
    L.total = batch > 0 ? off : 0;
    return L;
  }
  WsLayout L;
  size_t es = (size_t)p->es, B = (size_t)batch;
  size_t off = 0;
  L.a = off; off = align256(off + B * (size_t)p->ws_a_elems * es);
  L.b = off; off = align256(off + B * (size_t)p->ws_b_elems * es);
  L.e = off;
  if (((op == WL_OP_SYNTHESIZE || op == WL_OP_GRAD || op == WL_OP_FISTA || op == WL_OP_LIPSCHITZ) &&
       p->bc == WL_BC_SYMMETRIC_EDAG) ||
      (op == WL_OP_ANALYZE_ADJOINT && (p->bc == WL_BC_SYMMETRIC_EDAG || p->bc == WL_BC_SYMMETRIC)))
    off = align256(off + B * (size_t)p->edag_elems * es);
  L.u = off;
  L.s = off;
  if (op == WL_OP_GRAD || op == WL_OP_FISTA || op == WL_OP_LIPSCHITZ) {
    size_t img = B * (size_t)p->h * (size_t)p->w * es;
    L.u = off; off = align256(off + img);
    L.s = off; off = align256(off + img);
  }
  (void)bl;
  if (op == WL_OP_FISTA) {  // + g = grad f(y)
    L.g = off;
    off = align256(off + B * (size_t)p->p_alloc * es);
  }
  if (op == WL_OP_LIPSCHITZ) {  // + v, g (one image), a zero image b0, two fp64 scalars
    L.v = off; off = align256(off + (size_t)p->p_alloc * es);
    L.g = off; off = align256(off + (size_t)p->p_alloc * es);
    L.b0 = off; off = align256(off + (size_t)p->h * p->w * es);
    L.d = off; off = align256(off + 2 * sizeof(double));
  }
  L.total = off;
  return L;
}

// level buffers ---------------------------------------------------------------
struct Buf {
  char *ptr;
  int64_t pitch, bstride;
};

Buf ll_buf(const wl_plan *p, char *ws, const WsLayout &L, int j) {  // LL_j, 1 <= j < J
  Buf b;
  b.ptr = ws + ((j % 2) ? L.a : L.b);
  b.pitch = p->ll_pitch[j];
  b.bstride = (j % 2) ? p->ws_a_elems : p->ws_b_elems;
  return b;
}

Buf band_buf(const wl_plan *p, const void *x, int idx) {
  Buf b;
  b.ptr = (char *)x + (size_t)p->band[idx].offset * (size_t)p->es;
  b.pitch = p->band[idx].pitch;
  b.bstride = p->p_alloc;
  return b;
}

int lh_index(const wl_plan *p, int j) { return 1 + 3 * (p->J - j); }

// analysis chain (W-dagger when adjoint = false, W* when true) -----------------
// fused FISTA epilogue for the W* chain: x is the coefficient array written by run_analysis (= y of
// the iteration), xo the other state vector; every stored coefficient is g of grad f(y).
struct FistaFuse {
  void *xo;
  double inv_lip, tau, mom;
  const double *tdev;  // non-null: mom from the device-resident t
};

wl_status run_analysis(const wl_plan *p, int64_t batch, const void *img, void *x, char *ws, const WsLayout &L,
                       bool adjoint, cudaStream_t s, const FistaFuse *fz = nullptr) {
  int ext;
  if (adjoint)
    ext = p->bc == WL_BC_PERIODIC ? EXT_PER : (p->bc == WL_BC_SYMMETRIC_EDAG ? EXT_SYM_PADJ : EXT_ZERO);
  else
    ext = p->bc == WL_BC_PERIODIC ? EXT_PER : (p->bc == WL_BC_ZERO ? EXT_ZERO : EXT_SYM);
  AnalysisArgs chain[WL_MAX_LEVELS];
  for (int j = 1; j <= p->J; j++) {
    AnalysisArgs &a = chain[j - 1];
    a = AnalysisArgs();
    if (j == 1) {
      a.in = img;
      a.in_pitch = p->w;
      a.in_bstride = p->h * p->w;
    } else {
      Buf in = ll_buf(p, ws, L, j - 1);
      a.in = in.ptr;
      a.in_pitch = in.pitch;
      a.in_bstride = in.bstride;
    }
    a.n0 = (int)p->n0[j - 1];
    a.n1 = (int)p->n1[j - 1];
    Buf ll = (j == p->J) ? band_buf(p, x, 0) : ll_buf(p, ws, L, j);
    Buf lh = band_buf(p, x, lh_index(p, j)), hl = band_buf(p, x, lh_index(p, j) + 1),
        hh = band_buf(p, x, lh_index(p, j) + 2);
    Buf outs[4] = {ll, lh, hl, hh};
    for (int i = 0; i < 4; i++) {
      a.out[i] = outs[i].ptr;
      a.out_pitch[i] = outs[i].pitch;
      a.out_bstride[i] = outs[i].bstride;
    }
    a.m0 = (int)p->n0[j];
    a.m1 = (int)p->n1[j];
    a.ext = ext;
    a.lo = adjoint ? p->fb.d_lo : p->fb.a_lo;
    a.hi = adjoint ? p->fb.d_hi : p->fb.a_hi;
    a.L = p->fb.L;
    a.batch = (int)batch;
    a.ll_keep = j < p->J;  // LL_j is read by level j+1 right away
    if (fz) {  // LH/HL/HH of every level and LL of the last land in x
      a.fista_mask = (j == p->J) ? 15 : 14;
      a.fista_xdelta = ((char *)fz->xo - (char *)x) / (int64_t)p->es;
      a.fista_inv_lip = fz->inv_lip;
      a.fista_tau = fz->tau;
      a.fista_mom = fz->mom;
      a.fista_tdev = fz->tdev;
      cudaError_t e = launch_analysis(p->dtype, a, s);
      if (e != cudaSuccess) return cuda_fail(e, "analysis level launch");
    }
  }
  if (!fz) {  // long levels one launch each, the short coarse tail as one persistent launch
    cudaError_t e = launch_analysis_chain(p->dtype, chain, p->J, s);
    if (e != cudaSuccess) return cuda_fail(e, "analysis chain launch");
  }
  return WL_OK;
}

bool full_fold() {
  static const bool v = getenv("WL_FULL_FOLD") != nullptr;  // A/B: synthesize the whole frame, fold it all
  return v;
}

// synthesis chain (W) ------------------------------------------------------------
// Multi-level upsample-convolve chain, coarse -> fine.  transpose_of_analysis = false: W
// (dual filters; crop / periodic / weighted EDAG fold); true: (W-dagger)* (analysis filters;
// crop / periodic / unweighted reflect-add fold, the adjoint of W-dagger's E_bc).
wl_status run_synthesis(const wl_plan *p, int64_t batch, const void *x, void *img, char *ws, const WsLayout &L,
                        cudaStream_t s, bool transpose_of_analysis = false) {
  const int Lp = p->fb.L - 1;
  const bool sym = p->bc == WL_BC_SYMMETRIC_EDAG || (transpose_of_analysis && p->bc == WL_BC_SYMMETRIC);
  SynthesisArgs chain[WL_MAX_LEVELS];  // coarse -> fine, launched together when no fold interleaves
  for (int j = p->J; j >= 1; j--) {
    SynthesisArgs &a = chain[p->J - j];
    a = SynthesisArgs();
    Buf ll = (j == p->J) ? band_buf(p, x, 0) : ll_buf(p, ws, L, j);
    Buf bands[4] = {ll, band_buf(p, x, lh_index(p, j)), band_buf(p, x, lh_index(p, j) + 1),
                    band_buf(p, x, lh_index(p, j) + 2)};
    for (int i = 0; i < 4; i++) {
      a.in[i] = bands[i].ptr;
      a.in_pitch[i] = bands[i].pitch;
      a.in_bstride[i] = bands[i].bstride;
    }
    a.m0 = (int)p->n0[j];
    a.m1 = (int)p->n1[j];
    a.coef_mod = p->bc == WL_BC_PERIODIC;
    a.lo = transpose_of_analysis ? p->fb.a_lo : p->fb.d_lo;
    a.hi = transpose_of_analysis ? p->fb.a_hi : p->fb.d_hi;
    a.L = p->fb.L;
    a.batch = (int)batch;
    a.out_keep = j > 1;  // LL_{j-1} is read by level j-1 right away
    int64_t n0 = p->n0[j - 1], n1 = p->n1[j - 1];
    Buf out;
    if (j == 1) {
      out.ptr = (char *)img;
      out.pitch = p->w;
      out.bstride = p->h * p->w;
    } else {
      out = ll_buf(p, ws, L, j - 1);
    }
    if (sym) {
      // synthesize onto [-L', n+L') per axis, then fold: E_sym^dagger (W of EDAG) or
      // E_sym^T ((W-dagger)* under symmetric BC).  U columns start one position earlier, at t = -L
      // (even): output column pairs then sit at even U indices and stay aligned pairs.  Split
      // output: the in-image positions go straight to the level's output, U keeps only the frame
      // outside it, and the fold touches the L'-wide border only (WL_FULL_FOLD: the whole frame
      // in U and a full-image fold pass, A/B).
      int64_t ep = round_up(n1 + 2 * Lp + 1, 16 / p->es);
      a.out = ws + L.e;
      a.out_pitch = ep;
      a.out_bstride = p->edag_elems;
      a.N0 = (int)(n0 + 2 * Lp);
      a.N1 = (int)(n1 + 2 * Lp + 1);
      a.o0 = -Lp;
      a.o1 = -Lp - 1;
      const bool split = !full_fold();
      if (split) {
        a.y = out.ptr;
        a.y_pitch = out.pitch;
        a.y_bstride = out.bstride;
        a.yn0 = (int)n0;
        a.yn1 = (int)n1;
      }
      cudaError_t e = launch_synthesis(p->dtype, a, s);
      if (e != cudaSuccess) return cuda_fail(e, "synthesis level launch");
      FoldArgs f;
      f.in = ws + L.e;
      f.in_pitch = ep;
      f.in_bstride = p->edag_elems;
      f.out = out.ptr;
      f.out_pitch = out.pitch;
      f.out_bstride = out.bstride;
      f.n0 = (int)n0;
      f.n1 = (int)n1;
      f.Lp = Lp;
      f.weighted = transpose_of_analysis ? 0 : 1;
      f.batch = (int)batch;
      f.col_off = 1;
      f.border_only = split ? 1 : 0;
      e = launch_fold(p->dtype, f, s);
      if (e != cudaSuccess) return cuda_fail(e, "fold launch");
    } else {
      a.out = out.ptr;
      a.out_pitch = out.pitch;
      a.out_bstride = out.bstride;
      a.N0 = (int)n0;
      a.N1 = (int)n1;
      a.o0 = 0;
      a.o1 = 0;
    }
  }
  if (!sym) {  // the short coarse head as one persistent launch, then the long levels
    cudaError_t e = launch_synthesis_chain(p->dtype, chain, p->J, s);
    if (e != cudaSuccess) return cuda_fail(e, "synthesis chain launch");
  }
  return WL_OK;
}

wl_status check_plan(const wl_plan *p) {
  if (!p) return fail(WL_EINVAL, "plan is NULL");
  return WL_OK;
}

wl_status check_ws(const wl_plan *p, const wl_blur_plan *bl, wl_op op, int64_t batch, void *ws) {
  size_t need = ws_layout(p, bl, op, batch).total;
  if (need == 0) return WL_OK;
  return check_dev(ws, "ws", 256);
}

wl_status check_io(const void *in, size_t in_bytes, const char *in_name, const void *out, size_t out_bytes,
                   const char *out_name) {
  wl_status st = check_dev(in, in_name);
  if (st) return st;
  st = check_dev(out, out_name);
  if (st) return st;
  if (overlap(in, in_bytes, out, out_bytes)) return fail(WL_EINVAL, "%s and %s overlap", in_name, out_name);
  return WL_OK;
}

// g = W* R* (R W x - b) into g (W chain -> fused residual -> W* chain; W-dagger chain when
// true_adjoint = false), no validation.
wl_status grad_core(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *x, const void *b, void *g,
                    double *f_dev, char *w, const WsLayout &L, cudaStream_t s, bool true_adjoint = true);

}  // namespace

// =============================================================== public API
extern "C" {

const char *wl_last_error(void) { return t_err.c_str(); }
int64_t wl_launch_count(void) { return g_launches.load(); }
const char *wl_version(void) { return "wl 0.1 (sm_100a)"; }

wl_status wl_plan_create(wl_plan **out, int64_t h, int64_t w, int levels, wl_filter filter, wl_bc bc,
                         wl_dtype dtype) {
  if (!out) return fail(WL_EINVAL, "out is NULL");
  *out = nullptr;
  if (h < 1 || w < 1) return fail(WL_ESIZE, "image size h=%lld w=%lld must be >= 1", (long long)h, (long long)w);
  if (h > (1LL << 30) || w > (1LL << 30)) return fail(WL_ESIZE, "image side > 2^30");
  if (levels < 1 || levels > WL_MAX_LEVELS)
    return fail(WL_ESIZE, "levels=%d must be in [1, %d]", levels, WL_MAX_LEVELS);
  if (bc < WL_BC_ZERO || bc > WL_BC_SYMMETRIC_EDAG) return fail(WL_EINVAL, "unknown bc %d", (int)bc);
  if (dtype != WL_F32 && dtype != WL_F64) return fail(WL_EINVAL, "unknown dtype %d", (int)dtype);
  wl_plan *p = new (std::nothrow) wl_plan();
  if (!p) return fail(WL_ENOMEM, "plan allocation failed");
  if (!build_filter_bank(filter, p->fb)) {
    delete p;
    return fail(WL_EINVAL, "unknown filter %d", (int)filter);
  }
  p->h = h; p->w = w; p->J = levels; p->filter = filter; p->bc = bc; p->dtype = dtype;
  p->es = dtype == WL_F64 ? 8 : 4;
  const int L = p->fb.L;
  const int64_t align = 16 / p->es;
  p->n0[0] = h;
  p->n1[0] = w;
  for (int j = 1; j <= levels; j++) {
    for (int ax = 0; ax < 2; ax++) {
      int64_t n = ax == 0 ? p->n0[j - 1] : p->n1[j - 1];
      const char *an = ax == 0 ? "h" : "w";
      if (bc == WL_BC_PERIODIC && (n % 2)) {
        delete p;
        return fail(WL_ESIZE, "level %d cannot be formed: periodic BC needs an even length, axis %s has %lld", j,
                    an, (long long)n);
      }
      if ((bc == WL_BC_SYMMETRIC || bc == WL_BC_SYMMETRIC_EDAG) && n < L - 1) {
        delete p;
        return fail(WL_ESIZE, "level %d cannot be formed: symmetric BC needs length >= L-1 = %d, axis %s has %lld",
                    j, L - 1, an, (long long)n);
      }
      int64_t m = bc == WL_BC_PERIODIC ? n / 2 : (n + L - 1) / 2;
      if (m < 1) {
        delete p;
        return fail(WL_ESIZE, "level %d cannot be formed: axis %s length %lld", j, an, (long long)n);
      }
      (ax == 0 ? p->n0 : p->n1)[j] = m;
    }
  }
  // subband table: LL_J, then (LH, HL, HH) for j = J..1
  int64_t off = 0, pv = 0;
  auto add = [&](int idx, int64_t rows, int64_t cols) {
    p->band[idx].offset = off;
    p->band[idx].rows = rows;
    p->band[idx].cols = cols;
    p->band[idx].pitch = round_up(cols, align);
    off += rows * p->band[idx].pitch;
    pv += rows * cols;
  };
  add(0, p->n0[levels], p->n1[levels]);
  for (int j = levels; j >= 1; j--)
    for (int k = 0; k < 3; k++) add(1 + 3 * (levels - j) + k, p->n0[j], p->n1[j]);
  p->p_alloc = off;
  p->p_valid = pv;
  // workspace: LL_1..LL_{J-1}, ping-pong by level parity
  for (int j = 1; j < levels; j++) {
    p->ll_pitch[j] = round_up(p->n1[j], align);
    int64_t e = p->n0[j] * p->ll_pitch[j];
    if (j % 2) p->ws_a_elems = std::max(p->ws_a_elems, e);
    else p->ws_b_elems = std::max(p->ws_b_elems, e);
  }
  if (bc == WL_BC_SYMMETRIC_EDAG || bc == WL_BC_SYMMETRIC)  // extended synthesis buffer (W of EDAG, (W-dagger)*)
    for (int j = 1; j <= levels; j++)
      p->edag_elems = std::max(p->edag_elems, (p->n0[j - 1] + 2 * (L - 1)) * round_up(p->n1[j - 1] + 2 * (L - 1) + 1, align));
  *out = p;
  return ok();
}

void wl_plan_destroy(wl_plan *plan) { delete plan; }

wl_status wl_plan_query(const wl_plan *p, wl_plan_info *info) {
  if (check_plan(p)) return WL_EINVAL;
  if (!info) return fail(WL_EINVAL, "info is NULL");
  memset(info, 0, sizeof *info);
  info->levels = p->J;
  info->filter_length = p->fb.L;
  info->p_valid = p->p_valid;
  info->p_alloc = p->p_alloc;
  for (int j = 0; j <= p->J; j++) {
    info->h[j] = p->n0[j];
    info->w[j] = p->n1[j];
  }
  for (int i = 0; i < 1 + 3 * p->J; i++) info->band[i] = p->band[i];
  return ok();
}

wl_status wl_plan_filters(const wl_plan *p, double *a_lo, double *a_hi, double *d_lo, double *d_hi) {
  if (check_plan(p)) return WL_EINVAL;
  size_t n = sizeof(double) * (size_t)p->fb.L;
  if (a_lo) memcpy(a_lo, p->fb.a_lo, n);
  if (a_hi) memcpy(a_hi, p->fb.a_hi, n);
  if (d_lo) memcpy(d_lo, p->fb.d_lo, n);
  if (d_hi) memcpy(d_hi, p->fb.d_hi, n);
  return ok();
}

size_t wl_workspace_bytes(const wl_plan *p, const wl_blur_plan *bl, wl_op op, int64_t batch) {
  if (!p || batch < 0) return 0;
  return ws_layout(p, bl, op, batch).total;
}

static wl_status analysis_entry(const wl_plan *p, int64_t batch, const void *img, void *x, void *ws, void *stream,
                                bool adjoint, const char *name) {
  if (check_plan(p)) return WL_EINVAL;
  if (batch < 0) return fail(WL_EINVAL, "%s: batch=%lld < 0", name, (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "%s: batch=%lld exceeds %d", name, (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * p->h * p->w * p->es, xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st = check_io(img, ib, "img", x, xb, "x");
  if (st) return st;
  if ((st = check_ws(p, nullptr, adjoint ? WL_OP_ADJOINT : WL_OP_ANALYZE, batch, ws))) return st;
  WsLayout L = ws_layout(p, nullptr, adjoint ? WL_OP_ADJOINT : WL_OP_ANALYZE, batch);
  if (L.total && (overlap(ws, L.total, img, ib) || overlap(ws, L.total, x, xb)))
    return fail(WL_EINVAL, "%s: ws overlaps img or x", name);
  st = run_analysis(p, batch, img, x, (char *)ws, L, adjoint, (cudaStream_t)stream);
  return st ? st : ok();
}

wl_status wl_adjoint(const wl_plan *p, int64_t batch, const void *img, void *x, void *ws, void *stream) {
  return analysis_entry(p, batch, img, x, ws, stream, true, "wl_adjoint");
}

wl_status wl_analyze(const wl_plan *p, int64_t batch, const void *img, void *x, void *ws, void *stream) {
  return analysis_entry(p, batch, img, x, ws, stream, false, "wl_analyze");
}

wl_status wl_synthesize(const wl_plan *p, int64_t batch, const void *x, void *img, void *ws, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (batch < 0) return fail(WL_EINVAL, "wl_synthesize: batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "wl_synthesize: batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * p->h * p->w * p->es, xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st = check_io(x, xb, "x", img, ib, "img");
  if (st) return st;
  if ((st = check_ws(p, nullptr, WL_OP_SYNTHESIZE, batch, ws))) return st;
  WsLayout L = ws_layout(p, nullptr, WL_OP_SYNTHESIZE, batch);
  if (L.total && (overlap(ws, L.total, img, ib) || overlap(ws, L.total, x, xb)))
    return fail(WL_EINVAL, "wl_synthesize: ws overlaps img or x");
  st = run_synthesis(p, batch, x, img, (char *)ws, L, (cudaStream_t)stream);
  return st ? st : ok();
}

wl_status wl_analyze_adjoint(const wl_plan *p, int64_t batch, const void *x, void *img, void *ws, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (batch < 0) return fail(WL_EINVAL, "wl_analyze_adjoint: batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "wl_analyze_adjoint: batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * p->h * p->w * p->es, xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st = check_io(x, xb, "x", img, ib, "img");
  if (st) return st;
  if ((st = check_ws(p, nullptr, WL_OP_ANALYZE_ADJOINT, batch, ws))) return st;
  WsLayout L = ws_layout(p, nullptr, WL_OP_ANALYZE_ADJOINT, batch);
  if (L.total && (overlap(ws, L.total, img, ib) || overlap(ws, L.total, x, xb)))
    return fail(WL_EINVAL, "wl_analyze_adjoint: ws overlaps img or x");
  st = run_synthesis(p, batch, x, img, (char *)ws, L, (cudaStream_t)stream, true);
  return st ? st : ok();
}

// ------------------------------------------------------------------- blur
wl_status wl_blur_create(wl_blur_plan **out, int64_t h, int64_t w, const double *taps, int ntaps, wl_bc bc,
                         wl_dtype dtype) {
  if (!out) return fail(WL_EINVAL, "out is NULL");
  *out = nullptr;
  if (!taps) return fail(WL_EINVAL, "taps_host is NULL");
  if (ntaps < 1 || ntaps > kMaxTaps || ntaps % 2 == 0)
    return fail(WL_EINVAL, "ntaps=%d must be odd and <= %d", ntaps, kMaxTaps);
  if (bc != WL_BC_SYMMETRIC) return fail(WL_EINVAL, "blur supports bc=symmetric only (got %s)", bc_name(bc));
  if (dtype != WL_F32 && dtype != WL_F64) return fail(WL_EINVAL, "unknown dtype %d", (int)dtype);
  int hw = ntaps / 2;
  if (h < 1 || w < 1 || h < hw || w < hw)
    return fail(WL_ESIZE, "blur needs h, w >= ntaps/2 = %d (got h=%lld w=%lld)", hw, (long long)h, (long long)w);
  double mx = 0;
  for (int i = 0; i < ntaps; i++) {
    if (!std::isfinite(taps[i])) return fail(WL_EINVAL, "tap %d is not finite", i);
    mx = std::fmax(mx, std::fabs(taps[i]));
  }
  for (int i = 0; i < ntaps; i++)
    if (std::fabs(taps[i] - taps[ntaps - 1 - i]) > 1e-15 * mx)
      return fail(WL_EINVAL, "taps must be symmetric (k[t] = k[-t]); tap %d differs from tap %d", i, ntaps - 1 - i);
  wl_blur_plan *b = new (std::nothrow) wl_blur_plan();
  if (!b) return fail(WL_ENOMEM, "blur plan allocation failed");
  b->h = h; b->w = w; b->dtype = dtype; b->es = dtype == WL_F64 ? 8 : 4; b->ntaps = ntaps;
  for (int i = 0; i < ntaps; i++) b->taps[i] = taps[i];
  *out = b;
  return ok();
}

wl_status wl_blur_create_gaussian(wl_blur_plan **out, int64_t h, int64_t w, int ntaps, double sigma, wl_bc bc,
                                  wl_dtype dtype) {
  if (!(sigma > 0) || !std::isfinite(sigma)) return fail(WL_EINVAL, "sigma=%g must be > 0", sigma);
  if (ntaps < 1 || ntaps > kMaxTaps || ntaps % 2 == 0)
    return fail(WL_EINVAL, "ntaps=%d must be odd and <= %d", ntaps, kMaxTaps);
  double k[kMaxTaps], sum = 0;
  int hw = ntaps / 2;
  for (int t = -hw; t <= hw; t++) sum += (k[t + hw] = std::exp(-(double)(t * t) / (2.0 * sigma * sigma)));
  for (int i = 0; i < ntaps; i++) k[i] /= sum;
  return wl_blur_create(out, h, w, k, ntaps, bc, dtype);
}

void wl_blur_destroy(wl_blur_plan *b) { delete b; }

wl_status wl_blur_taps(const wl_blur_plan *b, double *taps, int *ntaps) {
  if (!b) return fail(WL_EINVAL, "blur is NULL");
  if (ntaps) *ntaps = b->ntaps;
  if (taps) memcpy(taps, b->taps, sizeof(double) * (size_t)b->ntaps);
  return ok();
}

static wl_status blur_entry(const wl_blur_plan *bl, int64_t batch, const void *in, void *out, void *stream,
                            const char *name) {
  if (!bl) return fail(WL_EINVAL, "%s: blur plan is NULL", name);
  if (batch < 0) return fail(WL_EINVAL, "%s: batch=%lld < 0", name, (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "%s: batch=%lld exceeds %d", name, (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * bl->h * bl->w * bl->es;
  wl_status st = check_io(in, ib, "in", out, ib, "out");
  if (st) return st;
  BlurArgs a;
  a.in = in; a.b = nullptr; a.out = out; a.f = nullptr; a.h = bl->h; a.w = bl->w;
  a.ntaps = bl->ntaps; a.taps = bl->taps; a.batch = (int)batch;
  cudaError_t e = launch_blur(bl->dtype, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, name);
  return ok();
}

wl_status wl_blur(const wl_blur_plan *bl, int64_t batch, const void *in, void *out, void *stream) {
  return blur_entry(bl, batch, in, out, stream, "wl_blur");
}

wl_status wl_blur_adjoint(const wl_blur_plan *bl, int64_t batch, const void *in, void *out, void *stream) {
  // R* = E_sym^T o correlation = R for the symmetric PSFs wl_blur_create accepts (pinned by tests)
  return blur_entry(bl, batch, in, out, stream, "wl_blur_adjoint");
}

static wl_status residual_core(const wl_blur_plan *bl, int64_t batch, const void *u, const void *b, void *s,
                               double *f, cudaStream_t stream, bool f_zeroed = false) {
  BlurArgs a;
  a.in = u; a.b = b; a.out = s; a.f = f; a.h = bl->h; a.w = bl->w;
  a.ntaps = bl->ntaps; a.taps = bl->taps; a.batch = (int)batch;
  a.f_zeroed = f_zeroed ? 1 : 0;
  cudaError_t e = launch_blur_residual(bl->dtype, a, stream);
  if (e != cudaSuccess) return cuda_fail(e, "blur residual launch");
  return WL_OK;
}

}  // extern "C"

namespace {
wl_status grad_core(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *x, const void *b, void *g,
                    double *f_dev, char *w, const WsLayout &L, cudaStream_t s, bool true_adjoint) {
  wl_status st;
  if (f_dev) {  // f is accumulated by the residual kernel: zeroed here, ahead of the W chain, so no memset sits
                // between W's last level and the residual on the stream
    cudaError_t e = launch_zero(f_dev, sizeof(double) * (size_t)batch, s);
    if (e != cudaSuccess) return cuda_fail(e, "zero f");
  }
  if ((st = run_synthesis(p, batch, x, w + L.u, w, L, s))) return st;          // u = W x
  if ((st = residual_core(bl, batch, w + L.u, b, w + L.s, f_dev, s, true))) return st;  // s = R*(R u - b)
  return run_analysis(p, batch, w + L.s, g, w, L, true_adjoint, s);             // g = W* s (or W-dagger s)
}
}  // namespace

extern "C" {

wl_status wl_blur_residual_adjoint(const wl_blur_plan *bl, int64_t batch, const void *u, const void *b, void *s,
                                   double *f_dev, void *stream) {
  if (!bl) return fail(WL_EINVAL, "blur plan is NULL");
  if (batch < 0) return fail(WL_EINVAL, "batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * bl->h * bl->w * bl->es;
  wl_status st = check_io(u, ib, "u", s, ib, "s");
  if (st) return st;
  if ((st = check_dev(b, "b"))) return st;
  if (overlap(b, ib, s, ib)) return fail(WL_EINVAL, "b and s overlap");
  if (f_dev && (st = check_dev(f_dev, "f_dev", 8))) return st;
  st = residual_core(bl, batch, u, b, s, f_dev, (cudaStream_t)stream);
  return st ? st : ok();
}

wl_status wl_grad(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *x, const void *b, void *g,
                  double *f_dev, void *ws, void *stream) {
  return wl_grad_adj(p, bl, batch, x, b, g, f_dev, WL_ADJ_TRUE, ws, stream);
}

wl_status wl_grad_adj(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *x, const void *b, void *g,
                      double *f_dev, wl_adj adj, void *ws, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (adj != WL_ADJ_TRUE && adj != WL_ADJ_PINV) return fail(WL_EINVAL, "wl_grad: adj=%d is not a wl_adj", (int)adj);
  if (!bl) return fail(WL_EINVAL, "wl_grad: blur plan is NULL");
  if (bl->h != p->h || bl->w != p->w)
    return fail(WL_EINVAL, "wl_grad: blur plan is %lldx%lld but wavelet plan is %lldx%lld", (long long)bl->h,
                (long long)bl->w, (long long)p->h, (long long)p->w);
  if (bl->dtype != p->dtype) return fail(WL_EDTYPE, "wl_grad: blur and wavelet plans have different dtypes");
  if (batch < 0) return fail(WL_EINVAL, "wl_grad: batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "wl_grad: batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  size_t ib = (size_t)batch * p->h * p->w * p->es, xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st = check_io(x, xb, "x", g, xb, "g");
  if (st) return st;
  if ((st = check_dev(b, "b"))) return st;
  if (overlap(b, ib, g, xb)) return fail(WL_EINVAL, "wl_grad: b and g overlap");
  if (f_dev && (st = check_dev(f_dev, "f_dev", 8))) return st;
  if ((st = check_ws(p, bl, WL_OP_GRAD, batch, ws))) return st;
  WsLayout L = ws_layout(p, bl, WL_OP_GRAD, batch);
  if (overlap(ws, L.total, x, xb) || overlap(ws, L.total, g, xb) || overlap(ws, L.total, b, ib))
    return fail(WL_EINVAL, "wl_grad: ws overlaps an argument");
  st = grad_core(p, bl, batch, x, b, g, f_dev, (char *)ws, L, (cudaStream_t)stream, adj == WL_ADJ_TRUE);
  return st ? st : ok();
}

wl_status wl_grad_host(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *x_host,
                       const void *b_host, void *g_host, double *f_host, void *ws, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (!bl) return fail(WL_EINVAL, "wl_grad_host: blur plan is NULL");
  if (bl->h != p->h || bl->w != p->w || bl->dtype != p->dtype)
    return fail(WL_EINVAL, "wl_grad_host: blur plan does not match the wavelet plan");
  if (batch < 0) return fail(WL_EINVAL, "wl_grad_host: batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "wl_grad_host: batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (batch == 0) return ok();
  if (!x_host || !b_host || !g_host) return fail(WL_EINVAL, "wl_grad_host: x_host, b_host and g_host must be non-NULL");
  wl_status st;
  if ((st = check_ws(p, bl, WL_OP_GRAD_HOST, batch, ws))) return st;
  const WsLayout L = ws_layout(p, bl, WL_OP_GRAD_HOST, batch);
  const size_t es = (size_t)p->es, xs = (size_t)p->p_alloc * es, is = (size_t)p->h * p->w * es;
  cudaStream_t s = (cudaStream_t)stream;
  // copy streams and events: created once per (thread, device) and reused by every call
  struct HostPipe {
    int dev = -1;
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t ev[7] = {};  // start, in[2], done[2], free[2]
  };
  thread_local HostPipe pipes[8];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "wl_grad_host device");
  HostPipe *hp = nullptr;
  for (auto &q : pipes)
    if (q.dev == dev || q.dev < 0) {
      hp = &q;
      break;
    }
  if (!hp) return fail(WL_EINVAL, "wl_grad_host: more than 8 devices used from one thread");
  if (hp->dev < 0) {
    e = cudaStreamCreateWithFlags(&hp->cin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&hp->cout, cudaStreamNonBlocking);
    for (int i = 0; i < 7 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&hp->ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "wl_grad_host stream setup");
    hp->dev = dev;
  }
  cudaStream_t cin = hp->cin, cout = hp->cout;
  cudaEvent_t *ev = hp->ev;
  char *w = (char *)ws;
  e = cudaEventRecord(ev[0], s);  // the call is ordered after prior work on `stream`
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cin, ev[0], 0);
  for (int64_t i = 0; i < batch && e == cudaSuccess && !st; i++) {
    const int k = (int)(i & 1);
    char *dx = w + L.hx + k * xs, *db = w + L.hb + k * is, *dg = w + L.hg + k * xs;
    double *df = reinterpret_cast<double *>(w + L.hf) + k;
    if (i >= 2) e = cudaStreamWaitEvent(cin, ev[5 + k], 0);  // slot k copied out (image i-2)
    if (e == cudaSuccess) e = cudaMemcpyAsync(dx, (const char *)x_host + i * xs, xs, cudaMemcpyHostToDevice, cin);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, (const char *)b_host + i * is, is, cudaMemcpyHostToDevice, cin);
    if (e == cudaSuccess) e = cudaEventRecord(ev[1 + k], cin);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[1 + k], 0);
    if (e != cudaSuccess) break;
    st = grad_core(p, bl, 1, dx, db, dg, f_host ? df : nullptr, w, L, s);
    if (st) break;
    e = cudaEventRecord(ev[3 + k], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cout, ev[3 + k], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char *)g_host + i * xs, dg, xs, cudaMemcpyDeviceToHost, cout);
    if (e == cudaSuccess && f_host) e = cudaMemcpyAsync(f_host + i, df, sizeof(double), cudaMemcpyDeviceToHost, cout);
    if (e == cudaSuccess) e = cudaEventRecord(ev[5 + k], cout);
  }
  // `stream` resumes after every copy this call queued, on success and on failure alike, so the
  // caller never reuses ws or the host buffers while a copy is in flight
  cudaError_t e2 = cudaEventRecord(ev[0], cout);
  if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(s, ev[0], 0);
  if (e2 == cudaSuccess) e2 = cudaEventRecord(ev[0], cin);
  if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(s, ev[0], 0);
  if (e2 != cudaSuccess) {
    cudaStreamSynchronize(cin);
    cudaStreamSynchronize(cout);
  }
  if (st) return st;
  if (e != cudaSuccess) return cuda_fail(e, "wl_grad_host pipeline");
  if (e2 != cudaSuccess) return cuda_fail(e2, "wl_grad_host pipeline");
  return ok();
}

wl_status wl_fista_update(const wl_plan *p, int64_t batch, const void *g, void *x, void *y, double t, double lambda,
                          double lip, double *t_next_host, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (batch < 0) return fail(WL_EINVAL, "wl_fista_update: batch=%lld < 0", (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "wl_fista_update: batch=%lld exceeds %d", (long long)batch, kMaxBatch);
  if (!(lip > 0) || !std::isfinite(lip)) return fail(WL_EINVAL, "wl_fista_update: lip=%g must be > 0", lip);
  if (!(lambda >= 0) || !std::isfinite(lambda)) return fail(WL_EINVAL, "wl_fista_update: lambda=%g must be >= 0", lambda);
  if (!(t >= 1) || !std::isfinite(t)) return fail(WL_EINVAL, "wl_fista_update: t=%g must be >= 1", t);
  if (t_next_host) *t_next_host = fista_next_t(t);
  if (batch == 0) return ok();
  const size_t xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st;
  if ((st = check_dev(g, "g")) || (st = check_dev(x, "x")) || (st = check_dev(y, "y"))) return st;
  if (overlap(g, xb, x, xb) || overlap(g, xb, y, xb) || overlap(x, xb, y, xb))
    return fail(WL_EINVAL, "wl_fista_update: g, x and y must not overlap");
  cudaError_t e = launch_fista_update(p->dtype, g, x, y, (long long)batch * p->p_alloc, t, lambda, lip,
                                      (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fista update launch");
  return ok();
}

static wl_status fista_step_core(const char *fn, const wl_plan *p, const wl_blur_plan *bl, int64_t batch,
                                 const void *b, void *x, void *y, double t, double *t_dev, double lambda, double lip,
                                 double *f_dev, wl_adj adj, void *ws, double *t_next_host, void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (adj != WL_ADJ_TRUE && adj != WL_ADJ_PINV) return fail(WL_EINVAL, "%s: adj=%d is not a wl_adj", fn, (int)adj);
  if (!bl) return fail(WL_EINVAL, "%s: blur plan is NULL", fn);
  if (bl->h != p->h || bl->w != p->w || bl->dtype != p->dtype)
    return fail(WL_EINVAL, "%s: blur plan does not match the wavelet plan", fn);
  if (batch < 0) return fail(WL_EINVAL, "%s: batch=%lld < 0", fn, (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "%s: batch=%lld exceeds %d", fn, (long long)batch, kMaxBatch);
  if (!(lip > 0) || !(lambda >= 0) || !(t_dev || t >= 1))
    return fail(WL_EINVAL, "%s: need lip > 0, lambda >= 0, t >= 1", fn);
  if (!t_dev && t_next_host) *t_next_host = fista_next_t(t);
  if (batch == 0) return ok();
  const size_t ib = (size_t)batch * p->h * p->w * p->es, xb = (size_t)batch * p->p_alloc * p->es;
  wl_status st;
  if ((st = check_dev(b, "b")) || (st = check_dev(x, "x")) || (st = check_dev(y, "y"))) return st;
  if (t_dev && (st = check_dev(t_dev, "t_dev", 8))) return st;
  if (overlap(x, xb, y, xb) || overlap(b, ib, x, xb) || overlap(b, ib, y, xb))
    return fail(WL_EINVAL, "%s: b, x and y must not overlap", fn);
  if (f_dev && (st = check_dev(f_dev, "f_dev", 8))) return st;
  if ((st = check_ws(p, bl, WL_OP_FISTA, batch, ws))) return st;
  WsLayout L = ws_layout(p, bl, WL_OP_FISTA, batch);
  if (overlap(ws, L.total, x, xb) || overlap(ws, L.total, y, xb) || overlap(ws, L.total, b, ib))
    return fail(WL_EINVAL, "%s: ws overlaps an argument", fn);
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  // g = grad f(y) = W* R* (R W y - b), with the prox + momentum update fused into W*'s stores
  // (g never reaches HBM).  W reads y before the W* chain rewrites it (stream order).
  if ((st = run_synthesis(p, batch, y, w + L.u, w, L, s))) return st;
  if ((st = residual_core(bl, batch, w + L.u, b, w + L.s, f_dev, s))) return st;
  const double t_new = fista_next_t(t);
  const FistaFuse fz{x, 1.0 / lip, lambda / lip, t_dev ? 0.0 : (t - 1.0) / t_new, t_dev};
  if ((st = run_analysis(p, batch, w + L.s, y, w, L, adj == WL_ADJ_TRUE, s, &fz))) return st;
  if (t_dev) {
    cudaError_t e = launch_fista_advance_t(t_dev, s);
    if (e != cudaSuccess) return cuda_fail(e, "fista t update");
  }
  return ok();
}

wl_status wl_fista_step(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *b, void *x, void *y,
                        double t, double lambda, double lip, double *f_dev, wl_adj adj, void *ws, double *t_next_host,
                        void *stream) {
  return fista_step_core("wl_fista_step", p, bl, batch, b, x, y, t, nullptr, lambda, lip, f_dev, adj, ws, t_next_host,
                         stream);
}

wl_status wl_fista_step_dev(const wl_plan *p, const wl_blur_plan *bl, int64_t batch, const void *b, void *x, void *y,
                            double *t_dev, double lambda, double lip, double *f_dev, wl_adj adj, void *ws,
                            void *stream) {
  if (!t_dev) return fail(WL_EINVAL, "wl_fista_step_dev: t_dev is NULL");
  return fista_step_core("wl_fista_step_dev", p, bl, batch, b, x, y, 1.0, t_dev, lambda, lip, f_dev, adj, ws, nullptr,
                         stream);
}

wl_status wl_lipschitz(const wl_plan *p, const wl_blur_plan *bl, int iters, uint64_t seed, double *lip_host, void *ws,
                       void *stream) {
  if (check_plan(p)) return WL_EINVAL;
  if (!bl) return fail(WL_EINVAL, "wl_lipschitz: blur plan is NULL");
  if (bl->h != p->h || bl->w != p->w || bl->dtype != p->dtype)
    return fail(WL_EINVAL, "wl_lipschitz: blur plan does not match the wavelet plan");
  if (iters < 1) return fail(WL_EINVAL, "wl_lipschitz: iters=%d must be >= 1", iters);
  if (!lip_host) return fail(WL_EINVAL, "wl_lipschitz: lip_host is NULL");
  wl_status st;
  if ((st = check_ws(p, bl, WL_OP_LIPSCHITZ, 1, ws))) return st;
  WsLayout L = ws_layout(p, bl, WL_OP_LIPSCHITZ, 1);
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  void *v = w + L.v, *g = w + L.g, *b0 = w + L.b0;
  double *d = reinterpret_cast<double *>(w + L.d);
  const long long n = p->p_alloc;
  cudaError_t e = cudaMemsetAsync(b0, 0, (size_t)p->h * p->w * p->es, s);
  if (e == cudaSuccess) e = launch_fill_seeded(p->dtype, v, n, (unsigned long long)seed, s);
  if (e != cudaSuccess) return cuda_fail(e, "wl_lipschitz init");
  double est = 0.0;
  for (int it = 0; it < iters; it++) {
    double h[2];
    e = launch_dot(p->dtype, v, v, n, 1, d, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "wl_lipschitz norm");
    if (!(h[0] > 0)) {  // zero operator
      *lip_host = 0.0;
      return ok();
    }
    e = launch_scale(p->dtype, v, n, 1.0 / std::sqrt(h[0]), s);
    if (e != cudaSuccess) return cuda_fail(e, "wl_lipschitz scale");
    if ((st = grad_core(p, bl, 1, v, b0, g, nullptr, w, L, s))) return st;  // g = W* R* R W v
    e = launch_dot(p->dtype, v, g, n, 1, d + 1, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h + 1, d + 1, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "wl_lipschitz rayleigh");
    est = h[1];  // <v, G v> with ||v|| = 1
    e = cudaMemcpyAsync(v, g, (size_t)n * p->es, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "wl_lipschitz copy");
  }
  *lip_host = est;
  return ok();
}

// ------------------------------------------------------------- Example 2
static wl_status bce_sizes(const char *fn, wl_dtype dtype, int64_t batch, int64_t K, int64_t N) {
  if (dtype != WL_F32 && dtype != WL_F64) return fail(WL_EDTYPE, "%s: dtype=%d", fn, (int)dtype);
  if (batch < 0) return fail(WL_EINVAL, "%s: batch=%lld < 0", fn, (long long)batch);
  if (batch > kMaxBatch) return fail(WL_ESIZE, "%s: batch=%lld exceeds %d", fn, (long long)batch, kMaxBatch);
  if (K < 1 || N < 1) return fail(WL_ESIZE, "%s: K=%lld and N=%lld must be >= 1", fn, (long long)K, (long long)N);
  if (K + N > (int64_t)1 << 24) return fail(WL_ESIZE, "%s: K+N=%lld too long", fn, (long long)(K + N));
  return WL_OK;
}

static wl_status xcorr_call(const char *fn, wl_dtype dtype, int64_t batch, const void *a, int64_t a_len, int a_rev,
                            const void *b, int64_t b_len, int64_t b_off, void *out, int64_t n_out, void *stream) {
  const size_t es = dtype == WL_F64 ? 8 : 4;
  const size_t smem = xcorr_smem_bytes(dtype, (int)a_len, (int)n_out);
  if (smem > kMaxSmemOptin)
    return fail(WL_ESIZE, "%s: operands need %zu bytes of shared memory (max %zu)", fn, smem, kMaxSmemOptin);
  wl_status st;
  if ((st = check_dev(a, "a", es)) || (st = check_dev(b, "b", es)) || (st = check_dev(out, "out", es))) return st;
  const size_t ob = (size_t)batch * n_out * es;
  if (overlap(a, (size_t)batch * a_len * es, out, ob) || overlap(b, (size_t)batch * b_len * es, out, ob))
    return fail(WL_EINVAL, "%s: out overlaps an input", fn);
  XcorrArgs x;
  x.a = a;
  x.a_bstride = a_len;
  x.ta = (int)a_len;
  x.a_rev = a_rev;
  x.b = b;
  x.b_bstride = b_len;
  x.lb = (int)b_len;
  x.b_off = (int)b_off;
  x.out = out;
  x.out_bstride = n_out;
  x.n_out = (int)n_out;
  x.batch = batch;
  cudaError_t e = launch_xcorr(dtype, x, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, fn);
  return ok();
}

wl_status wl_conv_full(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *h, const void *s, void *x,
                       void *stream) {
  wl_status st = bce_sizes("wl_conv_full", dtype, batch, K, N);
  if (st) return st;
  if (batch == 0) return ok();
  // x[m] = sum_k h[k] s[m-k] = sum_j h[K-1-j] s_pad[m+j], s_pad = s shifted by K-1
  return xcorr_call("wl_conv_full", dtype, batch, h, K, 1, s, N, K - 1, x, K + N - 1, stream);
}

wl_status wl_conv_adjoint_h(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *s, const void *r,
                            void *gh, void *stream) {
  wl_status st = bce_sizes("wl_conv_adjoint_h", dtype, batch, K, N);
  if (st) return st;
  if (batch == 0) return ok();
  return xcorr_call("wl_conv_adjoint_h", dtype, batch, s, N, 0, r, K + N - 1, 0, gh, K, stream);
}

wl_status wl_conv_adjoint_s(wl_dtype dtype, int64_t batch, int64_t K, int64_t N, const void *h, const void *r,
                            void *gs, void *stream) {
  wl_status st = bce_sizes("wl_conv_adjoint_s", dtype, batch, K, N);
  if (st) return st;
  if (batch == 0) return ok();
  return xcorr_call("wl_conv_adjoint_s", dtype, batch, h, K, 0, r, K + N - 1, 0, gs, N, stream);
}

wl_status wl_bce_grad(wl_dtype dtype, int64_t problems, int channels, int64_t K, int64_t N, const void *h,
                      const void *s, const void *x, int x_shared, double lam_tv, double delta, void *gh, void *gs,
                      double *f_dev, void *stream) {
  wl_status st = bce_sizes("wl_bce_grad", dtype, problems, K, N);
  if (st) return st;
  if (channels < 1 || channels > 64) return fail(WL_EINVAL, "wl_bce_grad: channels=%d not in [1, 64]", channels);
  if (!(delta > 0) || !std::isfinite(delta)) return fail(WL_EINVAL, "wl_bce_grad: delta=%g must be > 0", delta);
  if (!(lam_tv >= 0) || !std::isfinite(lam_tv)) return fail(WL_EINVAL, "wl_bce_grad: lam_tv=%g must be >= 0", lam_tv);
  if (problems == 0) return ok();
  BceArgs a;
  a.h = h;
  a.s = s;
  a.x = x;
  a.x_shared = x_shared ? 1 : 0;
  a.gh = gh;
  a.gs = gs;
  a.f = f_dev;
  a.C = channels;
  a.K = (int)K;
  a.N = (int)N;
  a.problems = problems;
  a.lam_tv = lam_tv;
  a.delta = delta;
  const size_t es = dtype == WL_F64 ? 8 : 4;
  const size_t smem = bce_smem_bytes(dtype, a);
  if (smem > kMaxSmemOptin)
    return fail(WL_ESIZE, "wl_bce_grad: C=%d K=%lld N=%lld need %zu bytes of shared memory (max %zu)", channels,
                (long long)K, (long long)N, smem, kMaxSmemOptin);
  if ((st = check_dev(h, "h", es)) || (st = check_dev(s, "s", es)) || (st = check_dev(x, "x", es)) ||
      (st = check_dev(gh, "gh", es)) || (st = check_dev(gs, "gs", es)))
    return st;
  if (f_dev && (st = check_dev(f_dev, "f_dev", 8))) return st;
  const size_t hb = (size_t)problems * channels * K * es, sb = (size_t)problems * N * es;
  const size_t xb = (size_t)(x_shared ? 1 : problems) * channels * (K + N - 1) * es;
  const void *ins[3] = {h, s, x};
  const size_t inb[3] = {hb, sb, xb};
  for (int i = 0; i < 3; i++)
    if (overlap(ins[i], inb[i], gh, hb) || overlap(ins[i], inb[i], gs, sb))
      return fail(WL_EINVAL, "wl_bce_grad: an output overlaps an input");
  if (overlap(gh, hb, gs, sb)) return fail(WL_EINVAL, "wl_bce_grad: gh and gs overlap");
  cudaError_t e = launch_bce_grad(dtype, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "wl_bce_grad launch");
  return ok();
}

}  // extern "C"
