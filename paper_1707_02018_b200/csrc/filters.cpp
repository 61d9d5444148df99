// Filter-bank construction for the product library (host, fp64 / long double).
//
// Independent of oracle/ (which uses numpy companion-matrix roots and complex
// polynomial products): here the roots of P_N come from a Durand-Kerner iteration
// polished by Newton steps in long double, and the CDF 9/7 cubic is solved with
// Cardano's formula and real quadratic factors.
//
// Families: P:101-102 ("Haar and more generally Daubechies wavelets")
// ("CDF 9/7"); taps are not printed in the paper.  Array conventions (DESIGN.md
// readings R3-R5): common frame of L taps, analysis out[k] = sum_j f[j] yhat[2k+1-j],
// a_lo = d_lo = reverse(h) for Daubechies; CDF 9/7: a_lo = [0, h9], d_lo = [0,0,h7,0];
// a_hi[j] = (-1)^(j+1) d_lo[L-1-j], d_hi[j] = (-1)^(j+1) a_lo[L-1-j].
#include <cmath>
#include <complex>
#include <vector>

#include "wl_internal.h"

namespace wl {
namespace {

using cld = std::complex<long double>;

// Horner evaluation of sum_k c[k] y^k.
template <typename V>
V horner(const std::vector<long double> &c, V y) {
  V acc = V(0);
  for (int k = (int)c.size() - 1; k >= 0; k--) acc = acc * y + V(c[(size_t)k]);
  return acc;
}

// All roots of sum_k c[k] y^k (degree c.size()-1) by Durand-Kerner + Newton polish.
std::vector<cld> poly_roots(const std::vector<long double> &c) {
  int deg = (int)c.size() - 1;
  std::vector<cld> z((size_t)deg);
  if (deg <= 0) return z;
  std::vector<long double> mon(c.size());
  for (size_t k = 0; k < c.size(); k++) mon[k] = c[k] / c[(size_t)deg];
  cld seed(0.4L, 0.9L), s(1.0L, 0.0L);
  for (int i = 0; i < deg; i++) { s *= seed; z[(size_t)i] = s; }
  for (int it = 0; it < 2000; it++) {
    long double delta = 0;
    for (int i = 0; i < deg; i++) {
      cld den(1.0L, 0.0L);
      for (int j = 0; j < deg; j++)
        if (j != i) den *= (z[(size_t)i] - z[(size_t)j]);
      cld step = horner(mon, z[(size_t)i]) / den;
      z[(size_t)i] -= step;
      delta = std::max(delta, std::abs(step));
    }
    if (delta < 1e-30L) break;
  }
  // Newton polish on the original polynomial
  std::vector<long double> der;
  for (size_t k = 1; k < c.size(); k++) der.push_back(c[k] * (long double)k);
  for (auto &r : z)
    for (int it = 0; it < 8; it++) {
      cld d = horner(der, r);
      if (std::abs(d) == 0) break;
      r -= horner(c, r) / d;
    }
  return z;
}

// Multiply polynomial a (in z^-1) by (1 - r z^-1).
void mul_linear(std::vector<cld> &a, cld r) {
  a.push_back(cld(0));
  for (size_t k = a.size() - 1; k > 0; k--) a[k] -= r * a[k - 1];
}

// Minimum-phase Daubechies lowpass, length 2N, sum sqrt(2).
std::vector<long double> daubechies(int N) {
  std::vector<long double> P((size_t)N);
  for (int k = 0; k < N; k++) {  // binomial C(N-1+k, k)
    long double b = 1;
    for (int i = 1; i <= k; i++) b = b * (long double)(N - 1 + i) / (long double)i;
    P[(size_t)k] = b;
  }
  std::vector<cld> h{cld(1)};
  for (int i = 0; i < N; i++) mul_linear(h, cld(-1.0L));  // (1 + z^-1)^N
  for (cld yr : poly_roots(P)) {
    // y = (2 - z - 1/z)/4  ->  z^2 - (2 - 4 y_r) z + 1 = 0 ; keep the root inside |z| < 1
    cld bq = 2.0L - 4.0L * yr;
    cld disc = std::sqrt(bq * bq - 4.0L);
    cld z1 = (bq + disc) / 2.0L, z2 = (bq - disc) / 2.0L;
    mul_linear(h, std::abs(z1) < 1.0L ? z1 : z2);
  }
  std::vector<long double> out(h.size());
  long double s = 0;
  for (size_t i = 0; i < h.size(); i++) { out[i] = h[i].real(); s += out[i]; }
  for (auto &v : out) v *= std::sqrt(2.0L) / s;
  return out;
}

// Symmetric polynomial products in u = z + 1/z represented by centred coefficient arrays.
std::vector<long double> conv(const std::vector<long double> &a, const std::vector<long double> &b) {
  std::vector<long double> c(a.size() + b.size() - 1, 0.0L);
  for (size_t i = 0; i < a.size(); i++)
    for (size_t j = 0; j < b.size(); j++) c[i + j] += a[i] * b[j];
  return c;
}

void cdf97(std::vector<long double> &h9, std::vector<long double> &h7) {
  // 20 y^3 + 10 y^2 + 4 y + 1 = 0  ->  y^3 + a y^2 + b y + c with a = 1/2, b = 1/5, c = 1/20
  const long double a = 0.5L, b = 0.2L, c = 0.05L;
  long double p = b - a * a / 3.0L, q = 2.0L * a * a * a / 27.0L - a * b / 3.0L + c;
  long double D = q * q / 4.0L + p * p * p / 27.0L;  // > 0: one real root
  long double sD = std::sqrt(D);
  long double yr = std::cbrt(-q / 2.0L + sD) + std::cbrt(-q / 2.0L - sD) - a / 3.0L;
  // y^3 + a y^2 + b y + c = (y - yr)(y^2 + s1 y + p1)
  long double s1 = a + yr, p1 = b + yr * (a + yr);
  // y = (2 - z - 1/z)/4 as the centred array [-1/4, 1/2, -1/4]; cos^2(w/2) = [1/4, 1/2, 1/4]
  std::vector<long double> Y{-0.25L, 0.5L, -0.25L}, C2{0.25L, 0.5L, 0.25L};
  std::vector<long double> C4 = conv(C2, C2);
  // h7 ∝ cos^4 * (y - yr)
  std::vector<long double> lin{-0.25L, 0.5L - yr, -0.25L};
  h7 = conv(C4, lin);
  // h9 ∝ cos^4 * (y^2 + s1 y + p1)
  std::vector<long double> Y2 = conv(Y, Y);  // 5 taps
  std::vector<long double> quad(5, 0.0L);
  for (int i = 0; i < 5; i++) quad[(size_t)i] = Y2[(size_t)i];
  for (int i = 0; i < 3; i++) quad[(size_t)i + 1] += s1 * Y[(size_t)i];
  quad[2] += p1;
  h9 = conv(C4, quad);
  for (auto *f : {&h7, &h9}) {
    long double s = 0;
    for (auto v : *f) s += v;
    for (auto &v : *f) v *= std::sqrt(2.0L) / s;
  }
}

}  // namespace

bool build_filter_bank(int filter, FilterBank &fb) {
  std::vector<long double> alo, dlo;
  int L;
  if (filter == WL_HAAR || filter == WL_DB2 || filter == WL_DB4 || filter == WL_DB8) {
    int N = filter == WL_HAAR ? 1 : filter;
    std::vector<long double> h = N == 1 ? std::vector<long double>{1.0L / std::sqrt(2.0L), 1.0L / std::sqrt(2.0L)}
                                        : daubechies(N);
    L = 2 * N;
    alo.assign(h.rbegin(), h.rend());
    dlo = alo;
  } else if (filter == WL_CDF97) {
    std::vector<long double> h9, h7;
    cdf97(h9, h7);
    L = 10;
    alo.assign(10, 0.0L);
    dlo.assign(10, 0.0L);
    for (int i = 0; i < 9; i++) alo[(size_t)i + 1] = h9[(size_t)i];
    for (int i = 0; i < 7; i++) dlo[(size_t)i + 2] = h7[(size_t)i];
  } else {
    return false;
  }
  fb.L = L;
  for (int j = 0; j < L; j++) {
    long double sgn = (j % 2 == 0) ? -1.0L : 1.0L;  // (-1)^(j+1)
    fb.a_lo[j] = (double)alo[(size_t)j];
    fb.d_lo[j] = (double)dlo[(size_t)j];
    fb.a_hi[j] = (double)(sgn * dlo[(size_t)(L - 1 - j)]);
    fb.d_hi[j] = (double)(sgn * alo[(size_t)(L - 1 - j)]);
  }
  return true;
}

}  // namespace wl
