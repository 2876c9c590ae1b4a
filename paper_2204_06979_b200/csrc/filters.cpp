// Host-side Daubechies filter derivation and DWT plan for libhyde.
//
// The wavelet is SPEC.md:179 D4 (Haar, db4 = 8 taps, db8 = 16 taps; default
// db8).  Filters are derived here, independently of oracle/, by spectral
// factorisation in long double: |H(w)|^2 = 2 cos^{2N}(w/2) P(sin^2(w/2)),
// P(y) = sum_{k<N} C(N-1+k, k) y^k; roots of P by Durand-Kerner, each mapped
// to the root z of z^2 - 2(1-2y) z + 1 = 0 inside the unit circle (minimum
// phase); H(z) ~ (1+z)^N prod (z - z_i); sum h = sqrt(2).  The high-pass is
// g_k = (-1)^k h_{T-1-k}.
#include <cmath>
#include <complex>
#include <mutex>
#include <vector>

#include "common.cuh"

typedef long double ld;
typedef std::complex<ld> cld;

static std::vector<cld> poly_roots(const std::vector<ld>& c_high_first) {
  // monic normalisation
  int deg = (int)c_high_first.size() - 1;
  std::vector<cld> a(deg + 1);
  for (int i = 0; i <= deg; ++i) a[i] = c_high_first[i] / c_high_first[0];
  std::vector<cld> z(deg);
  cld seed(0.4L, 0.9L), p(1.0L, 0.0L);
  for (int i = 0; i < deg; ++i) { z[i] = p; p *= seed; }
  for (int it = 0; it < 2000; ++it) {
    ld delta = 0;
    for (int i = 0; i < deg; ++i) {
      cld num = a[0];
      for (int k = 1; k <= deg; ++k) num = num * z[i] + a[k];
      cld den(1.0L, 0.0L);
      for (int j = 0; j < deg; ++j)
        if (j != i) den *= (z[i] - z[j]);
      cld step = num / den;
      z[i] -= step;
      delta = std::max(delta, (ld)std::abs(step));
    }
    if (delta < 1e-30L) break;
  }
  return z;
}

static int daubechies(int nmom, std::vector<ld>& h) {
  if (nmom < 1) return -1;
  if (nmom == 1) {
    h.assign(2, 1.0L / std::sqrt(2.0L));
    return 0;
  }
  const int N = nmom;
  std::vector<ld> c(N);  // highest degree first: C(N-1+k, k), k = N-1..0
  for (int k = N - 1; k >= 0; --k) {
    ld b = 1;
    for (int i = 1; i <= k; ++i) b = b * (N - 1 + i) / i;
    c[N - 1 - k] = b;
  }
  std::vector<cld> yr = poly_roots(c);
  std::vector<cld> poly(1, cld(1.0L, 0.0L));  // highest power first
  auto mul = [&](cld r0, cld r1) {          // poly *= (r0 z + r1)
    std::vector<cld> out(poly.size() + 1, cld(0, 0));
    for (size_t i = 0; i < poly.size(); ++i) {
      out[i] += poly[i] * r0;
      out[i + 1] += poly[i] * r1;
    }
    poly.swap(out);
  };
  for (int i = 0; i < N; ++i) mul(cld(1, 0), cld(1, 0));
  for (const cld& y : yr) {
    cld cc = cld(1, 0) - cld(2, 0) * y;
    cld s = std::sqrt(cc * cc - cld(1, 0));
    cld z1 = cc + s, z2 = cc - s;
    cld zi = std::abs(z1) < 1 ? z1 : z2;
    mul(cld(1, 0), -zi);
  }
  ld tot = 0;
  for (auto& v : poly) tot += v.real();
  h.resize(poly.size());
  for (size_t i = 0; i < poly.size(); ++i) h[i] = poly[i].real() * std::sqrt(2.0L) / tot;
  return 0;
}

// The derivation (Durand-Kerner in long double) costs ~1 ms of host time, so
// each filter is derived once per process and cached; every hyres call used to
// pay it on the critical path before its first launch.
static const std::vector<ld>* cached_filter(int taps) {
  static std::once_flag once[3];
  static std::vector<ld> h[3];
  static int ok[3];
  const int i = taps == 2 ? 0 : taps == 8 ? 1 : 2;
  std::call_once(once[i], [&] { ok[i] = daubechies(taps / 2, h[i]) == 0 && (int)h[i].size() == taps; });
  return ok[i] ? &h[i] : nullptr;
}

int hyde_build_filters(int taps, FilterBank* fb, double* h64) {
  if (taps != 2 && taps != 8 && taps != 16) return -1;
  const std::vector<ld>* hp = cached_filter(taps);
  if (!hp) return -1;
  const std::vector<ld>& h = *hp;
  if (fb) {
    fb->taps = taps;
    for (int k = 0; k < HYDE_MAX_TAPS; ++k) {
      fb->h[k] = k < taps ? (float)h[k] : 0.f;
      ld gk = k < taps ? ((k & 1) ? -h[taps - 1 - k] : h[taps - 1 - k]) : 0;
      fb->g[k] = (float)gk;
      fb->hg[k].x = fb->h[k];
      fb->hg[k].y = fb->g[k];
    }
  }
  if (h64)
    for (int k = 0; k < taps; ++k) h64[k] = (double)h[k];
  return 0;
}

void hyde_make_plan(int rows, int cols, int levels, DwtPlan* p) {
  p->levels = levels;
  p->rows = rows;
  p->cols = cols;
  int h = rows, w = cols;
  long long off = 0;
  for (int l = 0; l < levels; ++l) {
    p->lv[l].h_in = h;
    p->lv[l].w_in = w;
    p->lv[l].hs = (h + 1) / 2;
    p->lv[l].ws = (w + 1) / 2;
    p->sub_off[l] = off;
    off += 3LL * p->lv[l].hs * p->lv[l].ws;
    h = p->lv[l].hs;
    w = p->lv[l].ws;
  }
  p->ll_off = off;
  p->n_coeffs = off + (long long)h * w;
}

extern "C" hyde_status hyde_filter(int taps, double* h_out) {
  if (!h_out) return HYDE_EPARAM;
  return hyde_build_filters(taps, nullptr, h_out) == 0 ? HYDE_OK : HYDE_EPARAM;
}

extern "C" int hyde_dwt_coeff_count(int rows, int cols, int levels) {
  if (rows < 1 || cols < 1 || levels < 1 || levels > HYDE_MAX_LEVELS) return -1;
  DwtPlan p;
  hyde_make_plan(rows, cols, levels, &p);
  return (int)p.n_coeffs;
}

extern "C" int hyde_auto_levels(int rows, int cols, int taps) {
  // largest L with (taps-1) 2^L <= min(R, C), clamped to [1, 5]
  long long m = rows < cols ? rows : cols;
  long long t = taps > 1 ? taps - 1 : 1;
  int lv = 0;
  while (lv < 5 && (t << (lv + 1)) <= m) ++lv;
  if (lv < 1) lv = 1;
  return lv;
}
