// K2 (SURVEY.md §8(a) A1 tail + A2; north_star stages (1)-(2)): per-band
// noise, whitening, eigendecomposition of the whitened Gram -- one CTA.
//
//  (1) sigma_b^2 = 1/(N M_bb), M = (G + ridge I)^-1 (HySime's
//      regression estimator).  diag(M) comes from the
//      symmetric sweep operator (Gauss-Jordan on the packed lower triangle;
//      sweeping every pivot of an SPD matrix leaves -M, no pivoting needed).
//  (2) G_w = diag(sigma)^-1 G diag(sigma)^-1 / N, eigenpairs in descending
//      order, each vector sign-fixed (largest-|.| entry positive, lowest index
//      on ties; SPEC.md:181 D6 applied to V).
//
// B200 design note (DESIGN.md §4 K2): a dense fp64 B x B matrix is 401 KB at
// B = 224, more than one SM's 227 KB of shared memory, so the Jacobi rotation
// of A *and* V that the north_star names cannot stay on chip in one CTA.  The
// packed lower triangle (201 KB at B = 224) can: the solver is Householder
// tridiagonalisation in shared memory (reflectors streamed to an L2-resident
// column-major buffer), multisection bisection on the tridiagonal (all warps,
// ballot-based), inverse iteration for the needed eigenvectors only, and the
// back-transform through the stored reflectors.  Everything is fp64.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int NT = 1024;
constexpr int NW = NT / 32;

// clock64() stamps of the last noise_eig_kernel run (diagnostics, hyde_debug_eig_clocks):
// [0] start [1] sweep done [2] tridiagonal done [3] eigenvalues [4] inverse iteration
// [5] back-transform done
__device__ long long g_eig_clk[8];
__device__ __forceinline__ void stamp(int i) {
  if (threadIdx.x == 0) g_eig_clk[i] = clock64();
}

__device__ __forceinline__ long long pk(int i, int j) {  // packed lower, i >= j
  return (long long)i * (i + 1) / 2 + j;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, result broadcast to all threads.  `red` holds NW+1 doubles.
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = l < NW ? red[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) red[NW] = t;
  }
  __syncthreads();
  return red[NW];
}

__device__ double block_minmax(double v, double* red, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : fmin(v, u);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = l < NW ? red[l] : (is_max ? -INFINITY : INFINITY);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = is_max ? fmax(t, u) : fmin(t, u);
    }
    if (l == 0) red[NW] = t;
  }
  __syncthreads();
  return red[NW];
}

// number of eigenvalues of T (d, e2 = squared off-diagonal) strictly below x
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) <= pivmin) q = -pivmin;
    if (q < 0) ++cnt;
  }
  return cnt;
}

// Eigenvalues with descending indices k0 .. k0+K-1 of the symmetric
// tridiagonal T (d, e2) by multisection: tpe lanes per eigenvalue evaluate tpe
// interior points per step; the sub-interval containing the target is chosen
// with a warp ballot.  Results to lam_out[k - k0].
__device__ void bisect_eigs(const double* d, const double* e2, int n, double glo, double ghi,
                            double pivmin, int k0, int K, double* lam_out) {
  int tpe = 32;
  while (tpe > 1 && tpe * K > NT) tpe >>= 1;
  const int lane = threadIdx.x & 31;
  const int group = threadIdx.x / tpe;        // eigenvalue slot handled by this lane group
  const int sub = threadIdx.x % tpe;
  const int gbase = (lane / tpe) * tpe;
  const int groups_total = NT / tpe;
  // the same iteration count everywhere keeps the full-warp ballot legal
  const double range = fmax(ghi - glo, 1e-300);
  const double tol = 4.0 * 2.220446049250313e-16 * fmax(fabs(glo), fabs(ghi)) + 4.0 * pivmin;
  int iters = (int)ceil(log2(range / tol) / log2((double)tpe + 1.0)) + 2;
  if (iters > 200) iters = 200;
  for (int base = 0; base < K; base += groups_total) {
    const int slot = base + group;
    const bool active = slot < K;
    const int kdesc = k0 + (active ? slot : 0);
    const int asc = n - 1 - kdesc;            // ascending index of the target eigenvalue
    double lo = glo, hi = ghi;
    for (int it = 0; it < iters; ++it) {
      double x = lo + (hi - lo) * (double)(sub + 1) / (double)(tpe + 1);
      int c = sturm_count(d, e2, n, x, pivmin);
      unsigned bal = __ballot_sync(0xffffffffu, c > asc);
      unsigned gb = (tpe == 32) ? bal : ((bal >> gbase) & ((1u << tpe) - 1u));
      int q = gb ? (__ffs(gb) - 1) : tpe;      // first point with count > asc
      // every lane executes both shuffles (clamped sources), then selects
      double xq = __shfl_sync(0xffffffffu, x, gbase + min(q, tpe - 1));
      double xp = __shfl_sync(0xffffffffu, x, gbase + max(q - 1, 0));
      double nlo = (q > 0) ? xp : lo;
      double nhi = (q < tpe) ? xq : hi;
      lo = nlo;
      hi = nhi;
    }
    if (active && sub == 0) lam_out[slot] = 0.5 * (lo + hi);
  }
}

// Inverse iteration for eigenvalue lam of T: solve (T - lam I) x = x_prev three
// times with the partial-pivot tridiagonal LU (stored per vector in scratch).
// One thread per vector.  x has stride 1, length n.
__device__ void inv_iter(const double* d, const double* e, int n, double lam, double tnorm,
                         double* x, double* dd, double* u1, double* u2, double* ml,
                         unsigned char* piv, unsigned seed) {
  // pivot floor eps ||T|| (for T == 0 every vector is an eigenvector: floor 1)
  const double tiny = tnorm > 0.0 ? 2.220446049250313e-16 * tnorm : 1.0;
  // factorise T - lam I = P L U (U has two super-diagonals)
  double a = d[0] - lam, b = (n > 1) ? e[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    double c = e[i];                       // sub-diagonal (i+1, i)
    double a1 = d[i + 1] - lam;
    double b1 = (i + 1 < n - 1) ? e[i + 1] : 0.0;
    if (fabs(a) >= fabs(c)) {
      if (fabs(a) < tiny) a = (a < 0 ? -tiny : tiny);
      double m = c / a;
      dd[i] = a; u1[i] = b; u2[i] = 0.0; ml[i] = m; piv[i] = 0;
      a = a1 - m * b;
      b = b1;
    } else {
      double m = a / c;
      dd[i] = c; u1[i] = a1; u2[i] = b1; ml[i] = m; piv[i] = 1;
      a = b - m * a1;
      b = -m * b1;
    }
  }
  if (fabs(a) < tiny) a = (a < 0 ? -tiny : tiny);
  dd[n - 1] = a;
  // deterministic start vector
  for (int i = 0; i < n; ++i) {
    unsigned h = (unsigned)(i * 2654435761u) ^ (seed * 40503u + 0x9E3779B9u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    x[i] = 0.5 + (double)(h & 0xFFFF) / 65536.0;
  }
  for (int it = 0; it < 3; ++it) {
    // forward: apply P L^-1
    for (int i = 0; i < n - 1; ++i) {
      if (piv[i]) {
        double t = x[i];
        x[i] = x[i + 1];
        x[i + 1] = t - ml[i] * x[i + 1];
      } else {
        x[i + 1] -= ml[i] * x[i];
      }
    }
    // back substitution with U
    x[n - 1] /= dd[n - 1];
    if (n > 1) x[n - 2] = (x[n - 2] - u1[n - 2] * x[n - 1]) / dd[n - 2];
    for (int i = n - 3; i >= 0; --i) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / dd[i];
    double mx = 0.0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(x[i]));
    mx = 1.0 / mx;                       // scale before squaring: no overflow
    double s = 0.0;
    for (int i = 0; i < n; ++i) { x[i] *= mx; s += x[i] * x[i]; }
    s = 1.0 / sqrt(s);
    for (int i = 0; i < n; ++i) x[i] *= s;
  }
}

// Phases shared by the first-chunk kernel and the later-chunk kernel:
// eigenvalues k0..k0+K-1, inverse iteration, back-transform Q y (reflectors in
// house_col[k*B + i], betas in house_beta[k]), sign fix, outputs.
__device__ void vectors_phase(const double* d, const double* e, const double* e2, int B,
                              double glo, double ghi, double pivmin, int k0, int K,
                              double* lamk /*smem K*/, double* scratch /*smem*/,
                              const double* __restrict__ house_col,
                              const double* __restrict__ house_beta, const double* sig_s,
                              double* lam_top_out, double* V, int ldv, float* W, float* U,
                              int ldwu, double* red) {
  bisect_eigs(d, e2, B, glo, ghi, pivmin, k0, K, lamk);
  __syncthreads();
  stamp(3);
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  // per-vector scratch: x, dd, u1, u2, ml (5B doubles) + piv (B bytes)
  double* xs = scratch;
  double* fs = scratch + (size_t)K * B;
  unsigned char* pv = (unsigned char*)(fs + (size_t)K * 4 * B);
  if (threadIdx.x < K) {
    int k = threadIdx.x;
    double* f = fs + (size_t)k * 4 * B;
    inv_iter(d, e, B, lamk[k], tnorm, xs + (size_t)k * B, f, f + B, f + 2 * B, f + 3 * B,
             pv + (size_t)k * B, (unsigned)(k0 + k));
  }
  __syncthreads();
  // re-orthogonalise numerically coincident eigenvalues (cluster tolerance
  // 1e-9 ||T||: above it inverse iteration alone is accurate to ~1e-7)
  if (threadIdx.x == 0) {
    for (int j = 1; j < K; ++j) {
      double* xj = xs + (size_t)j * B;
      bool touched = false;
      for (int i = 0; i < j; ++i) {
        if (fabs(lamk[i] - lamk[j]) > 1e-9 * tnorm) continue;
        const double* xi = xs + (size_t)i * B;
        double dot = 0.0;
        for (int t = 0; t < B; ++t) dot += xi[t] * xj[t];
        for (int t = 0; t < B; ++t) xj[t] -= dot * xi[t];
        touched = true;
      }
      if (touched) {
        double s = 0.0;
        for (int t = 0; t < B; ++t) s += xj[t] * xj[t];
        s = 1.0 / sqrt(s);
        for (int t = 0; t < B; ++t) xj[t] *= s;
      }
    }
  }
  __syncthreads();
  stamp(4);
  // back-transform: one warp per vector, reflectors k = B-3 .. 0
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int k = w; k < K; k += NW) {
    double* y = xs + (size_t)k * B;
    for (int r = B - 3; r >= 0; --r) {
      const double beta = house_beta[r];
      if (beta == 0.0) continue;
      const double* v = house_col + (size_t)r * B;
      double s = 0.0;
      for (int i = r + 1 + l; i < B; i += 32) s += v[i] * y[i];
      s = warp_sum(s) * beta;
      for (int i = r + 1 + l; i < B; i += 32) y[i] -= s * v[i];
      __syncwarp();
    }
    // sign convention: largest |y_i| positive, lowest index on ties
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = l; i < B; i += 32) {
      double a = fabs(y[i]);
      if (a > best) { best = a; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sgn = (y[bi] < 0) ? -1.0 : 1.0;
    const int kk = k0 + k;
    for (int i = l; i < B; i += 32) {
      double vi = sgn * y[i];
      if (V) V[(size_t)i * ldv + k] = vi;
      W[(size_t)i * ldwu + kk] = (float)(vi / sig_s[i]);
      U[(size_t)i * ldwu + kk] = (float)(vi * sig_s[i]);
    }
    if (l == 0 && lam_top_out) lam_top_out[kk] = lamk[k];
  }
  __syncthreads();
  stamp(5);
}

// tri layout (global): d[B], e[B], e2[B], misc[4] = {glo, ghi, pivmin, 0}
__global__ void __launch_bounds__(NT, 1) noise_eig_kernel(
    const double* __restrict__ G, long long n, int B, double ridge, int ncomp, int all_lam,
    double* sigma_out, double* lam_all, double* lam_top, double* V, double* house_col,
    double* house_beta, double* tri, float* W, float* U, int ldwu, double* A_glob) {
  extern __shared__ double sm[];
  const int EXT = 8 * B + NW + 2;   // col vv pp sig d e e2 red lamk
  double* ext = sm;
  double* A = A_glob ? A_glob : sm + EXT;
  double* col = ext;            // B
  double* vv = col + B;         // B
  double* pp = vv + B;          // B
  double* sig = pp + B;         // B
  double* d = sig + B;          // B
  double* e = d + B;            // B
  double* e2 = e + B;           // B
  double* red = e2 + B;         // NW + 2
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  stamp(0);

  // ---- (1) sweep operator on G + ridge I (packed lower) ----
  for (int i = w; i < B; i += NW)
    for (int j = l; j <= i; j += 32) A[pk(i, j)] = G[(size_t)i * B + j] + (i == j ? ridge : 0.0);
  __syncthreads();
  for (int k = 0; k < B; ++k) {
    for (int i = tid; i < B; i += NT) col[i] = (i >= k) ? A[pk(i, k)] : A[pk(k, i)];
    __syncthreads();
    const double rd = 1.0 / col[k];
    for (int i = w; i < B; i += NW) {
      const double ci = col[i] * rd;
      const long long base = (long long)i * (i + 1) / 2;
      if (i == k) {
        for (int j = l; j <= i; j += 32) A[base + j] = (j == k) ? -rd : col[j] * rd;
      } else {
        for (int j = l; j <= i; j += 32) {
          if (j == k) A[base + j] = ci;
          else A[base + j] -= ci * col[j];
        }
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < B; i += NT) {
    double mbb = -A[pk(i, i)];
    double s = sqrt(1.0 / ((double)n * mbb));
    sig[i] = s;
    sigma_out[i] = s;
  }
  __syncthreads();
  stamp(1);
  if (ncomp < 0) return;   // noise estimate only (hyde_estimate_noise)

  // ---- (2) G_w = S G S / N, Householder tridiagonalisation (lower) ----
  const double invn = 1.0 / (double)n;
  for (int i = w; i < B; i += NW)
    for (int j = l; j <= i; j += 32) A[pk(i, j)] = G[(size_t)i * B + j] / (sig[i] * sig[j]) * invn;
  __syncthreads();
  for (int k = 0; k < B - 2; ++k) {
    double part = 0.0;
    for (int i = k + 1 + tid; i < B; i += NT) {
      double x = A[pk(i, k)];
      vv[i] = x;
      part += x * x;
    }
    const double sumsq = block_sum(part, red);   // syncs: vv visible
    const double x0 = A[pk(k + 1, k)];          // untouched this step; vv[k+1] is rewritten below
    const double tail = sumsq - x0 * x0;
    double beta = 0.0, alpha = x0;
    if (tail > 0.0) {
      alpha = -copysign(sqrt(sumsq), x0);
      const double v0 = x0 - alpha;
      beta = 2.0 / (tail + v0 * v0);
      if (tid == 0) vv[k + 1] = v0;
    }
    if (tid == 0) { d[k] = A[pk(k, k)]; e[k] = alpha; house_beta[k] = beta; }
    __syncthreads();
    // stream the reflector to the column-major global buffer (zeros above)
    for (int i = tid; i < B; i += NT) house_col[(size_t)k * B + i] = (i > k) ? vv[i] : 0.0;
    if (beta != 0.0) {
      // p = beta A22 v
      for (int i = k + 1 + w; i < B; i += NW) {
        double s = 0.0;
        const long long base = (long long)i * (i + 1) / 2;
        for (int j = k + 1 + l; j < B; j += 32) {
          double a = (j <= i) ? A[base + j] : A[pk(j, i)];
          s += a * vv[j];
        }
        s = warp_sum(s);
        if (l == 0) pp[i] = beta * s;
      }
      __syncthreads();
      double pv = 0.0;
      for (int i = k + 1 + tid; i < B; i += NT) pv += pp[i] * vv[i];
      const double Kc = 0.5 * beta * block_sum(pv, red);
      // A22 -= v w^T + w v^T,  w = p - Kc v
      for (int i = k + 1 + w; i < B; i += NW) {
        const double vi = vv[i], wi = pp[i] - Kc * vi;
        const long long base = (long long)i * (i + 1) / 2;
        for (int j = k + 1 + l; j <= i; j += 32) {
          const double vj = vv[j], wj = pp[j] - Kc * vj;
          A[base + j] -= vi * wj + wi * vj;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[B - 2] = A[pk(B - 2, B - 2)];
    e[B - 2] = A[pk(B - 1, B - 2)];
    d[B - 1] = A[pk(B - 1, B - 1)];
    e[B - 1] = 0.0;
    house_beta[B - 2] = 0.0;
    house_beta[B - 1] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < 2 * B; i += NT) house_col[(size_t)(B - 2) * B + i] = 0.0;
  double lo = INFINITY, hi = -INFINITY, emax = 0.0;
  for (int i = tid; i < B; i += NT) {
    e2[i] = e[i] * e[i];
    double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < B - 1 ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    emax = fmax(emax, e2[i]);
  }
  const double glo = block_minmax(lo, red, false);
  const double ghi = block_minmax(hi, red, true);
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, block_minmax(emax, red, true));
  for (int i = tid; i < B; i += NT) { tri[i] = d[i]; tri[B + i] = e[i]; tri[2 * B + i] = e2[i]; }
  if (tid == 0) { tri[3 * B] = glo; tri[3 * B + 1] = ghi; tri[3 * B + 2] = pivmin; }
  __syncthreads();
  stamp(2);

  // ---- (3) eigenvalues (all if requested), vectors for the top ncomp ----
  double* lamk = red + NW + 2;                 // B doubles
  double* scratch = sm + EXT;                  // A (if on chip) is dead once reflectors are out
  if (all_lam && lam_all) {
    bisect_eigs(d, e2, B, glo, ghi, pivmin, 0, B, lamk);
    __syncthreads();
    for (int i = tid; i < B; i += NT) lam_all[i] = lamk[i];
    __syncthreads();
  }
  vectors_phase(d, e, e2, B, glo, ghi, pivmin, 0, ncomp, lamk, scratch, house_col, house_beta,
                sig, lam_top, V, ncomp, W, U, ldwu, red);
}

// Later chunks: eigenpairs k0 .. k0+ncomp-1 from the stored tridiagonal and reflectors.
__global__ void __launch_bounds__(NT, 1) eigvec_more_kernel(
    const double* __restrict__ tri, const double* __restrict__ house_col,
    const double* __restrict__ house_beta, const double* __restrict__ sigma, int B, int k0,
    int ncomp, double* lam_top, double* V, float* W, float* U, int ldwu) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e = d + B;
  double* e2 = e + B;
  double* sig = e2 + B;
  double* red = sig + B;
  double* lamk = red + NW + 2;
  double* scratch = lamk + B;
  for (int i = threadIdx.x; i < B; i += NT) {
    d[i] = tri[i]; e[i] = tri[B + i]; e2[i] = tri[2 * B + i]; sig[i] = sigma[i];
  }
  __syncthreads();
  vectors_phase(d, e, e2, B, tri[3 * B], tri[3 * B + 1], tri[3 * B + 2], k0, ncomp, lamk, scratch,
                house_col, house_beta, sig, lam_top, V, ncomp, W, U, ldwu, red);
}

// residual_b = (M Y)_b / M_bb: M from G + ridge I by the same sweep (one CTA),
// written to work[B*B]; then a plain mat-mat kernel.
__global__ void __launch_bounds__(NT, 1) inverse_kernel(const double* __restrict__ G, int B,
                                                        double ridge, double* A, double* Mfull) {
  extern __shared__ double sm[];
  double* col = sm;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int i = w; i < B; i += NW)
    for (int j = l; j <= i; j += 32) A[pk(i, j)] = G[(size_t)i * B + j] + (i == j ? ridge : 0.0);
  __syncthreads();
  for (int k = 0; k < B; ++k) {
    for (int i = tid; i < B; i += NT) col[i] = (i >= k) ? A[pk(i, k)] : A[pk(k, i)];
    __syncthreads();
    const double rd = 1.0 / col[k];
    for (int i = w; i < B; i += NW) {
      const double ci = col[i] * rd;
      const long long base = (long long)i * (i + 1) / 2;
      for (int j = l; j <= i; j += 32) {
        if (i == k) A[base + j] = (j == k) ? -rd : col[j] * rd;
        else if (j == k) A[base + j] = ci;
        else A[base + j] -= ci * col[j];
      }
    }
    __syncthreads();
  }
  for (int i = w; i < B; i += NW)
    for (int j = l; j < B; j += 32) {
      double m = -((j <= i) ? A[pk(i, j)] : A[pk(j, i)]);
      Mfull[(size_t)i * B + j] = m;
    }
}

__global__ void residual_kernel(const float* __restrict__ Y, long long n, int B,
                                const double* __restrict__ M, float* __restrict__ out) {
  long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int b = blockIdx.y;
  if (p >= n) return;
  double s = 0.0;
  for (int j = 0; j < B; ++j) s += M[(size_t)b * B + j] * (double)Y[(size_t)j * n + p];
  out[(size_t)b * n + p] = (float)(s / M[(size_t)b * B + b]);
}

}  // namespace

extern "C" hyde_status hyde_debug_eig_clocks(long long* out) {
  if (!out) return HYDE_EPARAM;
  return cudaMemcpyFromSymbol(out, g_eig_clk, sizeof(long long) * 8) == cudaSuccess ? HYDE_OK : HYDE_ECUDA;
}

static size_t eig_ext_bytes(int B) { return (size_t)(8 * B + NW + 2) * sizeof(double); }
static size_t eig_scr_bytes(int B, int ncomp) {
  return (size_t)ncomp * B * 5 * sizeof(double) + (size_t)ncomp * B + 16;
}

// shared memory of noise_eig_kernel with the packed matrix on chip
size_t eig_smem_bytes(int B, int ncomp) {
  size_t P = (size_t)B * (B + 1) / 2 * sizeof(double);
  size_t scr = eig_scr_bytes(B, ncomp);
  return eig_ext_bytes(B) + (P > scr ? P : scr);
}

static const size_t kMaxSmem = 227 * 1024;

cudaError_t launch_noise_eig(const double* G, long long n, int B, double ridge, int ncomp,
                             int all_lam, double* sigma, double* lam, double* V, double* house,
                             double* tri, float* W, float* U, int ldwu, cudaStream_t st) {
  // house: [B*B column-major reflectors][B betas][B top eigenvalues][P packed A fallback]
  double* house_col = house;
  double* house_beta = house + (size_t)B * B;
  double* lam_top = house_beta + B;
  double* A_glob = nullptr;
  size_t smem = eig_smem_bytes(B, ncomp < 0 ? 0 : ncomp);
  if (smem > kMaxSmem) {
    A_glob = lam_top + B;
    smem = eig_ext_bytes(B) + eig_scr_bytes(B, ncomp < 0 ? 0 : ncomp);
  }
  if (smem > kMaxSmem) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(noise_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kMaxSmem);
  if (e != cudaSuccess) return e;
  noise_eig_kernel<<<1, NT, smem, st>>>(G, n, B, ridge, ncomp, all_lam, sigma, lam, lam_top, V,
                                        house_col, house_beta, tri, W, U, ldwu, A_glob);
  return cudaGetLastError();
}

cudaError_t launch_eigvec_more(const double* tri, const double* house, const double* sigma, int B,
                               int k0, int ncomp, double* lam_top_unused, double* V, float* W,
                               float* U, int ldwu, cudaStream_t st) {
  const double* house_col = house;
  const double* house_beta = house + (size_t)B * B;
  double* lam_top = const_cast<double*>(house_beta + B);
  size_t smem = (size_t)(4 * B + NW + 2 + B) * sizeof(double) +
                (size_t)ncomp * B * 5 * sizeof(double) + (size_t)ncomp * B + 16;
  if (smem > kMaxSmem) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(eigvec_more_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
  if (e != cudaSuccess) return e;
  eigvec_more_kernel<<<1, NT, smem, st>>>(tri, house_col, house_beta, sigma, B, k0, ncomp, lam_top,
                                          V, W, U, ldwu);
  return cudaGetLastError();
}

cudaError_t launch_noise_residual(const float* Y, long long n, int B, const double* G, double ridge,
                                  double* work, float* out, cudaStream_t st) {
  // work: packed A (P) + M (B*B)
  double* A = work;
  double* M = work + (size_t)B * (B + 1) / 2;
  cudaError_t e = cudaFuncSetAttribute(inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(B * sizeof(double)));
  if (e != cudaSuccess) return e;
  inverse_kernel<<<1, NT, B * sizeof(double), st>>>(G, B, ridge, A, M);
  dim3 grid((unsigned)((n + 255) / 256), B);
  residual_kernel<<<grid, 256, 0, st>>>(Y, n, B, M, out);
  return cudaGetLastError();
}
