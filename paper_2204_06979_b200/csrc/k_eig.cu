// K2 (SURVEY.md §8(a) A1 tail + A2; north_star stages (1)-(2)): per-band
// noise and the eigendecomposition of the whitened Gram, as a short chain of
// kernels that each map to what B200 is good at:
//
//  K2a chol_kernel     (1 CTA)   G + delta I = L L^T, blocked right-looking
//                                Cholesky on the packed triangle in shared
//                                memory (panel 16, 4x4 register tiles).
//  K2b invdiag_kernel  (B/8 CTAs) one warp per band: forward substitution
//                                L x = e_b, M_bb = |x|^2 = [(G+dI)^-1]_bb,
//                                sigma_b = sqrt(1 / (N M_bb))  (
//                                HySime's regression estimator).
//  K2c tridiag_kernel  (1 CTA)   G_w = S G S / N (S = diag(sigma)^-1) in
//                                shared memory, Householder reduction to
//                                tridiagonal T; reflectors to an L2-resident
//                                column-major buffer.
//  K2d eigpair_kernel  (1 CTA per eigenpair) multisection bisection of T
//                                (division-free Sturm counts, 512 points per
//                                step), inverse iteration, back-transform,
//                                sign fix (largest-|.| entry positive, lowest
//                                index on ties: S:181 D6 applied to V), and
//                                W = S v, U = S^-1 v in fp32 for K3 / K6b.
//  K2e reorth_kernel   (1 CTA)   Gram-Schmidt inside clusters of numerically
//                                coincident eigenvalues (|dl| <= 1e-9 ||T||).
//
// Why not the north_star's single-CTA Jacobi (DESIGN.md §4 K2): a dense fp64
// B x B matrix is 401 KB at B = 224 -- more than one SM's 227 KB of shared
// memory -- so rotating A *and* V cannot stay on chip in one CTA, and Jacobi's
// ~8 sweeps x 5 B^3/2 flops would be ~20x the Householder path's work.  The
// packed triangle (201 KB) fits, and only the chunk's eigenpairs are formed,
// each on its own SM.  Everything is fp64.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int NT = 1024;
constexpr int NW = NT / 32;
constexpr int CNB = 16;        // Cholesky panel width
constexpr int CT = 512;        // Cholesky threads (4x4 fp64 register tiles need > 64 registers)
constexpr int CW = CT / 32;

// clock64() stamps (diagnostics, hyde_debug_eig_clocks): [0] chol start [1] chol end
// [2] tridiag start [3] tridiag end [4] eigpair start (CTA 0) [5] bisection done
// [6] inverse iteration done [7] back-transform done
__device__ long long g_eig_clk[16];
__device__ __forceinline__ void stamp(int i) {
  if (threadIdx.x == 0) g_eig_clk[i] = clock64();
}
// accumulate (clock64() - t0) into slot i (thread 0); returns the new t0
__device__ __forceinline__ long long acc_clk(int i, long long t0) {
  const long long t = clock64();
  if (threadIdx.x == 0) g_eig_clk[i] += t - t0;
  return t;
}

__device__ __forceinline__ int off(int i) { return (i * (i + 1)) >> 1; }   // packed lower row start

// 1/a to full fp64 accuracy without the division's long dependent sequence:
// MUFU reciprocal seed + two Newton steps (a finite, |a| >= 1e-300)
__device__ __forceinline__ double rcp64(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum (NT threads), broadcast; `red` holds NW + 1 doubles
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = l < NW ? red[l] : 0.0;
  t = warp_sum(t);
  __syncthreads();          // everyone has read red before it is reused
  return t;
}

// Workspace carve-up of the K2 buffer `house` (doubles):
struct EigWs {
  double* house_col;   // B*B  column k = Householder vector k (zeros at i <= k)
  double* vtop;        // B*B  fp64 eigenvectors, column k (row-major B x B)
  double* house_beta;  // B
  double* lam_top;     // B    eigenvalues by descending index
  double* rdiag;       // B    1 / L_ii
  double* flags;       // 8    [0] Cholesky failure
  double* Lp;          // P    packed Cholesky factor (also global fallback storage)
  double* Aw;          // B*B  global fallback storage for the tridiagonalisation / M
};
__host__ __device__ inline EigWs carve(double* house, int B) {
  EigWs w;
  const long long P = (long long)B * (B + 1) / 2;
  w.house_col = house;
  w.vtop = house + (long long)B * B;
  w.house_beta = w.vtop + (long long)B * B;
  w.lam_top = w.house_beta + B;
  w.rdiag = w.lam_top + B;
  w.flags = w.rdiag + B;
  w.Lp = w.flags + 8;
  w.Aw = w.Lp + P;
  return w;
}

// =====================================================================
// K2a: blocked right-looking Cholesky of G + ridge I (packed lower)
// =====================================================================
template <bool SMEM>
__global__ void __launch_bounds__(CT, 1) chol_kernel(const double* __restrict__ G, int B, double ridge, EigWs ws) {
  extern __shared__ double sm[];
  double* A = SMEM ? sm : ws.Lp;
  __shared__ double dinv_sh;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  stamp(0);
  for (int i = w; i < B; i += CW)
    for (int j = l; j <= i; j += 32) A[off(i) + j] = G[(size_t)i * B + j] + (i == j ? ridge : 0.0);
  __syncthreads();
  if (threadIdx.x == 0) { g_eig_clk[8] = 0; g_eig_clk[9] = 0; g_eig_clk[10] = 0; }
  long long tc0 = clock64();
  for (int k0 = 0; k0 < B; k0 += CNB) {
    const int kb = min(CNB, B - k0);
    // ---- panel: (a) kb x kb diagonal block by warp 0, rows in registers ----
    if (w == 0) {
      double a[CNB];
      const int r = l;
#pragma unroll
      for (int c = 0; c < CNB; ++c) a[c] = (r < kb && c <= r) ? A[off(k0 + r) + k0 + c] : 0.0;
#pragma unroll
      for (int c = 0; c < CNB; ++c) {
        if (c < kb) {
          double dc = __shfl_sync(0xffffffffu, a[c], c);
          if (!(dc > 0.0)) {   // not positive definite (cannot happen for G + dI, d > 0, G PSD)
            if (l == 0) ws.flags[0] = 1.0;
            dc = 1e-300;
          }
          const double piv = sqrt(dc);
          const double rinv = 1.0 / piv;
          if (r == c) a[c] = piv;
          else if (r > c) a[c] *= rinv;
          if (l == 0) ws.rdiag[k0 + c] = rinv;
#pragma unroll
          for (int j = c + 1; j < CNB; ++j) {
            const double ljc = __shfl_sync(0xffffffffu, a[c], j);
            if (j < kb && r >= j && r < kb) a[j] = fma(-a[c], ljc, a[j]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CNB; ++c)
        if (r < kb && c <= r) A[off(k0 + r) + k0 + c] = a[c];
    }
    __syncthreads();
    tc0 = acc_clk(8, tc0);
    // ---- panel: (b) rows below the block, one thread per row (triangular solve) ----
    for (int i = k0 + kb + tid; i < B; i += CT) {
      double li[CNB];
      const int oi = off(i);
#pragma unroll
      for (int c = 0; c < CNB; ++c) {
        if (c < kb) {
          double x = A[oi + k0 + c];
          const int oc = off(k0 + c);
#pragma unroll
          for (int q = 0; q < CNB; ++q)
            if (q < c) x = fma(-li[q], A[oc + k0 + q], x);
          li[c] = x * ws.rdiag[k0 + c];
          A[oi + k0 + c] = li[c];
        }
      }
    }
    __syncthreads();
    tc0 = acc_clk(9, tc0);
    // ---- trailing update A22 -= P P^T with 4x4 register tiles ----
    const int k1 = k0 + kb;
    const int m = B - k1;
    if (m <= 0) break;
    const int nt = (m + 3) >> 2;
    const int ntiles = nt * (nt + 1) / 2;
    for (int t = tid; t < ntiles; t += CT) {
      int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
      while (off(ti + 1) <= t) ++ti;
      while (off(ti) > t) --ti;
      const int tj = t - off(ti);
      const int i0 = k1 + 4 * ti, j0 = k1 + 4 * tj;
      double acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[r][s] = 0.0;
      int oi[4], oj[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        oi[r] = (i0 + r < B) ? off(i0 + r) + k0 : -1;
        oj[r] = (j0 + r < B) ? off(j0 + r) + k0 : -1;
      }
      for (int c = 0; c < kb; ++c) {
        double li[4], lj[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          li[r] = oi[r] >= 0 ? A[oi[r] + c] : 0.0;
          lj[r] = oj[r] >= 0 ? A[oj[r] + c] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int s = 0; s < 4; ++s) acc[r][s] = fma(li[r], lj[s], acc[r][s]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int i = i0 + r, j = j0 + s;
          if (i < B && j <= i) A[off(i) + j] -= acc[r][s];
        }
    }
    __syncthreads();
    tc0 = acc_clk(10, tc0);
  }
  if (SMEM) {
    const int P = off(B);
    for (int t = tid; t < P; t += CT) ws.Lp[t] = A[t];
  }
  stamp(1);
}

// =====================================================================
// K2b: M_bb = |L^-1 e_b|^2 by forward substitution, one warp per band
// =====================================================================
__global__ void __launch_bounds__(256) invdiag_kernel(EigWs ws, int B, long long n, double* sigma_out) {
  __shared__ double xs[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + w;
  if (b >= B) return;
  double* x = xs[w];
  const double* L = ws.Lp;
  const double* rd = ws.rdiag;
  const double xb = rd[b];
  if (l == 0) x[b] = xb;
  double ss = xb * xb;
  __syncwarp();
  // prefetch row b+1's entries (j in [b, i)) held strided by lane
  double cur[8];
  int i = b + 1;
  auto load_row = [&](int row, double (&dst)[8]) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = b + l + 32 * t;
      dst[t] = (row < B && j < row) ? L[off(row) + j] : 0.0;
    }
  };
  if (i < B) load_row(i, cur);
  for (; i < B; ++i) {
    double nxt[8];
    load_row(i + 1, nxt);
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = b + l + 32 * t;
      if (j < i) s = fma(cur[t], x[j], s);
    }
    s = warp_sum(s);
    const double xi = -s * rd[i];
    if (l == 0) x[i] = xi;
    ss = fma(xi, xi, ss);
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) cur[t] = nxt[t];
  }
  if (l == 0) sigma_out[b] = sqrt(1.0 / ((double)n * ss));
}

// =====================================================================
// K2c: whitening + Householder tridiagonalisation (one CTA)
// =====================================================================
constexpr int TT = 1024;        // tridiagonalisation threads
constexpr int TW = TT / 32;

// Warp 0 only: from the (final) column c below its diagonal, x = A[c+1.., c],
// form the Householder reflector H = I - beta v v^T with H x = alpha e_1;
// writes v (entries > c) into vout, d[c] / e[c] / beta to tri / ws, the
// reflector to ws.house_col and beta to *beta_sh.
__device__ void make_reflector(const double* A, int B, int c, double dcc, double* vout, double* tri, EigWs& ws,
                               double* beta_sh) {
  const int l = threadIdx.x & 31;
  double part = 0.0, x0 = 0.0;
  for (int i = c + 1 + l; i < B; i += 32) {
    const double x = A[off(i) + c];
    vout[i] = x;
    if (i == c + 1) x0 = x;
    else part = fma(x, x, part);             // |x[1:]|^2 directly: exactly 0 when x has one entry
  }
  const double tail = warp_sum(part);
  x0 = warp_sum(x0);                         // only the lane holding i = c+1 contributed
  double beta = 0.0, alpha = x0;
  // the last column (c = B-2) is already tridiagonal: no reflector (only 0..B-3 are applied)
  if (tail > 0.0 && c < B - 2) {
    const double sumsq = fma(x0, x0, tail);
    alpha = -copysign(sqrt(sumsq), x0);
    const double v0 = x0 - alpha;
    beta = 2.0 / (tail + v0 * v0);
    __syncwarp();
    if (l == 0) vout[c + 1] = v0;
  }
  __syncwarp();
  for (int i = l; i < B; i += 32) ws.house_col[(size_t)c * B + i] = (i > c) ? vout[i] : 0.0;
  if (l == 0) {
    tri[c] = dcc;
    tri[B + c] = alpha;
    ws.house_beta[c] = beta;
    *beta_sh = beta;
  }
  __syncwarp();
}

// Householder tridiagonalisation of G_w (one CTA, TT threads), look-ahead form:
// per column k two barriers -- (1) p = beta A22 v on blocks of 4 rows (four
// independent dot products per lane) plus the p.v partials; (2) the rank-2
// update A22 -= v w^T + w v^T by warps 1.. while warp 0 updates column k+1
// itself and immediately forms reflector k+1 into the other v buffer.
template <bool SMEM>
__global__ void __launch_bounds__(TT, 1) tridiag_kernel(const double* __restrict__ G, const double* __restrict__ sigma,
                                                        long long n, int B, EigWs ws, double* tri) {
  extern __shared__ double sm[];
  // shared layout: vbuf[2][B] pp[B] sig[B] red[TW+8] | A (packed) if SMEM
  double* vbuf0 = sm;
  double* vbuf1 = sm + B;
  double* pp = sm + 2 * B;
  double* sig = pp + B;
  double* red = sig + B;
  double* A = SMEM ? (red + TW + 8) : ws.Aw;
  __shared__ double beta_sh;
  __shared__ double hi_red[TW], lo_red[TW];
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  stamp(2);
  for (int i = tid; i < B; i += TT) sig[i] = sigma[i];
  __syncthreads();
  const double invn = 1.0 / (double)n;
  for (int i = w; i < B; i += TW)
    for (int j = l; j <= i; j += 32) A[off(i) + j] = G[(size_t)i * B + j] / (sig[i] * sig[j]) * invn;
  __syncthreads();
  if (threadIdx.x == 0) { g_eig_clk[11] = 0; g_eig_clk[12] = 0; g_eig_clk[13] = 0; }
  long long tt0 = clock64();
  if (w == 0) make_reflector(A, B, 0, A[0], vbuf0, tri, ws, &beta_sh);
  __syncthreads();
  for (int k = 0; k < B - 2; ++k) {
    double* vv = (k & 1) ? vbuf1 : vbuf0;
    double* vn = (k & 1) ? vbuf0 : vbuf1;
    const double beta = beta_sh;
    // ---- (1) p = beta A22 v, rows k+1 .. B-1, and p.v partials ----
    const int nblk = (B - k - 1 + 3) >> 2;
    double pvp = 0.0;
    for (int blk = w; blk < nblk; blk += TW) {
      const int i0 = k + 1 + 4 * blk;
      const int nr = min(4, B - i0);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      const int o0 = off(i0), o1 = off(i0 + 1), o2 = off(i0 + 2), o3 = off(i0 + 3);
      for (int j = k + 1 + l; j < i0; j += 32) {
        const double vj = vv[j];
        s0 = fma(A[o0 + j], vj, s0);
        if (nr > 1) s1 = fma(A[o1 + j], vj, s1);
        if (nr > 2) s2 = fma(A[o2 + j], vj, s2);
        if (nr > 3) s3 = fma(A[o3 + j], vj, s3);
      }
      for (int j = i0 + 4 + l; j < B; j += 32) {
        const double vj = vv[j];
        const int bj = off(j) + i0;
        s0 = fma(A[bj], vj, s0);
        s1 = fma(A[bj + 1], vj, s1);
        s2 = fma(A[bj + 2], vj, s2);
        s3 = fma(A[bj + 3], vj, s3);
      }
      if (l < nr) {   // diagonal 4x4 block: lane r adds row r's part
        double add = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nr) {
            const double a = (c <= l) ? A[off(i0 + l) + i0 + c] : A[off(i0 + c) + i0 + l];
            add = fma(a, vv[i0 + c], add);
          }
        if (l == 0) s0 += add;
        else if (l == 1) s1 += add;
        else if (l == 2) s2 += add;
        else s3 += add;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
      }
      if (l < nr) {
        const double sr = l == 0 ? s0 : (l == 1 ? s1 : (l == 2 ? s2 : s3));
        const double pr = beta * sr;
        pp[i0 + l] = pr;
        pvp = fma(pr, vv[i0 + l], pvp);
      }
    }
    pvp = warp_sum(pvp);
    if (l == 0) red[w] = pvp;
    __syncthreads();
    tt0 = acc_clk(12, tt0);
    const double Kc = 0.5 * beta * warp_sum(l < TW ? red[l] : 0.0);
    // ---- (2) rank-2 update; warp 0 owns column k+1 and the next reflector ----
    if (w == 0) {
      const double vk1 = vv[k + 1], wk1 = pp[k + 1] - Kc * vk1;
      double dnext = 0.0;
      for (int i = k + 1 + l; i < B; i += 32) {
        const double vi = vv[i], wi = pp[i] - Kc * vi;
        const double a = A[off(i) + k + 1] - fma(vi, wk1, wi * vk1);
        A[off(i) + k + 1] = a;
        if (i == k + 1) dnext = a;
      }
      dnext = warp_sum(dnext);
      __syncwarp();
      make_reflector(A, B, k + 1, dnext, vn, tri, ws, &beta_sh);
    } else {
      for (int blk = w - 1; blk < nblk; blk += TW - 1) {
        const int i0 = k + 1 + 4 * blk;
        const int nr = min(4, B - i0);
        double vi[4], wi[4];
        int oi[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          vi[r] = r < nr ? vv[i0 + r] : 0.0;
          wi[r] = r < nr ? pp[i0 + r] - Kc * vi[r] : 0.0;
          oi[r] = off(i0 + r);
        }
        for (int j = k + 2 + l; j < i0 + nr; j += 32) {
          const double vj = vv[j], wj = pp[j] - Kc * vj;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (r < nr && j <= i0 + r) A[oi[r] + j] -= fma(vi[r], wj, wi[r] * vj);
        }
      }
    }
    __syncthreads();
    tt0 = acc_clk(13, tt0);
  }
  if (tid == 0) {
    tri[B - 1] = A[off(B - 1) + B - 1];
    tri[B + B - 1] = 0.0;
    ws.house_beta[B - 1] = 0.0;
  }
  for (int i = tid; i < B; i += TT) ws.house_col[(size_t)(B - 1) * B + i] = 0.0;
  __syncthreads();
  double lo = INFINITY, hi = -INFINITY;
  for (int i = tid; i < B; i += TT) {
    const double ei = tri[B + i];
    tri[2 * B + i] = ei * ei;
    const double r = (i > 0 ? fabs(tri[B + i - 1]) : 0.0) + (i < B - 1 ? fabs(ei) : 0.0);
    lo = fmin(lo, tri[i] - r);
    hi = fmax(hi, tri[i] + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (l == 0) { lo_red[w] = lo; hi_red[w] = hi; }
  __syncthreads();
  if (tid == 0) {
    double a = INFINITY, b2 = -INFINITY;
    for (int q = 0; q < TW; ++q) { a = fmin(a, lo_red[q]); b2 = fmax(b2, hi_red[q]); }
    tri[3 * B] = a;
    tri[3 * B + 1] = b2;
  }
  stamp(3);
}

// =====================================================================
// K2d: one eigenpair per CTA
// =====================================================================
constexpr int EP_T = 256;           // threads per eigenpair CTA
constexpr int EP_W = EP_T / 32;
constexpr int RB = 16;              // reflectors per staged block (back-transform)

// Sign changes of the Sturm sequence p_0 = 1, p_i = det(T_i - x I) =
// (d_i - x) p_{i-1} - e2_{i-1} p_{i-2} at two points (= eigenvalues below x).
// Division-free (one dependent FMA per step), power-of-two rescaling every 4
// steps, exact zeros take the sign opposite to their predecessor (LAPACK's
// -pivmin convention for q_i = p_i / p_{i-1}).
__device__ __forceinline__ void sturm2(const double* d, const double* e2, int n, double x0, double x1, int& c0,
                                       int& c1) {
  double a0 = 1.0, b0 = d[0] - x0;
  double a1 = 1.0, b1 = d[0] - x1;
  if (b0 == 0.0) b0 = -1e-300;
  if (b1 == 0.0) b1 = -1e-300;
  int n0 = b0 < 0.0, n1 = b1 < 0.0;
#pragma unroll 4
  for (int i = 1; i < n; ++i) {
    const double di = d[i], ei = e2[i - 1];
    const double u0 = ei * a0, u1 = ei * a1;
    double t0 = fma(di - x0, b0, -u0);
    double t1 = fma(di - x1, b1, -u1);
    if (t0 == 0.0) t0 = b0 < 0.0 ? 1e-300 * fabs(b0) : -1e-300 * fabs(b0);
    if (t1 == 0.0) t1 = b1 < 0.0 ? 1e-300 * fabs(b1) : -1e-300 * fabs(b1);
    n0 += (t0 < 0.0) != (b0 < 0.0);
    n1 += (t1 < 0.0) != (b1 < 0.0);
    a0 = b0; b0 = t0;
    a1 = b1; b1 = t1;
    if ((i & 3) == 3) {
      const double m0 = fmax(fabs(a0), fabs(b0)), m1 = fmax(fabs(a1), fabs(b1));
      if (m0 > 0x1p+500) { a0 *= 0x1p-500; b0 *= 0x1p-500; }
      else if (m0 < 0x1p-500) { a0 *= 0x1p+500; b0 *= 0x1p+500; }
      if (m1 > 0x1p+500) { a1 *= 0x1p-500; b1 *= 0x1p-500; }
      else if (m1 < 0x1p-500) { a1 *= 0x1p+500; b1 *= 0x1p+500; }
    }
  }
  c0 = n0;
  c1 = n1;
}

// Eigenvalue with ascending index `asc` of T by (2*EP_T)-section; all threads
// of the CTA cooperate and end with the same (lo, hi).
__device__ double bisect_one(const double* d, const double* e2, int n, double glo, double ghi, int asc, int* qsh) {
  constexpr int NP = 2 * EP_T;
  const double range = fmax(ghi - glo, 1e-300);
  const double tol = 4.0 * 2.220446049250313e-16 * fmax(fabs(glo), fabs(ghi)) + 1e-300;
  int iters = (int)ceil(log2(range / tol) / log2((double)NP + 1.0)) + 1;
  if (iters > 64) iters = 64;
  double lo = glo, hi = ghi;
  const int t = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const double h = (hi - lo) / (double)(NP + 1);
    const double x0 = lo + h * (double)(2 * t + 1);
    const double x1 = lo + h * (double)(2 * t + 2);
    int ca, cb;
    sturm2(d, e2, n, x0, x1, ca, cb);
    int q = NP;
    if (cb > asc) q = 2 * t + 1;
    if (ca > asc) q = 2 * t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q = min(q, __shfl_xor_sync(0xffffffffu, q, o));
    if ((t & 31) == 0) qsh[t >> 5] = q;
    __syncthreads();
    int qq = qsh[0];
#pragma unroll
    for (int wv = 1; wv < EP_W; ++wv) qq = min(qq, qsh[wv]);
    __syncthreads();
    // point p sits at lo + h (p + 1): the target lies in (x_{q-1}, x_q]
    const double nlo = qq > 0 ? lo + h * (double)qq : lo;
    const double nhi = qq < NP ? lo + h * (double)(qq + 1) : hi;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

// Inverse iteration for eigenvalue lam of T (one thread): partial-pivot LU of
// T - lam I (two super-diagonals), two solves from a fixed start vector.
__device__ void inv_iter(const double* d, const double* e, int n, double lam, double tnorm, double* x,
                         double* dd, double* u1, double* u2, double* ml, unsigned char* piv, unsigned seed) {
  const double tiny = tnorm > 0.0 ? 2.220446049250313e-16 * tnorm : 1.0;
  double a = d[0] - lam, b = (n > 1) ? e[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    const double c = e[i];
    const double a1 = d[i + 1] - lam;
    const double b1 = (i + 1 < n - 1) ? e[i + 1] : 0.0;
    if (fabs(a) >= fabs(c)) {
      if (fabs(a) < tiny) a = (a < 0 ? -tiny : tiny);
      const double ra = rcp64(a);
      const double m = c * ra;
      dd[i] = ra; u1[i] = b; u2[i] = 0.0; ml[i] = m; piv[i] = 0;
      a = a1 - m * b;
      b = b1;
    } else {
      const double rc = rcp64(c);
      const double m = a * rc;
      dd[i] = rc; u1[i] = a1; u2[i] = b1; ml[i] = m; piv[i] = 1;
      a = b - m * a1;
      b = -m * b1;
    }
  }
  if (fabs(a) < tiny) a = (a < 0 ? -tiny : tiny);
  dd[n - 1] = rcp64(a);
  for (int i = 0; i < n; ++i) {
    unsigned h = (unsigned)(i * 2654435761u) ^ (seed * 40503u + 0x9E3779B9u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    x[i] = 0.5 + (double)(h & 0xFFFF) / 65536.0;
  }
  for (int it = 0; it < 2; ++it) {
    for (int i = 0; i < n - 1; ++i) {
      if (piv[i]) {
        const double t = x[i];
        x[i] = x[i + 1];
        x[i + 1] = t - ml[i] * x[i + 1];
      } else {
        x[i + 1] -= ml[i] * x[i];
      }
    }
    x[n - 1] *= dd[n - 1];
    if (n > 1) x[n - 2] = (x[n - 2] - u1[n - 2] * x[n - 1]) * dd[n - 2];
    for (int i = n - 3; i >= 0; --i) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) * dd[i];
    double mx = 0.0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(x[i]));
    mx = 1.0 / mx;
    double s = 0.0;
    for (int i = 0; i < n; ++i) { x[i] *= mx; s = fma(x[i], x[i], s); }
    s = 1.0 / sqrt(s);
    for (int i = 0; i < n; ++i) x[i] *= s;
  }
}

// one CTA = eigenpair k0 + blockIdx.x (descending order); vectors_only = 0
// also computes the vector, 1 = eigenvalue only (all-eigenvalue diagnostics)
__global__ void __launch_bounds__(EP_T) eigpair_kernel(const double* __restrict__ tri, EigWs ws,
                                                       const double* __restrict__ sigma, int B, int k0,
                                                       int values_only, double* lam_out, double* V, int ldv,
                                                       float* W, float* U, int ldwu) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e = d + B;
  double* e2 = e + B;
  double* y = e2 + B;
  double* dd = y + B;
  double* u1 = dd + B;
  double* u2 = u1 + B;
  double* ml = u2 + B;
  unsigned char* piv = reinterpret_cast<unsigned char*>(ml + B);
  __shared__ int qsh[EP_W];
  const int kdesc = k0 + blockIdx.x;
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) stamp(4);
  for (int i = tid; i < B; i += EP_T) { d[i] = tri[i]; e[i] = tri[B + i]; e2[i] = tri[2 * B + i]; }
  __syncthreads();
  const double glo = tri[3 * B], ghi = tri[3 * B + 1];
  const double lam = bisect_one(d, e2, B, glo, ghi, B - 1 - kdesc, qsh);
  if (blockIdx.x == 0) stamp(5);
  if (values_only) {
    if (tid == 0) lam_out[kdesc] = lam;
    return;
  }
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  if (tid == 0) inv_iter(d, e, B, lam, tnorm, y, dd, u1, u2, ml, piv, (unsigned)kdesc);
  __syncthreads();
  if (blockIdx.x == 0) stamp(6);
  // back-transform y <- H_0 ... H_{B-3} y: reflectors staged through shared
  // memory in blocks of RB (double-buffered: warps 1.. load the next block
  // while warp 0 applies the current one)
  double* rbuf = reinterpret_cast<double*>(piv + ((B + 15) & ~15));   // 2 x RB x B
  const int l = tid & 31;
  double yl[8];
  if (tid < 32) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = l + 32 * t;
      yl[t] = i < B ? y[i] : 0.0;
    }
  }
  const int nref = B - 2;                       // reflectors 0 .. B-3
  const int nblkr = (nref + RB - 1) / RB;       // blocks from the top (r = B-3 downwards)
  auto load_block = [&](int bb, int buf, int t0, int tstep) {
    const int rhi = nref - 1 - bb * RB;         // first reflector of the block
    for (int t = t0; t < RB * B; t += tstep) {
      const int q = t / B, i = t % B;
      const int r = rhi - q;
      rbuf[(size_t)buf * RB * B + t] = (r >= 0) ? ws.house_col[(size_t)r * B + i] : 0.0;
    }
  };
  load_block(0, 0, tid, EP_T);
  __syncthreads();
  for (int bb = 0; bb < nblkr; ++bb) {
    if (tid >= 32) {
      if (bb + 1 < nblkr) load_block(bb + 1, (bb + 1) & 1, tid - 32, EP_T - 32);
    } else {
      const double* rb = rbuf + (size_t)(bb & 1) * RB * B;
      const int rhi = nref - 1 - bb * RB;
      for (int q = 0; q < RB; ++q) {
        const int r = rhi - q;
        if (r < 0) break;
        const double beta = ws.house_beta[r];
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int i = l + 32 * t;
          if (i < B) s = fma(rb[q * B + i], yl[t], s);
        }
        s = warp_sum(s) * beta;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int i = l + 32 * t;
          if (i < B) yl[t] = fma(-s, rb[q * B + i], yl[t]);
        }
      }
    }
    __syncthreads();
  }
  if (tid < 32) {
    // sign convention: largest |y_i| positive, lowest index on ties
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = l + 32 * t;
      if (i < B && fabs(yl[t]) > best) { best = fabs(yl[t]); bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    double ysel = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (l + 32 * t == bi) ysel = yl[t];
    ysel = warp_sum(ysel);   // exactly one lane holds it
    const double sgn = ysel < 0.0 ? -1.0 : 1.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = l + 32 * t;
      if (i < B) {
        const double vi = sgn * yl[t];
        ws.vtop[(size_t)i * B + kdesc] = vi;
        if (V) V[(size_t)i * ldv + (kdesc - k0)] = vi;
        const double si = sigma[i];
        W[(size_t)i * ldwu + kdesc] = (float)(vi / si);
        U[(size_t)i * ldwu + kdesc] = (float)(vi * si);
      }
    }
    if (l == 0) {
      ws.lam_top[kdesc] = lam;
      if (lam_out) lam_out[kdesc] = lam;
    }
  }
  if (blockIdx.x == 0) stamp(7);
}

// =====================================================================
// K2e: re-orthogonalise numerically coincident eigenvalues (usually no-op)
// =====================================================================
__global__ void __launch_bounds__(256) reorth_kernel(const double* __restrict__ tri, EigWs ws,
                                                     const double* __restrict__ sigma, int B, int k0, int K,
                                                     double* V, int ldv, float* W, float* U, int ldwu) {
  const double tnorm = fmax(fabs(tri[3 * B]), fabs(tri[3 * B + 1]));
  const int l = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  for (int j = max(k0, 1); j < k0 + K; ++j) {
    bool touched = false;
    for (int i = 0; i < j; ++i) {
      if (fabs(ws.lam_top[i] - ws.lam_top[j]) > 1e-9 * tnorm) continue;
      double dot = 0.0;
      for (int t = l; t < B; t += 32) dot = fma(ws.vtop[(size_t)t * B + i], ws.vtop[(size_t)t * B + j], dot);
      dot = warp_sum(dot);
      for (int t = l; t < B; t += 32) ws.vtop[(size_t)t * B + j] -= dot * ws.vtop[(size_t)t * B + i];
      __syncwarp();
      touched = true;
    }
    if (!touched) continue;
    double s = 0.0;
    for (int t = l; t < B; t += 32) s = fma(ws.vtop[(size_t)t * B + j], ws.vtop[(size_t)t * B + j], s);
    s = 1.0 / sqrt(warp_sum(s));
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int t = l; t < B; t += 32) {
      const double a = fabs(ws.vtop[(size_t)t * B + j]);
      if (a > best) { best = a; bi = t; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sg = ws.vtop[(size_t)bi * B + j] < 0.0 ? -s : s;
    __syncwarp();
    for (int t = l; t < B; t += 32) {
      const double vi = ws.vtop[(size_t)t * B + j] * sg;
      ws.vtop[(size_t)t * B + j] = vi;
      if (V && j >= k0) V[(size_t)t * ldv + (j - k0)] = vi;
      W[(size_t)t * ldwu + j] = (float)(vi / sigma[t]);
      U[(size_t)t * ldwu + j] = (float)(vi * sigma[t]);
    }
    __syncwarp();
  }
}

// residual_b = (M Y)_b / M_bb with M = (G + ridge I)^-1 (noise estimate output)
__global__ void __launch_bounds__(256) inverse_cols_kernel(EigWs ws, int B, double* Minv) {
  // column b of M = L^-T L^-1 e_b: one warp per column: x = L^-1 e_b, then M e_b = L^-T x
  __shared__ double xs[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + w;
  if (b >= B) return;
  double* x = xs[w];
  for (int i = l; i < B; i += 32) x[i] = 0.0;
  __syncwarp();
  const double* L = ws.Lp;
  for (int i = b; i < B; ++i) {
    double s = 0.0;
    for (int j = b + l; j < i; j += 32) s = fma(L[off(i) + j], x[j], s);
    s = warp_sum(s);
    if (l == 0) x[i] = ((i == b ? 1.0 : 0.0) - s) * ws.rdiag[i];
    __syncwarp();
  }
  // back substitution with L^T: z_i = (x_i - sum_{j>i} L_ji z_j) / L_ii
  for (int i = B - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1 + l; j < B; j += 32) s = fma(L[off(j) + i], x[j], s);
    s = warp_sum(s);
    if (l == 0) x[i] = (x[i] - s) * ws.rdiag[i];
    __syncwarp();
  }
  for (int i = l; i < B; i += 32) Minv[(size_t)i * B + b] = x[i];
}

__global__ void residual_kernel(const float* __restrict__ Y, long long n, int B, const double* __restrict__ M,
                                float* __restrict__ out) {
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
  return cudaMemcpyFromSymbol(out, g_eig_clk, sizeof(long long) * 16) == cudaSuccess ? HYDE_OK : HYDE_ECUDA;
}

static const size_t kMaxSmem = 227 * 1024 - 1024;   // dynamic budget (static smem is separate)

size_t eig_workspace_doubles(int B) {
  const size_t P = (size_t)B * (B + 1) / 2;
  return 3 * (size_t)B * B + 3 * (size_t)B + 8 + P + 64;
}

static cudaError_t run_chol(const double* G, int B, double ridge, const EigWs& ws, cudaStream_t st) {
  const size_t P = (size_t)B * (B + 1) / 2;
  const size_t smem = P * sizeof(double);
  cudaError_t e;
  if (smem <= kMaxSmem) {
    e = cudaFuncSetAttribute(chol_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    chol_kernel<true><<<1, CT, smem, st>>>(G, B, ridge, ws);
  } else {
    chol_kernel<false><<<1, CT, 0, st>>>(G, B, ridge, ws);
  }
  return cudaGetLastError();
}

static size_t eigpair_smem(int B) {
  return (size_t)B * 8 * sizeof(double) + (size_t)((B + 15) & ~15) + 2 * (size_t)RB * B * sizeof(double) + 64;
}

static cudaError_t run_eigpairs(const double* tri, const EigWs& ws, const double* sigma, int B, int k0, int K,
                                double* lam, double* V, int ldv, float* W, float* U, int ldwu, cudaStream_t st) {
  const size_t smem = eigpair_smem(B);
  cudaError_t e = cudaFuncSetAttribute(eigpair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  eigpair_kernel<<<K, EP_T, smem, st>>>(tri, ws, sigma, B, k0, 0, lam, V, ldv, W, U, ldwu);
  reorth_kernel<<<1, 256, 0, st>>>(tri, ws, sigma, B, k0, K, V, ldv, W, U, ldwu);
  return cudaGetLastError();
}

// sigma (+ optionally the eigenpairs of the first ncomp components; ncomp < 0 = sigma only)
cudaError_t launch_noise_eig(const double* G, long long n, int B, double ridge, int ncomp, int all_lam,
                             double* sigma, double* lam, double* V, double* house, double* tri, float* W, float* U,
                             int ldwu, cudaStream_t st) {
  const EigWs ws = carve(house, B);
  cudaError_t e = cudaMemsetAsync(ws.flags, 0, 8 * sizeof(double), st);
  if (e != cudaSuccess) return e;
  e = run_chol(G, B, ridge, ws, st);
  if (e != cudaSuccess) return e;
  invdiag_kernel<<<(B + 7) / 8, 256, 0, st>>>(ws, B, n, sigma);
  e = cudaGetLastError();
  if (e != cudaSuccess || ncomp < 0) return e;
  const size_t P = (size_t)B * (B + 1) / 2;
  const size_t ext = (size_t)(4 * B + TW + 8) * sizeof(double);
  if (ext + P * sizeof(double) <= kMaxSmem) {
    e = cudaFuncSetAttribute(tridiag_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(ext + P * sizeof(double)));
    if (e != cudaSuccess) return e;
    tridiag_kernel<true><<<1, TT, ext + P * sizeof(double), st>>>(G, sigma, n, B, ws, tri);
  } else {
    tridiag_kernel<false><<<1, TT, ext, st>>>(G, sigma, n, B, ws, tri);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (all_lam && lam) {
    const size_t smem = eigpair_smem(B);
    e = cudaFuncSetAttribute(eigpair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    eigpair_kernel<<<B, EP_T, smem, st>>>(tri, ws, sigma, B, 0, 1, lam, nullptr, 0, W, U, ldwu);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (ncomp > 0) return run_eigpairs(tri, ws, sigma, B, 0, ncomp, nullptr, V, ncomp, W, U, ldwu, st);
  return cudaSuccess;
}

cudaError_t launch_eigvec_more(const double* tri, const double* house, const double* sigma, int B, int k0,
                               int ncomp, double* lam_top_unused, double* V, float* W, float* U, int ldwu,
                               cudaStream_t st) {
  (void)lam_top_unused;
  const EigWs ws = carve(const_cast<double*>(house), B);
  return run_eigpairs(tri, ws, sigma, B, k0, ncomp, nullptr, V, ncomp, W, U, ldwu, st);
}

cudaError_t launch_noise_residual(const float* Y, long long n, int B, const double* G, double ridge, double* work,
                                  float* out, cudaStream_t st) {
  // work: the K2 buffer (Cholesky factor already computed by launch_noise_eig) + B*B for M
  (void)G;
  (void)ridge;
  const EigWs ws = carve(work, B);
  double* M = ws.Aw;   // P >= ... use the trailing region (B*B doubles needed)
  inverse_cols_kernel<<<(B + 7) / 8, 256, 0, st>>>(ws, B, M);
  dim3 grid((unsigned)((n + 255) / 256), B);
  residual_kernel<<<grid, 256, 0, st>>>(Y, n, B, M, out);
  return cudaGetLastError();
}
