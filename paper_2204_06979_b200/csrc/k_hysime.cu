// F1 (the first NEXT row; PAPER.md:105-106
// "HySime ... implemented in HyDe"): HySime signal-subspace identification on
// the same A1/A2 data as HyRes.
//   R_y = G / N  (G = Y Y^T, K1's exact-integer Gram)
//   R_n = N~ N~^T / N with N~_b = (M Y)_b / M_bb the regression residual of
//         band b on all others, M = (G + delta I)^-1 (K2's sweep).  Without a
//         second pass over the cube: N~ N~^T = D^-1 M G M D^-1 and
//         M G M = M (M^-1 - delta I) M = M - delta M^2, so
//         R_n = D^-1 (M - delta M^2) D^-1 / N,  D = diag(M);
//   R_x = R_y - R_n = E diag(mu) E^T  (K2 in raw mode + more eigenpairs);
//   p_i = e_i^T R_y e_i, s_i^2 = e_i^T R_n e_i, delta_i = -p_i + 2 s_i^2;
//   k = #{delta_i < -1e-9 max|p|} (R13), basis = those e_i in
//   ascending-delta order.
#include "common.cuh"

namespace {

constexpr int NT = 256;

// one thread per (i, j); the pair is evaluated as (min, max) so R_n and R_x
// are exactly symmetric
__global__ void hysime_prep_kernel(const double* __restrict__ G, const double* __restrict__ M, int B, double n,
                                   double ridge, double* __restrict__ Ry, double* __restrict__ Rn,
                                   double* __restrict__ Rx) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * B) return;
  const int i0 = idx / B, j0 = idx % B;
  const int i = min(i0, j0), j = max(i0, j0);
  double m2 = 0.0;
  for (int k = 0; k < B; ++k) m2 = fma(M[(size_t)i * B + k], M[(size_t)k * B + j], m2);
  const double mij = 0.5 * (M[(size_t)i * B + j] + M[(size_t)j * B + i]);
  const double rn = (mij - ridge * m2) / (M[(size_t)i * B + i] * M[(size_t)j * B + j] * n);
  const double ry = 0.5 * (G[(size_t)i * B + j] + G[(size_t)j * B + i]) / n;
  Ry[idx] = ry;
  Rn[idx] = rn;
  Rx[idx] = ry - rn;
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < NT / 32; ++w) t += red[w];
  return t;
}

// one CTA per eigenvector c (column c of V, row-major B x ldv): p_c, s_c^2, delta_c
__global__ void __launch_bounds__(NT) hysime_delta_kernel(const double* __restrict__ V, int ldv,
                                                          const double* __restrict__ Ry,
                                                          const double* __restrict__ Rn, int B, double* p,
                                                          double* s2, double* delta) {
  __shared__ double v[256];
  __shared__ double red[NT / 32];
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < B; i += NT) v[i] = V[(size_t)i * ldv + c];
  __syncthreads();
  double ay = 0.0, an = 0.0;
  for (int i = threadIdx.x; i < B; i += NT) {
    double wy = 0.0, wn = 0.0;
    for (int k = 0; k < B; ++k) {
      wy = fma(Ry[(size_t)i * B + k], v[k], wy);
      wn = fma(Rn[(size_t)i * B + k], v[k], wn);
    }
    ay = fma(v[i], wy, ay);
    an = fma(v[i], wn, an);
  }
  const double py = block_sum(ay, red);
  const double pn = block_sum(an, red);
  if (threadIdx.x == 0) {
    p[c] = py;
    s2[c] = pn;
    delta[c] = -py + 2.0 * pn;
  }
}

// one CTA: k and the basis (columns of V in ascending-delta order, stable)
__global__ void __launch_bounds__(NT) hysime_select_kernel(const double* __restrict__ delta,
                                                           const double* __restrict__ p, int B, double tol_rel,
                                                           const double* __restrict__ V, int ldv,
                                                           double* __restrict__ basis, int* k_out) {
  __shared__ double red[NT / 32];
  __shared__ int rank_of[256];
  double pm = 0.0;
  for (int i = threadIdx.x; i < B; i += NT) pm = fmax(pm, fabs(p[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pm;
  __syncthreads();
  double tol = 0.0;
  for (int w = 0; w < NT / 32; ++w) tol = fmax(tol, red[w]);
  tol *= tol_rel;
  int kk = 0;
  for (int i = threadIdx.x; i < B; i += NT) {
    const double di = delta[i];
    int r = 0;
    for (int j = 0; j < B; ++j) {
      const double dj = delta[j];
      r += (dj < di || (dj == di && j < i)) ? 1 : 0;
    }
    rank_of[i] = r;
    kk += di < -tol ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = (double)kk;
  __syncthreads();
  int k = 0;
  for (int w = 0; w < NT / 32; ++w) k += (int)red[w];
  if (threadIdx.x == 0) *k_out = k;
  if (basis)
    for (int x = threadIdx.x; x < B * B; x += NT) {
      const int i = x / B, c = x % B;   // basis[i][rank_of[c]] = V[i][c] for the selected c
      const int r = rank_of[c];
      if (r < k) basis[(size_t)i * B + r] = V[(size_t)i * ldv + c];
    }
}

// l = the smallest eigenvalue of R_n (lam_n[B-1], from the raw-mode bisection)
// and m = #{mu_i > l (1 - 1e-6)}: an eigenvector of R_x with mu_i <= l has
// delta_i = s_i^2 - mu_i >= l - mu_i >= 0 (p_i = mu_i + s_i^2, s_i^2 >= l), so it
// can never be selected and needs no eigenvector
__global__ void hysime_bound_kernel(const double* __restrict__ lam_n, const double* __restrict__ mu, int B,
                                    double* lb, int* m_out) {
  if (threadIdx.x != 0) return;
  const double l = lam_n[B - 1];
  int m = B;
  if (l > 0.0) {
    const double cut = l * (1.0 - 1e-6);
    m = 0;
    for (int i = 0; i < B; ++i) m += mu[i] > cut ? 1 : 0;
  }
  *lb = l;
  *m_out = m;
}

// delta_i = l - mu_i (a lower bound, >= 0) for the eigenpairs without a vector
__global__ void hysime_fill_kernel(const double* mu, const double* lb, int m, int B, double* p, double* delta) {
  const int i = m + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  delta[i] = *lb - mu[i];
  p[i] = 0.0;
}

}  // namespace

cudaError_t launch_hysime_bound(const double* lam_n, const double* mu, int B, double* lb, int* m_out, cudaStream_t st) {
  hysime_bound_kernel<<<1, 32, 0, st>>>(lam_n, mu, B, lb, m_out);
  return cudaGetLastError();
}

cudaError_t launch_hysime_fill(const double* mu, const double* lb, int m, int B, double* p, double* delta,
                               cudaStream_t st) {
  if (m >= B) return cudaSuccess;
  hysime_fill_kernel<<<(B - m + 255) / 256, 256, 0, st>>>(mu, lb, m, B, p, delta);
  return cudaGetLastError();
}

cudaError_t launch_hysime_prep(const double* G, const double* M, int B, long long n, double ridge, double* Ry,
                               double* Rn, double* Rx, cudaStream_t st) {
  const int tot = B * B;
  hysime_prep_kernel<<<(tot + NT - 1) / NT, NT, 0, st>>>(G, M, B, (double)n, ridge, Ry, Rn, Rx);
  return cudaGetLastError();
}

cudaError_t launch_hysime_delta(const double* V, int ldv, const double* Ry, const double* Rn, int B, double* p,
                                double* s2, double* delta, cudaStream_t st, int ncols) {
  hysime_delta_kernel<<<ncols > 0 ? ncols : B, NT, 0, st>>>(V, ldv, Ry, Rn, B, p, s2, delta);
  return cudaGetLastError();
}

cudaError_t launch_hysime_select(const double* delta, const double* p, int B, double tol_rel, const double* V,
                                 int ldv, double* basis, int* k_out, cudaStream_t st) {
  hysime_select_kernel<<<1, NT, 0, st>>>(delta, p, B, tol_rel, V, ldv, basis, k_out);
  return cudaGetLastError();
}
