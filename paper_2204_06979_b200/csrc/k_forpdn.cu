// F2 (SURVEY.md §8(f) NEXT; SPEC.md:388-396, :432 D16; "FORPDN is a
// full-rank, wavelet-based method"): X = W (I + lam D^T D)^-1 with W the
// per-band DWT coefficients (N_c x B) and D the first-order spectral
// difference.  A = I + lam D^T D is TRIDIAGONAL (diagonal 1+lam, 1+2lam, ...,
// 1+2lam, 1+lam; off-diagonals -lam), symmetric and strictly diagonally
// dominant, so every coefficient row is one Thomas solve along the bands --
// O(B) per row instead of the dense N_c x B x B product, no pivoting needed.
//
// Default lam (D16): the grid value whose coefficient-domain residual power
// ||W - W A^-1||^2 / (N B) = trace(K^2 G_W) / (N B), K = I - A^-1 and
// G_W = W^T W (the band Gram of the coefficients -- equal to K1's G when the
// DWT is orthonormal on the image, i.e. 2^L divides R and C), is closest to
// HySime's noise power trace(R_n) / B, R_n,bb = (M_bb - delta (M^2)_bb) /
// (M_bb^2 N) (F1 identity).  All of it is O(B^3) on B x B matrices.
#include "common.cuh"

namespace {

constexpr int NT = 256;
constexpr int NGRID = 4;
__constant__ double kGrid[NGRID] = {0.1, 1.0, 10.0, 100.0};

// Thomas factors of A(lam): inv_m[i] = 1 / (b_i - a_i c'_{i-1}), cp[i] = c'_i
__device__ void thomas_factor(int B, double lam, double* inv_m, double* cp) {
  double cprev = 0.0;
  for (int i = 0; i < B; ++i) {
    const double bi = (i == 0 || i == B - 1) ? 1.0 + lam : 1.0 + 2.0 * lam;
    const double ai = i > 0 ? -lam : 0.0;
    const double m = bi - ai * cprev;
    inv_m[i] = 1.0 / m;
    cprev = (i < B - 1 ? -lam : 0.0) / m;
    cp[i] = cprev;
  }
}

// noise power (HySime): mean_b (M_bb - delta (M^2)_bb) / (M_bb^2 N)
__global__ void __launch_bounds__(NT) noise_power_kernel(const double* __restrict__ M, int B, double n, double ridge,
                                                         double* out) {
  __shared__ double red[NT / 32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < B; b += NT) {
    double m2 = 0.0;
    for (int k = 0; k < B; ++k) m2 = fma(M[(size_t)b * B + k], M[(size_t)k * B + b], m2);
    const double mbb = M[(size_t)b * B + b];
    acc += (mbb - ridge * m2) / (mbb * mbb * n);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    *out = t / B;
  }
}

// one CTA per grid value, one thread per column j of G_W:
//   trace(K^2 G) = trace(G) - 2 trace(A^-1 G) + trace(A^-1 A^-1 G),
// z_j = A^-1 g_j and y_j = A^-1 z_j by two in-place Thomas solves on the
// column (scratch Z: NGRID x B x B doubles); rp[g] = trace(K^2 G_W) / (N B)
__global__ void __launch_bounds__(NT) lambda_residual_kernel(const double* __restrict__ Gw, int B, double n,
                                                             double* __restrict__ Zs, double* rp) {
  __shared__ double inv_m[256], cp[256];
  __shared__ double red[NT / 32];
  const double lam = kGrid[blockIdx.x];
  if (threadIdx.x == 0) thomas_factor(B, lam, inv_m, cp);
  __syncthreads();
  double* Z = Zs + (size_t)blockIdx.x * B * B;
  double acc = 0.0;
  const int j = threadIdx.x;
  if (j < B) {
    auto solve = [&]() {   // column j of Z in place: Z[:, j] <- A^-1 Z[:, j]
      double d = 0.0;
      for (int i = 0; i < B; ++i) {
        d = (Z[(size_t)i * B + j] + (i > 0 ? lam * d : 0.0)) * inv_m[i];
        Z[(size_t)i * B + j] = d;
      }
      double x = d;
      for (int i = B - 2; i >= 0; --i) {
        x = Z[(size_t)i * B + j] - cp[i] * x;
        Z[(size_t)i * B + j] = x;
      }
    };
    for (int i = 0; i < B; ++i) Z[(size_t)i * B + j] = Gw[(size_t)i * B + j];
    const double gjj = Gw[(size_t)j * B + j];
    solve();
    const double zjj = Z[(size_t)j * B + j];
    solve();
    const double yjj = Z[(size_t)j * B + j];
    acc = gjj - 2.0 * zjj + yjj;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    rp[blockIdx.x] = t / (n * B);
  }
}

// lam* = the grid value with the residual power closest to the noise power (first on ties)
__global__ void lambda_pick_kernel(const double* rp, const double* npow, double* lam_out) {
  if (threadIdx.x != 0) return;
  int best = 0;
  for (int g = 1; g < NGRID; ++g)
    if (fabs(rp[g] - *npow) < fabs(rp[best] - *npow)) best = g;
  *lam_out = kGrid[best];
}

// X = W A^-1 in place, one coefficient index per thread: Thomas forward sweep
// (d' written over W), backward sweep (x written over d').  C is band-major
// (B rows of ldc coefficients): consecutive threads read consecutive
// coefficients of a band.  lam from device memory (the picked value) or the
// argument when lam_dev is NULL.
__global__ void __launch_bounds__(NT) thomas_solve_kernel(float* __restrict__ C, long long ldc, long long nc, int B,
                                                          double lam_arg, const double* __restrict__ lam_dev) {
  __shared__ float s_inv_m[256], s_cp[256];
  __shared__ float s_lam;
  if (threadIdx.x == 0) {
    const double lam = lam_dev ? *lam_dev : lam_arg;
    double cprev = 0.0;
    for (int i = 0; i < B; ++i) {
      const double bi = (i == 0 || i == B - 1) ? 1.0 + lam : 1.0 + 2.0 * lam;
      const double m = bi + (i > 0 ? lam * cprev : 0.0);
      s_inv_m[i] = (float)(1.0 / m);
      cprev = (i < B - 1 ? -lam : 0.0) / m;
      s_cp[i] = (float)cprev;
    }
    s_lam = (float)lam;
  }
  __syncthreads();
  const long long j = blockIdx.x * (long long)NT + threadIdx.x;
  if (j >= nc) return;
  const float lam = s_lam;
  float* col = C + j;
  // forward: d'_i = (w_i + lam d'_{i-1}) / m_i, loads issued 8 bands ahead
  constexpr int PF = 8;
  float buf[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) buf[u] = u < B ? __ldcg(col + (long long)u * ldc) : 0.f;
  float d = 0.f;
  for (int i0 = 0; i0 < B; i0 += PF) {
    float nxt[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int i = i0 + PF + u;
      nxt[u] = i < B ? __ldcg(col + (long long)i * ldc) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int i = i0 + u;
      if (i < B) {
        d = fmaf(lam, d, buf[u]) * s_inv_m[i];
        col[(long long)i * ldc] = d;
      }
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) buf[u] = nxt[u];
  }
  // backward: x_i = d'_i - c'_i x_{i+1}
  float x = d;
  for (int i = B - 2; i >= 0; --i) {
    x = fmaf(-s_cp[i], x, __ldcg(col + (long long)i * ldc));
    col[(long long)i * ldc] = x;
  }
}

}  // namespace

// Zs: scratch of 4 B^2 doubles
cudaError_t launch_forpdn_lambda(const double* M, const double* Gw, int B, long long n, double ridge, double* npow,
                                 double* rp, double* lam_out, double* Zs, cudaStream_t st) {
  if (B > 256) return cudaErrorInvalidValue;
  noise_power_kernel<<<1, NT, 0, st>>>(M, B, (double)n, ridge, npow);
  lambda_residual_kernel<<<NGRID, NT, 0, st>>>(Gw, B, (double)n, Zs, rp);
  lambda_pick_kernel<<<1, 32, 0, st>>>(rp, npow, lam_out);
  return cudaGetLastError();
}

cudaError_t launch_forpdn_solve(float* C, long long ldc, long long nc, int B, double lam, const double* lam_dev,
                                cudaStream_t st) {
  const unsigned blocks = (unsigned)((nc + NT - 1) / NT);
  thomas_solve_kernel<<<blocks, NT, 0, st>>>(C, ldc, nc, B, lam, lam_dev);
  return cudaGetLastError();
}
