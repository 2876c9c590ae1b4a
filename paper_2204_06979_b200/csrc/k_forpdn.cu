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

// noise power (HySime): mean_b (M_bb - delta (M^2)_bb) / (M_bb^2 N).  One CTA
// of 1024 threads, warp w takes rows b = w, w + 32, ...: lanes split k (all
// loads of a row in flight), a warp sum, then the per-warp partials in a fixed
// order.  (One thread per row walked 224 dependent-latency loads: 100 us.)
constexpr int NPT = 1024;
__global__ void __launch_bounds__(NPT) noise_power_kernel(const double* __restrict__ M, int B, double n, double ridge,
                                                          double* out) {
  __shared__ double red[NPT / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double acc = 0.0;
  for (int b = w; b < B; b += NPT / 32) {
    double m2 = 0.0;
    for (int k = l; k < B; k += 32) m2 = fma(M[(size_t)b * B + k], M[(size_t)k * B + b], m2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    const double mbb = M[(size_t)b * B + b];
    acc += (mbb - ridge * m2) / (mbb * mbb * n);   // same value in every lane
  }
  if (l == 0) red[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < NPT / 32; ++q) t += red[q];
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
    // column j of Z in place: Z[:, j] <- A^-1 Z[:, j].  Both sweeps in blocks
    // of LB rows with the next block's loads issued before this block's
    // stores (a load cannot be hoisted over a store to Z by the compiler: one
    // L2 round trip per row otherwise -- 200 us for the 4 grid values)
    constexpr int LB = 16;
    auto solve = [&]() {
      double d = 0.0;
      double zc[LB], zn[LB];
#pragma unroll
      for (int u = 0; u < LB; ++u) zc[u] = u < B ? Z[(size_t)u * B + j] : 0.0;
      for (int i0 = 0; i0 < B; i0 += LB) {
#pragma unroll
        for (int u = 0; u < LB; ++u) zn[u] = i0 + LB + u < B ? Z[(size_t)(i0 + LB + u) * B + j] : 0.0;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int i = i0 + u;
          if (i < B) {
            d = (zc[u] + (i > 0 ? lam * d : 0.0)) * inv_m[i];
            Z[(size_t)i * B + j] = d;
          }
        }
#pragma unroll
        for (int u = 0; u < LB; ++u) zc[u] = zn[u];
      }
      double x = d;
      // backward over rows B-2 .. 0, blocks from the top
#pragma unroll
      for (int u = 0; u < LB; ++u) zc[u] = B - 2 - u >= 0 ? Z[(size_t)(B - 2 - u) * B + j] : 0.0;
      for (int i1 = B - 2; i1 >= 0; i1 -= LB) {
#pragma unroll
        for (int u = 0; u < LB; ++u) zn[u] = i1 - LB - u >= 0 ? Z[(size_t)(i1 - LB - u) * B + j] : 0.0;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int i = i1 - u;
          if (i >= 0) {
            x = zc[u] - cp[i] * x;
            Z[(size_t)i * B + j] = x;
          }
        }
#pragma unroll
        for (int u = 0; u < LB; ++u) zc[u] = zn[u];
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

// X = W A^-1 in place.  A CTA takes 32 consecutive coefficients (the lanes)
// and all B bands: warp w owns the band segment [w SEG, (w+1) SEG) in
// registers (coalesced 128-byte band rows, every load of the tile in flight
// at once).  Thomas as two affine recurrences -- forward y_i = alpha_i
// (y_{i-1} + w_i), backward x_i = y_i - c'_i x_{i+1} -- composed per warp
// segment, chained across the 8 warps through shared memory, then applied:
// one read and one write of W.
constexpr int SEGMAX = 32;   // bands per warp (B <= 256)
// Thomas factors of A(lam) once per call: coef[0..256) = alpha_i, coef[256..512) = c'_i, coef[512] = lam
__global__ void thomas_factor_kernel(int B, double lam_arg, const double* __restrict__ lam_dev, float* coef) {
  if (threadIdx.x != 0) return;
  const double lam = lam_dev ? *lam_dev : lam_arg;
  double cprev = 0.0;
  for (int i = 0; i < 256; ++i) {
    if (i < B) {
      const double bi = (i == 0 || i == B - 1) ? 1.0 + lam : 1.0 + 2.0 * lam;
      const double m = bi + (i > 0 ? lam * cprev : 0.0);
      coef[i] = (float)(1.0 / m);
      cprev = (i < B - 1 ? -lam : 0.0) / m;
      coef[256 + i] = (float)cprev;
    } else {
      coef[i] = 0.f;
      coef[256 + i] = 0.f;
    }
  }
  coef[512] = (float)lam;
}

__global__ void __launch_bounds__(NT, 3) thomas_solve_kernel(float* __restrict__ C, long long ldc, long long nc, int B,
                                                          const float* __restrict__ coef) {
  __shared__ float s_alpha[256], s_cp[256];
  __shared__ float s_P[8][32], s_Q[8][32];
  {
    s_alpha[threadIdx.x] = coef[threadIdx.x];
    s_cp[threadIdx.x] = coef[256 + threadIdx.x];
  }
  __syncthreads();
  const float lamf = coef[512];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int seg = (B + 7) / 8;
  const int b0 = w * seg;
  const long long j = blockIdx.x * 32LL + l;
  const bool ok = j < nc;
  float v[SEGMAX];
#pragma unroll
  for (int s = 0; s < SEGMAX; ++s) {
    const int i = b0 + s;
    v[s] = (s < seg && i < B && ok) ? C[(size_t)i * ldc + j] : 0.f;
  }
  // forward: y_i = a_i y_{i-1} + a_i lam... (sub-diagonal -lam): y_i = a_i (w_i + lam y_{i-1})
  float P = 1.f, Q = 0.f;
#pragma unroll
  for (int s = 0; s < SEGMAX; ++s) {
    const int i = b0 + s;
    if (s < seg && i < B) {
      const float a = s_alpha[i];
      Q = a * fmaf(lamf, Q, v[s]);
      P = a * lamf * P;
    }
  }
  s_P[w][l] = P;
  s_Q[w][l] = Q;
  __syncthreads();
  float y = 0.f;   // y at the end of the previous segment
  for (int u = 0; u < w; ++u) y = fmaf(s_P[u][l], y, s_Q[u][l]);
#pragma unroll
  for (int s = 0; s < SEGMAX; ++s) {
    const int i = b0 + s;
    if (s < seg && i < B) {
      y = s_alpha[i] * fmaf(lamf, y, v[s]);
      v[s] = y;
    }
  }
  __syncthreads();
  // backward: x_i = y_i - c'_i x_{i+1}
  P = 1.f;
  Q = 0.f;
#pragma unroll
  for (int s = SEGMAX - 1; s >= 0; --s) {
    const int i = b0 + s;
    if (s < seg && i < B) {
      Q = fmaf(-s_cp[i], Q, v[s]);
      P = -s_cp[i] * P;
    }
  }
  s_P[w][l] = P;
  s_Q[w][l] = Q;
  __syncthreads();
  float x = 0.f;   // x at the start of the next segment
  for (int u = 7; u > w; --u) x = fmaf(s_P[u][l], x, s_Q[u][l]);
#pragma unroll
  for (int s = SEGMAX - 1; s >= 0; --s) {
    const int i = b0 + s;
    if (s < seg && i < B) {
      x = fmaf(-s_cp[i], x, v[s]);
      if (ok) C[(size_t)i * ldc + j] = x;
    }
  }
}

}  // namespace

// Zs: scratch of 4 B^2 doubles
cudaError_t launch_forpdn_lambda(const double* M, const double* Gw, int B, long long n, double ridge, double* npow,
                                 double* rp, double* lam_out, double* Zs, cudaStream_t st) {
  if (B > 256) return cudaErrorInvalidValue;
  noise_power_kernel<<<1, NPT, 0, st>>>(M, B, (double)n, ridge, npow);
  lambda_residual_kernel<<<NGRID, NT, 0, st>>>(Gw, B, (double)n, Zs, rp);
  lambda_pick_kernel<<<1, 32, 0, st>>>(rp, npow, lam_out);
  return cudaGetLastError();
}

// coef: device scratch of 513 floats
cudaError_t launch_forpdn_solve(float* C, long long ldc, long long nc, int B, double lam, const double* lam_dev,
                                float* coef, cudaStream_t st) {
  if (B > 8 * SEGMAX) return cudaErrorInvalidValue;
  thomas_factor_kernel<<<1, 32, 0, st>>>(B, lam, lam_dev, coef);
  const unsigned blocks = (unsigned)((nc + 31) / 32);
  thomas_solve_kernel<<<blocks, NT, 0, st>>>(C, ldc, nc, B, coef);
  return cudaGetLastError();
}
