// F4 (SURVEY.md §8(f) NEXT; SPEC.md:397-405, :433 D17; §2.1
// "Wavelet-Based Sparse Reduced-Rank Regression"): min_{C,V} ||W - C V^T||^2 +
// lam ||C||_1, V^T V = I, W (N_c x B) the per-band DWT coefficients (stored
// band-major: B rows of N_c).  Per sweep: C = soft(W V, lam/2) (K3's
// projection kernel + the fused soft/statistics kernel here), M = W^T C
// (wtc: one read of W, C staged in shared memory), V = M (M^T M)^-1/2 -- the
// orthogonal polar factor P Q^T of M = P S Q^T, from the r x r eigenproblem of
// M^T M (cyclic Jacobi, r <= 32) -- and the objective
// ||W||^2 - 2 tr(V^T M) + ||C||^2 + lam ||C||_1 (V^T V = I).
#include "common.cuh"

namespace {

constexpr int NT = 256;
// coefficients per wtc chunk (C chunk staged in dynamic shared memory: R x JC floats)
template <int R> __host__ __device__ constexpr int jc() { return R <= 8 ? 4096 : 1536; }

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

// lam = sqrt(mean_b sigma_b^2) sqrt(2 ln N_c)  (D17 default)
__global__ void wsrrr_lambda_kernel(const double* sigma, int B, double nc, double* lam) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += sigma[b] * sigma[b];
  *lam = sqrt(s / B) * sqrt(2.0 * log(nc));
}

// per-CTA fp64 partial sums of x^2 (fixed order), then one CTA adds them.
// 16-byte loads, four in flight per thread, over SUMSQ_CTAS CTAs (8 per SM: a
// 940 MB stream needs ~40 KB in flight per SM; 296 CTAs of four scalar loads
// per thread ran at 4.3 TB/s)
constexpr int SUMSQ_CTAS = 1184;
__global__ void __launch_bounds__(NT) sumsq_kernel(const float* __restrict__ x, long long n, double* partial) {
  __shared__ double red[NT / 32];
  double s = 0.0;
  const long long G = (long long)gridDim.x * NT;
  const long long tid = blockIdx.x * (long long)NT + threadIdx.x;
  const bool vec = ((reinterpret_cast<unsigned long long>(x) & 15) == 0);
  const long long n4 = vec ? n / 4 : 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  long long i = tid;
  for (; i + 3 * G < n4; i += 4 * G) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + i + u * G);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s = fma((double)v[u].x, (double)v[u].x, s);
      s = fma((double)v[u].y, (double)v[u].y, s);
      s = fma((double)v[u].z, (double)v[u].z, s);
      s = fma((double)v[u].w, (double)v[u].w, s);
    }
  }
  for (; i < n4; i += G) {
    const float4 v = __ldcs(x4 + i);
    s = fma((double)v.x, (double)v.x, s);
    s = fma((double)v.y, (double)v.y, s);
    s = fma((double)v.z, (double)v.z, s);
    s = fma((double)v.w, (double)v.w, s);
  }
  for (long long k = 4 * n4 + tid; k < n; k += G) {
    const double v = x[k];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void __launch_bounds__(NT) reduce_kernel(const double* partial, int np, double* out) {
  __shared__ double red[NT / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += NT) s += partial[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// C <- soft(C, lam/2) in place; per-CTA partials of ||C||^2 and ||C||_1
__global__ void __launch_bounds__(NT) soft_stats_kernel(float* __restrict__ c, long long n, const double* lam,
                                                        double* p2, double* p1) {
  __shared__ double red[NT / 32];
  const float t = (float)(0.5 * *lam);
  double s2 = 0.0, s1 = 0.0;
  for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) {
    const float v = c[i];
    const float a = fmaxf(fabsf(v) - t, 0.f);
    const float o = copysignf(a, v);
    c[i] = o;
    s2 = fma((double)a, (double)a, s2);
    s1 += (double)a;
  }
  s2 = block_sum(s2, red);
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) { p2[blockIdx.x] = s2; p1[blockIdx.x] = s1; }
}

// partial[chunk][b][k] = sum_{j in chunk} W[b][j] C[k][j]: C chunk in shared
// memory, warp w takes bands w, w+8, ..., lanes stride the chunk, fp64 accumulators
template <int R>
__global__ void __launch_bounds__(NT) wtc_kernel(const float* __restrict__ W, const float* __restrict__ C,
                                                 long long nc, int B, int r, double* __restrict__ partial) {
  constexpr int JC = jc<R>();
  extern __shared__ float csm[];
  float (*cs)[JC] = reinterpret_cast<float (*)[JC]>(csm);
  const long long j0 = (long long)blockIdx.x * JC;
  const int len = (int)min((long long)JC, nc - j0);
  for (int x = threadIdx.x; x < r * JC; x += NT) {
    const int k = x / JC, j = x - k * JC;
    cs[k][j] = j < len ? C[(size_t)k * nc + j0 + j] : 0.f;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int b = w; b < B; b += NT / 32) {
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    const float* wr = W + (size_t)b * nc + j0;
    int j = l;
    // four loads of the band row in flight per lane (same accumulation order)
    for (; j + 96 < len; j += 128) {
      float w4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w4[u] = __ldg(wr + j + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double wv = w4[u];
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < r) acc[k] = fma(wv, (double)cs[k][j + 32 * u], acc[k]);
      }
    }
    for (; j < len; j += 32) {
      const double wv = wr[j];
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) acc[k] = fma(wv, (double)cs[k][j], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double v = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0 && k < r) partial[((size_t)blockIdx.x * B + b) * r + k] = v;
    }
  }
}

__global__ void __launch_bounds__(NT) wtc_reduce_kernel(const double* partial, int nchunk, int Br, double* M) {
  const int x = blockIdx.x * NT + threadIdx.x;
  if (x >= Br) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += partial[(size_t)c * Br + x];
  M[x] = s;
}

// V = M (M^T M)^-1/2 (polar factor), single CTA; r <= 32.  Also the objective
// f = ||W||^2 - 2 tr(V^T M) + ||C||^2 + lam ||C||_1 into *f, V^T as fp32 for K3.
__global__ void __launch_bounds__(NT) procrustes_kernel(const double* __restrict__ M, int B, int r,
                                                        double* __restrict__ V, float* __restrict__ V32, int ldv32,
                                                        const double* w2, const double* c2, const double* c1,
                                                        const double* lam, double* f) {
  __shared__ double S[32][33], Q[32][33], T[32][33];
  __shared__ double ev[32];
  __shared__ double red[NT / 32];
  const int tid = threadIdx.x;
  for (int x = tid; x < r * r; x += NT) {   // S = M^T M
    const int a = x / r, b = x % r;
    double s = 0.0;
    for (int i = 0; i < B; ++i) s = fma(M[(size_t)i * r + a], M[(size_t)i * r + b], s);
    S[a][b] = s;
    Q[a][b] = a == b ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {   // cyclic Jacobi on the r x r symmetric S (tiny)
    for (int sweep = 0; sweep < 60; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (int a = 0; a < r; ++a)
        for (int b = 0; b < r; ++b) { tot += S[a][b] * S[a][b]; if (a != b) off += S[a][b] * S[a][b]; }
      if (off <= 1e-30 * tot) break;
      for (int p = 0; p < r - 1; ++p)
        for (int q = p + 1; q < r; ++q) {
          const double apq = S[p][q];
          if (fabs(apq) < 1e-300) continue;
          const double theta = (S[q][q] - S[p][p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
          for (int k = 0; k < r; ++k) {
            const double skp = S[k][p], skq = S[k][q];
            S[k][p] = c * skp - s * skq;
            S[k][q] = s * skp + c * skq;
          }
          for (int k = 0; k < r; ++k) {
            const double spk = S[p][k], sqk = S[q][k];
            S[p][k] = c * spk - s * sqk;
            S[q][k] = s * spk + c * sqk;
          }
          for (int k = 0; k < r; ++k) {
            const double qkp = Q[k][p], qkq = Q[k][q];
            Q[k][p] = c * qkp - s * qkq;
            Q[k][q] = s * qkp + c * qkq;
          }
        }
    }
    double mx = 0.0;
    for (int a = 0; a < r; ++a) mx = fmax(mx, S[a][a]);
    for (int a = 0; a < r; ++a) ev[a] = S[a][a] > 1e-30 * mx ? 1.0 / sqrt(S[a][a]) : 0.0;
  }
  __syncthreads();
  for (int x = tid; x < r * r; x += NT) {   // T = Q diag(ev) Q^T
    const int a = x / r, b = x % r;
    double s = 0.0;
    for (int k = 0; k < r; ++k) s += Q[a][k] * ev[k] * Q[b][k];
    T[a][b] = s;
  }
  __syncthreads();
  double tr = 0.0;
  for (int x = tid; x < B * r; x += NT) {   // V = M T
    const int i = x / r, b = x % r;
    double s = 0.0;
    for (int k = 0; k < r; ++k) s = fma(M[(size_t)i * r + k], T[k][b], s);
    V[x] = s;
    V32[(size_t)i * ldv32 + b] = (float)s;
    tr = fma(s, M[x], tr);
  }
  tr = block_sum(tr, red);
  if (tid == 0) *f = *w2 - 2.0 * tr + *c2 + *lam * *c1;
}

// fp32 copy of V (B x r) with leading dimension ld
__global__ void v32_kernel(const double* V, int B, int r, float* V32, int ld) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < B * r) V32[(size_t)(x / r) * ld + x % r] = (float)V[x];
}

}  // namespace

cudaError_t launch_wsrrr_lambda(const double* sigma, int B, long long nc, double* lam, cudaStream_t st) {
  wsrrr_lambda_kernel<<<1, 32, 0, st>>>(sigma, B, (double)nc, lam);
  return cudaGetLastError();
}

// *out = sum x^2 (fp64, fixed order); partial: >= SUMSQ_CTAS doubles
cudaError_t launch_sumsq(const float* x, long long n, double* partial, double* out, cudaStream_t st) {
  sumsq_kernel<<<SUMSQ_CTAS, NT, 0, st>>>(x, n, partial);
  reduce_kernel<<<1, NT, 0, st>>>(partial, SUMSQ_CTAS, out);
  return cudaGetLastError();
}

// partial: >= 2 * 296 doubles; c2 / c1 sums into c2, c1
cudaError_t launch_soft_stats(float* c, long long n, const double* lam, double* partial, double* c2, double* c1,
                              cudaStream_t st) {
  soft_stats_kernel<<<296, NT, 0, st>>>(c, n, lam, partial, partial + 296);
  reduce_kernel<<<1, NT, 0, st>>>(partial, 296, c2);
  reduce_kernel<<<1, NT, 0, st>>>(partial + 296, 296, c1);
  return cudaGetLastError();
}

int wtc_chunks(long long nc, int r) {
  const int J = r <= 8 ? jc<8>() : jc<32>();
  return (int)((nc + J - 1) / J);
}

// M (B x r row-major) = W^T C; partial: wtc_chunks(nc, r) * B * r doubles
cudaError_t launch_wtc(const float* W, const float* C, long long nc, int B, int r, double* partial, double* M,
                       cudaStream_t st) {
  const int nch = wtc_chunks(nc, r);
  cudaError_t e;
  if (r <= 8) {
    const int sm = r * jc<8>() * 4;   // only the r live rows of the C chunk
    // instantiation by the live rank (the accumulators of a wider one are predicated off)
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      if (e2 != cudaSuccess) return e2;
      kern<<<nch, NT, sm, st>>>(W, C, nc, B, r, partial);
      return cudaGetLastError();
    };
    e = r == 1 ? go(wtc_kernel<1>) : r == 2 ? go(wtc_kernel<2>) : r <= 4 ? go(wtc_kernel<4>) : go(wtc_kernel<8>);
    if (e != cudaSuccess) return e;
  } else if (r <= 32) {
    const int sm = r * jc<32>() * 4;
    e = cudaFuncSetAttribute(wtc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    wtc_kernel<32><<<nch, NT, sm, st>>>(W, C, nc, B, r, partial);
  } else {
    return cudaErrorInvalidValue;
  }
  wtc_reduce_kernel<<<(B * r + NT - 1) / NT, NT, 0, st>>>(partial, nch, B * r, M);
  return cudaGetLastError();
}

cudaError_t launch_procrustes(const double* M, int B, int r, double* V, float* V32, int ldv32, const double* w2,
                              const double* c2, const double* c1, const double* lam, double* f, cudaStream_t st) {
  if (r > 32) return cudaErrorInvalidValue;
  procrustes_kernel<<<1, NT, 0, st>>>(M, B, r, V, V32, ldv32, w2, c2, c1, lam, f);
  return cudaGetLastError();
}

cudaError_t launch_v32(const double* V, int B, int r, float* V32, int ld, cudaStream_t st) {
  v32_kernel<<<(B * r + 255) / 256, 256, 0, st>>>(V, B, r, V32, ld);
  return cudaGetLastError();
}
