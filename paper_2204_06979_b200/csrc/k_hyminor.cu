// F3 (SPEC.md:415-423 D19; §2.1 "the remaining
// sparse noise is removed by solving an l1-l1 optimization problem with a
// modified split-Bregman technique"): per pixel spectrum m (B bands) of the
// HyRes output, min_x ||m - x||_1 + lam ||D x||_1 by split Bregman
// (a = x - m, d = D x):
//   x = (I + D^T D)^-1 (a + m - b_a + D^T (d - b_d))
//   a = shrink(x - m + b_a, 1/mu), b_a += x - m - a
//   d = shrink(D x + b_d, lam/mu), b_d += D x - d
// ONE WARP PER PIXEL, the whole state in registers: lane l owns the S = B/32
// consecutive bands [l S, l S + S).  The tridiagonal x-update (I + D^T D is
// tridiagonal, strictly diagonally dominant) is the Thomas algorithm written
// as two first-order affine recurrences -- forward y_i = alpha_i (y_{i-1} +
// r_i), backward x_i = y_i - c'_i x_{i+1} -- each evaluated as a lane-local
// composition of affine maps plus a 5-step warp scan (no shared memory, no
// serial 224-step chain).  A pixel stops when ||x_new - x_old|| <= tol ||x_old||.
#include "common.cuh"

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NT = 256;

__device__ __forceinline__ float shrinkf(float v, float t) { return copysignf(fmaxf(fabsf(v) - t, 0.f), v); }

// inclusive scan of affine maps y -> P y + Q from lane 0 upwards (earlier first)
__device__ __forceinline__ void scan_up(float& P, float& Q, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float pp = __shfl_up_sync(FULL, P, o), qq = __shfl_up_sync(FULL, Q, o);
    if (lane >= o) { Q = fmaf(P, qq, Q); P *= pp; }
  }
}
// inclusive scan from lane 31 downwards (later lanes first)
__device__ __forceinline__ void scan_down(float& P, float& Q, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float pp = __shfl_down_sync(FULL, P, o), qq = __shfl_down_sync(FULL, Q, o);
    if (lane + o < 32) { Q = fmaf(P, qq, Q); P *= pp; }
  }
}

// Thomas factors of I + D^T D (diag 2, 3, ..., 3, 2; off-diagonal -1): they
// depend on B only, so the host computes them once per call (fp64, the same
// IEEE operations a device loop would do) and every CTA copies them to shared
// memory (a serial fp64 loop in thread 0 of every CTA cost ~256 divisions
// per 32-pixel tile).
struct ThomasF {
  float alpha[256];
  float cp[256];
};

template <int S>
__global__ void __launch_bounds__(NT) l1spec_kernel(const float* __restrict__ M, float* __restrict__ X, long long n,
                                                    int B, float lam, float mu, int max_iters, float tol,
                                                    int* __restrict__ iters_out, const ThomasF tf) {
  __shared__ float s_alpha[32 * S], s_cp[32 * S];
  for (int i = threadIdx.x; i < 32 * S; i += NT) {
    s_alpha[i] = tf.alpha[i];
    s_cp[i] = tf.cp[i];
  }
  __syncthreads();
  // the CTA stages a tile of TP consecutive pixels x all bands through shared
  // memory (coalesced 128-byte band rows in and out); warp w solves pixels
  // w, w + 8, ... of the tile from it
  extern __shared__ float tile[];   // [32 S][TP + 1]
  constexpr int TP = 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long p0 = (long long)blockIdx.x * TP;
  const int np = (int)min((long long)TP, n - p0);
  for (int x = threadIdx.x; x < B * TP; x += NT) {
    const int i = x / TP, q = x % TP;
    tile[i * (TP + 1) + q] = q < np ? M[(size_t)i * n + p0 + q] : 0.f;
  }
  __syncthreads();
  const float ta = 1.f / mu, td = lam / mu;
  for (int q = wid; q < np; q += NT / 32) {
    float m[S], x[S], a[S], ba[S], d[S], bd[S], al[S], cp[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane * S + s;
      m[s] = i < B ? tile[i * (TP + 1) + q] : 0.f;
      x[s] = m[s];
      a[s] = ba[s] = d[s] = bd[s] = 0.f;
      al[s] = s_alpha[i];
      cp[s] = s_cp[i];
    }
    int it = 0;
    for (; it < max_iters; ++it) {
      // rhs_i = a_i + m_i - ba_i + v_{i-1} - v_i, v = d - bd (v_{B-1} = 0, v_{-1} = 0)
      float v[S];
  #pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = lane * S + s;
        v[s] = i < B - 1 ? d[s] - bd[s] : 0.f;
      }
      float vprev = __shfl_up_sync(FULL, v[S - 1], 1);
      if (lane == 0) vprev = 0.f;
      float r[S];
  #pragma unroll
      for (int s = 0; s < S; ++s) {
        r[s] = a[s] + m[s] - ba[s] + (s == 0 ? vprev : v[s - 1]) - v[s];
      }
      // forward: y_i = al_i y_{i-1} + al_i r_i
      float P = 1.f, Q = 0.f;
  #pragma unroll
      for (int s = 0; s < S; ++s) { Q = al[s] * (Q + r[s]); P *= al[s]; }
      scan_up(P, Q, lane);
      float yin = __shfl_up_sync(FULL, Q, 1);   // y at the end of the previous lane (y_{-1} = 0)
      if (lane == 0) yin = 0.f;
      float y[S];
      {
        float yy = yin;
  #pragma unroll
        for (int s = 0; s < S; ++s) { yy = al[s] * (yy + r[s]); y[s] = yy; }
      }
      // backward: x_i = -cp_i x_{i+1} + y_i
      float P2 = 1.f, Q2 = 0.f;
  #pragma unroll
      for (int s = S - 1; s >= 0; --s) { Q2 = fmaf(-cp[s], Q2, y[s]); P2 *= -cp[s]; }
      scan_down(P2, Q2, lane);
      float xin = __shfl_down_sync(FULL, Q2, 1);   // x at the start of the next lane (x_B = 0)
      if (lane == 31) xin = 0.f;
      float dx2 = 0.f, xo2 = 0.f;
      {
        float xx = xin;
  #pragma unroll
        for (int s = S - 1; s >= 0; --s) {
          xx = fmaf(-cp[s], xx, y[s]);
          const int i = lane * S + s;
          const float xn = i < B ? xx : 0.f;
          dx2 = fmaf(xn - x[s], xn - x[s], dx2);
          xo2 = fmaf(x[s], x[s], xo2);
          x[s] = xn;
        }
      }
      // a, b_a
  #pragma unroll
      for (int s = 0; s < S; ++s) {
        const float t = x[s] - m[s] + ba[s];
        a[s] = shrinkf(t, ta);
        ba[s] = t - a[s];
      }
      // D x: x_{i+1} - x_i (i < B-1), x_{i+1} of the last slot from the next lane
      float xnext = __shfl_down_sync(FULL, x[0], 1);
  #pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = lane * S + s;
        const float x1 = s + 1 < S ? x[s + 1] : xnext;
        if (i < B - 1) {
          const float u = (x1 - x[s]) + bd[s];
          d[s] = shrinkf(u, td);
          bd[s] = u - d[s];
        }
      }
  #pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dx2 += __shfl_xor_sync(FULL, dx2, o);
        xo2 += __shfl_xor_sync(FULL, xo2, o);
      }
      if (sqrtf(dx2) <= tol * sqrtf(xo2)) { ++it; break; }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane * S + s;
      if (i < B) tile[i * (TP + 1) + q] = x[s];
    }
    if (iters_out && lane == 0) iters_out[p0 + q] = it;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < B * TP; x += NT) {
    const int i = x / TP, q = x % TP;
    if (q < np) X[(size_t)i * n + p0 + q] = tile[i * (TP + 1) + q];
  }
}

}  // namespace

cudaError_t launch_l1spec(const float* M, float* X, long long n, int B, float lam, float mu, int max_iters, float tol,
                          int* iters, cudaStream_t st) {
  const unsigned blocks = (unsigned)((n + 31) / 32);
  const int S = (B + 31) / 32;
  if (S > 8) return cudaErrorInvalidValue;
  const size_t sm = (size_t)32 * S * 33 * sizeof(float);
  ThomasF tf;
  {
    double cprev = 0.0;
    for (int i = 0; i < 256; ++i) {
      if (i < B) {
        const double bi = (i == 0 || i == B - 1) ? (B == 1 ? 1.0 : 2.0) : 3.0;
        const double m = bi + cprev;              // b_i - a_i c'_{i-1}, a_i = -1
        tf.alpha[i] = (float)(1.0 / m);
        cprev = (i < B - 1 ? -1.0 : 0.0) / m;
        tf.cp[i] = (float)cprev;
      } else {
        tf.alpha[i] = 0.f;
        tf.cp[i] = 0.f;
      }
    }
  }
  if (S <= 2) l1spec_kernel<2><<<blocks, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, tf);
  else if (S <= 4) l1spec_kernel<4><<<blocks, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, tf);
  else l1spec_kernel<8><<<blocks, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, tf);
  return cudaGetLastError();
}
