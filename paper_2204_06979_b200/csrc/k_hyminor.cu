// F3 (SPEC.md:415-423 D19; §2.1 "the remaining
// sparse noise is removed by solving an l1-l1 optimization problem with a
// modified split-Bregman technique"): per pixel spectrum m (B bands) of the
// HyRes output, min_x ||m - x||_1 + lam ||D x||_1 by split Bregman
// (a = x - m, d = D x):
//   x = (I + D^T D)^-1 (a + m - b_a + D^T (d - b_d))
//   a = shrink(x - m + b_a, 1/mu), b_a += x - m - a
//   d = shrink(D x + b_d, lam/mu), b_d += D x - d
// Two kernels.  (1) l1spec_first_kernel: ONE THREAD PER PIXEL for the first
// iteration, which starts from x = m, a = d = b = 0 so its right-hand side is m
// itself: a sequential Thomas sweep along the bands (forward y_i = alpha_i
// (y_{i-1} + m_i) stored in X as scratch, backward x_i = y_i - c'_i x_{i+1}
// written over it), the stopping test ||x - m|| <= tol ||m|| on the way back.
// Band rows are read and written by consecutive threads (coalesced, no
// staging), so the stage streams M once and X once (the backward re-reads are
// L2 hits): the D19 defaults stop every pixel of the BJ cubes here.  Every
// pixel that has not stopped is marked in a per-32-pixel tile mask.
// (2) l1spec_kernel continues the marked tiles' unstopped pixels from
// x_1 (a_1, b_a, d_1, b_d follow from x_1 and m):
// ONE WARP PER PIXEL, the whole state in registers: lane l owns the S = B/32
// consecutive bands [l S, l S + S).  The tridiagonal x-update (I + D^T D is
// tridiagonal, strictly diagonally dominant) is the Thomas algorithm written
// as two first-order affine recurrences -- forward y_i = alpha_i (y_{i-1} +
// r_i), backward x_i = y_i - c'_i x_{i+1} -- each evaluated as a lane-local
// composition of affine maps plus a 5-step warp scan (no shared memory, no
// serial 224-step chain).  A pixel stops when ||x_new - x_old|| <= tol ||x_old||.
#include "common.cuh"

#include <cstdio>
#include <cstdlib>
#include <vector>

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

// (1) first iteration, one thread per pixel.  From x_0 = m and zero state the
// right-hand side is m itself: a sequential Thomas sweep along the bands,
// forward y_i = alpha_i (y_{i-1} + m_i) stored in X as scratch, backward
// x_i = y_i - c'_i x_{i+1} written over it; ||m|| on the way forward and
// ||x_1 - m|| on the way back from x - m = -(D^T D) x, so M is read once (and
// M == X works).  Consecutive threads touch consecutive pixels of a band row
// (coalesced, no staging).  (A 41-tap band filter of rows of A^-1 -- one pass,
// no scratch -- measured slower: 1.8 vs 0.8 ms at `large`, long-scoreboard and
// instruction-fetch bound.)
__global__ void __launch_bounds__(128) l1spec_first_kernel(const float* __restrict__ M, float* __restrict__ X,
                                                          long long n, int B, float tol, int max_iters,
                                                          int* __restrict__ iters_out,
                                                          unsigned* __restrict__ tile_todo, const ThomasF tf) {
  __shared__ float s_alpha[256], s_cp[256];
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    s_alpha[i] = tf.alpha[i];
    s_cp[i] = tf.cp[i];
  }
  __syncthreads();
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool live = p < n;
  // Both sweeps run in blocks of L1B bands with the NEXT block's loads issued
  // (in program order) before this block's stores: the compiler may not hoist
  // a load of M / X above a store to X (M == X is allowed), so a plain loop
  // waited one DRAM / L2 round trip per band (0.97 ms at `large`).  Same
  // arithmetic, same order as the band-by-band loop.
  constexpr int L1B = 32;
  float y = 0.f, xo2 = 0.f;
  if (live) {
    float mc[L1B], mn[L1B];
#pragma unroll
    for (int u = 0; u < L1B; ++u) mc[u] = u < B ? M[(size_t)u * n + p] : 0.f;
    for (int i0 = 0; i0 < B; i0 += L1B) {
#pragma unroll
      for (int u = 0; u < L1B; ++u) {
        const int i = i0 + L1B + u;
        mn[u] = i < B ? M[(size_t)i * n + p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < L1B; ++u) {
        const int i = i0 + u;
        if (i < B) {
          const float m = mc[u];
          xo2 = fmaf(m, m, xo2);
          y = s_alpha[i] * (y + m);
          X[(size_t)i * n + p] = y;
        }
      }
#pragma unroll
      for (int u = 0; u < L1B; ++u) mc[u] = mn[u];
    }
  }
  float dx2 = 0.f;
  if (live) {
    float x1 = 0.f, x2 = 0.f;   // x_{i+1}, x_{i+2}
    // blocks from the top: [i1 - L1B + 1, i1]
    float yc[L1B], yn[L1B];
    const int itop = B - 1;
#pragma unroll
    for (int u = 0; u < L1B; ++u) {
      const int i = itop - u;
      yc[u] = i >= 0 ? X[(size_t)i * n + p] : 0.f;
    }
    for (int i1 = itop; i1 >= 0; i1 -= L1B) {
#pragma unroll
      for (int u = 0; u < L1B; ++u) {
        const int i = i1 - L1B - u;
        yn[u] = i >= 0 ? X[(size_t)i * n + p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < L1B; ++u) {
        const int i = i1 - u;
        if (i >= 0) {
          const float x = fmaf(-s_cp[i], x1, yc[u]);
          __stcs(X + (size_t)i * n + p, x);
          if (i + 1 <= B - 1) {   // (D^T D x)_{i+1} now that x_i is known
            const float t = (i + 1 == B - 1) ? x1 - x : (2.f * x1 - x - x2);
            dx2 = fmaf(t, t, dx2);
          }
          x2 = x1;
          x1 = x;
        }
      }
#pragma unroll
      for (int u = 0; u < L1B; ++u) yc[u] = yn[u];
    }
    if (B >= 2) {
      const float t = x1 - x2;   // row 0: x_0 - x_1
      dx2 = fmaf(t, t, dx2);
    }
  }
  const bool stop = live && (max_iters <= 1 || sqrtf(dx2) <= tol * sqrtf(xo2));
  if (live && iters_out) iters_out[p] = 1;
  const unsigned more = __ballot_sync(0xffffffffu, live && !stop);
  if ((threadIdx.x & 31) == 0 && live) tile_todo[p >> 5] = more;
}

// (1b) the same first iteration with the forward-sweep scratch y in SHARED
// memory ([B][CP] per CTA of CP pixels) instead of X: the stage then moves the
// method's minimum bytes (read M once, write X once) -- the X-scratch kernel's
// y spills past the L2 (ncu at `large`: 2.55 GB of DRAM traffic for 1.88 GB).
// Fewer pixels fit per SM (~7 CTAs of 32), so the forward sweep keeps a
// deeper window of M loads in flight (L1S bands, double-buffered in
// registers).  Same arithmetic in the same order as (1): bit-identical.
template <int CP, int L1S>
__global__ void __launch_bounds__(CP) l1spec_first_smem_kernel(const float* __restrict__ M, float* __restrict__ X,
                                                               long long n, int B, float tol, int max_iters,
                                                               int* __restrict__ iters_out,
                                                               unsigned* __restrict__ tile_todo, const ThomasF tf) {
  extern __shared__ float l1sh[];
  float* s_alpha = l1sh;
  float* s_cp = l1sh + 256;
  float* ys = l1sh + 512;   // y[i][t] at ys[i * CP + t]
  for (int i = threadIdx.x; i < B; i += CP) {
    s_alpha[i] = tf.alpha[i];
    s_cp[i] = tf.cp[i];
  }
  __syncthreads();
  const int t = threadIdx.x;
  const long long p = blockIdx.x * (long long)CP + t;
  const bool live = p < n;
  float xo2 = 0.f, dx2 = 0.f;
  if (live) {
    float y = 0.f;
    float mc[L1S], mn[L1S];
#pragma unroll
    for (int u = 0; u < L1S; ++u) mc[u] = u < B ? __ldcs(M + (size_t)u * n + p) : 0.f;
    for (int i0 = 0; i0 < B; i0 += L1S) {
#pragma unroll
      for (int u = 0; u < L1S; ++u) {
        const int i = i0 + L1S + u;
        mn[u] = i < B ? __ldcs(M + (size_t)i * n + p) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < L1S; ++u) {
        const int i = i0 + u;
        if (i < B) {
          const float m = mc[u];
          xo2 = fmaf(m, m, xo2);
          y = s_alpha[i] * (y + m);
          ys[i * CP + t] = y;
        }
      }
#pragma unroll
      for (int u = 0; u < L1S; ++u) mc[u] = mn[u];
    }
    float x1 = 0.f, x2 = 0.f;   // x_{i+1}, x_{i+2}
    for (int i = B - 1; i >= 0; --i) {
      const float x = fmaf(-s_cp[i], x1, ys[i * CP + t]);
      __stcs(X + (size_t)i * n + p, x);
      if (i + 1 <= B - 1) {   // (D^T D x)_{i+1} now that x_i is known
        const float tt = (i + 1 == B - 1) ? x1 - x : (2.f * x1 - x - x2);
        dx2 = fmaf(tt, tt, dx2);
      }
      x2 = x1;
      x1 = x;
    }
    if (B >= 2) {
      const float tt = x1 - x2;   // row 0: x_0 - x_1
      dx2 = fmaf(tt, tt, dx2);
    }
  }
  const bool stop = live && (max_iters <= 1 || sqrtf(dx2) <= tol * sqrtf(xo2));
  if (live && iters_out) iters_out[p] = 1;
  const unsigned more = __ballot_sync(0xffffffffu, live && !stop);
  if ((t & 31) == 0 && live) tile_todo[p >> 5] = more;
}

// (2) later iterations of the marked pixels, one warp per pixel, from x_1
template <int S>
__global__ void __launch_bounds__(NT) l1spec_kernel(const float* __restrict__ M, float* __restrict__ X, long long n,
                                                    int B, float lam, float mu, int max_iters, float tol,
                                                    int* __restrict__ iters_out, const unsigned* __restrict__ tile_todo,
                                                    const ThomasF tf) {
  __shared__ float s_alpha[32 * S], s_cp[32 * S];
  __shared__ unsigned long long s_tile;
  const long long ntile = (n + 31) / 32;
  for (long long tile_i = blockIdx.x;; tile_i += gridDim.x) {
  // next tile of this CTA with a pixel to continue (most CTAs find none)
  __syncthreads();
  if (threadIdx.x == 0) s_tile = ~0ull;
  __syncthreads();
  // the first tile >= tile_i (stride gridDim) with work: NT candidates at a time
  for (long long t0 = tile_i; t0 < ntile; t0 += (long long)NT * gridDim.x) {
    const long long t = t0 + (long long)threadIdx.x * gridDim.x;
    const bool has = t < ntile && tile_todo[t] != 0u;
    if (has) atomicMin(&s_tile, (unsigned long long)t);   // ~0 (none) is the largest u64
    if (__syncthreads_or(has)) break;
  }
  if (s_tile == ~0ull) return;
  tile_i = (long long)s_tile;
  const unsigned todo = tile_todo[tile_i];
  for (int i = threadIdx.x; i < 32 * S; i += NT) {
    s_alpha[i] = tf.alpha[i];
    s_cp[i] = tf.cp[i];
  }
  __syncthreads();
  // the CTA stages a tile of TP consecutive pixels x all bands through shared
  // memory (coalesced 128-byte band rows in and out); warp w solves pixels
  // w, w + 8, ... of the tile from it
  extern __shared__ float tile[];   // m: [32 S][TP + 1], then x_1: [32 S][TP + 1]
  constexpr int TP = 32;
  float* tx = tile + 32 * S * (TP + 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long p0 = tile_i * TP;
  const int np = (int)min((long long)TP, n - p0);
  for (int x = threadIdx.x; x < B * TP; x += NT) {
    const int i = x / TP, q = x % TP;
    if (M != X) tile[i * (TP + 1) + q] = q < np ? M[(size_t)i * n + p0 + q] : 0.f;
    tx[i * (TP + 1) + q] = q < np ? X[(size_t)i * n + p0 + q] : 0.f;
  }
  __syncthreads();
  if (M == X) {
    // in place: m was overwritten by x_1; m = (I + D^T D) x_1 (to fp32 rounding)
    for (int x = threadIdx.x; x < B * TP; x += NT) {
      const int i = x / TP, q = x % TP;
      const float xc = tx[i * (TP + 1) + q];
      const float xl = i > 0 ? tx[(i - 1) * (TP + 1) + q] : xc;
      const float xr = i < B - 1 ? tx[(i + 1) * (TP + 1) + q] : xc;
      tile[i * (TP + 1) + q] = xc + (xc - xl) + (xc - xr);
    }
    __syncthreads();
  }
  const float ta = 1.f / mu, td = lam / mu;
  for (int q = wid; q < np; q += NT / 32) {
    if (!((todo >> q) & 1u)) continue;   // stopped after the first iteration
    float m[S], x[S], a[S], ba[S], d[S], bd[S], al[S], cp[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane * S + s;
      m[s] = i < B ? tile[i * (TP + 1) + q] : 0.f;
      x[s] = i < B ? tx[i * (TP + 1) + q] : 0.f;
      al[s] = s_alpha[i];
      cp[s] = s_cp[i];
    }
    // the first iteration's a, b_a, d, b_d from x_1 and m (x_0 = m, zero state)
    {
      float xnext = __shfl_down_sync(FULL, x[0], 1);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = lane * S + s;
        const float t = x[s] - m[s];
        a[s] = shrinkf(t, ta);
        ba[s] = t - a[s];
        const float x1 = s + 1 < S ? x[s + 1] : xnext;
        if (i < B - 1) {
          const float u = x1 - x[s];
          d[s] = shrinkf(u, td);
          bd[s] = u - d[s];
        } else {
          d[s] = bd[s] = 0.f;
        }
      }
    }
    int it = 1;
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
      if (i < B) tx[i * (TP + 1) + q] = x[s];
    }
    if (iters_out && lane == 0) iters_out[p0 + q] = it;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < B * TP; x += NT) {
    const int i = x / TP, q = x % TP;
    if (q < np && ((todo >> q) & 1u)) X[(size_t)i * n + p0 + q] = tx[i * (TP + 1) + q];
  }
  }
}

}  // namespace

size_t l1spec_ws_bytes(long long n) { return (size_t)((n + 31) / 32) * sizeof(unsigned); }

// todo_ws: l1spec_ws_bytes(n) bytes of device scratch (the per-tile masks).
// M and X may alias only when equal (in place): the first iteration never
// re-reads M; a pixel continued past it then works from m = (I + D^T D) x_1
// (equal to m up to fp32 rounding) instead of the overwritten input.
cudaError_t launch_l1spec(const float* M, float* X, long long n, int B, float lam, float mu, int max_iters, float tol,
                          int* iters, void* todo_ws, cudaStream_t st) {
  const unsigned blocks = (unsigned)((n + 31) / 32);
  const int S = (B + 31) / 32;
  if (S > 8) return cudaErrorInvalidValue;
  const int St = S <= 2 ? 2 : (S <= 4 ? 4 : 8);   // the instantiated register width
  const unsigned g2 = blocks < 1184u ? blocks : 1184u;   // continuation: grid-stride over 32-pixel tiles
  const size_t sm = (size_t)2 * 32 * St * 33 * sizeof(float);
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
  unsigned* todo = (unsigned*)todo_ws;
  // At most 8 resident CTAs per SM (an unused dynamic shared-memory
  // reservation): measured at `large`, 3 / 4 / 6 / 8 / 16 per SM gave 0.86 /
  // 0.67 / 0.57 / 0.57 / 0.57 ms and no cap 0.66 ms (more pixels in flight
  // than the L2 holds scratch for).  (A register-resident variant -- 32 pixels
  // per CTA, band segments per warp chained by affine scans, like FORPDN's
  // solve -- measured 0.97 ms: too few pixels in flight per SM.)
  // HYDE_L1_CTAS_PER_SM overrides (experiments).
  static const int cap = [] {
    const char* ev = getenv("HYDE_L1_CTAS_PER_SM");
    return ev ? atoi(ev) : 8;
  }();
  size_t pad = 0;
  if (cap > 0) {
    pad = (size_t)(227 * 1024) / (size_t)cap > 2048 ? (size_t)(227 * 1024) / (size_t)cap - 2048 : 0;
    static bool attr_done = false;
    if (!attr_done) {
      cudaFuncSetAttribute(l1spec_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_done = true;
    }
  }
  static const int smem_mode = [] {
    const char* ev = getenv("HYDE_L1_SMEM");   // experiments: 0 = X scratch, 32 / 64 = y in shared memory
    return ev ? atoi(ev) : 0;
  }();
  if (smem_mode == 32 || smem_mode == 64) {
    const size_t shb = (size_t)(512 + B * smem_mode) * sizeof(float);
    if (smem_mode == 32) {
      cudaFuncSetAttribute(l1spec_first_smem_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb);
      l1spec_first_smem_kernel<32, 64><<<(unsigned)((n + 31) / 32), 32, shb, st>>>(M, X, n, B, tol, max_iters, iters,
                                                                                  todo, tf);
    } else {
      cudaFuncSetAttribute(l1spec_first_smem_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb);
      l1spec_first_smem_kernel<64, 64><<<(unsigned)((n + 63) / 64), 64, shb, st>>>(M, X, n, B, tol, max_iters, iters,
                                                                                  todo, tf);
    }
  } else {
    l1spec_first_kernel<<<(unsigned)((n + 127) / 128), 128, pad, st>>>(M, X, n, B, tol, max_iters, iters, todo, tf);
  }
  cudaError_t e = cudaGetLastError();
  if (getenv("HYDE_DEBUG_SYNC")) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { fprintf(stderr, "l1spec_first_kernel: %s\n", cudaGetErrorString(e)); return e; }
  }
  if (e != cudaSuccess || max_iters <= 1) return e;
  if (S <= 2) {
    e = cudaFuncSetAttribute(l1spec_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    l1spec_kernel<2><<<g2, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, todo, tf);
  } else if (S <= 4) {
    e = cudaFuncSetAttribute(l1spec_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    l1spec_kernel<4><<<g2, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, todo, tf);
  } else {
    e = cudaFuncSetAttribute(l1spec_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    l1spec_kernel<8><<<g2, NT, sm, st>>>(M, X, n, B, lam, mu, max_iters, tol, iters, todo, tf);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
