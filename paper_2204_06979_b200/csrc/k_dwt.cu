// K4 / K6a (north_star stages (4) and (6)):
// one level of the separable, periodised, orthonormal 2-D DWT and its inverse,
// batched over `count` eigen-images (blockIdx.z).
//
// Forward (per-level pad-to-even SPEC.md:182 D7): an odd
// extent is first padded by duplicating the last row/column; along an axis of
// even length n, a_j = sum_m h_m x_{(2j+m) mod n}, d_j = sum_m g_m x_{(2j+m) mod n};
// the contiguous axis (columns) is filtered first, then rows.  Subbands
// (axis-0 filter, axis-1 filter): LL, LH, HL, HH.
// Inverse: the adjoint synthesis
//   x_i = sum_{m = i mod 2} h_m a_{((i-m) mod n)/2} + g_m d_{((i-m) mod n)/2},
// rows first then columns, then crop to the level's input extent.
//
// Each CTA stages its input tile (with the periodic halo, read once with
// modular indexing) in shared memory and does both separable passes there:
// one read and one write of the level's data.
#include "common.cuh"

namespace {

constexpr int FR = 16;   // forward: subband rows per tile
constexpr int FC = 32;   // forward: subband cols per tile
constexpr int IR = 32;   // inverse: output rows per tile
constexpr int IC = 64;   // inverse: output cols per tile

template <int T>
__global__ void __launch_bounds__(256) dwt_fwd_kernel(const float* __restrict__ in, long long in_stride,
                                                      int h_in, int w_in, float* __restrict__ ll,
                                                      long long ll_stride, float* __restrict__ sub,
                                                      long long sub_stride, FilterBank fb) {
  constexpr int NR = 2 * FR + T - 2;
  constexpr int NC = 2 * FC + T - 2;
  __shared__ float xin[NR][NC + 1];
  __shared__ float lo[NR][FC + 1];
  __shared__ float hi[NR][FC + 1];
  const int H = h_in + (h_in & 1), Wd = w_in + (w_in & 1);
  const int hs = H >> 1, ws = Wd >> 1;
  const int i0 = blockIdx.y * FR, j0 = blockIdx.x * FC;
  const float* x = in + (long long)blockIdx.z * in_stride;
  for (int idx = threadIdx.x; idx < NR * NC; idx += 256) {
    int r = idx / NC, c = idx % NC;
    int gr = (2 * i0 + r) % H;
    int gc = (2 * j0 + c) % Wd;
    gr = min(gr, h_in - 1);
    gc = min(gc, w_in - 1);
    xin[r][c] = x[(long long)gr * w_in + gc];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NR * FC; idx += 256) {
    int r = idx / FC, j = idx % FC;
    float a = 0.f, d = 0.f;
#pragma unroll
    for (int m = 0; m < T; ++m) {
      float v = xin[r][2 * j + m];
      a = fmaf(fb.h[m], v, a);
      d = fmaf(fb.g[m], v, d);
    }
    lo[r][j] = a;
    hi[r][j] = d;
  }
  __syncthreads();
  const long long nsb = (long long)hs * ws;
  float* lh = sub + (long long)blockIdx.z * sub_stride;
  float* hl = lh + nsb;
  float* hh = hl + nsb;
  float* llo = ll + (long long)blockIdx.z * ll_stride;
  for (int idx = threadIdx.x; idx < FR * FC; idx += 256) {
    int i = idx / FC, j = idx % FC;
    int gi = i0 + i, gj = j0 + j;
    if (gi >= hs || gj >= ws) continue;
    float s_ll = 0.f, s_hl = 0.f, s_lh = 0.f, s_hh = 0.f;
#pragma unroll
    for (int m = 0; m < T; ++m) {
      float a = lo[2 * i + m][j], d = hi[2 * i + m][j];
      s_ll = fmaf(fb.h[m], a, s_ll);
      s_hl = fmaf(fb.g[m], a, s_hl);
      s_lh = fmaf(fb.h[m], d, s_lh);
      s_hh = fmaf(fb.g[m], d, s_hh);
    }
    long long o = (long long)gi * ws + gj;
    llo[o] = s_ll;
    lh[o] = s_lh;
    hl[o] = s_hl;
    hh[o] = s_hh;
  }
}

__device__ __forceinline__ float soft(float v, float t) {
  const float a = fabsf(v) - t;
  return a > 0.f ? copysignf(a, v) : 0.f;
}

// thresholds applied on load (K5's t* per subband): tstar
// [image][nsub], this level's LH/HL/HH at s_lh .. s_lh+2, LL at s_ll (-1 = none)
struct SoftSpec {
  const float* tstar;
  int nsub, s_lh, s_ll;
};

template <int T>
__global__ void __launch_bounds__(256) dwt_inv_kernel(const float* __restrict__ llp, long long ll_stride,
                                                      const float* __restrict__ sub, long long sub_stride,
                                                      int h_out, int w_out, float* __restrict__ out,
                                                      long long out_stride, FilterBank fb, SoftSpec sp) {
  constexpr int CR = IR / 2 + T / 2 - 1;
  constexpr int CC = IC / 2 + T / 2 - 1;
  __shared__ float t_ll[CR][CC + 1], t_hl[CR][CC + 1], t_lh[CR][CC + 1], t_hh[CR][CC + 1];
  __shared__ float lo1[IR][CC + 1], hi1[IR][CC + 1];
  const int H = h_out + (h_out & 1), Wd = w_out + (w_out & 1);
  const int hs = H >> 1, ws = Wd >> 1;
  const int r0 = blockIdx.y * IR, c0 = blockIdx.x * IC;
  const int ilo = (r0 >> 1) - (T / 2 - 1);
  const int jlo = (c0 >> 1) - (T / 2 - 1);
  const long long nsb = (long long)hs * ws;
  const float* a_ll = llp + (long long)blockIdx.z * ll_stride;
  const float* a_lh = sub + (long long)blockIdx.z * sub_stride;
  const float* a_hl = a_lh + nsb;
  const float* a_hh = a_hl + nsb;
  float th_ll = 0.f, th_lh = 0.f, th_hl = 0.f, th_hh = 0.f;
  if (sp.tstar) {
    const float* tz = sp.tstar + (long long)blockIdx.z * sp.nsub;
    th_lh = tz[sp.s_lh];
    th_hl = tz[sp.s_lh + 1];
    th_hh = tz[sp.s_lh + 2];
    if (sp.s_ll >= 0) th_ll = tz[sp.s_ll];
  }
  for (int idx = threadIdx.x; idx < CR * CC; idx += 256) {
    int r = idx / CC, c = idx % CC;
    int gi = ((ilo + r) % hs + hs) % hs;
    int gj = ((jlo + c) % ws + ws) % ws;
    long long o = (long long)gi * ws + gj;
    t_ll[r][c] = soft(a_ll[o], th_ll);
    t_lh[r][c] = soft(a_lh[o], th_lh);
    t_hl[r][c] = soft(a_hl[o], th_hl);
    t_hh[r][c] = soft(a_hh[o], th_hh);
  }
  __syncthreads();
  // synthesis along axis 0: lo1 <- (LL, HL), hi1 <- (LH, HH)
  for (int idx = threadIdx.x; idx < IR * CC; idx += 256) {
    int rr = idx / CC, c = idx % CC;
    int r = r0 + rr;
    float s_lo = 0.f, s_hi = 0.f;
    const int par = r & 1;   // taps m with m = r (mod 2) contribute
#pragma unroll
    for (int q = 0; q < T / 2; ++q) {
      const int m = 2 * q + par;
      const float hm = par ? fb.h[2 * q + 1] : fb.h[2 * q];
      const float gm = par ? fb.g[2 * q + 1] : fb.g[2 * q];
      const int ti = ((r - m) >> 1) - ilo;
      s_lo = fmaf(hm, t_ll[ti][c], s_lo);
      s_lo = fmaf(gm, t_hl[ti][c], s_lo);
      s_hi = fmaf(hm, t_lh[ti][c], s_hi);
      s_hi = fmaf(gm, t_hh[ti][c], s_hi);
    }
    lo1[rr][c] = s_lo;
    hi1[rr][c] = s_hi;
  }
  __syncthreads();
  float* o = out + (long long)blockIdx.z * out_stride;
  for (int idx = threadIdx.x; idx < IR * IC; idx += 256) {
    int rr = idx / IC, cc = idx % IC;
    int r = r0 + rr, c = c0 + cc;
    if (r >= h_out || c >= w_out) continue;
    float s = 0.f;
    const int par = c & 1;
#pragma unroll
    for (int q = 0; q < T / 2; ++q) {
      const int m = 2 * q + par;
      const float hm = par ? fb.h[2 * q + 1] : fb.h[2 * q];
      const float gm = par ? fb.g[2 * q + 1] : fb.g[2 * q];
      const int tj = ((c - m) >> 1) - jlo;
      s = fmaf(hm, lo1[rr][tj], s);
      s = fmaf(gm, hi1[rr][tj], s);
    }
    o[(long long)r * w_out + c] = s;
  }
}

}  // namespace

cudaError_t launch_dwt_level(const float* in, long long in_stride, int h_in, int w_in, float* ll,
                             long long ll_stride, float* sub, long long sub_stride, int count,
                             const FilterBank& fb, cudaStream_t st) {
  const int hs = (h_in + 1) / 2, ws = (w_in + 1) / 2;
  dim3 grid((ws + FC - 1) / FC, (hs + FR - 1) / FR, count);
  switch (fb.taps) {
    case 2: dwt_fwd_kernel<2><<<grid, 256, 0, st>>>(in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb); break;
    case 8: dwt_fwd_kernel<8><<<grid, 256, 0, st>>>(in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb); break;
    case 16: dwt_fwd_kernel<16><<<grid, 256, 0, st>>>(in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_idwt_level(const float* ll, long long ll_stride, const float* sub,
                              long long sub_stride, int h_out, int w_out, float* out,
                              long long out_stride, int count, const FilterBank& fb,
                              const float* tstar, int nsub, int s_lh, int s_ll, cudaStream_t st) {
  const int H = h_out + (h_out & 1), Wd = w_out + (w_out & 1);
  dim3 grid((Wd + IC - 1) / IC, (H + IR - 1) / IR, count);
  const SoftSpec sp{tstar, nsub, s_lh, s_ll};
  switch (fb.taps) {
    case 2: dwt_inv_kernel<2><<<grid, 256, 0, st>>>(ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp); break;
    case 8: dwt_inv_kernel<8><<<grid, 256, 0, st>>>(ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp); break;
    case 16: dwt_inv_kernel<16><<<grid, 256, 0, st>>>(ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
