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

constexpr int FR = 24;   // forward: subband rows per tile (row pass: (2 FR + T - 2) x FC/FJ = 248 items, one round of 256 threads)
constexpr int FC = 32;   // forward: subband cols per tile
constexpr int FJ = 8;    // forward row pass: outputs per thread (register window 2FJ+T-2)
constexpr int FI = 3;    // forward column pass: output rows per thread (FC x FR/FI = 256 items)
constexpr int IR = 32;   // inverse: output rows per tile
constexpr int IC = 64;   // inverse: output cols per tile

// Packed fp32x2 FMA (FFMA2): two lanes of arithmetic per issue slot.  The
// forward filter passes are issue-bound, and FFMA2 halves their FMA
// instructions; each half of the pair is the same fp32 fma as before (so the
// coefficients are bit-identical).  The inverse packs the two output parities
// of a window position along axis 1 (same window entries, taps 2q / 2q + 1)
// and the {LL, LH} / {HL, HH} subband pairs along axis 0.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(f2_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// g mod n for g >= -n (the common case g in [0, n) costs one compare)
__device__ __forceinline__ int wrap(int g, int n) {
  if (g >= n) return g < 2 * n ? g - n : g % n;
  if (g < 0) { g += n; return g >= 0 ? g : (g % n + n) % n; }
  return g;
}

// Forward level.  Each thread of the row pass slides a register window of
// 2 FJ + T - 2 inputs along one staged row and produces FJ (lo, hi) pairs; each
// thread of the column pass does the same down one column for FI output rows
// of all four subbands -- ~1 shared-memory load per 8 FMAs instead of 1:1.
template <int T>
__global__ void __launch_bounds__(256) dwt_fwd_kernel(const float* __restrict__ in, long long in_stride,
                                                      int h_in, int w_in, float* __restrict__ ll,
                                                      long long ll_stride, float* __restrict__ sub,
                                                      long long sub_stride, FilterBank fb) {
  pdl_wait();
  constexpr int NR = 2 * FR + T - 2;
  constexpr int NC = 2 * FC + T - 2;
  constexpr int WR = 2 * FJ + T - 2;   // row-pass window
  constexpr int WC = 2 * FI + T - 2;   // column-pass window
  __shared__ float xin[NR][NC + 1];
  __shared__ float lo[NR][FC + 1];
  __shared__ float hi[NR][FC + 1];
  const int H = h_in + (h_in & 1), Wd = w_in + (w_in & 1);
  const int hs = H >> 1, ws = Wd >> 1;
  const int i0 = blockIdx.y * FR, j0 = blockIdx.x * FC;
  const float* x = in + (long long)blockIdx.z * in_stride;
  {
    // stage the tile: warp w takes rows w, w + 8, ...; lane l columns l + 32u
    // (coalesced rows; the periodic indices are computed once per row and
    // once per column -- the per-element index math of a linear mapping cost
    // more than the loads); every load of this thread is issued before the
    // first shared store, so the L2/HBM round trips overlap
    constexpr int NCI = (NC + 31) / 32;
    constexpr int NRI = (NR + 7) / 8;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int gcol[NCI];
#pragma unroll
    for (int u = 0; u < NCI; ++u) gcol[u] = min(wrap(2 * j0 + l + 32 * u, Wd), w_in - 1);   // odd extent: duplicate the last column
    float v[NRI][NCI];
    // interior tile (no periodic wrap, no odd-extent padding): plain strided
    // addressing; boundary tiles take the general path
    const bool interior = 2 * i0 + NR <= h_in && 2 * j0 + NC <= w_in;
    if (interior) {
      const float* base = x + (long long)(2 * i0 + w) * w_in + 2 * j0 + l;
#pragma unroll
      for (int ri = 0; ri < NRI; ++ri) {
        const int r = w + 8 * ri;
#pragma unroll
        for (int u = 0; u < NCI; ++u)
          v[ri][u] = (r < NR && l + 32 * u < NC) ? __ldg(base + (long long)(8 * ri) * w_in + 32 * u) : 0.f;
      }
    } else {
#pragma unroll
      for (int ri = 0; ri < NRI; ++ri) {
        const int r = w + 8 * ri;
        const float* rowp = x + (long long)min(wrap(2 * i0 + r, H), h_in - 1) * w_in;
#pragma unroll
        for (int u = 0; u < NCI; ++u)
          v[ri][u] = (r < NR && l + 32 * u < NC) ? __ldg(rowp + gcol[u]) : 0.f;
      }
    }
#pragma unroll
    for (int ri = 0; ri < NRI; ++ri) {
      const int r = w + 8 * ri;
#pragma unroll
      for (int u = 0; u < NCI; ++u)
        if (r < NR && l + 32 * u < NC) xin[r][l + 32 * u] = v[ri][u];
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < NR * (FC / FJ); it += 256) {
    // lanes run down the rows (odd row stride NC + 1: conflict-free window loads)
    const int q = it / NR, r = it - q * NR;
    float v[WR];
#pragma unroll
    for (int t = 0; t < WR; ++t) v[t] = xin[r][2 * FJ * q + t];
#pragma unroll
    for (int jj = 0; jj < FJ; ++jj) {
      f2_t ad = 0ull;   // {a, d}
#pragma unroll
      for (int m = 0; m < T; ++m) ad = ffma2(pk2(fb.hg[m].x, fb.hg[m].y), pk2(v[2 * jj + m], v[2 * jj + m]), ad);
      const float2 o = up2(ad);
      lo[r][FJ * q + jj] = o.x;
      hi[r][FJ * q + jj] = o.y;
    }
  }
  __syncthreads();
  const long long nsb = (long long)hs * ws;
  float* lh = sub + (long long)blockIdx.z * sub_stride;
  float* hl = lh + nsb;
  float* hh = hl + nsb;
  float* llo = ll + (long long)blockIdx.z * ll_stride;
  for (int it = threadIdx.x; it < FC * (FR / FI); it += 256) {
    const int j = it % FC, p = it / FC;   // lanes run along j: coalesced stores
    float L[WC], Hh[WC];
#pragma unroll
    for (int t = 0; t < WC; ++t) {
      L[t] = lo[2 * FI * p + t][j];
      Hh[t] = hi[2 * FI * p + t][j];
    }
    const int gj = j0 + j;
#pragma unroll
    for (int ii = 0; ii < FI; ++ii) {
      f2_t pl = 0ull, ph = 0ull;   // {s_ll, s_hl}, {s_lh, s_hh}
#pragma unroll
      for (int m = 0; m < T; ++m) {
        const f2_t c = pk2(fb.hg[m].x, fb.hg[m].y);
        pl = ffma2(c, pk2(L[2 * ii + m], L[2 * ii + m]), pl);
        ph = ffma2(c, pk2(Hh[2 * ii + m], Hh[2 * ii + m]), ph);
      }
      const float2 vl = up2(pl), vh = up2(ph);
      const float s_ll = vl.x, s_hl = vl.y, s_lh = vh.x, s_hh = vh.y;
      const int gi = i0 + FI * p + ii;
      if (gi < hs && gj < ws) {
        const long long o = (long long)gi * ws + gj;
        llo[o] = s_ll;
        lh[o] = s_lh;
        hl[o] = s_hl;
        hh[o] = s_hh;
      }
    }
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
  const RankState* rs;   // non-NULL: images z >= kept (rank rule, decided on the device) are skipped
  int k0, cnt;           // first component of the chunk, components in it
};

constexpr int II = 4;    // inverse axis-0 pass: output rows per thread (even)
constexpr int IJ = 8;    // inverse axis-1 pass: output cols per thread (even)

// Inverse level, register-tiled like the forward: output rows r = 2u + par
// take taps m = 2q + par, coefficient index u - q, so II consecutive rows of
// one column read a window of II/2 + T/2 - 1 coefficients per subband.
template <int T>
__global__ void __launch_bounds__(256) dwt_inv_kernel(const float* __restrict__ llp, long long ll_stride,
                                                      const float* __restrict__ sub, long long sub_stride,
                                                      int h_out, int w_out, float* __restrict__ out,
                                                      long long out_stride, FilterBank fb, SoftSpec sp) {
  pdl_wait();
  constexpr int HT = T / 2;
  constexpr int CR = IR / 2 + HT - 1;
  constexpr int CC = IC / 2 + HT - 1;
  constexpr int W0 = II / 2 + HT - 1;   // axis-0 window
  constexpr int W1 = IJ / 2 + HT - 1;   // axis-1 window
  __shared__ float t_ll[CR][CC + 1], t_hl[CR][CC + 1], t_lh[CR][CC + 1], t_hh[CR][CC + 1];
  // row stride = 1 mod 4: the axis-1 pass (lanes = 4 rows x 8 column groups
  // 4 apart) reads 32 distinct banks
  constexpr int LS = CC + ((1 - CC) % 4 + 4) % 4;
  __shared__ float lo1[IR][LS], hi1[IR][LS];
  // output tile, written back with coalesced float4 rows.  Swizzled so that
  // both its writers (float2 pairs: 4 rows x 8 column groups per warp) and its
  // readers (float4, a row's 16 slots per half-warp) are conflict-free: slot
  // c4 of row r lives at r * IC / 4 + oslot(c4) and, in odd rows, its two
  // float2 halves are swapped.
  __shared__ __align__(16) float otile[IR * IC];
  auto oslot = [](int c4) { return c4 ^ ((c4 >> 3) & 1); };
  auto oidx = [&](int rr, int c) { return rr * IC + 4 * oslot(c >> 2) + ((c & 3) ^ ((rr & 1) << 1)); };
  if (sp.rs) {
    const int kept = sp.rs->found ? sp.rs->rank - sp.k0 : sp.cnt;
    if ((int)blockIdx.z >= kept) return;
  }
  const int H = h_out + (h_out & 1), Wd = w_out + (w_out & 1);
  const int hs = H >> 1, ws = Wd >> 1;
  const int r0 = blockIdx.y * IR, c0 = blockIdx.x * IC;
  const int ilo = (r0 >> 1) - (HT - 1);
  const int jlo = (c0 >> 1) - (HT - 1);
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
  {
    // stage the four coefficient tiles (linear index, constant divide, cheap
    // periodic wrap), all loads in flight before the stores, soft-thresholded
    // as they land
    constexpr int NL = (CR * CC + 255) / 256;
    float v0[NL], v1[NL], v2[NL], v3[NL];
    // interior tiles (no periodic wrap): one base offset, the element's
    // (row, col) from the constant divide only
    const bool interior = ilo >= 0 && jlo >= 0 && ilo + CR <= hs && jlo + CC <= ws;
    const long long obase = (long long)ilo * ws + jlo;
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int idx = threadIdx.x + 256 * u;
      v0[u] = v1[u] = v2[u] = v3[u] = 0.f;
      if (idx < CR * CC) {
        const int r = idx / CC, c = idx - r * CC;
        const long long o = interior ? obase + (long long)r * ws + c
                                     : (long long)wrap(ilo + r, hs) * ws + wrap(jlo + c, ws);
        v0[u] = a_ll[o];
        v1[u] = a_lh[o];
        v2[u] = a_hl[o];
        v3[u] = a_hh[o];
      }
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int idx = threadIdx.x + 256 * u;
      if (idx < CR * CC) {
        const int r = idx / CC, c = idx - r * CC;
        t_ll[r][c] = soft(v0[u], th_ll);
        t_lh[r][c] = soft(v1[u], th_lh);
        t_hl[r][c] = soft(v2[u], th_hl);
        t_hh[r][c] = soft(v3[u], th_hh);
      }
    }
  }
  __syncthreads();
  // synthesis along axis 0: lo1 <- (LL, HL), hi1 <- (LH, HH); II rows per thread
  for (int it = threadIdx.x; it < CC * (IR / II); it += 256) {
    const int c = it % CC, p = it / CC;
    const int ub = (II / 2) * p;   // first coefficient row of the window (tile-relative, + HT - 1 offset)
    f2_t wa[W0], wd[W0];   // {LL, LH} and {HL, HH} of one coefficient row
#pragma unroll
    for (int t = 0; t < W0; ++t) {
      wa[t] = pk2(t_ll[ub + t][c], t_lh[ub + t][c]);
      wd[t] = pk2(t_hl[ub + t][c], t_hh[ub + t][c]);
    }
#pragma unroll
    for (int k = 0; k < II; ++k) {
      const int par = k & 1, u = k >> 1;   // output row rr = II p + k = 2 (ub + u) + par (r0 even)
      f2_t s2 = 0ull;                      // {s_lo, s_hi}: same fma order as the scalar form
#pragma unroll
      for (int q = 0; q < HT; ++q) {
        const int m = 2 * q + par;
        const int ti = u - q + HT - 1;   // window index of coefficient row (ub + u) - q
        s2 = ffma2(pk2(fb.h[m], fb.h[m]), wa[ti], s2);
        s2 = ffma2(pk2(fb.g[m], fb.g[m]), wd[ti], s2);
      }
      const float2 o = up2(s2);
      lo1[II * p + k][c] = o.x;
      hi1[II * p + k][c] = o.y;
    }
  }
  __syncthreads();
  float* o = out + (long long)blockIdx.z * out_stride;
  for (int it = threadIdx.x; it < IR * (IC / IJ); it += 256) {
    const int q8 = it % (IC / IJ), rr = it / (IC / IJ);
    const int vb = (IJ / 2) * q8;
    float wl[W1], wh[W1];
#pragma unroll
    for (int t = 0; t < W1; ++t) {
      wl[t] = lo1[rr][vb + t];
      wh[t] = hi1[rr][vb + t];
    }
    // outputs 2u (taps 2q) and 2u + 1 (taps 2q + 1) read the SAME window
    // entries: one packed FMA per (q, subband) computes both, each half the
    // scalar fma sequence of its output (bit-identical)
#pragma unroll
    for (int u = 0; u < IJ / 2; ++u) {
      f2_t s2 = 0ull;   // {s_2u, s_2u+1}
#pragma unroll
      for (int q = 0; q < HT; ++q) {
        const int tj = u - q + HT - 1;
        s2 = ffma2(pk2(fb.h[2 * q], fb.h[2 * q + 1]), pk2(wl[tj], wl[tj]), s2);
        s2 = ffma2(pk2(fb.g[2 * q], fb.g[2 * q + 1]), pk2(wh[tj], wh[tj]), s2);
      }
      const float2 o2 = up2(s2);
      *reinterpret_cast<float2*>(&otile[oidx(rr, IJ * q8 + 2 * u)]) = o2;
    }
  }
  __syncthreads();
  // write-back: lanes along the row (a register-tiled thread's own outputs
  // are 8 apart -- 32 sectors per store instruction)
  if ((w_out & 3) == 0 && (reinterpret_cast<unsigned long long>(o) & 15) == 0) {
    for (int e = threadIdx.x; e < IR * (IC / 4); e += 256) {
      const int rr = e / (IC / 4), c4 = e - rr * (IC / 4);
      const int r = r0 + rr, cc = c0 + 4 * c4;
      if (r < h_out && cc < w_out) {
        float4 v = *reinterpret_cast<const float4*>(&otile[rr * IC + 4 * oslot(c4)]);
        if (rr & 1) v = make_float4(v.z, v.w, v.x, v.y);
        *reinterpret_cast<float4*>(o + (long long)r * w_out + cc) = v;
      }
    }
  } else {
    for (int e = threadIdx.x; e < IR * IC; e += 256) {
      const int rr = e / IC, c = e - rr * IC;
      const int r = r0 + rr, cc = c0 + c;
      if (r < h_out && cc < w_out) o[(long long)r * w_out + cc] = otile[oidx(rr, c)];
    }
  }
}

}  // namespace

cudaError_t launch_dwt_level(const float* in, long long in_stride, int h_in, int w_in, float* ll,
                             long long ll_stride, float* sub, long long sub_stride, int count,
                             const FilterBank& fb, cudaStream_t st) {
  const int hs = (h_in + 1) / 2, ws = (w_in + 1) / 2;
  dim3 grid((ws + FC - 1) / FC, (hs + FR - 1) / FR, count);
  switch (fb.taps) {
    case 2: return launch_pdl(dwt_fwd_kernel<2>, grid, dim3(256), 0, st, in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb);
    case 8: return launch_pdl(dwt_fwd_kernel<8>, grid, dim3(256), 0, st, in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb);
    case 16: return launch_pdl(dwt_fwd_kernel<16>, grid, dim3(256), 0, st, in, in_stride, h_in, w_in, ll, ll_stride, sub, sub_stride, fb);
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_idwt_level(const float* ll, long long ll_stride, const float* sub,
                              long long sub_stride, int h_out, int w_out, float* out,
                              long long out_stride, int count, const FilterBank& fb,
                              const float* tstar, int nsub, int s_lh, int s_ll, const RankState* rs, int k0,
                              cudaStream_t st) {
  const int H = h_out + (h_out & 1), Wd = w_out + (w_out & 1);
  dim3 grid((Wd + IC - 1) / IC, (H + IR - 1) / IR, count);
  const SoftSpec sp{tstar, nsub, s_lh, s_ll, rs, k0, count};
  switch (fb.taps) {
    case 2: return launch_pdl(dwt_inv_kernel<2>, grid, dim3(256), 0, st, ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp);
    case 8: return launch_pdl(dwt_inv_kernel<8>, grid, dim3(256), 0, st, ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp);
    case 16: return launch_pdl(dwt_inv_kernel<16>, grid, dim3(256), 0, st, ll, ll_stride, sub, sub_stride, h_out, w_out, out, out_stride, fb, sp);
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
