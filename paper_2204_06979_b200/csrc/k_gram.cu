// K1 (north_star stage (1)): G = Y Y^T over all pixels.
//
// Y is the BSQ cube viewed as a bands x N row-major matrix (pixel-contiguous,
// "K-major" for the contraction over pixels).  G is B x B, symmetric,
// uncentered, accumulated in fp64: sigma_b^2 = 1/(N [(G+dI)^-1]_bb) amplifies
// the Gram's relative error by roughly the band SNR (SURVEY.md §7 hard part
// 1), so the sums must be far more accurate than an fp32 accumulation.
//
// This kernel is the fp64 SIMT formulation (fallback for B > 224; the
// tensor-core path is k_gram_tc.cu): 64x64 output blocks (upper
// block triangle only), the pixel axis split into `nsplit`
// slices whose fp64 partial Grams are summed in a fixed order by a second
// kernel, so the result is bit-deterministic.  It also raises the device
// non-finite-input flag ("finite values").
#include "common.cuh"

namespace {

constexpr int TB = 64;   // output block edge
constexpr int TP = 32;   // pixels per smem stage

__global__ void __launch_bounds__(256) gram_partial_kernel(const float* __restrict__ Y, long long n,
                                                           int B, int nb, double* __restrict__ partial,
                                                           long long per_split, int* nonfinite) {
  __shared__ double As[TP][TB + 1];
  __shared__ double Bs[TP][TB + 1];
  // decode upper-triangular block pair
  int pair = blockIdx.x, bi = 0;
  while (pair >= nb - bi) { pair -= nb - bi; ++bi; }
  const int bj = bi + pair;
  const int i0 = bi * TB, j0 = bj * TB;
  const int split = blockIdx.y;
  const long long p_begin = (long long)split * per_split;
  const long long p_end = min(n, p_begin + per_split);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  bool bad = false;
  for (long long p0 = p_begin; p0 < p_end; p0 += TP) {
    // load 64 rows x 32 pixels of both operands (coalesced along pixels)
#pragma unroll
    for (int it = 0; it < (TB * TP) / 256; ++it) {
      int idx = threadIdx.x + it * 256;
      int r = idx / TP, c = idx % TP;
      long long p = p0 + c;
      float va = 0.f, vb = 0.f;
      if (p < p_end) {
        if (i0 + r < B) va = Y[(long long)(i0 + r) * n + p];
        if (j0 + r < B) vb = Y[(long long)(j0 + r) * n + p];
      }
      bad |= !isfinite(va) || !isfinite(vb);
      As[c][r] = (double)va;
      Bs[c][r] = (double)vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int pp = 0; pp < TP; ++pp) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[pp][ty * 4 + q]; b[q] = Bs[pp][tx * 4 + q]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  if (bad) atomicOr(nonfinite, 1);
  double* P = partial + (long long)split * B * B;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int i = i0 + ty * 4 + u, j = j0 + tx * 4 + v;
      if (i < B && j < B) {
        P[(long long)i * B + j] = acc[u][v];   // upper block triangle; the reduce reads (min,max)
      }
    }
}

// G = sum of the per-split partial Grams.  One block = 32 consecutive
// elements (coalesced lanes) x 8 warps; warp w sums splits k = w, w + 8, ...
// with its loads in flight together, then the 8 warp sums are added in a
// fixed order -- deterministic, and not one 74-deep chain of L2 round trips
// per element.  The (min, max) element is read so G is exactly symmetric.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double* __restrict__ partial, int nsplit, int B,
                                                          double* __restrict__ G, int sym) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long tot = (long long)B * B;
  const long long idx = blockIdx.x * 32LL + lane;
  double s = 0.0;
  // sym > 0: only i <= j is computed (both G[i][j] and G[j][i] are written)
  const int i0 = idx < tot ? (int)(idx / B) : 0, j0 = idx < tot ? (int)(idx % B) : 0;
  const bool active = idx < tot && (sym == 0 || i0 <= j0);
  if (active) {
    const int i = i0, j = j0;
    const long long src = (long long)min(i, j) * B + max(i, j);
    // sym > 0: partials of the diagonal blocks ([0, sym) and [sym, B)) are not
    // symmetric -- G = (sum P + sum P^T) / 2 there (tensor-core Gram, K1)
    const bool both = sym > 0 && ((i < sym) == (j < sym));
    const long long srt = (long long)max(i, j) * B + min(i, j);
    double v[16];
    for (int k0 = w; k0 < nsplit; k0 += 8 * 16) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = k0 + 8 * u;
        v[u] = k < nsplit ? __ldcs(partial + (long long)k * tot + src) : 0.0;
        if (both && k < nsplit) v[u] += __ldcs(partial + (long long)k * tot + srt);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    if (both) s *= 0.5;
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && active) {
    double t = part[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += part[q][lane];
    G[idx] = t;
    if (sym > 0 && i0 != j0) G[(long long)j0 * B + i0] = t;
  }
}

}  // namespace

int gram_nsplit(long long n, int B) {
  int nb = (B + TB - 1) / TB;
  int pairs = nb * (nb + 1) / 2;
  long long want = (3LL * 148 + pairs - 1) / pairs;
  long long maxs = (n + 2047) / 2048;
  if (want > maxs) want = maxs;
  if (want < 1) want = 1;
  return (int)want;
}

cudaError_t launch_gram(const float* Y, long long n, int B, double* partial, int nsplit, double* G,
                        int* nonfinite, cudaStream_t st) {
  int nb = (B + TB - 1) / TB;
  int pairs = nb * (nb + 1) / 2;
  long long per = (n + nsplit - 1) / nsplit;
  per = (per + TP - 1) / TP * TP;
  dim3 grid(pairs, nsplit);
  gram_partial_kernel<<<grid, 256, 0, st>>>(Y, n, B, nb, partial, per, nonfinite);
  return launch_gram_reduce(partial, nsplit, B, G, st);
}

cudaError_t launch_gram_reduce(const double* partial, int nsplit, int B, double* G, cudaStream_t st, int sym) {
  long long tot = (long long)B * B;
  gram_reduce_kernel<<<(unsigned)((tot + 31) / 32), 256, 0, st>>>(partial, nsplit, B, G, sym);
  return cudaGetLastError();
}
