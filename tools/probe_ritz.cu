// Microbenchmark of the phase-2L Ritz-check helpers in isolation (one CTA,
// the K2 kernel's helpers included verbatim): cycles of tri_bounds,
// bisect_warp (1e-10), twisted_prod, twisted_vec on a Lanczos-like T_n.
#include "../paper_2204_06979_b200/csrc/k_eig.cu"
#include <cstdio>
namespace {
struct PS {
  double d[BM], e[BM], e2[BM], ds[BM], e2s[BM], red[4 * NW];
  double z[8][64], scr[8][4][64];
};
__global__ void probe(int n, long long* out) {
  __shared__ PS S;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int i = tid; i < n; i += NT) {
    S.d[i] = i == 0 ? 7279.0 : (i < 4 ? 0.5 / i : 0.02 * sin(1.0 * i));
    S.e[i] = 0.015 + 0.001 * cos(2.0 * i);
  }
  __syncthreads();
  long long t0 = clock64();
  double glo, ghi;
  tri_bounds(S.d, S.e, S.e2, n, S.red, glo, ghi);
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  const double tsc = tri_scale(tnorm);
  tri_scaled(S.d, S.e2, n, tsc, S.ds, S.e2s);
  long long t1 = clock64();
  double lo = glo * tsc, hi = ghi * tsc, th = 0;
  long long t2 = t1, t3 = t1, t4 = t1, t5 = t1;
  if (w < 4) {
    bisect_warp(S.ds, S.e2s, n, lo, hi, n - 1 - w, 1e-10 * fmax(fabs(glo), fabs(ghi)) * tsc);
    th = 0.5 * (lo + hi) / tsc;
    t2 = clock64();
    twisted_prod(S.d, S.e, n, th, S.z[w], S.scr[w][0], S.scr[w][1], S.scr[w][2], S.scr[w][3]);
    t3 = clock64();
    twisted_vec(S.d, S.e, n, th, tnorm, S.z[w + 4], S.scr[w + 4][0], S.scr[w + 4][1], S.scr[w + 4][2], S.scr[w + 4][3]);
    t4 = clock64();
    int c0, c1;
    sturm_count2(S.ds, S.e2s, n, lo, hi, c0, c1);
    t5 = clock64();
    if (lane == 0 && c0 == -7) out[9] = c1;
  }
  if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = (long long)(th * 1e6); }
}
}  // namespace
int main() {
  long long* o;
  cudaMallocManaged(&o, 16 * sizeof(long long));
  for (int n : {12, 28, 54}) {
    probe<<<1, NT>>>(n, o);
    cudaDeviceSynchronize();
    probe<<<1, NT>>>(n, o);
    cudaDeviceSynchronize();
    printf("n=%d: bounds+scale %lld, bisect %lld, twisted_prod %lld, twisted_vec %lld, one sturm2 pass %lld cycles (theta %.6f)\n",
           n, o[0], o[1], o[2], o[3], o[4], o[5] * 1e-6);
  }
  return 0;
}
