// K6b (north_star stage (6)): reconstruction to bands
//   X^[b][p] = sum_{k < r*} U[b][k] E^[k][p],   U = diag(sigma) V[:, :r*]
// (SPEC.md:380 step (6) "inverse transforms and de-whitening").  r* is small
// (1-5 at the BASELINE configs), so this is a K = r* outer-product GEMM whose
// cost is the single BSQ write of the output (4 N B bytes): each thread keeps
// its pixels' r* denoised eigen-image values in registers and streams all B
// bands out with 16-byte stores.
#include "common.cuh"

namespace {

constexpr int RK = 8;  // components held in registers per pass

template <int PIX, bool VEC>
__global__ void __launch_bounds__(256) recon_kernel(const float* __restrict__ E, long long ldE, long long n,
                                                    int B, const float* __restrict__ U, int ldu, int k0,
                                                    int kcount, int accumulate, float* __restrict__ out,
                                                    const RankState* __restrict__ rs) {
  pdl_wait();
  if (rs) {   // rank decided on the device: nothing until it is found, then r* - k0 components
    if (!rs->found) return;
    kcount = min(kcount, rs->rank - k0);
    if (kcount <= 0) return;
  }
  extern __shared__ float Us[];  // B x RK
  for (int i = threadIdx.x; i < B * RK; i += blockDim.x) {
    int b = i / RK, k = i % RK;
    Us[i] = (k < kcount) ? U[(size_t)b * ldu + k0 + k] : 0.f;
  }
  __syncthreads();
  const long long p0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * PIX;
  if (p0 >= n) return;
  const bool full = p0 + PIX <= n;
  float e[RK][PIX];
#pragma unroll
  for (int k = 0; k < RK; ++k) {
#pragma unroll
    for (int q = 0; q < PIX; ++q) e[k][q] = 0.f;
    if (k < kcount) {
      const float* src = E + (size_t)(k0 + k) * ldE + p0;
      if (VEC && full) {
        float4 v = __ldcs(reinterpret_cast<const float4*>(src));
        e[k][0] = v.x; e[k][1] = v.y; e[k][2] = v.z; e[k][3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < PIX; ++q) e[k][q] = (p0 + q < n) ? src[q] : 0.f;
      }
    }
  }
  for (int b = 0; b < B; ++b) {
    float acc[PIX];
#pragma unroll
    for (int q = 0; q < PIX; ++q) acc[q] = 0.f;
    const float* ub = Us + b * RK;
#pragma unroll
    for (int k = 0; k < RK; ++k) {
      const float u = ub[k];
#pragma unroll
      for (int q = 0; q < PIX; ++q) acc[q] = fmaf(u, e[k][q], acc[q]);
    }
    float* dst = out + (size_t)b * n + p0;
    if (VEC && full) {
      float4 v = make_float4(acc[0], acc[1], acc[2], acc[3]);
      if (accumulate) {
        float4 o = *reinterpret_cast<const float4*>(dst);
        v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
      }
      __stcs(reinterpret_cast<float4*>(dst), v);
    } else {
#pragma unroll
      for (int q = 0; q < PIX; ++q)
        if (p0 + q < n) dst[q] = accumulate ? dst[q] + acc[q] : acc[q];
    }
  }
}

}  // namespace

// rs == NULL: rank is the component count.  rs != NULL: rank is an upper bound
// and the kernels read r* from the device rank state (no-ops until it is found).
cudaError_t launch_reconstruct(const float* E, long long ldE, long long n, int B, const float* U,
                               int ldu, int rank, float* out, cudaStream_t st, const RankState* rs) {
  constexpr int PIX = 4;
  const long long threads = (n + PIX - 1) / PIX;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  const size_t smem = (size_t)B * RK * sizeof(float);
  const bool vec = (n % 4 == 0) && (ldE % 4 == 0) && ((uintptr_t)E % 16 == 0) && ((uintptr_t)out % 16 == 0);
  for (int k0 = 0; k0 < rank; k0 += RK) {
    const int kc = rank - k0 < RK ? rank - k0 : RK;
    const int acc = k0 > 0;
    if (vec)
      launch_pdl(recon_kernel<PIX, true>, dim3(blocks), dim3(256), smem, st, E, ldE, n, B, U, ldu, k0, kc, acc, out, rs);
    else
      launch_pdl(recon_kernel<PIX, false>, dim3(blocks), dim3(256), smem, st, E, ldE, n, B, U, ldu, k0, kc, acc, out, rs);
  }
  return cudaGetLastError();
}
