// K3 (north_star stage (3)): eigen-image projection
//   E[k][p] = sum_b W[b][k] Y[b][p],   W = diag(sigma)^-1 V[:, chunk]
// a dense N x B . B x r contraction with r = chunk (<= 32).  At r = 16 it is
// 16 FMA per 4-byte load (4 flop/B): HBM-bound on the fp32 pipe (B200: ~75
// TFLOP/s fp32 vs 6.5 TB/s x 8 flop/B = 52 TFLOP/s needed at r = 16), so it
// runs on CUDA cores in exact fp32 FMA -- no tensor-core reshaping of an
// HBM-bound stream (SURVEY.md §8(d) "A3/A6 GEMMs: HBM-bound").
// One pass over the cube: each thread owns PIX consecutive pixels for all r
// outputs, W is broadcast from shared memory, loads are 16 B (float4) when
// the band stride allows it.
#include "common.cuh"

namespace {

template <int NC, int PIX, bool VEC, int UB>
__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ Y, long long n, int B,
                                                      const float* __restrict__ W, int ldw, int ncomp,
                                                      float* __restrict__ E, long long ldE) {
  pdl_wait();
  extern __shared__ float Ws[];  // B x NC
  for (int i = threadIdx.x; i < B * NC; i += blockDim.x) {
    int b = i / NC, k = i % NC;
    Ws[i] = (k < ncomp) ? W[(size_t)b * ldw + k] : 0.f;
  }
  __syncthreads();
  // blocks walk the cube from its END: K1's pass finishes on the last pixels,
  // which are still in L2 when this kernel starts
  const long long p0 = ((long long)(gridDim.x - 1 - blockIdx.x) * blockDim.x + threadIdx.x) * PIX;
  if (p0 >= n) return;
  float acc[NC][PIX];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int q = 0; q < PIX; ++q) acc[k][q] = 0.f;
  const bool full = p0 + PIX <= n;
  // UB bands per step: UB independent 16-byte loads in flight per thread
  int b = 0;
  for (; b + UB <= B; b += UB) {
    float y[UB][PIX];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const float* row = Y + (size_t)(b + u) * n + p0;
      if (VEC && full) {
        if constexpr (PIX == 4) {
          const float4 v = __ldcs(reinterpret_cast<const float4*>(row));
          y[u][0] = v.x; y[u][1] = v.y; y[u][2] = v.z; y[u][3] = v.w;
        } else if constexpr (PIX == 2) {
          const float2 v = __ldcs(reinterpret_cast<const float2*>(row));
          y[u][0] = v.x; y[u][1] = v.y;
        } else {
#pragma unroll
          for (int q = 0; q < PIX; ++q) y[u][q] = row[q];
        }
      } else {
#pragma unroll
        for (int q = 0; q < PIX; ++q) y[u][q] = (p0 + q < n) ? row[q] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const float* wb = Ws + (b + u) * NC;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const float wk = wb[k];
#pragma unroll
        for (int q = 0; q < PIX; ++q) acc[k][q] = fmaf(wk, y[u][q], acc[k][q]);
      }
    }
  }
  for (; b < B; ++b) {
    float y[PIX];
    const float* row = Y + (size_t)b * n + p0;
#pragma unroll
    for (int q = 0; q < PIX; ++q) y[q] = (p0 + q < n) ? row[q] : 0.f;
    const float* wb = Ws + b * NC;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const float wk = wb[k];
#pragma unroll
      for (int q = 0; q < PIX; ++q) acc[k][q] = fmaf(wk, y[q], acc[k][q]);
    }
  }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    if (k >= ncomp) break;
    float* out = E + (size_t)k * ldE + p0;
    if (VEC && full && PIX == 4) {
      *reinterpret_cast<float4*>(out) = make_float4(acc[k][0], acc[k][1], acc[k][2], acc[k][3]);
    } else {
#pragma unroll
      for (int q = 0; q < PIX; ++q)
        if (p0 + q < n) out[q] = acc[k][q];
    }
  }
}

template <int NC, int PIX, int UB = 8>
cudaError_t launch_nc(const float* Y, long long n, int B, const float* W, int ldw, int ncomp,
                      float* E, long long ldE, cudaStream_t st) {
  const long long threads = (n + PIX - 1) / PIX;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  const size_t smem = (size_t)B * NC * sizeof(float);
  const bool vec = (n % 4 == 0) && (ldE % 4 == 0) && ((uintptr_t)Y % 16 == 0) && ((uintptr_t)E % 16 == 0);
  if (vec) {
    cudaFuncSetAttribute(project_kernel<NC, PIX, true, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(project_kernel<NC, PIX, true, UB>, dim3(blocks), dim3(256), smem, st, Y, n, B, W, ldw, ncomp, E, ldE);
  } else {
    cudaFuncSetAttribute(project_kernel<NC, PIX, false, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(project_kernel<NC, PIX, false, UB>, dim3(blocks), dim3(256), smem, st, Y, n, B, W, ldw, ncomp, E, ldE);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_project(const float* Y, long long n, int B, const float* W, int ldw, int ncomp,
                           float* E, long long ldE, cudaStream_t st) {
  // the rank loop's first chunk is 4 components: fewer accumulators, more loads in flight
  if (ncomp <= 4) return launch_nc<4, 4, 16>(Y, n, B, W, ldw, ncomp, E, ldE, st);
  if (ncomp <= 8) return launch_nc<8, 4>(Y, n, B, W, ldw, ncomp, E, ldE, st);
  if (ncomp <= 16) return launch_nc<16, 4>(Y, n, B, W, ldw, ncomp, E, ldE, st);
  return launch_nc<32, 2>(Y, n, B, W, ldw, ncomp, E, ldE, st);
}
