// Measured roofline denominators the driver's MEASURED_PEAKS.json lacks
// (VERDICT r01 item 2): fp64 FMA throughput of the whole GPU and of one SM,
// and the dense tcgen05.mma kind::i8 throughput (cta_group::2, the Gram's
// shape M=128 x N=128 and the largest M=256 x N=256), operands resident in
// shared memory (no data movement: the tensor-pipe ceiling).  Prints one JSON
// line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 \
//   -o /tmp/probe_peaks tools/probe_peaks.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_2204_06979_b200/csrc/tc_util.cuh"

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

template <int CH>
__global__ void __launch_bounds__(1024) dfma_kernel(double* out, int iters) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = (double)(threadIdx.x + c) * 1e-3;
  const double m = 0.9999, b = 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma(a[c], m, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one cluster of 2 CTAs; thread 0 of CTA 0 issues `iters` x 4 k-steps of
// cta_group::2 kind::i8 MMAs (M = MT rows over the pair, N columns)
template <int MT, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_i8_kernel(int iters, int* sink) {
  constexpr int MR = MT / 2, NR = N / 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tbase;
  unsigned char* sA = smem;
  unsigned char* sB = smem + MR * 128;
  for (int i = threadIdx.x; i < (MR + NR) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0u, 0u, 0u);
  tc::fence_proxy_async_smem();
  const uint32_t rank = tc::cluster_ctarank();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar_done, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    tc::tmem_alloc<2>(&tbase, 512);
    tc::tmem_relinquish<2>();
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_i8(MT, N, true, true);
    const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        tc::mma_i8<2>(tmem, tc::sdesc_kmajor_sw128(a0 + ks * 32), tc::sdesc_kmajor_sw128(b0 + ks * 32), idesc,
                      (it | ks) ? 1u : 0u);
    tc::mma_commit<2>(&bar_done, 0x3);
  }
  if (threadIdx.x == 0) tc::mbar_wait_cluster(&bar_done, 0);
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) {
    uint32_t v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(0) << 16), v);
    tc::tmem_ld_wait();
    if (v[0] == 0x7fffffffu) sink[0] = 1;
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (threadIdx.x < 32) {
    tc::tc_fence_after();
    tc::tmem_dealloc<2>(tmem, 512);
  }
}

template <typename F>
float time_ms(F f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double* out;
  int* sink;
  CK(cudaMalloc(&out, (size_t)sms * 8 * 1024 * 8));
  CK(cudaMalloc(&sink, 64));
  const int it64 = 1 << 14;
  // whole GPU: 2 CTAs x 1024 threads per SM, 8 independent chains each
  const float ms_all = time_ms([&] { dfma_kernel<8><<<2 * sms, 1024>>>(out, it64); });
  const double f_all = 2.0 * 2 * sms * 1024.0 * it64 * 8;
  // one SM
  const float ms_one = time_ms([&] { dfma_kernel<8><<<1, 1024>>>(out, it64); });
  const double f_one = 2.0 * 1024.0 * it64 * 8;
  // tcgen05 kind::i8: every SM pair issuing back to back
  const int itm = 4096;
  auto mma = [&](auto kern, int mt, int n, size_t smem) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const float ms = time_ms([&] { kern<<<sms, 128, smem>>>(itm, sink); });
    CK(cudaGetLastError());
    const double ops = 2.0 * mt * n * 128.0 * itm * (sms / 2);   // 4 k-steps of K = 32 per iteration
    return ops / (ms * 1e-3) / 1e12;
  };
  const double i8_128 = mma(mma_i8_kernel<128, 128>, 128, 128, (64 + 64) * 128);
  const double i8_256 = mma(mma_i8_kernel<256, 256>, 256, 256, (128 + 128) * 128);
  printf("{\"fp64_tflops\": %.3f, \"fp64_tflops_per_sm\": %.4f, \"fp64_dfma_per_clk_per_sm\": %.1f, "
         "\"i8_tops_m128n128_cg2\": %.1f, \"i8_tops_m256n256_cg2\": %.1f, \"sms\": %d, \"clock_mhz_attr\": %d, "
         "\"how\": \"fp64: dfma chains, 2 x 1024 threads per SM (all SMs) and 1024 threads on one SM; "
         "i8: tcgen05.mma.cta_group::2.kind::i8, K=32 per instruction, smem-resident operands, one issuing "
         "thread per SM pair, all pairs; CUDA events, second of two runs\"}\n",
         f_all / (ms_all * 1e-3) / 1e12, f_one / (ms_one * 1e-3) / 1e12,
         f_one / 2.0 / (ms_one * 1e-3) / (clk_khz * 1e3), i8_128, i8_256, sms, clk_khz / 1000);
  return 0;
}
