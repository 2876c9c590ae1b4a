// Standalone probe of the tcgen05 building blocks in csrc/tc_util.cuh:
// K-major no-swizzle smem descriptors, kind::i8 MMA (cta_group::1 M=128 and
// cta_group::2 M=128 / M=256), multicast commit, TMEM allocation and the
// accumulator layout read back with tcgen05.ld.  Prints PASS/FAIL per case.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o probe probe_tcgen05.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2204_06979_b200/csrc/tc_util.cuh"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int K = 64;  // two K-steps of 32 bytes

__device__ inline int canon(int r, int k, int rows) {  // K-major no-swizzle byte offset
  return (k / 16) * (rows * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 16);
}

// CG = cta group; MT = total M; N = total N.  Each CTA holds MT/CG rows of A and N/CG rows of B.
template <int CG, int MT, int N>
__global__ void probe_kernel(const signed char* A, const signed char* B, int* out) {
  constexpr int MR = MT / CG, NR = N / CG;
  __shared__ __align__(1024) signed char sA[MR * K];
  __shared__ __align__(1024) signed char sB[NR * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t rank = (CG == 2) ? tc::cluster_ctarank() : 0;
  for (int i = threadIdx.x; i < MR * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    sA[canon(r, k, MR)] = A[(rank * MR + r) * K + k];
  }
  for (int i = threadIdx.x; i < NR * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    sB[canon(r, k, NR)] = B[(rank * NR + r) * K + k];
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    tc::tmem_alloc<CG>(&tbase, 128);
    tc::tmem_relinquish<CG>();
  }
  tc::tc_fence_before();
  if (CG == 2) tc::cluster_sync(); else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_i8(MT, N);
    for (int ks = 0; ks < K / 32; ++ks) {
      uint64_t ad = tc::sdesc_kmajor_noswz(tc::smem_u32(sA) + ks * 2 * MR * 16, MR * 16, 128);
      uint64_t bd = tc::sdesc_kmajor_noswz(tc::smem_u32(sB) + ks * 2 * NR * 16, NR * 16, 128);
      tc::mma_i8<CG>(tmem, ad, bd, idesc, ks > 0);
    }
    tc::mma_commit<CG>(&bar, 0x3);
  }
  tc::mbar_wait_cluster(&bar, 0);
  tc::tc_fence_after();
  // each warp reads its 32-lane quadrant, all 128 allocated columns (first N*MR/128 meaningful)
  if (warp < 4) {
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      tc::tmem_ld_wait();
      int lane = warp * 32 + (threadIdx.x & 31);
      for (int j = 0; j < 32; ++j) out[(rank * 128 + lane) * 128 + c0 + j] = (int)v[j];
    }
  }
  tc::tc_fence_before();
  if (CG == 2) tc::cluster_sync(); else __syncthreads();
  if (warp == 0) tc::tmem_dealloc<CG>(tmem, 128);
}

template <int CG, int MT, int N>
bool run(const char* name) {
  std::vector<signed char> A(MT * K), B(N * K);
  srand(1234 + MT + N + CG);
  for (auto& a : A) a = (signed char)(rand() % 11 - 5);
  for (auto& b : B) b = (signed char)(rand() % 11 - 5);
  std::vector<int> D(MT * N);
  for (int m = 0; m < MT; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int k = 0; k < K; ++k) s += A[m * K + k] * B[n * K + k];
      D[m * N + n] = s;
    }
  signed char *dA, *dB;
  int* dO;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dO, 2 * 128 * 128 * sizeof(int)));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dO, 0, 2 * 128 * 128 * sizeof(int)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CG, 1, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, probe_kernel<CG, MT, N>, (const signed char*)dA, (const signed char*)dB, dO));
  CK(cudaDeviceSynchronize());
  std::vector<int> O(2 * 128 * 128);
  CK(cudaMemcpy(O.data(), dO, O.size() * sizeof(int), cudaMemcpyDeviceToHost));
  // hypotheses for (cta, lane, col) -> (m, n)
  const int MR = MT / CG;
  int bad_h1 = 0, bad_h2 = 0, bad_h3 = 0;
  for (int r = 0; r < CG; ++r)
    for (int m = 0; m < MR; ++m)
      for (int n = 0; n < N; ++n) {
        int want = D[(r * MR + m) * N + n];
        // H1: row m -> lane m, col n  (M per CTA == 128)
        if (MR == 128) { if (O[(r * 128 + m) * 128 + n] != want) ++bad_h1; } else ++bad_h1;
        // H2: M per CTA == 64: lane m + 64*(n / (N/2)), col n % (N/2)
        if (MR == 64) {
          int lane = m + 64 * (n / (N / 2)), col = n % (N / 2);
          if (O[(r * 128 + lane) * 128 + col] != want) ++bad_h2;
        } else ++bad_h2;
        // H3: M per CTA == 64: lane m (0..63), col n
        if (MR == 64) { if (O[(r * 128 + m) * 128 + n] != want) ++bad_h3; } else ++bad_h3;
      }
  printf("%-28s H1(lane=m,col=n,M128) bad=%d  H2(2x2 interleaved) bad=%d  H3(lane=m<64,col=n) bad=%d  -> %s\n", name,
         bad_h1, bad_h2, bad_h3, (bad_h1 == 0 || bad_h2 == 0 || bad_h3 == 0) ? "PASS" : "FAIL");
  if (bad_h1 && bad_h2 && bad_h3) {
    for (int l = 0; l < 4; ++l) {
      printf("  cta0 lane %d:", l);
      for (int c = 0; c < 8; ++c) printf(" %d", O[l * 128 + c]);
      printf("   want row %d:", l);
      for (int c = 0; c < 8; ++c) printf(" %d", D[l * N + c]);
      printf("\n");
    }
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return bad_h1 == 0 || bad_h2 == 0 || bad_h3 == 0;
}

int main() {
  bool ok = true;
  ok &= run<1, 128, 64>("cta_group::1 M128 N64");
  ok &= run<1, 128, 96>("cta_group::1 M128 N96");
  ok &= run<2, 256, 64>("cta_group::2 M256 N64");
  ok &= run<2, 128, 64>("cta_group::2 M128 N64");
  ok &= run<2, 128, 96>("cta_group::2 M128 N96");
  ok &= run<2, 128, 128>("cta_group::2 M128 N128");
  printf(ok ? "ALL PASS\n" : "SOME FAIL\n");
  return ok ? 0 : 1;
}
