// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput per SM (sm_100a).
#include <cstdio>
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int CH>
__global__ void k1(float* out, int iters, float m, float b, long long* cyc) {
  float a[CH];
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fmaf(a[c], m, b);
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
__global__ void k2(float* out, int iters, float m, float b, long long* cyc) {
  unsigned long long a[CH];
  unsigned long long mm, bb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(mm) : "f"(m));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  for (int c = 0; c < CH; ++c) { float x = threadIdx.x * 1e-3f + c; asm("mov.b64 %0, {%1, %1};" : "=l"(a[c]) : "f"(x)); }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = f2(a[c], mm, bb);
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[c])); s += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int nt : {256, 512, 1024}) {
    long long h;
    k1<8><<<148, nt>>>(out, iters, 0.999f, 1e-4f, cyc); cudaDeviceSynchronize();
    k1<8><<<148, nt>>>(out, iters, 0.999f, 1e-4f, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double f1 = (double)nt * iters * 8 / h;
    k2<8><<<148, nt>>>(out, iters, 0.999f, 1e-4f, cyc); cudaDeviceSynchronize();
    k2<8><<<148, nt>>>(out, iters, 0.999f, 1e-4f, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double f2v = (double)nt * iters * 8 * 2 / h;
    printf("threads %4d: FFMA %.1f fma/clk/SM   FFMA2 %.1f fma/clk/SM\n", nt, f1, f2v);
  }
  return 0;
}
