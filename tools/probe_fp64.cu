// Microbenchmark: fp64 / fp32 FMA latency and throughput per SM, smem bandwidth.
#include <cstdio>
template <typename T, int CH>
__global__ void fma_kernel(T* out, int iters, long long* cyc) {
  T a[CH];
  for (int c = 0; c < CH; ++c) a[c] = (T)(threadIdx.x + c) * (T)1e-3;
  const T m = (T)0.9999, b = (T)1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m + b;
  }
  __syncthreads();
  long long t1 = clock64();
  T s = 0;
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void div_kernel(double* out, int iters, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 3.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = b / (a + 1.0);
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <typename T, int CH>
void run(const char* name, int threads) {
  T* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 64);
  int iters = 4096;
  fma_kernel<T, CH><<<1, threads>>>(out, iters, cyc);
  fma_kernel<T, CH><<<1, threads>>>(out, iters, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)threads * iters * CH;
  printf("%-6s chains=%d threads=%4d: %8.2f FMA/clk/SM   %.2f clk per dependent FMA\n", name, CH, threads, ops / c,
         (double)c / iters / CH * (CH == 1 ? 1 : 1));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<double, 1>("fp64", 32);
  run<double, 1>("fp64", 1024);
  run<double, 8>("fp64", 1024);
  run<float, 1>("fp32", 32);
  run<float, 8>("fp32", 1024);
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
  div_kernel<<<1, 32>>>(out, 4096, cyc); div_kernel<<<1, 32>>>(out, 4096, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("fp64 division latency: %.1f clk\n", (double)c / 4096);
  return 0;
}
