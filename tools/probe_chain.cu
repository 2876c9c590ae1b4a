// Dependent fp64 recurrence latency on one warp: which part of a Sturm step
// costs (pure DFMA chain; the Sturm step with operands in registers; with
// shared-memory operands; with the sign count).
#include <cstdio>
__global__ void k(const double* __restrict__ gd, int n, int reps, long long* out, double* sink) {
  __shared__ double d[1024], e2[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { d[i] = gd[i]; e2[i] = gd[1024 + i] * 1e-3; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const double x = 0.37 + threadIdx.x * 1e-3;
  double r = 0;
  long long t0, t1;
  // 1: pure dependent DFMA chain
  double b = 1.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) b = fma(b, 0.999, 1e-3);
  t1 = clock64(); r += b; if (threadIdx.x == 0) out[0] = t1 - t0;
  // 2: Sturm step, operands in registers (constants)
  double a = 1.0; b = 0.5;
  int c = 0;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double t = fma(0.3 - x, b, -0.01 * a);
    c += (int)((unsigned)(__double2hiint(t) ^ __double2hiint(b)) >> 31);
    a = b; b = t;
  }
  t1 = clock64(); r += b + c; if (threadIdx.x == 0) out[1] = t1 - t0;
  // 3: Sturm step, operands from shared memory
  a = 1.0; b = 0.5; c = 0;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double t = fma(d[i & 1023] - x, b, -e2[i & 1023] * a);
    c += (int)((unsigned)(__double2hiint(t) ^ __double2hiint(b)) >> 31);
    a = b; b = t;
  }
  t1 = clock64(); r += b + c; if (threadIdx.x == 0) out[2] = t1 - t0;
  // 4: as 3 without the count
  a = 1.0; b = 0.5;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double t = fma(d[i & 1023] - x, b, -e2[i & 1023] * a);
    a = b; b = t;
  }
  t1 = clock64(); r += b; if (threadIdx.x == 0) out[3] = t1 - t0;
  // 5: as 3 with the rescale every 8 steps
  a = 1.0; b = 0.5; c = 0;
  t0 = clock64();
  for (int i = 0; i + 7 < n; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double t = fma(d[(i + u) & 1023] - x, b, -e2[(i + u) & 1023] * a);
      c += (int)((unsigned)(__double2hiint(t) ^ __double2hiint(b)) >> 31);
      a = b; b = t;
    }
    const double m = fmax(fabs(a), fabs(b));
    const double sc = m > 0x1p+500 ? 0x1p-500 : (m < 0x1p-500 ? 0x1p+500 : 1.0);
    a *= sc; b *= sc;
  }
  t1 = clock64(); r += b + c; if (threadIdx.x == 0) out[4] = t1 - t0;
  // 6: fp32 version of 3
  float af = 1.f, bf = 0.5f; c = 0;
  const float xf = (float)x;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const float t = fmaf((float)d[i & 1023] - xf, bf, -(float)e2[i & 1023] * af);
    c += (int)(__float_as_uint(t) ^ __float_as_uint(bf)) >> 31;
    af = bf; bf = t;
  }
  t1 = clock64(); r += bf + c; if (threadIdx.x == 0) out[5] = t1 - t0;
  sink[threadIdx.x] = r;
}
int main() {
  double* gd; long long* o; double* sink;
  cudaMallocManaged(&gd, 2048 * sizeof(double)); cudaMallocManaged(&o, 16 * sizeof(long long)); cudaMallocManaged(&sink, 64 * sizeof(double));
  for (int i = 0; i < 2048; ++i) gd[i] = 0.5 + 0.001 * (i % 97);
  const int n = 224;
  for (int r = 0; r < 2; ++r) { k<<<1, 256>>>(gd, n, 1, o, sink); cudaDeviceSynchronize(); }
  const char* nm[6] = {"pure DFMA chain", "Sturm step, register operands", "Sturm step, smem operands", "smem operands, no count", "smem + rescale/8", "fp32 Sturm step, smem"};
  for (int i = 0; i < 6; ++i) printf("%-34s %6.1f cycles/step\n", nm[i], (double)o[i] / n);
  return 0;
}
