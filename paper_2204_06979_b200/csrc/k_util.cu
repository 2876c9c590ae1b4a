// Small kernels of the E1 sharded path.
#include "common.cuh"

namespace {

// flag |= any non-finite element of x[0, n): after the Gram all-reduce every
// rank holds the same G, so every rank raises the same flag (a NaN on one
// rank's slab reaches every rank's G through the sum) and all ranks stop
// together at the first host check -- no rank waits in a collective the
// others skipped.
__global__ void check_finite_kernel(const double* __restrict__ x, long long n, int* flag) {
  pdl_wait();
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// dst[map[r]][:] = src[r][:] for r < nrows (rows of ncols doubles); dst rows not
// in the map are zeroed (the chunk's per-subband SURE statistics of this rank's
// components, placed at their chunk positions before the all-reduce); the slot
// after the rows carries this rank's flag (SURE overflow) into the same sum
struct RowMap {
  int to[HYDE_MAX_CHUNK];
};
__global__ void scatter_rows_kernel(const double* __restrict__ src, int nrows, int ncols, RowMap m, double* dst,
                                    int dst_rows, const int* flag_in) {
  pdl_wait();
  const int tot = dst_rows * ncols;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) dst[i] = 0.0;
  if (threadIdx.x == 0) dst[tot] = (flag_in && *flag_in) ? 1.0 : 0.0;   // this rank's flag, summed with the rows
  __syncthreads();
  for (int i = threadIdx.x; i < nrows * ncols; i += blockDim.x) {
    const int r = i / ncols, c = i % ncols;
    dst[m.to[r] * ncols + c] = src[i];
  }
}

__global__ void check_finite_f32_kernel(const float* __restrict__ x, long long n, int* flag) {
  bool bad = false;
  const long long n4 = ((uintptr_t)x & 15) == 0 ? n / 4 : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

// flag |= any non-finite value of the fp32 array x[0, n) (HYDE_VALIDATE: one read)
cudaError_t launch_check_finite_f32(const float* x, long long n, int* flag, cudaStream_t st) {
  check_finite_f32_kernel<<<592, 256, 0, st>>>(x, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double* x, long long n, int* flag, cudaStream_t st) {
  const unsigned g = (unsigned)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64);
  return launch_pdl(check_finite_kernel, dim3(g > 0 ? g : 1), dim3(256), 0, st, x, n, flag);
}

cudaError_t launch_scatter_rows(const double* src, int nrows, int ncols, const int* to, double* dst, int dst_rows,
                                const int* flag_in, cudaStream_t st) {
  RowMap m;
  for (int i = 0; i < HYDE_MAX_CHUNK; ++i) m.to[i] = i < nrows ? to[i] : 0;
  return launch_pdl(scatter_rows_kernel, dim3(1), dim3(256), 0, st, src, nrows, ncols, m, dst, dst_rows, flag_in);
}

namespace {
__global__ void flag_from_sum_kernel(const double* x, int* flag) {
  pdl_wait();
  if (threadIdx.x == 0 && *x > 0.0) *flag = 1;
}
}  // namespace

cudaError_t launch_flag_from_sum(const double* x, int* flag, cudaStream_t st) {
  return launch_pdl(flag_from_sum_kernel, dim3(1), dim3(32), 0, st, x, flag);
}
