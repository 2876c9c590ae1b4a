// Microbenchmark of k_sure.cu's shared-memory block sort (tools only).
#include "../paper_2204_06979_b200/csrc/k_sure.cu"
#include <cstdio>
#include <vector>
#include <algorithm>

template <int IT>
__global__ void sortk(const unsigned* in, unsigned* out, int P, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* keys = reinterpret_cast<unsigned*>(sm);
  unsigned* buf = keys + 8192;
  for (int i = threadIdx.x; i < P; i += NT) keys[sw(i)] = in[blockIdx.x * P + i];
  __syncthreads();
  long long t0 = clock64();
  unsigned* r = block_sort<IT>(keys, buf, P);
  __syncthreads();
  long long t1 = clock64();
  for (int i = threadIdx.x; i < P; i += NT) out[blockIdx.x * P + i] = r[sw(i)];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int nb = 148;
  for (int P : {16, 32, 64, 256, 1024, 4096, 8192}) {
    std::vector<unsigned> h(nb * P);
    unsigned s = 12345;
    for (auto& v : h) { s = s * 1664525u + 1013904223u; v = s >> 1; }
    unsigned *din, *dout; long long* dc;
    cudaMalloc(&din, h.size() * 4); cudaMalloc(&dout, h.size() * 4); cudaMalloc(&dc, nb * 8);
    cudaMemcpy(din, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(sortk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(sortk<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int rep = 0; rep < 2; ++rep) {
      if (P <= 4096) sortk<16><<<nb, NT, 65536>>>(din, dout, P, dc);
      else sortk<32><<<nb, NT, 65536>>>(din, dout, P, dc);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned> o(h.size()); std::vector<long long> c(nb);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), dc, nb * 8, cudaMemcpyDeviceToHost);
    bool ok = true;
    for (int b = 0; b < nb; ++b) {
      std::vector<unsigned> ref(h.begin() + b * P, h.begin() + (b + 1) * P);
      std::sort(ref.begin(), ref.end());
      for (int i = 0; i < P; ++i) ok &= ref[i] == o[b * P + i];
    }
    std::sort(c.begin(), c.end());
    printf("P %d err %s ok %d cycles median %lld max %lld\n", P, cudaGetErrorString(e), ok, c[nb / 2], c[nb - 1]);
  }
  return 0;
}
