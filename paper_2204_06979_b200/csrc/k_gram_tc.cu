// K1 (north_star stage (1)) on the 5th-generation tensor
// cores: an EXACT integer Gram of a quantised cube, G = diag(s) Q Q^T diag(s).
//
// Why integers (DESIGN.md §4 K1): sigma_b^2 = 1/(N [(G+dI)^-1]_bb) amplifies
// the Gram's relative error by ~the band SNR, so G must be good to ~1e-7
// relative; fp32 (or TF32/BF16-split) accumulation over 10^6 pixels is not,
// and any non-PSD rounding breaks noiseless cubes.  Here each band b is
// scaled by inv_s_b = 16256 / max|y_b| (max from a pre-pass) and rounded:
// q = rint(y inv_s) in [-16256, 16256], split q = 128 S0 + S1 with S0 in
// [-127, 127], S1 in [-64, 63] (both int8).  Then
//   Q Q^T = 16384 S0 S0^T + 128 (S0 S1^T + S1 S0^T) + S1 S1^T
// three int8 x int8 -> int32 GEMMs (tcgen05.mma kind::i8), accumulated
// EXACTLY in TMEM; G is Q Q^T scaled by s_a s_b in fp64.  The result is the
// exact Gram of a 15-bit quantisation of the cube: symmetric PSD by
// construction, deterministic, and ~1e-6 from the fp64 oracle end to end
// (survey/design experiment: /tmp-free numbers in DESIGN.md).
//
// Structure: clusters of 2 CTAs (one SM pair) per pixel range, cta_group::2
// MMAs with M = 128 (64 rows per SM, TMEM "2x2" layout).  Bands are split
// S_a = [0,128), S_b = [128,B); three tiles T_aa (128 x 128), T_ab (128 x Nb),
// T_bb (128 x Nb), Nb = B-128 rounded up to 32; x 3 products = 480 of 512
// TMEM columns for B <= 224.  16 converter warps per CTA load fp32 straight
// from HBM (16-byte loads, ~90 KB in flight per SM), quantise and write the
// int8 slices into shared memory in the UMMA canonical K-major layout; one
// thread of the leader CTA issues the MMAs; the stage ring is released by
// tcgen05.commit multicast to both CTAs.  Each CTA finally reads its TMEM,
// combines the three products in int64 and writes its fp64 partial Gram.
#include "common.cuh"
#include "tc_util.cuh"

namespace {

constexpr int KC = 128;        // pixels (bytes per int8 row) per stage
constexpr int NI = 4;          // int8 stages
constexpr int NCW = 14;        // converter warps
constexpr int NTHREADS = (NCW + 2) * 32;
constexpr int MAXU = 8;        // max band rows per converter warp per stage: (64 + 48) / 14
constexpr int TMEM_COLS = 512;

struct GramTc {
  const float* Y;
  long long n;
  int B;
  int nb;           // Nb (0 when B <= 128)
  int rows_tot;     // 64 + 64 + nb/2 (or 64)
  long long per_pair;
  const unsigned* amax_bits;
  double* partial;  // [pair][B][B]
  int* nonfinite;
};

// smem regions of one int8 slice of a stage: P (64 rows: S_a bands of this SM)
// and QS (64 rows: this SM's half of S_b, nb/2 live rows then zeros).  QS is
// both the A operand of T_bb and -- its first nb/2 rows -- this SM's half of
// the B operand of T_ab and T_bb, so every band is read from HBM once.
__device__ __forceinline__ int region_rows(int rg, int nb) { return 64; }
__device__ __forceinline__ int region_base(int rg) { return rg * 64 * KC; }

__device__ __forceinline__ int band_of(int region, int r, int rank, int B, int nb) {
  int b;
  if (region == 0) {
    b = rank * 64 + r;                                      // P : S_a rows of this SM
    return b < (B < 128 ? B : 128) ? b : -1;
  }
  if (r >= nb / 2) return -1;                               // QS padding rows
  b = 128 + rank * (nb / 2) + r;                            // QS: S_b rows of this SM
  return b < B ? b : -1;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    gram_tc_kernel(GramTc P) {
  pdl_wait();
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar_full[NI];
  __shared__ __align__(8) uint64_t bar_empty[NI];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float inv_s[2][64];
  __shared__ double s_of[2][64];

  const int rank = (int)tc::cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = P.B, nb = P.nb;
  const int nreg = B > 128 ? 2 : 1;
  const int slice_bytes = P.rows_tot * KC;
  const int stage_bytes = 2 * slice_bytes;
  const long long p_begin = (long long)pair * P.per_pair;
  const long long p_end = min(P.n, p_begin + P.per_pair);
  const int nst = p_end > p_begin ? (int)((p_end - p_begin + KC - 1) / KC) : 0;

  // per-band quantisation scales of the rows this SM handles
  for (int i = threadIdx.x; i < 2 * 64; i += NTHREADS) {
    const int rg = i / 64, r = i % 64;
    float is = 0.f;
    double sv = 0.0;
    if (rg < nreg && r < region_rows(rg, nb)) {
      const int b = band_of(rg, r, rank, B, nb);
      if (b >= 0) {
        const float m = __uint_as_float(P.amax_bits[b]);
        is = m > 0.f ? fminf((float)(16256.0 / (double)m), 1e30f) : 1.f;
        sv = 1.0 / (double)is;
      }
    }
    inv_s[rg][r] = is;
    s_of[rg][r] = sv;
  }
  // dead rows (QS padding, bands >= B) are never written: zero the ring once
  for (int i = threadIdx.x; i < NI * stage_bytes / 16; i += NTHREADS)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NI; ++i) {
      tc::mbar_init(&bar_full[i], 2);   // one forwarded arrival per CTA
      tc::mbar_init(&bar_empty[i], 1);
    }
    tc::mbar_init(&bar_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) {
    tc::tmem_alloc<2>(&tmem_base_sh, TMEM_COLS);
    tc::tmem_relinquish<2>();
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  // TMEM column map per product level: T_aa 64 cols, T_ab nb/2, T_bb nb/2
  const int CL = 64 + nb;
  const int off_ab = 64, off_bb = 64 + nb / 2;

  if (warp == 0) {
    // ================= forwarder: converters' stage s -> leader's bar_full ===
    for (int s = 0; s < nst; ++s) {
      const int is = s % NI;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + is), "r"((NCW + 1) * 32) : "memory");
      if (lane == 0) tc::mbar_arrive_cluster(&bar_full[is], 0);
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, one thread) =================
    if (rank == 0 && lane == 0 && nst > 0) {
      const uint32_t id_aa = tc::idesc_i8(128, 128);
      const uint32_t id_b = nb > 0 ? tc::idesc_i8(128, nb) : 0u;
      const uint32_t sbase = tc::smem_u32(smem);
      for (int s = 0; s < nst; ++s) {
        const int is = s % NI;
        tc::mbar_wait_cluster(&bar_full[is], (uint32_t)((s / NI) & 1));
        tc::tc_fence_after();
        const uint32_t st0 = sbase + is * stage_bytes;   // S0 slice
        const uint32_t st1 = st0 + slice_bytes;           // S1 slice
        for (int ks = 0; ks < KC / 32; ++ks) {
          auto dsc = [&](uint32_t slice, int rg, int row0) -> uint64_t {
            (void)row0;
            return tc::sdesc_kmajor_sw128(slice + region_base(rg) + ks * 32);
          };
          const uint32_t first = (s == 0 && ks == 0) ? 0u : 1u;
          // T_aa: A = P, B = P
          tc::mma_i8<2>(tmem + 0 * CL, dsc(st0, 0, 0), dsc(st0, 0, 0), id_aa, first);
          // diagonal tiles: only X = S0 S1^T (the cross term is X + X^T,
          // symmetrised in the reduction) -- one MMA of four saved
          tc::mma_i8<2>(tmem + 1 * CL, dsc(st0, 0, 0), dsc(st1, 0, 0), id_aa, first);
          tc::mma_i8<2>(tmem + 2 * CL, dsc(st1, 0, 0), dsc(st1, 0, 0), id_aa, first);
          if (nb > 0) {
            // T_ab: A = P, B = QB ; T_bb: A = QA, B = QB
            tc::mma_i8<2>(tmem + 0 * CL + off_ab, dsc(st0, 0, 0), dsc(st0, 1, 0), id_b, first);
            tc::mma_i8<2>(tmem + 1 * CL + off_ab, dsc(st0, 0, 0), dsc(st1, 1, 0), id_b, first);
            tc::mma_i8<2>(tmem + 1 * CL + off_ab, dsc(st1, 0, 0), dsc(st0, 1, 0), id_b, 1u);
            tc::mma_i8<2>(tmem + 2 * CL + off_ab, dsc(st1, 0, 0), dsc(st1, 1, 0), id_b, first);
            tc::mma_i8<2>(tmem + 0 * CL + off_bb, dsc(st0, 1, 0), dsc(st0, 1, 0), id_b, first);
            tc::mma_i8<2>(tmem + 1 * CL + off_bb, dsc(st0, 1, 0), dsc(st1, 1, 0), id_b, first);
            tc::mma_i8<2>(tmem + 2 * CL + off_bb, dsc(st1, 1, 0), dsc(st1, 1, 0), id_b, first);
          }
        }
        tc::mma_commit<2>(&bar_empty[is], 0x3);
      }
      tc::mma_commit<2>(&bar_done, 0x3);
    }
  } else if (warp >= 2) {
    // ================= converters: HBM fp32 -> int8 slices in smem ==========
    // (non-finite input is detected by the amax pre-pass)
    // One unit = one live band row of the stage: the warp's 32 lanes load its
    // 128 pixels as 32 contiguous 16-byte pieces (512 B per load instruction)
    // and write the 128 int8 bytes of each slice as one swizzled 128-B line
    // (conflict-free).  The per-unit offsets and scale are stage-invariant.
    const int cw = warp - 2;
    const int hb = nb / 2;
    const int nrow_p = max(0, min(64, (B < 128 ? B : 128) - rank * 64));
    const int nrow_q = nreg == 2 ? max(0, min(hb, B - 128 - rank * hb)) : 0;
    const int nunits = nrow_p + nrow_q;
    const bool vec_ok = (P.n % 4 == 0) && (((uintptr_t)P.Y & 15) == 0);
    long long src0[MAXU];
    int soff[MAXU];
    float isc[MAXU];
#pragma unroll
    for (int t = 0; t < MAXU; ++t) {
      const int u = cw + t * NCW;
      src0[t] = -1;
      soff[t] = 0;
      isc[t] = 0.f;
      if (u < nunits) {
        const int rg = u < nrow_p ? 0 : 1;
        const int r = rg ? u - nrow_p : u;
        const int b = rg ? 128 + rank * hb + r : rank * 64 + r;
        src0[t] = (long long)b * P.n + p_begin + 4 * lane;
        soff[t] = region_base(rg) + r * 128 + (((lane >> 2) ^ (r & 7)) << 4) + 4 * (lane & 3);
        isc[t] = inv_s[rg][r];
      }
    }
    const long long n_end = p_end - p_begin;   // pixels of this pair
    float4 va[MAXU], vb[MAXU];
    // issue every load of stage s for this warp (memory-level parallelism)
    auto load_stage = [&](int s, float4 (&v)[MAXU]) {
      const long long sh = (long long)s * KC;
      const bool full = vec_ok && sh + KC <= n_end;
#pragma unroll
      for (int t = 0; t < MAXU; ++t) {
        v[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src0[t] >= 0 && s < nst) {
          const float* src = P.Y + src0[t] + sh;
          if (full) {
            v[t] = __ldcs(reinterpret_cast<const float4*>(src));
          } else {
            const long long pix = sh + 4 * lane;   // pixel index within the pair
            v[t].x = pix < n_end ? src[0] : 0.f;
            v[t].y = pix + 1 < n_end ? src[1] : 0.f;
            v[t].z = pix + 2 < n_end ? src[2] : 0.f;
            v[t].w = pix + 3 < n_end ? src[3] : 0.f;
          }
        }
      }
    };
    // quantise the registers of stage s into its smem slot:
    // q = rint(y / s_b) via the 1.5*2^23 rounding constant (exact RN of the
    // product), t = q + 64, S0 = t >> 7 in [-127, 127], S1 = (t & 127) - 64
    // in [-64, 63]; four values packed per 32-bit word with byte permutes
    auto store_stage = [&](int s, const float4 (&v)[MAXU]) {
      const int is = s % NI;
      tc::mbar_wait(&bar_empty[is], (uint32_t)(((s / NI) & 1) ^ 1));   // local barrier (commit multicast)
      unsigned char* st0 = smem + is * stage_bytes;
      unsigned char* st1 = st0 + slice_bytes;
#pragma unroll
      for (int t = 0; t < MAXU; ++t) {
        if (cw + t * NCW >= nunits) break;
        const float x[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
        int h[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tq = __float_as_int(fmaf(x[j], isc[t], 12582912.0f)) - (0x4B400000 - 64);
          h[j] = tq >> 7;
          l[j] = (tq & 127) - 64;
        }
        const uint32_t w0 = __byte_perm(__byte_perm(h[0], h[1], 0x0040), __byte_perm(h[2], h[3], 0x0040), 0x5410);
        const uint32_t w1 = __byte_perm(__byte_perm(l[0], l[1], 0x0040), __byte_perm(l[2], l[3], 0x0040), 0x5410);
        *reinterpret_cast<uint32_t*>(st0 + soff[t]) = w0;
        *reinterpret_cast<uint32_t*>(st1 + soff[t]) = w1;
      }
      tc::fence_proxy_async_smem();
      // named barrier 1+slot: the forwarder warp (no loads in flight) makes the
      // single cluster-scope release-arrive for the whole CTA
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + is), "r"((NCW + 1) * 32) : "memory");
    };
    load_stage(0, va);
    for (int s = 0; s < nst; s += 2) {
      load_stage(s + 1, vb);          // next stage's loads fly while this one converts
      store_stage(s, va);
      if (s + 1 >= nst) break;
      load_stage(s + 2, va);
      store_stage(s + 1, vb);
    }

    // ================= epilogue: TMEM -> exact int64 -> fp64 partial ========
    if (cw < 4) {
      const int q4 = warp & 3;                    // TMEM lane quadrant of this warp
      const int L = q4 * 32 + lane;               // TMEM lane = this thread's row slot
      const int m = L & 63, half = L >> 6;
      long long* Pq = reinterpret_cast<long long*>(P.partial) + (long long)pair * B * B;
      if (nst > 0) {
        tc::mbar_wait_cluster(&bar_done, 0);
        tc::tc_fence_after();
      }
      const int ntile = nb > 0 ? 3 : 1;
      for (int t = 0; t < ntile; ++t) {
        const int Nt = t == 0 ? 128 : nb;
        const int coff = t == 0 ? 0 : (t == 1 ? off_ab : off_bb);
        // row band i and its scale; column bands j
        const int rg_i = t == 2 ? 1 : 0;
        const int bi = band_of(rg_i, m, rank, B, nb);
        for (int c0 = 0; c0 < Nt / 2; c0 += 16) {
          uint32_t a0[16], a1[16], a2[16];
          const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + coff + c0;
          if (nst > 0) {
            tc::tmem_ld16(ta + 0 * CL, a0);
            tc::tmem_ld16(ta + 1 * CL, a1);
            tc::tmem_ld16(ta + 2 * CL, a2);
            tc::tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) a0[j] = a1[j] = a2[j] = 0u;
          }
          if (bi < 0) continue;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int nn = c0 + j + (Nt / 2) * half;    // column within the tile
            const int bj = t == 0 ? (nn < (B < 128 ? B : 128) ? nn : -1) : (128 + nn < B ? 128 + nn : -1);
            if (bj < 0) continue;
            // T_ab holds S0 S1^T + S1 S0^T; the diagonal tiles hold X = S0 S1^T only:
            // 256 X here, (P + P^T) / 2 in the reduction gives 128 (X + X^T).
            // The partial is the EXACT integer (Q Q^T over this pair's pixels):
            // the reduction sums integers and scales once, so G does not depend
            // on how the pixels were split over pairs.
            const long long qq = 16384LL * (long long)(int)a0[j] + (t == 1 ? 128LL : 256LL) * (long long)(int)a1[j] +
                                 (long long)(int)a2[j];
            Pq[(long long)bi * B + bj] = qq;
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<2>(tmem, TMEM_COLS);
  }
}

__global__ void amax_kernel(const float* __restrict__ Y, long long n, unsigned* amax_bits, int* nonfinite) {
  pdl_wait();
  const int b = blockIdx.y;
  const float* row = Y + (long long)b * n;
  unsigned m = 0;
  bool bad = false;
  const bool vec = (n % 4 == 0) && (((uintptr_t)Y & 15) == 0);
  if (vec) {
    // eight independent 16-byte loads in flight per thread per step
    const long long n4 = n / 4;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n4; i += 8 * stride) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(row) + i + u * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        m = max(m, __float_as_uint(fabsf(v[u].x)));
        m = max(m, __float_as_uint(fabsf(v[u].y)));
        m = max(m, __float_as_uint(fabsf(v[u].z)));
        m = max(m, __float_as_uint(fabsf(v[u].w)));
      }
    }
    for (; i < n4; i += stride) {
      float4 v = __ldcs(reinterpret_cast<const float4*>(row) + i);
      m = max(m, __float_as_uint(fabsf(v.x)));
      m = max(m, __float_as_uint(fabsf(v.y)));
      m = max(m, __float_as_uint(fabsf(v.z)));
      m = max(m, __float_as_uint(fabsf(v.w)));
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
      m = max(m, __float_as_uint(fabsf(__ldcs(row + i))));
  }
  bad = m >= 0x7F800000u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&amax_bits[b], m);
  if (bad) atomicOr(nonfinite, 1);
}

}  // namespace

bool gram_tc_supported(int B) { return B >= 1 && B <= 224; }

// SM pairs for n pixels: min_px = 0 -> as many as the GPU has (at most 74,
// >= 512 pixels each: latency); min_px > 0 -> at least min_px pixels each
// (throughput mode of the batched lanes)
int gram_tc_npairs(long long n, int min_px) {
  long long np = min_px > 0 ? n / min_px : (n + 4LL * KC - 1) / (4LL * KC);
  if (np > 74) np = 74;
  if (np < 1) np = 1;
  long long per = (n + np - 1) / np;
  if (per > 100000) {
    np = (n + 99999) / 100000;
    per = (n + np - 1) / np;
  }
  per = (per + KC - 1) / KC * KC;
  np = (n + per - 1) / per;
  return (int)np;
}

// per-band max |y| bit patterns (the quantisation scales of K1) + non-finite flag
// zero the per-band max words (and the caller's RankState, when given) as a
// kernel, so the whole step stays a chain of dependent launches (no memset node)
__global__ void zero_kernel(unsigned* a, int na, int* st4) {
  pdl_wait();
  for (int i = threadIdx.x; i < na; i += blockDim.x) a[i] = 0u;
  if (st4 && threadIdx.x < (int)(sizeof(RankState) / sizeof(int))) st4[threadIdx.x] = 0;
}

cudaError_t launch_gram_amax(const float* Y, long long n, int B, unsigned* amax_bits, int* nonfinite, cudaStream_t st,
                             int* state4) {
  cudaError_t e = launch_pdl(zero_kernel, dim3(1), dim3(256), 0, st, amax_bits, B, state4);
  if (e != cudaSuccess) return e;
  long long per_block = 256LL * 4 * 8;
  unsigned gx = (unsigned)((n + per_block - 1) / per_block);
  if (gx > 16) gx = 16;   // 16 x B blocks: 64K-element band segments at B = 224, N = 2^20
  if (gx < 1) gx = 1;
  return launch_pdl(amax_kernel, dim3(gx, B), dim3(256), 0, st, Y, n, amax_bits, nonfinite);
}

// exact integer Gram of Y with the given per-band scales (amax_bits)
cudaError_t launch_gram_tc_scaled(const float* Y, long long n, int B, const unsigned* amax_bits, double* partial,
                                  int npairs, double* G, int* nonfinite, cudaStream_t st) {
  cudaError_t e;
  GramTc P;
  P.Y = Y;
  P.n = n;
  P.B = B;
  P.nb = B > 128 ? ((B - 128 + 31) / 32) * 32 : 0;
  P.rows_tot = B > 128 ? 128 : 64;
  long long per = (n + npairs - 1) / npairs;
  per = (per + KC - 1) / KC * KC;
  P.per_pair = per;
  P.amax_bits = amax_bits;
  P.partial = partial;
  P.nonfinite = nonfinite;
  const size_t smem = (size_t)NI * 2 * P.rows_tot * KC;
  e = cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(gram_tc_kernel, dim3(2 * npairs), dim3(NTHREADS), smem, st, P);   // __cluster_dims__(2)
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_gram_reduce_i64(reinterpret_cast<const long long*>(partial), npairs, B, amax_bits, G, st);
}

cudaError_t launch_gram_tc(const float* Y, long long n, int B, unsigned* amax_bits, double* partial, int npairs,
                           double* G, int* nonfinite, cudaStream_t st, int* state4) {
  cudaError_t e = launch_gram_amax(Y, n, B, amax_bits, nonfinite, st, state4);
  if (e != cudaSuccess) return e;
  return launch_gram_tc_scaled(Y, n, B, amax_bits, partial, npairs, G, nonfinite, st);
}
