// K1 (north_star stage (1)) on the 5th-generation tensor
// cores: an EXACT integer Gram of a quantised cube, with every pixel the
// quantisation cannot represent added exactly in fp64.
//
// Why integers (DESIGN.md §4 K1): sigma_b^2 = 1/(N [(G+dI)^-1]_bb) amplifies
// the Gram's error by ~the band SNR, so G must be good to ~1e-8 relative;
// fp32 (or TF32/BF16-split) accumulation over 10^6 pixels is not, and any
// non-PSD rounding breaks noiseless cubes.
//
// Quantisation (robust to hot / dead / saturated pixels):
//   * gram_qscale_kernel reads a fixed sample of every band (64 blocks of the
//     pixel axis, <= 256 pixels each) and takes a centre m_b = median of the
//     block means and a range R_b = 2 x the 8th-largest block max |y - m_b|,
//     so a few outliers cannot widen the step (one CTA per band,
//     1.6 % of the cube read at `large`; the old full max pre-pass read all);
//   * inv_s = fp32(32767 / R_b), c_b = rint(m_b inv_s) (an integer centre),
//     q = rint(y inv_s - c_b) in [-32768, 32767] (16 bits), y ~ s (q + c);
//   * a value outside that range (outlier, NaN, Inf) sets its PIXEL's bit in a
//     clip bitmap (its bytes still go through the MMAs; the fix replaces them).
// Split q = 256 S0 + S1 (S0 in [-128, 127] signed, S1 in [0, 255] unsigned int8,
// read straight off the bits of one fma -- see `convert`):
//   Q Q^T = 65536 S0 S0^T + 256 (S0 S1^T + S1 S0^T) + S1 S1^T
// int8 x int8 -> int32 GEMMs (tcgen05.mma kind::i8), accumulated EXACTLY in
// TMEM; the per-pair partials (and sum_p q_p per band) are exact int64.
// gram_fix_kernel then walks the bitmap and, for the flagged pixels P only,
// forms F = sum_P y y^T in fp64 and D = sum_P q q^T, sum_P q in int64, and
// the finalize kernel assembles, with N' = N - |P| and Q1' = sum_{p not in P} q,
//   G = diag(s) [ (QQ^T - D) + c Q1'^T + Q1' c^T + N' c c^T ] diag(s) + F
// (the bracket exact in 128-bit integers).  So G is the exact Gram of the
// cube with the unflagged values rounded to the 16-bit grid s (q + c) and the
// flagged pixels exact: symmetric PSD, deterministic, any dynamic range.
//
// Structure: clusters of 2 CTAs (one SM pair) per pixel range, cta_group::2
// MMAs with M = 128 (64 rows per SM, TMEM "2x2" layout).  Bands are split
// S_a = [0,128), S_b = [128,B), Nb = B-128 rounded up to 32; two tiles:
// T_a* = [T_aa | T_ab] (128 x (128 + Nb): A = S_a, B = S_a then S_b in ONE
// MMA per product) and T_bb (128 x Nb); x 3 products = 480 of 512 TMEM
// columns for B <= 224.  A TMA producer streams fp32 tiles into a 2-stage
// ring; 13 converter warps per CTA quantise them and write the int8 slices
// into shared memory in the UMMA canonical K-major layout; one thread of the
// leader CTA
// issues the MMAs; the stage ring is released by tcgen05.commit multicast to
// both CTAs.  Each CTA finally reads its TMEM, combines the three products in
// int64 and writes its exact integer partial.
#include "common.cuh"
#include "tc_util.cuh"

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <type_traits>

namespace {

constexpr int KC = 128;        // pixels (bytes per int8 row) per stage
constexpr int NTHREADS = 16 * 32;
// Two feeds of the converters: registers (each converter warp loads its band
// rows from HBM, one stage in flight: the fallback for unaligned pixel counts)
// or TMA (one producer thread streams fp32 tiles of the stage -- two 2-D boxes,
// the P and QS band ranges -- into a 2-stage smem ring, ~115 KB in flight per
// SM, and the converters read shared memory).
template <bool TMA> struct Feed;
template <> struct Feed<false> { static constexpr int NI = 4, NCW = 14, MAXU = 8, W0 = 2; };
template <> struct Feed<true>  { static constexpr int NI = 3, NCW = 13, MAXU = 9, W0 = 3; };
constexpr int NF = 2;                   // fp32 stages (TMA feed)
constexpr int FROWS = 64 + 48;          // fp32 rows per stage: P (64) + QS (<= 48)
constexpr int FSTAGE = FROWS * KC * 4;  // 57344 B
constexpr int TMEM_COLS = 512;

constexpr int GQ_MAX = 32767;  // v in [-32768, 32767]: the range maps to R = 32767 steps
constexpr int QS_NBLK = 64;    // sample blocks per band (qscale)
constexpr int FIX_SPLITS = 64; // pixel splits (CTAs) of the clipped-pixel correction
constexpr int FIX_TB = 64;     // correction output block edge
constexpr int FIX_TP = 32;     // correction pixels per stage
constexpr int FIX_CAP = 2048;  // flagged-pixel list entries per pass

struct FixOut {
  double* F;        // [FIX_SPLITS][B*B]
  long long* D;     // [FIX_SPLITS][B*B]
  long long* Q1;    // [FIX_SPLITS][B]
  int* cnt;         // [FIX_SPLITS]
};

// One cube of a batched Gram (hyde_hyres_batched's phased mode): the kernels
// take jobs[blockIdx.y] instead of their pointer arguments (same n and B).
struct GramJob {
  const float* Y;
  GramQScale* qs;
  unsigned* bitmap;
  long long* partial;
  FixOut fix;
  double* G;
  int* nonfinite;
  int* state4;     // rank-state words to zero (or NULL)
  double* zero8;   // 8 more words to zero (the eigensolver's flags), or NULL
};

struct GramTc {
  const float* Y;
  long long n;
  int B;
  int nb;           // Nb (0 when B <= 128)
  int rows_tot;     // 64 + 64 + nb/2 (or 64)
  long long per_pair;
  const GramQScale* qs;
  long long* partial;  // [pair][B*B + B]: Q Q^T over the pair's pixels, then sum q per band
  unsigned* bitmap;    // clipped-pixel bits
  int atomic_sum;      // 1: pairs add their exact partials into partial[0] (zeroed by qscale) -- no reduce kernel
  int exp;             // experiments only (HYDE_GRAM_EXP; wrong results, timing): 1 no MMAs, 2 no T_bb MMAs, 4 no conversion
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

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(tc::smem_u32(bar))
      : "memory");
}

template <bool TMA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    gram_tc_kernel(GramTc P, const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                   const GramJob* __restrict__ jobs) {
  enum : int { NI = Feed<TMA>::NI, NCW = Feed<TMA>::NCW, MAXU = Feed<TMA>::MAXU, W0 = Feed<TMA>::W0 };
  pdl_wait();
  if (!TMA && jobs) {
    const GramJob& j = jobs[blockIdx.y];
    P.Y = j.Y;
    P.qs = j.qs;
    P.partial = j.partial;
    P.bitmap = j.bitmap;
  }
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar_full[NI];
  __shared__ __align__(8) uint64_t bar_empty[NI];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ __align__(8) uint64_t f_full[NF];
  __shared__ __align__(8) uint64_t f_empty[NF];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float inv_s[2][64];
  __shared__ float kf_of[2][64];

  const int rank = (int)tc::cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = P.B, nb = P.nb;
  const int nreg = B > 128 ? 2 : 1;
  const int slice_bytes = P.rows_tot * KC;
  const int stage_bytes = 2 * slice_bytes;
  // Pixel tiles of KC.  TMA feed: tiles are dealt to the pairs cyclically
  // (tile s * npairs + pair), so the pass ends on the LAST pixels of the cube
  // -- a contiguous ~L2-sized tail that K3 (which walks the cube backwards)
  // then reads from L2.  Register feed: one contiguous range per pair.  (The
  // per-pair partials are exact integers: G does not depend on the split.)
  const long long p_begin = (long long)pair * P.per_pair;
  const long long p_end = min(P.n, p_begin + P.per_pair);
  const int npairs = (int)(gridDim.x >> 1);
  const long long ntiles = (P.n + KC - 1) / KC;
  const int nst = TMA ? (pair < ntiles ? (int)((ntiles - 1 - pair) / npairs + 1) : 0)
                      : (p_end > p_begin ? (int)((p_end - p_begin + KC - 1) / KC) : 0);
  // absolute first pixel of stage s and the pixel limit of this pair
  auto tile_px = [&](int s) -> long long {
    return TMA ? ((long long)s * npairs + pair) * KC : p_begin + (long long)s * KC;
  };
  const long long px_lim = TMA ? P.n : p_end;

  // per-band quantisation scales of the rows this SM handles
  for (int i = threadIdx.x; i < 2 * 64; i += NTHREADS) {
    const int rg = i / 64, r = i % 64;
    float is = 0.f, kf = 8421376.0f;
    if (rg < nreg && r < region_rows(rg, nb)) {
      const int b = band_of(rg, r, rank, B, nb);
      if (b >= 0) {
        is = P.qs[b].inv_s;
        kf = P.qs[b].kf;
      }
    }
    inv_s[rg][r] = is;
    kf_of[rg][r] = kf;
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
    for (int i = 0; i < NF; ++i) {
      tc::mbar_init(&f_full[i], 1);       // the producer's expect_tx arrival
      tc::mbar_init(&f_empty[i], NCW);    // one arrival per converter warp
    }
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
  const int off_bb = 64 + nb / 2;

  if (warp == 0) {
    // ================= forwarder: converters' stage s -> leader's bar_full ===
    for (int s = 0; s < nst; ++s) {
      const int is = s % NI;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + is), "r"((NCW + 1) * 32) : "memory");
      if (lane == 0) {
        // CTA-scope release (the converters' writes were fenced to the async
        // proxy and joined by the named barrier; a cluster-scope release
        // compiles to MEMBAR.ALL.GPU on this thread: 3-4 us per gram call)
        tc::mbar_arrive_cluster_cta(&bar_full[is], 0);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, one thread) =================
    if (rank == 0 && lane == 0 && nst > 0) {
      // S0 (high bytes) signed, S1 (low bytes) unsigned.  B <= 128: T_aa
      // (N = 128).  B > 128: T_a* = [T_aa | T_ab] with A = P and B = [P ; QS]
      // -- this CTA's 64 P rows then its nb/2 QS rows, contiguous in the slice
      // -- in ONE MMA per product (N = 128 + nb), plus T_bb (A = QS, B = the
      // live QS rows, N = nb): 7 MMAs per k-slice instead of 10 with a
      // separate T_ab (large: gram stage 254 -> 227 us on the same box).
      const int Na = 128 + nb;
      const uint32_t id_a00 = tc::idesc_i8(128, Na, true, true);
      const uint32_t id_a01 = tc::idesc_i8(128, Na, true, false);
      const uint32_t id_a10 = nb > 0 ? tc::idesc_i8(128, Na, false, true) : 0u;
      const uint32_t id_a11 = tc::idesc_i8(128, Na, false, false);
      const uint32_t id_b = nb > 0 ? tc::idesc_i8(128, nb, true, true) : 0u;
      const uint32_t id_b01 = nb > 0 ? tc::idesc_i8(128, nb, true, false) : 0u;
      const uint32_t id_b11 = nb > 0 ? tc::idesc_i8(128, nb, false, false) : 0u;
      const uint32_t sbase = tc::smem_u32(smem);
      for (int s = 0; s < nst; ++s) {
        const int is = s % NI;
        tc::mbar_wait_cluster(&bar_full[is], (uint32_t)((s / NI) & 1));
        tc::tc_fence_after();
        const uint32_t st0 = sbase + is * stage_bytes;   // S0 slice
        const uint32_t st1 = st0 + slice_bytes;           // S1 slice
        if (P.exp & 1) {   // experiment: no MMAs
          tc::mma_commit<2>(&bar_empty[is], 0x3);
          continue;
        }
        for (int ks = 0; ks < KC / 32; ++ks) {
          auto dsc = [&](uint32_t slice, int rg) -> uint64_t {
            return tc::sdesc_kmajor_sw128(slice + region_base(rg) + ks * 32);
          };
          const uint32_t first = (s == 0 && ks == 0) ? 0u : 1u;
          tc::mma_i8<2>(tmem + 0 * CL, dsc(st0, 0), dsc(st0, 0), id_a00, first);
          tc::mma_i8<2>(tmem + 1 * CL, dsc(st0, 0), dsc(st1, 0), id_a01, first);
          if (nb > 0) {
            // the cross accumulator of T_a* holds S0 S1^T + S1 S0^T (the T_ab
            // block needs both; on the diagonal block it is the symmetric sum)
            tc::mma_i8<2>(tmem + 1 * CL, dsc(st1, 0), dsc(st0, 0), id_a10, 1u);
          }
          // (B <= 128: the diagonal tile holds X = S0 S1^T only; the cross
          // term X + X^T is symmetrised in the reduction -- one MMA saved)
          tc::mma_i8<2>(tmem + 2 * CL, dsc(st1, 0), dsc(st1, 0), id_a11, first);
          if (nb > 0 && !(P.exp & 2)) {
            // T_bb: A = QS, B = the live QS rows; cross term X = S0 S1^T only
            tc::mma_i8<2>(tmem + 0 * CL + off_bb, dsc(st0, 1), dsc(st0, 1), id_b, first);
            tc::mma_i8<2>(tmem + 1 * CL + off_bb, dsc(st0, 1), dsc(st1, 1), id_b01, first);
            tc::mma_i8<2>(tmem + 2 * CL + off_bb, dsc(st1, 1), dsc(st1, 1), id_b11, first);
          }
        }
        tc::mma_commit<2>(&bar_empty[is], 0x3);
      }
      tc::mma_commit<2>(&bar_done, 0x3);
    }
  } else if (TMA && warp == 2) {
    // ================= TMA producer: fp32 stage tiles -> smem ring ==========
    if (lane == 0) {
      unsigned char* fring = smem + NI * stage_bytes;
      const int hb = nb / 2;
      const uint32_t bytes = (uint32_t)(64 + (nreg == 2 ? hb : 0)) * KC * 4;
      for (int s = 0; s < nst; ++s) {
        const int fs = s % NF;
        if (s >= NF) tc::mbar_wait(&f_empty[fs], (uint32_t)(((s / NF) - 1) & 1));
        tc::mbar_expect_tx(&f_full[fs], bytes);
        unsigned char* dst = fring + fs * FSTAGE;
        const int x = (int)tile_px(s);
        tma_load_2d(dst, &tmP, x, rank * 64, &f_full[fs]);
        if (nreg == 2) tma_load_2d(dst + 64 * KC * 4, &tmQ, x, 128 + rank * hb, &f_full[fs]);
      }
    }
  } else if (warp >= W0) {
    // ================= converters: HBM fp32 -> int8 slices in smem ==========
    // (non-finite input fails the range test and is flagged like an outlier;
    // gram_fix_kernel raises the non-finite flag when it reads the pixel)
    // One unit = one live band row of the stage: the warp's 32 lanes load its
    // 128 pixels as 32 contiguous 16-byte pieces (512 B per load instruction)
    // and write the 128 int8 bytes of each slice as one swizzled 128-B line
    // (conflict-free).  The per-unit offsets and scale are stage-invariant.
    const int cw = warp - W0;
    const int hb = nb / 2;
    const int nrow_p = max(0, min(64, (B < 128 ? B : 128) - rank * 64));
    const int nrow_q = nreg == 2 ? max(0, min(hb, B - 128 - rank * hb)) : 0;
    const int nunits = nrow_p + nrow_q;
    const bool vec_ok = (P.n % 4 == 0) && (((uintptr_t)P.Y & 15) == 0);
    int brow[MAXU];   // band of each unit (-1: none); TMA feed: its row in the fp32 stage
    const float* ybase = P.Y + p_begin + 4 * lane;
    int soff[MAXU];
    float isc[MAXU];
    const float* kfu = &kf_of[0][0];   // per-unit fma addend kf_of[rg][r], index soff >> 7 (register budget)
    int sq[MAXU];   // this lane's sum of q per unit (band): |.| <= 4 * 32768 * 256 stages
#pragma unroll
    for (int t = 0; t < MAXU; ++t) {
      const int u = cw + t * NCW;
      brow[t] = -1;
      soff[t] = 0;
      isc[t] = 0.f;
      sq[t] = 0;
      if (u < nunits) {
        const int rg = u < nrow_p ? 0 : 1;
        const int r = rg ? u - nrow_p : u;
        const int b = rg ? 128 + rank * hb + r : rank * 64 + r;
        brow[t] = TMA ? (rg ? 64 + r : r) : b;
        soff[t] = region_base(rg) + r * 128 + (((lane >> 2) ^ (r & 7)) << 4) + 4 * (lane & 3);
        isc[t] = inv_s[rg][r];
      }
    }
    const long long n_end = p_end - p_begin;   // pixels of this pair
    float4 va[MAXU], vb[MAXU];
    // issue every load of stage s for this warp (memory-level parallelism)
    auto load_stage = [&](int s, float4 (&v)[MAXU]) {
      if (TMA) {   // from the fp32 ring; the slot is released as soon as it is read
        if (s >= nst) return;
        const int fs = s % NF;
        tc::mbar_wait(&f_full[fs], (uint32_t)((s / NF) & 1));
        const float* fr = reinterpret_cast<const float*>(smem + NI * stage_bytes + fs * FSTAGE) + 4 * lane;
#pragma unroll
        for (int t = 0; t < MAXU; ++t)
          v[t] = brow[t] >= 0 ? *reinterpret_cast<const float4*>(fr + brow[t] * KC) : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&f_empty[fs]);
        return;
      }
      const long long sh = (long long)s * KC;
      const bool full = vec_ok && sh + KC <= n_end;
#pragma unroll
      for (int t = 0; t < MAXU; ++t) {
        v[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (brow[t] >= 0 && s < nst) {
          const float* src = ybase + (long long)brow[t] * P.n + sh;
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
    // quantise the registers of stage s into its smem slot.
    // Per value: r = fma(y, inv_s, 2^23 + 32768 - c) is the exact RN of
    // y inv_s - c + 32768 + 2^23, so for an in-range value bits(r) =
    // 0x4B000000 + u, u = v + 32768 in [0, 65535], v = rint(y inv_s - c).  The
    // int8 slices are read straight off those bits: S0 = byte1 ^ 0x80 (signed,
    // = floor(v / 256)), S1 = byte0 (unsigned), v = 256 S0 + S1.  For ANY bits
    // the MMAs consume v_used = (bits & 0xFFFF) - 32768; a value whose bits
    // leave [0x4B000000, 0x4B00FFFF] (out of range, NaN, Inf) flags its pixel
    // and gram_fix_kernel replaces the pixel's v_used terms by the exact ones.
    // Per 4 values: 4 FFMA, 4 LOP3 (range OR), 6 PRMT, 1 LOP3 (sign flip),
    // 2 IDP4A + IMAD (sum of v); the clip atomics run once per stage, rarely.
    auto convert = [&](auto full_tag, int s, const float4 (&v)[MAXU], unsigned char* st0, unsigned char* st1) {
      constexpr bool FULL = decltype(full_tag)::value;
      const long long sh = tile_px(s) + 4 * lane;   // absolute first pixel of this lane
      unsigned acc0 = 0u, acc1 = 0u, acc2 = 0u, acc3 = 0u;   // OR of (bits ^ 0x4B000000) per pixel
#pragma unroll
      for (int t = 0; t < MAXU; ++t) {
        if (cw + t * NCW >= nunits) break;
        const float kf = kfu[soff[t] >> 7];
        unsigned r0 = __float_as_uint(fmaf(v[t].x, isc[t], kf));
        unsigned r1 = __float_as_uint(fmaf(v[t].y, isc[t], kf));
        unsigned r2 = __float_as_uint(fmaf(v[t].z, isc[t], kf));
        unsigned r3 = __float_as_uint(fmaf(v[t].w, isc[t], kf));
        if (!FULL) {   // ragged tail: pixels past the pair's end are v = 0 (u = 32768)
          r0 = sh + 0 < px_lim ? r0 : 0x4B008000u;
          r1 = sh + 1 < px_lim ? r1 : 0x4B008000u;
          r2 = sh + 2 < px_lim ? r2 : 0x4B008000u;
          r3 = sh + 3 < px_lim ? r3 : 0x4B008000u;
        }
        acc0 |= r0 ^ 0x4B000000u;
        acc1 |= r1 ^ 0x4B000000u;
        acc2 |= r2 ^ 0x4B000000u;
        acc3 |= r3 ^ 0x4B000000u;
        const uint32_t w0 = __byte_perm(__byte_perm(r0, r1, 0x0051), __byte_perm(r2, r3, 0x0051), 0x5410) ^ 0x80808080u;
        const uint32_t w1 = __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
        sq[t] += 256 * __dp4a((int)w0, 0x01010101, 0) + (int)__dp4a(w1, 0x01010101u, 0u);
        *reinterpret_cast<uint32_t*>(st0 + soff[t]) = w0;
        *reinterpret_cast<uint32_t*>(st1 + soff[t]) = w1;
      }
      const unsigned pm = ((acc0 >> 16) ? 1u : 0u) | ((acc1 >> 16) ? 2u : 0u) | ((acc2 >> 16) ? 4u : 0u) |
                          ((acc3 >> 16) ? 8u : 0u);
      if (pm) {
#pragma unroll 1
        for (int j = 0; j < 4; ++j)
          if ((pm >> j) & 1u) {
            const long long px = sh + j;
            atomicOr(P.bitmap + (px >> 5), 1u << (px & 31));
          }
      }
    };
    auto store_stage = [&](int s, const float4 (&v)[MAXU]) {
      const int is = s % NI;
      tc::mbar_wait(&bar_empty[is], (uint32_t)(((s / NI) & 1) ^ 1));   // local barrier (commit multicast)
      unsigned char* st0 = smem + is * stage_bytes;
      unsigned char* st1 = st0 + slice_bytes;
      if (P.exp & 4) {
      } else if (tile_px(s) + KC <= px_lim)
        convert(std::true_type{}, s, v, st0, st1);
      else
        convert(std::false_type{}, s, v, st0, st1);
      tc::fence_proxy_async_smem();
      // named barrier 1+slot: the forwarder warp (no loads in flight) makes the
      // single cluster-scope release-arrive for the whole CTA
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + is), "r"((NCW + 1) * 32) : "memory");
    };
    if (TMA) {
      // smem-fed: read a stage, release its fp32 slot, convert
      for (int s = 0; s < nst; ++s) {
        load_stage(s, va);
        store_stage(s, va);
      }
    } else {
      load_stage(0, va);
      for (int s = 0; s < nst; s += 2) {
        load_stage(s + 1, vb);          // next stage's loads fly while this one converts
        store_stage(s, va);
        if (s + 1 >= nst) break;
        load_stage(s + 2, va);
        store_stage(s + 1, vb);
      }
    }
    // sum_p q of every unit's band over this pair's pixels (exact int64)
    {
      long long* Q1 = P.partial + (P.atomic_sum ? 0LL : (long long)pair * ((long long)B * B + B)) + (long long)B * B;
#pragma unroll
      for (int t = 0; t < MAXU; ++t) {
        const int u = cw + t * NCW;
        if (u >= nunits) break;
        long long v = sq[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          const int b = u < nrow_p ? rank * 64 + u : 128 + rank * hb + (u - nrow_p);
          if (!P.atomic_sum) Q1[b] = v;
          else if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(Q1 + b), (unsigned long long)v);
        }
      }
    }

    // ================= epilogue: TMEM -> exact int64 -> fp64 partial ========
    if (cw < 4) {
      const int q4 = warp & 3;                    // TMEM lane quadrant of this warp
      const int L = q4 * 32 + lane;               // TMEM lane = this thread's row slot
      const int m = L & 63, half = L >> 6;
      // atomic_sum: every pair adds its exact integer partial into partial[0]
      // (integer adds: the sum does not depend on their order)
      long long* Pq = P.partial + (P.atomic_sum ? 0LL : (long long)pair * ((long long)B * B + B));
      if (nst > 0) {
        tc::mbar_wait_cluster(&bar_done, 0);
        tc::tc_fence_after();
      }
      const int ntile = nb > 0 ? 3 : 1;
      const bool merged = nb > 0;   // tile 0 is T_a* = [T_aa | T_ab]
      const int hb = nb / 2;
      for (int t = 0; t < ntile; ++t) {
        if (t == 1) continue;          // (T_ab is part of tile 0)
        const int Nt = t == 0 ? 128 + nb : nb;
        const int coff = t == 0 ? 0 : off_bb;
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
            int bj;
            if (merged && t == 0) {   // column half h = CTA h's B rows: its 64 P bands, then its hb QS bands
              const int rho = c0 + j;
              bj = rho < 64 ? 64 * half + rho : 128 + hb * half + (rho - 64);
              bj = bj < B ? bj : -1;
            } else {
              bj = t == 0 ? (nn < (B < 128 ? B : 128) ? nn : -1) : (128 + nn < B ? 128 + nn : -1);
            }
            if (bj < 0) continue;
            // T_a* (B > 128) holds S0 S1^T + S1 S0^T: weight 256; T_bb and the
            // B <= 128 T_aa hold X = S0 S1^T only: 512 X here, (P + P^T) / 2 in
            // the reduction gives 256 (X + X^T).
            // The partial is the EXACT integer (Q Q^T over this pair's pixels):
            // the reduction sums integers and scales once, so G does not depend
            // on how the pixels were split over pairs.
            const long long qq = 65536LL * (long long)(int)a0[j] + (merged && t == 0 ? 256LL : 512LL) * (long long)(int)a1[j] +
                                 (long long)(int)a2[j];
            if (!P.atomic_sum) Pq[(long long)bi * B + bj] = qq;
            else if (qq != 0) atomicAdd(reinterpret_cast<unsigned long long*>(Pq + (long long)bi * B + bj), (unsigned long long)qq);
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


// ------------------------------------------------------------------ qscale
// One CTA per band; warp w samples blocks w, w + 8, ... (all eight of its
// blocks' loads in flight before the reductions).  Block k of the pixel
// axis ([kN/64, (k+1)N/64)) is sampled at <= 256 pixels (all of them, or two
// runs at the starts of its halves: 128 pixels each -- 1.6 % of the cube at
// `large` -- 64 or 32 for blocks under 8192 / 4096 pixels);
// per block: mean, min, max of the finite samples.  (An 8-CTA cluster per
// band with one block per warp cost 450 us for the 64 x 191 bands of the
// batched mode -- 98k CTAs of latency -- against 16 us for one cube.)  Then:
// m = lower median of the block
// means; dev_k = max(max_k - m, m - min_k); R = 2 x the 8th largest dev_k
// (rank min(7, nblk/8): the largest
// for fewer than 16 blocks; the largest when that is 0; |m|, else 1e-30, when
// all are 0: every nonzero value is then flagged and exact); widened so
// |c| <= 2^21 (the fma addend must stay in [2^23, 2^24)).
// Also zeroes a slice of the clip bitmap and, on CTA 0, the caller's
// rank-state words -- the first kernel of the step.
// UU = 32-pixel loads per half-block run (qscale_uu(n)): a template so the
// sample registers are sized to the run (107 registers for UU = 4 held the
// batched mode's UU = 1 launch of 12k CTAs to 2 CTAs per SM).
template <int UU>
__global__ void __launch_bounds__(256)
    gram_qscale_kernel(const float* __restrict__ Y, long long n, GramQScale* qs, unsigned* bitmap, long long nwords,
                       int* st4, int nst4, const GramJob* __restrict__ jobs, long long* zs = nullptr,
                       long long nzs = 0) {
  pdl_wait();
  if (jobs) {
    const GramJob& j = jobs[blockIdx.y];
    Y = j.Y;
    qs = j.qs;
    bitmap = j.bitmap;
    st4 = j.state4;
    if (j.zero8 && blockIdx.x == 0 && threadIdx.x < 8) j.zero8[threadIdx.x] = 0.0;
    if (nzs > 0) zs = j.partial;   // the cube's atomic-sum accumulator
  }
  const int b = blockIdx.x;
  {
    const long long w0 = nwords * blockIdx.x / gridDim.x, w1 = nwords * (blockIdx.x + 1) / gridDim.x;
    for (long long w = w0 + threadIdx.x; w < w1; w += blockDim.x) bitmap[w] = 0u;
    if (st4 && blockIdx.x == 0 && (int)threadIdx.x < nst4) st4[threadIdx.x] = 0;
    if (zs) {   // the atomic Gram sum's accumulator
      const long long z0 = nzs * blockIdx.x / gridDim.x, z1 = nzs * (blockIdx.x + 1) / gridDim.x;
      for (long long z = z0 + threadIdx.x; z < z1; z += blockDim.x) zs[z] = 0;
    }
  }
  __shared__ double bmean[QS_NBLK];
  __shared__ float bmin[QS_NBLK], bmax[QS_NBLK], bdev[QS_NBLK];
  __shared__ float m_sh;
  const int nblk = n < QS_NBLK ? (int)n : QS_NBLK;
  const float* row = Y + (long long)b * n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KPW = QS_NBLK / 8;   // blocks per warp
  // block k starts at n k / nblk: a shift for nblk = 64 (a 64-bit division is a
  // ~100-instruction routine; three per block made this kernel 0.42 ms for the
  // 64 x 191 bands of the batched mode)
  static_assert(QS_NBLK == 64, "blk_lo shifts by log2(QS_NBLK)");
  auto blk_lo = [&](int k) -> long long { return nblk == QS_NBLK ? (n * k) >> 6 : (long long)k; };
  // samples per half-block run: 128 (blocks of >= 8192 pixels: 1.6 % of the
  // cube at `large`), 64 / 32 for shorter blocks (the batched mode's
  // 1024-pixel blocks: 6 % of the band instead of 25 %, which made this
  // kernel 0.42 ms for 64 cubes)
  float v[KPW][2 * UU];
  bool full[KPW];
#pragma unroll
  for (int q = 0; q < KPW; ++q) {
    const int k = warp + 8 * q;
    const long long p0 = blk_lo(k), p1 = blk_lo(k + 1), len = p1 - p0;
    full[q] = k < nblk && len > 256;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float* src = row + p0 + ((len * j) >> 1);
#pragma unroll
      for (int u = 0; u < UU; ++u) v[q][UU * j + u] = full[q] ? __ldg(src + lane + 32 * u) : 0.f;
    }
  }
#pragma unroll
  for (int q = 0; q < KPW; ++q) {
    const int k = warp + 8 * q;
    if (k >= nblk) continue;
    const long long p0 = blk_lo(k), p1 = blk_lo(k + 1), len = p1 - p0;
    double sum = 0.0;
    int cnt = 0;
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    auto take = [&](float x) {
      const bool ok = isfinite(x);
      sum += ok ? (double)x : 0.0;
      cnt += ok;
      mn = ok ? fminf(mn, x) : mn;
      mx = ok ? fmaxf(mx, x) : mx;
    };
    if (!full[q]) {
      for (long long i = lane; i < len; i += 32) take(__ldg(row + p0 + i));
    } else {
#pragma unroll
      for (int u = 0; u < 2 * UU; ++u) take(v[q][u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      bmean[k] = cnt > 0 ? sum / cnt : 0.0;
      bmin[k] = cnt > 0 ? mn : 0.f;
      bmax[k] = cnt > 0 ? mx : 0.f;
    }
  }
  __syncthreads();

  // order statistics by rank counting (ties broken by block index)
  if ((int)threadIdx.x < nblk) {
    const int kk = threadIdx.x;
    int r = 0;
    for (int j = 0; j < nblk; ++j) r += (bmean[j] < bmean[kk]) || (bmean[j] == bmean[kk] && j < kk);
    if (r == (nblk - 1) / 2) m_sh = (float)bmean[kk];
  }
  __syncthreads();
  const float m = m_sh;
  if ((int)threadIdx.x < nblk) {
    const int kk = threadIdx.x;
    bdev[kk] = fminf(fmaxf(bmax[kk] - m, m - bmin[kk]), 3e38f);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // rank min(7, nblk/8) and rank 0 (largest) of bdev, descending
    const int want = (nblk >> 3) < 7 ? (nblk >> 3) : 7;
    float r7 = 0.f, r0 = 0.f;
    for (int kk = lane; kk < nblk; kk += 32) {
      int r = 0;
      for (int j = 0; j < nblk; ++j) r += (bdev[j] > bdev[kk]) || (bdev[j] == bdev[kk] && j < kk);
      if (r == want) r7 = bdev[kk];
      if (r == 0) r0 = bdev[kk];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r7 = fmaxf(r7, __shfl_xor_sync(0xffffffffu, r7, o));
      r0 = fmaxf(r0, __shfl_xor_sync(0xffffffffu, r0, o));
    }
    if (lane == 0) {
      double R = 2.0 * (double)r7;
      if (!(R > 0.0)) R = 2.0 * (double)r0;
      if (!(R > 0.0)) R = fabs((double)m);
      if (!(R > 0.0)) R = 1e-30;
      const double cmax = 2097152.0;   // 2^21
      if (fabs((double)m) * GQ_MAX / R > cmax) R = fabs((double)m) * GQ_MAX / cmax;
      if (R > 3e38) R = 3e38;
      const float is = (float)((double)GQ_MAX / R);
      double cd = rint((double)m * (double)is);
      cd = fmin(fmax(cd, -cmax), cmax);
      GramQScale o;
      o.inv_s = is;
      o.c = (int)cd;
      o.kf = (float)(8421376.0 - cd);   // 2^23 + 32768 - c, an exact integer in [2^22, 2^24)
      o.pad = 0;
      o.s = 1.0 / (double)is;
      qs[b] = o;
    }
  }
}

// ------------------------------------------------------------------ reduce
// Stage 1: S[e] = sum over pairs of P[k][e] for every element a pair writes
// (B x B without the block rows >= 128 / columns < 128, then the B sums of q),
// coalesced; 8 warps split k, fixed order.  S overwrites P[0] (each element is
// read and written by its own thread only).
__global__ void __launch_bounds__(256) gram_reduce_i64_kernel(long long* __restrict__ partial, int np, int B,
                                                              const GramJob* __restrict__ jobs) {
  pdl_wait();
  if (jobs) partial = jobs[blockIdx.y].partial;
  __shared__ long long part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long bb = (long long)B * B, tot = bb + B;
  if (np <= 16) {
    // few pairs (the batched mode's 8 per cube): one element per thread, all
    // np loads in flight -- 256 elements per CTA instead of 32 (the 32-wide
    // split below left 73k latency-bound CTAs for 64 cubes)
    const long long idx = blockIdx.x * 256LL + threadIdx.x;
    const int i = idx < bb ? (int)(idx / B) : 0, j = idx < bb ? (int)(idx % B) : 0;
    if (idx < tot && !(idx < bb && i >= 128 && j < 128)) {
      long long v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = k < np ? __ldcs(partial + (long long)k * tot + idx) : 0;
      long long s = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) s += v[k];
      partial[idx] = s;
    }
    return;
  }
  const long long idx = blockIdx.x * 32LL + lane;
  const int i = idx < bb ? (int)(idx / B) : 0, j = idx < bb ? (int)(idx % B) : 0;
  const bool active = idx < tot && !(idx < bb && i >= 128 && j < 128);
  long long s = 0;
  if (active) {
    for (int k0 = w; k0 < np; k0 += 8 * 16) {
      long long v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = k0 + 8 * u;
        v[u] = k < np ? __ldcs(partial + (long long)k * tot + idx) : 0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && active) {
    long long t = part[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += part[q][lane];
    partial[idx] = t;
  }
}

// ------------------------------------------------------------------ fix
// The flagged pixels P of one pixel split, in increasing order: F = sum y y^T
// (fp64), D = sum q q^T and, on the diagonal output blocks, sum q (int64),
// q recomputed exactly as the converters did.  Grid: fix_splits(n) CTAs, each
// walking the upper-triangular 64x64 output blocks of its split.  A split
// without a flagged pixel writes only its count (0) and exits after one scan
// of its bitmap words.

// the integer the converters fed to the MMAs for value y (any y, flagged or not)
__device__ __forceinline__ int quant_q(float y, const GramQScale& q) {
  return (int)(__float_as_uint(fmaf(y, q.inv_s, q.kf)) & 0xFFFFu) - 32768;
}

__global__ void __launch_bounds__(256) gram_fix_kernel(const float* __restrict__ Y, long long n, int B, int nbk,
                                                       const GramQScale* __restrict__ qsc,
                                                       const unsigned* __restrict__ bitmap, FixOut o,
                                                       int* nonfinite, const GramJob* __restrict__ jobs) {
  pdl_wait();
  if (jobs) {
    const GramJob& j = jobs[blockIdx.y];
    Y = j.Y;
    qsc = j.qs;
    bitmap = j.bitmap;
    o = j.fix;
    nonfinite = j.nonfinite;
  }
  __shared__ float As[FIX_TP][FIX_TB + 1];
  __shared__ float Bs[FIX_TP][FIX_TB + 1];
  __shared__ int Aq[FIX_TP][FIX_TB + 1];
  __shared__ int Bq[FIX_TP][FIX_TB + 1];
  __shared__ int list[FIX_CAP];
  __shared__ int wtot[8];
  const int split = blockIdx.x;
  const long long nw = (n + 31) / 32;
  const long long wper = ((nw + gridDim.x - 1) / gridDim.x + 3) / 4 * 4;   // gridDim.x = fix_splits(n)
  const long long w_begin = split * wper, w_end = min(nw, w_begin + wper);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntp = nbk * (nbk + 1) / 2;
  bool bad = false;
  // one CTA per pixel split walks every upper-triangular 64 x 64 output block;
  // the first walk finds whether the split has any flagged pixel at all
  for (int tp = 0; tp < ntp; ++tp) {
  int pr = tp, bi = 0;
  while (pr >= nbk - bi) { pr -= nbk - bi; ++bi; }
  const int bj = bi + pr;
  const int i0 = bi * FIX_TB, j0 = bj * FIX_TB;
  double f[4][4];
  long long d[4][4], q1[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    q1[a] = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) { f[a][c] = 0.0; d[a][c] = 0; }
  }
  int total = 0;
  // chunks of 1024 bitmap words: 4 consecutive words per thread, so thread
  // order = pixel order; a block scan of the bit counts places every flagged
  // pixel in the list in increasing order (one round trip when none is set)
  for (long long wc = w_begin; wc < w_end; wc += 1024) {
    unsigned wv[4];
    int c = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long w = wc + threadIdx.x * 4 + u;
      wv[u] = w < w_end ? bitmap[w] : 0u;
      c += __popc(wv[u]);
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    int before = 0, chunk = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      before += q < warp ? wtot[q] : 0;
      chunk += wtot[q];
    }
    __syncthreads();
    if (chunk == 0) continue;
    const int excl = before + incl - c;
    for (int base = 0; base < chunk; base += FIX_CAP) {
      int pos = excl;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned bits = wv[u];
        while (bits) {
          const int t = __ffs(bits) - 1;
          bits &= bits - 1;
          if (pos >= base && pos < base + FIX_CAP) list[pos - base] = (int)((wc + threadIdx.x * 4 + u) * 32 + t);
          ++pos;
        }
      }
      __syncthreads();
      const int nl = min(FIX_CAP, chunk - base);
      total += nl;
      for (int p0 = 0; p0 < nl; p0 += FIX_TP) {
#pragma unroll
        for (int it = 0; it < (FIX_TB * FIX_TP) / 256; ++it) {
          const int idx = threadIdx.x + it * 256;
          const int r = idx / FIX_TP, cc = idx % FIX_TP;
          float va = 0.f, vb = 0.f;
          int qa = 0, qb = 0;
          if (p0 + cc < nl) {
            const long long p = list[p0 + cc];
            if (i0 + r < B) { va = Y[(long long)(i0 + r) * n + p]; qa = quant_q(va, qsc[i0 + r]); }
            if (j0 + r < B) { vb = Y[(long long)(j0 + r) * n + p]; qb = quant_q(vb, qsc[j0 + r]); }
          }
          bad |= !isfinite(va) || !isfinite(vb);
          As[cc][r] = va;
          Bs[cc][r] = vb;
          Aq[cc][r] = qa;
          Bq[cc][r] = qb;
        }
        __syncthreads();
        for (int pp = 0; pp < FIX_TP; ++pp) {
          double a[4], bv[4];
          long long ia[4], ib[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[q] = (double)As[pp][ty * 4 + q];
            bv[q] = (double)Bs[pp][tx * 4 + q];
            ia[q] = Aq[pp][ty * 4 + q];
            ib[q] = Bq[pp][tx * 4 + q];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            q1[u] += ia[u];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              f[u][v] = fma(a[u], bv[v], f[u][v]);
              d[u][v] += ia[u] * ib[v];
            }
          }
        }
        __syncthreads();
      }
    }
  }
  if (tp == 0 && threadIdx.x == 0) o.cnt[split] = total;
  if (total == 0) return;
  double* F = o.F + (long long)split * B * B;
  long long* D = o.D + (long long)split * B * B;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ty * 4 + u;
    if (i >= B) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tx * 4 + v;
      if (j < B) {
        F[(long long)i * B + j] = f[u][v];
        D[(long long)i * B + j] = d[u][v];
      }
    }
    if (bi == bj && tx == 0) o.Q1[(long long)split * B + i] = q1[u];
  }
  }
  if (bad) atomicOr(nonfinite, 1);
}

__device__ __forceinline__ double i128_to_f64(__int128 x) {
  const bool neg = x < 0;
  const unsigned __int128 u = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;
  const double v = (double)(unsigned long long)(u >> 64) * 18446744073709551616.0 + (double)(unsigned long long)u;
  return neg ? -v : v;
}

// Stage 2: G_ij = G_ji = s_i s_j T_ij + F_ij (i <= j) with
//   T = (S - D) + c_i Q1'_j + c_j Q1'_i + N' c_i c_j   (exact, 128-bit)
// S_ij = sum of the pair partials, (S_ij + S_ji)/2 on the diagonal 128-blocks
// (exact: the pairs wrote 512 X there); D, F, Q1' from the non-empty fix splits
// in split order.
__global__ void __launch_bounds__(256) gram_finalize_kernel(const long long* __restrict__ S, int B, long long n,
                                                            const GramQScale* __restrict__ qsc, FixOut o,
                                                            double* __restrict__ G, const GramJob* __restrict__ jobs,
                                                            int nsplit) {
  pdl_wait();
  if (jobs) {
    const GramJob& j = jobs[blockIdx.y];
    S = j.partial;
    qsc = j.qs;
    o = j.fix;
    G = j.G;
  }
  __shared__ int live[FIX_SPLITS];
  __shared__ int nlive;
  __shared__ long long np_sh;
  static_assert(FIX_SPLITS == 64, "two splits per lane");
  if (threadIdx.x < 32) {   // the non-empty splits in split order: one warp, both loads in flight
    const int l = threadIdx.x;
    const int v0 = l < nsplit ? o.cnt[l] : 0, v1 = 32 + l < nsplit ? o.cnt[32 + l] : 0;
    const unsigned b0 = __ballot_sync(0xffffffffu, v0 != 0), b1 = __ballot_sync(0xffffffffu, v1 != 0);
    const unsigned below = (1u << l) - 1u;
    if (v0) live[__popc(b0 & below)] = l;
    if (v1) live[__popc(b0) + __popc(b1 & below)] = 32 + l;
    long long np = (long long)v0 + (long long)v1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) np += __shfl_xor_sync(0xffffffffu, np, off);
    if (l == 0) {
      nlive = __popc(b0) + __popc(b1);
      np_sh = np;
    }
  }
  __syncthreads();
  const long long idx = blockIdx.x * 256LL + threadIdx.x;
  if (idx >= (long long)B * B) return;
  const int i = (int)(idx / B), j = (int)(idx % B);
  if (i > j) return;
  long long t = S[idx];
  if ((i < 128) == (j < 128)) t = (t + S[(long long)j * B + i]) / 2;
  const long long* Q1 = S + (long long)B * B;
  long long q1i = Q1[i], q1j = Q1[j];
  const long long np = np_sh;
  double f = 0.0;
  for (int kk = 0; kk < nlive; ++kk) {
    const int k = live[kk];
    t -= o.D[(long long)k * B * B + idx];
    f += o.F[(long long)k * B * B + idx];
    q1i -= o.Q1[(long long)k * B + i];
    q1j -= o.Q1[(long long)k * B + j];
  }
  const long long ci = qsc[i].c, cj = qsc[j].c;
  const __int128 T = (__int128)t + (__int128)ci * q1j + (__int128)cj * q1i + (__int128)(n - np) * ci * cj;
  const double g = i128_to_f64(T) * qsc[i].s * qsc[j].s + f;
  G[(long long)i * B + j] = g;
  G[(long long)j * B + i] = g;
}

}  // namespace

bool gram_tc_supported(int B) { return B >= 1 && B <= 224; }

// SM pairs for n pixels: min_px = 0 -> as many as the GPU has (at most 74,
// >= 512 pixels each: latency); min_px > 0 -> at least min_px pixels each
// (throughput mode of the batched lanes).  At most 32768 pixels per pair: the
// int32 TMEM accumulators must hold the T_ab cross term S0 S1^T + S1 S0^T
// (|.| <= 2 * 128 * 255 per pixel) and S1 S1^T (<= 255^2 per pixel).
int gram_tc_npairs(long long n, int min_px) {
  long long np = min_px > 0 ? n / min_px : (n + 4LL * KC - 1) / (4LL * KC);
  if (np > 74) np = 74;
  if (np < 1) np = 1;
  long long per = (n + np - 1) / np;
  if (per > 32768) {
    np = (n + 32767) / 32768;
    per = (n + np - 1) / np;
  }
  per = (per + KC - 1) / KC * KC;
  np = (n + per - 1) / per;
  return (int)np;
}

namespace {
size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
struct TcWs {
  GramQScale* qs;
  unsigned* bitmap;
  long long nwords;
  long long* partial;
  FixOut fix;
};
TcWs carve(void* base, long long n, int B, int npairs) {
  char* p = (char*)base;
  TcWs w;
  const size_t bb = (size_t)B * B;
  w.qs = (GramQScale*)p;                          p += al256((size_t)B * sizeof(GramQScale));
  w.nwords = (n + 31) / 32;
  w.bitmap = (unsigned*)p;                        p += al256((size_t)w.nwords * 4);
  w.partial = (long long*)p;                      p += al256((size_t)npairs * (bb + B) * 8);
  w.fix.F = (double*)p;                           p += al256((size_t)FIX_SPLITS * bb * 8);
  w.fix.D = (long long*)p;                        p += al256((size_t)FIX_SPLITS * bb * 8);
  w.fix.Q1 = (long long*)p;                       p += al256((size_t)FIX_SPLITS * B * 8);
  w.fix.cnt = (int*)p;                            p += al256((size_t)FIX_SPLITS * 4);
  return w;
}
}  // namespace

size_t gram_tc_ws_bytes(long long n, int B, int npairs) {
  const size_t bb = (size_t)B * B;
  return al256((size_t)B * sizeof(GramQScale)) + al256((size_t)((n + 31) / 32) * 4) +
         al256((size_t)npairs * (bb + B) * 8) + 2 * al256((size_t)FIX_SPLITS * bb * 8) +
         al256((size_t)FIX_SPLITS * B * 8) + al256((size_t)FIX_SPLITS * 4);
}

// the quantisation scales and per-split flagged-pixel counts of the last call
// on this workspace (tests / diagnostics)
void gram_tc_debug_ptrs(void* ws, long long n, int B, int npairs, const GramQScale** qs, const int** cnt) {
  TcWs w = carve(ws, n, B, npairs);
  *qs = w.qs;
  *cnt = w.fix.cnt;
}
// CTAs of the clipped-pixel correction: one per 256 bitmap words (8192
// pixels), at most FIX_SPLITS (a 65536-pixel cube of the batched mode: 8, not
// 64 -- the kernel's 222 registers keep one CTA per SM, so 64 x 64 mostly
// empty CTAs took 107 us)
static int fix_splits(long long n) {
  const long long nw = (n + 31) / 32, k = nw / 256;
  return (int)(k < 1 ? 1 : (k > FIX_SPLITS ? FIX_SPLITS : k));
}
int gram_tc_fix_splits(long long n) { return fix_splits(n); }

// 2-D tensor maps of the cube viewed as B rows of n fp32 pixels: boxes of
// 128 pixels x 64 bands (P region) and x hb bands (QS region); bands past B
// and pixels past n are zero-filled by the TMA unit.
static bool make_maps(const float* Y, long long n, int B, int hb, CUtensorMap* tmP, CUtensorMap* tmQ) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  }
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)B};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
  const cuuint32_t estr[2] = {1, 1};
  auto one = [&](CUtensorMap* tm, int rows) {
    const cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)rows};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)Y, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!one(tmP, 64)) return false;
  return one(tmQ, hb >= 8 ? hb : 64);
}

// K1: qscale (+ zeroing) -> tcgen05 Gram (the pairs' exact partials summed by
// int64 atomics into one accumulator; HYDE_GRAM_REDUCE: per-pair partials and
// an integer reduction kernel) -> clipped-pixel fix -> finalize.  Four launches
// on `st`, all with programmatic dependent launch.
static int qscale_uu(long long n) {
  const long long blen = n / QS_NBLK;
  return blen >= 8192 ? 4 : (blen >= 4096 ? 2 : 1);
}
template <typename... Args>
static cudaError_t launch_qscale(long long n, dim3 grid, cudaStream_t st, Args... args) {
  switch (qscale_uu(n)) {
    case 4: return launch_pdl(gram_qscale_kernel<4>, grid, dim3(256), 0, st, args...);
    case 2: return launch_pdl(gram_qscale_kernel<2>, grid, dim3(256), 0, st, args...);
    default: return launch_pdl(gram_qscale_kernel<1>, grid, dim3(256), 0, st, args...);
  }
}

static bool gram_atomic_sum() {
  static const bool a = !getenv("HYDE_GRAM_REDUCE");   // experiments: the separate reduce kernel
  return a;
}
int gram_tc_launches() { return gram_atomic_sum() ? 4 : 5; }

cudaError_t launch_gram_tc(const float* Y, long long n, int B, void* ws, int npairs, double* G, int* nonfinite,
                           cudaStream_t st, int* state4) {
  TcWs w = carve(ws, n, B, npairs);
  const bool atomic_sum = gram_atomic_sum();
  const long long tot = (long long)B * B + B;
  cudaError_t e = launch_qscale(n, dim3(B), st, Y, n, w.qs, w.bitmap, w.nwords, state4,
                             (int)(sizeof(RankState) / sizeof(int)), (const GramJob*)nullptr,
                             atomic_sum ? w.partial : (long long*)nullptr, atomic_sum ? tot : 0LL);
  if (e != cudaSuccess) return e;
  GramTc P;
  P.Y = Y;
  P.n = n;
  P.B = B;
  P.nb = B > 128 ? ((B - 128 + 31) / 32) * 32 : 0;
  P.rows_tot = B > 128 ? 128 : 64;
  long long per = (n + npairs - 1) / npairs;
  per = (per + KC - 1) / KC * KC;
  P.per_pair = per;
  P.qs = w.qs;
  P.partial = w.partial;
  P.bitmap = w.bitmap;
  P.atomic_sum = atomic_sum ? 1 : 0;
  {
    static const int gexp = [] { const char* ev = getenv("HYDE_GRAM_EXP"); return ev ? atoi(ev) : 0; }();
    P.exp = gexp;
  }
  CUtensorMap tmP, tmQ;
  const bool tma = (n % 4 == 0) && (((uintptr_t)Y & 15) == 0) && !getenv("HYDE_GRAM_NO_TMA") &&
                   make_maps(Y, n, B, P.nb / 2, &tmP, &tmQ);
  if (tma) {
    const size_t smem = (size_t)Feed<true>::NI * 2 * P.rows_tot * KC + (size_t)NF * FSTAGE;
    e = cudaFuncSetAttribute(gram_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(gram_tc_kernel<true>, dim3(2 * npairs), dim3(NTHREADS), smem, st, P, tmP, tmQ,
                   (const GramJob*)nullptr);
  } else {
    memset(&tmP, 0, sizeof(tmP));
    const size_t smem = (size_t)Feed<false>::NI * 2 * P.rows_tot * KC;
    e = cudaFuncSetAttribute(gram_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(gram_tc_kernel<false>, dim3(2 * npairs), dim3(NTHREADS), smem, st, P, tmP, tmP,
                   (const GramJob*)nullptr);
  }
  if (e != cudaSuccess) return e;
  if (!atomic_sum) {
    e = launch_pdl(gram_reduce_i64_kernel, dim3((unsigned)(npairs <= 16 ? (tot + 255) / 256 : (tot + 31) / 32)),
                   dim3(256), 0, st, w.partial, npairs, B, (const GramJob*)nullptr);
    if (e != cudaSuccess) return e;
  }
  const int nbk = (B + FIX_TB - 1) / FIX_TB;
  e = launch_pdl(gram_fix_kernel, dim3(fix_splits(n)), dim3(256), 0, st, Y, n, B, nbk,
                 (const GramQScale*)w.qs, (const unsigned*)w.bitmap, w.fix, nonfinite, (const GramJob*)nullptr);
  if (e != cudaSuccess) return e;
  return launch_pdl(gram_finalize_kernel, dim3((unsigned)(((long long)B * B + 255) / 256)), dim3(256), 0, st,
                    (const long long*)w.partial, B, n, (const GramQScale*)w.qs, w.fix, G, (const GramJob*)nullptr,
                    fix_splits(n));
}

// The same five kernels for nb cubes of one shape in one launch each
// (blockIdx.y = cube; register feed): the phased batched path.  hjobs: pinned
// host scratch, djobs: device scratch, nb * sizeof(GramJob) each.
size_t gram_job_bytes() { return sizeof(GramJob); }
cudaError_t launch_gram_tc_batched(int nb, const float* const* Y, void* const* ws, double* const* G,
                                   int* const* nonfinite, int* const* state4, double* const* zero8, long long n,
                                   int B, int npairs, void* hjobs, void* djobs, cudaStream_t st) {
  GramJob* hj = reinterpret_cast<GramJob*>(hjobs);
  for (int b = 0; b < nb; ++b) {
    TcWs w = carve(ws[b], n, B, npairs);
    hj[b].Y = Y[b];
    hj[b].qs = w.qs;
    hj[b].bitmap = w.bitmap;
    hj[b].partial = w.partial;
    hj[b].fix = w.fix;
    hj[b].G = G[b];
    hj[b].nonfinite = nonfinite[b];
    hj[b].state4 = state4 ? state4[b] : nullptr;
    hj[b].zero8 = zero8 ? zero8[b] : nullptr;
  }
  const GramJob* dj = reinterpret_cast<const GramJob*>(djobs);
  cudaError_t e = cudaMemcpyAsync(djobs, hjobs, (size_t)nb * sizeof(GramJob), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  const long long nwords = (n + 31) / 32;
  e = launch_qscale(n, dim3(B, nb), st, (const float*)nullptr, n,
                 (GramQScale*)nullptr, (unsigned*)nullptr, nwords, (int*)nullptr,
                 (int)(sizeof(RankState) / sizeof(int)), dj, (long long*)nullptr,
                 gram_atomic_sum() ? (long long)B * B + B : 0LL);
  if (e != cudaSuccess) return e;
  GramTc P;
  memset(&P, 0, sizeof(P));
  P.n = n;
  P.B = B;
  P.nb = B > 128 ? ((B - 128 + 31) / 32) * 32 : 0;
  P.rows_tot = B > 128 ? 128 : 64;
  long long per = (n + npairs - 1) / npairs;
  per = (per + KC - 1) / KC * KC;
  P.per_pair = per;
  P.atomic_sum = gram_atomic_sum() ? 1 : 0;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  const size_t smem = (size_t)Feed<false>::NI * 2 * P.rows_tot * KC;
  e = cudaFuncSetAttribute(gram_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(gram_tc_kernel<false>, dim3(2 * npairs, nb), dim3(NTHREADS), smem, st, P, tm, tm, dj);
  if (e != cudaSuccess) return e;
  if (!gram_atomic_sum()) {
    const long long tot = (long long)B * B + B;
    e = launch_pdl(gram_reduce_i64_kernel, dim3((unsigned)(npairs <= 16 ? (tot + 255) / 256 : (tot + 31) / 32), nb),
                   dim3(256), 0, st, (long long*)nullptr, npairs, B, dj);
    if (e != cudaSuccess) return e;
  }
  const int nbk = (B + FIX_TB - 1) / FIX_TB;
  FixOut fo;
  memset(&fo, 0, sizeof(fo));
  e = launch_pdl(gram_fix_kernel, dim3(fix_splits(n), nb), dim3(256), 0, st, (const float*)nullptr, n, B, nbk,
                 (const GramQScale*)nullptr, (const unsigned*)nullptr, fo, (int*)nullptr, dj);
  if (e != cudaSuccess) return e;
  return launch_pdl(gram_finalize_kernel, dim3((unsigned)(((long long)B * B + 255) / 256), nb), dim3(256), 0, st,
                    (const long long*)nullptr, B, n, (const GramQScale*)nullptr, fo, (double*)nullptr, dj,
                    fix_splits(n));
}
