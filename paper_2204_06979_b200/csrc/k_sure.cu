// K5 (north_star stage (5)): exact per-subband SURE
// threshold and post-threshold energy.
//
// For a subband x of n coefficients (whitened units, noise sigma = 1) with
// sorted magnitudes a_(1) <= ... <= a_(n), a_(0) = 0:
//   S_k = n - 2k + sum_{i<=k} a_(i)^2 + (n-k) a_(k)^2,  k = 0..n,
//   k* = smallest argmin S_k,  t* = a_(k*)
// (Stein's unbiased risk of soft thresholding; soft threshold SPEC.md:136-137),
// E_post = sum over the subband of (max(|x| - t*, 0))^2 (rank rule, A5).
// The soft threshold itself is applied by the inverse DWT when it loads the
// coefficients (K6a), so this kernel only reads the subband.
//
// Exact argmin without sorting n elements.  One launch covers every
// (component, subband); a subband with n >= BIG_MIN is split over a cluster
// of G CTAs (slices of n/G), smaller ones take one CTA each (G per cluster).
//  * the fp32 bit pattern of |x| is an order-preserving uint32 key; the key
//    window starts as the exact [min, max] of the subband;
//  * pruning passes: every thread keeps PRIVATE (count, fp64 sum of squares)
//    accumulators for 32 bins -- 30 equal key-bins over the window (equal key
//    width = log-spaced magnitudes) plus two catch-alls -- in shared memory
//    (no atomics: shared-memory float/int64 atomics are CAS loops on sm_100),
//    reduced in a fixed order; each rank pushes its bins to the cluster
//    leader over DSMEM.  Exact counts and sums at the bin edges give, per bin j,
//      S_k >= LB_j = n - 2(c_j+m_j) + q_j + (n - c_j) lo_j^2,
//      min S <= UB_j = n - 2(c_j+m_j) + q_j + sq_j + (n-c_j-m_j) hi_j^2.
//    Bins whose LB exceeds the best UB cannot hold the argmin; the window
//    shrinks to the hull of the surviving bins (everything outside it was
//    pruned earlier: the best UB only decreases);
//  * the survivors are written to a scratch list, the window is cut at bin
//    edges into one key sub-range per rank, and each rank evaluates S_k
//    exactly over its sub-range in ascending chunks of <= CAPL keys (gathered,
//    sorted in shared memory by a register bitonic + merge-path sort, fp64
//    prefix sums in sorted order; products of fp32 values are exact in fp64),
//    starting from the exact count / sum below the sub-range.  A chunk that
//    is one repeated key is evaluated in closed form (S falls by 2 per step
//    along a run of equal magnitudes: its best is the run end).
// Every sum is taken in a fixed order, so the result is deterministic.
#include "common.cuh"
#include "tc_util.cuh"
#include <cstdio>

namespace {

constexpr int NT = 256;
constexpr int NWS = NT / 32;
constexpr int NBIN = 32;          // 0 = below, 1..30 inner, 31 = above
constexpr int NIN = NBIN - 2;
constexpr int G = 8;              // cluster size (CTAs per big subband)
constexpr int CAPL = NT * 32;     // keys one CTA sorts at a time (8192)
constexpr int BIG_MIN = 32768;    // subbands at least this long use a cluster
constexpr int MAXPASS = 12;
constexpr int SURV_GOAL = 2048;   // prune until at most this many keys survive (or no progress)
constexpr int PF = 16;            // loads in flight per thread in the streaming passes
constexpr int PFC = 8;            // ... in the compaction streams (more live state per value)
constexpr size_t SMEM_DYN = (size_t)NBIN * NT * sizeof(unsigned long long);   // == 2 x CAPL keys

struct SubTable {
  long long off[3 * HYDE_MAX_LEVELS + 1];
  int n[3 * HYDE_MAX_LEVELS + 1];
  int nsub;
  int nbig, nsmall;
  int big[3 * HYDE_MAX_LEVELS + 1];     // subband indices handled by a cluster
  int small[3 * HYDE_MAX_LEVELS + 1];   // subband indices handled by one CTA
};

// ------------------------------------------------------------ DSMEM helpers
__device__ __forceinline__ void st_dsm_u32(uint32_t a, unsigned v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_dsm_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_dsm_s64(uint32_t a, long long v) {
  asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

__device__ __forceinline__ double ld_dsm_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed tree), broadcast
__device__ double block_sum_d(double v, double* red) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = l < NWS ? red[l] : 0.0;
  return warp_sum_d(t);
}

// exclusive scan of per-thread fp64 values (fixed order); returns this thread's
// offset, *total = block total
__device__ double block_excl_scan(double v, double* scan, double* total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (l >= o) incl += t;
  }
  if (l == 31) scan[w] = incl;
  __syncthreads();
  if (w == 0) {
    const double x = l < NWS ? scan[l] : 0.0;
    double ix = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, ix, o);
      if (l >= o) ix += t;
    }
    if (l < NWS) scan[NWS + l] = ix - x;
    if (l == NWS - 1) scan[2 * NWS] = ix;
  }
  __syncthreads();
  const double r = scan[NWS + w] + (incl - v);
  *total = scan[2 * NWS];
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned keyof(float x) { return __float_as_uint(fabsf(x)); }
__device__ __forceinline__ double kval(unsigned k) { return (double)__uint_as_float(k); }

// Sort buffers are addressed through sw(): the low 5 index bits are XORed with
// the row (index / 32), so per-thread contiguous runs of 32 keys -- the
// register-sort runs, each thread's merge output, each thread's evaluation
// segment -- fall in distinct banks across a warp.
__device__ __forceinline__ int sw(int p) { return p ^ ((p >> 5) & 31); }

// Sort keys[0..P) ascending (P a power of two, ITEMS <= P <= NT*ITEMS; swizzled
// layout): each thread sorts ITEMS keys in registers (bitonic network), then
// runs are merged pairwise with merge-path partitions.  Returns the buffer
// holding the result.
template <int ITEMS>
__device__ unsigned* block_sort(unsigned* keys, unsigned* buf, int P) {
  const int tid = threadIdx.x;
  const int nthr = P / ITEMS;
  if (tid < nthr) {
    unsigned r[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) r[i] = keys[sw(tid * ITEMS + i)];
#pragma unroll
    for (int k = 2; k <= ITEMS; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const unsigned a = r[i], b = r[ixj];
            const unsigned mn = min(a, b), mx = max(a, b);
            if ((i & k) == 0) { r[i] = mn; r[ixj] = mx; } else { r[i] = mx; r[ixj] = mn; }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) keys[sw(tid * ITEMS + i)] = r[i];
  }
  __syncthreads();
  // ping-pong between keys and buf by offset from keys (buf - keys is a
  // multiple of 1024, so sw() commutes with the offset)
  const int boff = (int)(buf - keys);
  int so = 0, dof = boff;
  for (int L = ITEMS; L < P; L <<= 1) {
    if (tid < nthr) {
      const int base = (tid * ITEMS) & ~(2 * L - 1);
      const int d = tid * ITEMS - base;
      const int ab = so + base, bb = so + base + L;   // run A / run B origins
      int lo = max(0, d - L), hi = min(d, L);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[sw(ab + mid)] <= keys[sw(bb + d - 1 - mid)]) lo = mid + 1; else hi = mid;
      }
      int i = lo, j = d - lo;
      unsigned a = i < L ? keys[sw(ab + i)] : 0xFFFFFFFFu;
      unsigned b = j < L ? keys[sw(bb + j)] : 0xFFFFFFFFu;
      const int ob = dof + base + d;
#pragma unroll
      for (int t = 0; t < ITEMS; ++t) {
        const bool takeA = (j >= L) || (i < L && a <= b);
        keys[sw(ob + t)] = takeA ? a : b;
        if (takeA) ++i; else ++j;
        const int ni = takeA ? i : j;
        const int nb = takeA ? ab : bb;
        const unsigned nv = ni < L ? keys[sw(nb + ni)] : 0xFFFFFFFFu;
        if (takeA) a = nv; else b = nv;
      }
    }
    __syncthreads();
    const int t = so; so = dof; dof = t;
  }
  return keys + so;
}

// bin(k) = min(NIN-1, int(float(k-klo) * inv)) is monotone in k and THE bin
// definition; edge[] inverts it exactly (inner bin j holds keys
// [edge[j], edge[j+1]-1]), so bounds built on the edges hold whatever the
// rounding of inv.
__device__ __forceinline__ float bin_inv(unsigned klo, unsigned khi) {
  return (float)NIN * __frcp_rn((float)(khi - klo) + 1.0f);
}
__device__ __forceinline__ int bin_of(unsigned k, unsigned klo, unsigned khi, float inv) {
  if (k < klo) return 0;
  if (k > khi) return NBIN - 1;
  return 1 + min(NIN - 1, (int)((float)(k - klo) * inv));
}
// lane j of the calling warp computes edge[j]
__device__ __forceinline__ void bin_edges(unsigned klo, unsigned khi, unsigned* edge) {
  const int l = threadIdx.x & 31;
  const float inv = bin_inv(klo, khi);
  if (l == 0) { edge[0] = klo; edge[NIN] = khi + 1u; }
  if (l >= 1 && l < NIN) {
    unsigned lo = klo, hi = khi + 1u;
    while (lo < hi) {
      const unsigned mid = lo + ((hi - lo) >> 1);
      const int bm = min(NIN - 1, (int)((float)(mid - klo) * inv));
      if (bm >= l) hi = mid; else lo = mid + 1u;
    }
    edge[l] = lo;
  }
}

// Streams src[0..n) with PF loads in flight per thread, double-buffered so the
// next batch is in flight while f(i, value, valid) consumes the current one.
// Iteration is block-uniform (f may use warp collectives); a thread visits its
// elements in a fixed order.  CG: read through L2 only (data written earlier
// in this kernel by other CTAs), else the read-only path.
template <bool CG, typename F>
__device__ __forceinline__ void stream_u32(const unsigned* __restrict__ src, int n, F&& f) {
  const int tid = threadIdx.x;
  unsigned cur[PF], nxt[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) {
    const int i = u * NT + tid;
    cur[u] = i < n ? (CG ? __ldcg(src + i) : __ldg(src + i)) : 0u;
  }
  for (int b0 = 0; b0 < n; b0 += NT * PF) {
    const int b1 = b0 + NT * PF;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int i = b1 + u * NT + tid;
      nxt[u] = i < n ? (CG ? __ldcg(src + i) : __ldg(src + i)) : 0u;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int i = b0 + u * NT + tid;
      f(i, cur[u], i < n);
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) cur[u] = nxt[u];
  }
}

// Order-preserving single-stream compaction of the streamed values v with
// pred(v): per batch of NT*PFC values, per-warp counts (ballots) are published,
// every warp takes its exclusive offset, then writes -- no atomics, two block
// barriers per batch, deterministic output order (batch, warp, slot, lane).
// store(pos, v) receives the output position; acc(v) sees every valid value.
// Returns the total (all threads).
template <bool CG, typename P, typename S, typename A>
__device__ __forceinline__ int compact_stream(const unsigned* __restrict__ src, int n, P&& pred, S&& store, A&& acc,
                                              int* wcnt) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const unsigned lt = (1u << l) - 1u;
  unsigned cur[PFC], nxt[PFC];
#pragma unroll
  for (int u = 0; u < PFC; ++u) {
    const int i = u * NT + tid;
    cur[u] = i < n ? (CG ? __ldcg(src + i) : __ldg(src + i)) : 0u;
  }
  int total = 0;
  for (int b0 = 0; b0 < n; b0 += NT * PFC) {
    const int b1 = b0 + NT * PFC;
#pragma unroll
    for (int u = 0; u < PFC; ++u) {
      const int i = b1 + u * NT + tid;
      nxt[u] = i < n ? (CG ? __ldcg(src + i) : __ldg(src + i)) : 0u;
    }
    unsigned bal[PFC];
    int wc = 0;
#pragma unroll
    for (int u = 0; u < PFC; ++u) {
      const bool valid = b0 + u * NT + tid < n;
      bal[u] = __ballot_sync(0xffffffffu, valid && pred(cur[u]));
      wc += __popc(bal[u]);
      if (valid) acc(cur[u]);
    }
    if (l == 0) wcnt[w] = wc;
    __syncthreads();
    int off = total;
#pragma unroll
    for (int q = 0; q < NWS; ++q) {
      const int c = wcnt[q];
      off += q < w ? c : 0;
      total += c;
    }
#pragma unroll
    for (int u = 0; u < PFC; ++u) {
      if ((bal[u] >> l) & 1u) store(off + __popc(bal[u] & lt), cur[u]);
      off += __popc(bal[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PFC; ++u) cur[u] = nxt[u];
  }
  return total;
}

// Exact binning of n values over [klo, khi]: exact counts and sums of squares
// per bin into bcnt / bsq, edges into edge.  Each thread's private bin is one
// 64-bit word (u32 count | fp32 partial sum of squares), so an update is one
// LDS.64 + one STS.64; the fp32 partials (at most ept = ceil(n/NT) terms, so
// relative error <= ept * 2^-24) are reduced in fp64 in a fixed order -- the
// pruning bounds carry that error as slack.  KEYS: the source holds keys (a
// survivor list, read through L2), else fp32 coefficients.
template <bool KEYS>
__device__ __forceinline__ void bin_pass(const void* __restrict__ src, int n, unsigned klo, unsigned khi,
                                         unsigned long long* pb, unsigned* bcnt, double* bsq, unsigned* edge) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const float inv = bin_inv(klo, khi);
  for (int b = 0; b < NBIN; ++b) pb[b * NT + tid] = 0ull;
  stream_u32<KEYS>(static_cast<const unsigned*>(src), n, [&](int, unsigned v, bool valid) {
    if (valid) {
      const unsigned k = KEYS ? v : (v & 0x7FFFFFFFu);
      const int b = bin_of(k, klo, khi, inv);
      const unsigned long long e = pb[b * NT + tid];
      const float a = __uint_as_float(k);
      const float q = fmaf(a, a, __uint_as_float((unsigned)(e >> 32)));
      pb[b * NT + tid] = ((unsigned long long)__float_as_uint(q) << 32) | (unsigned)(e + 1ull);
    }
  });
  __syncthreads();
  for (int b = w; b < NBIN; b += NWS) {      // fixed-order reduction
    unsigned c = 0;
    double q = 0.0;
    for (int t = l; t < NT; t += 32) {
      const unsigned long long e = pb[b * NT + t];
      c += (unsigned)e;
      q += (double)__uint_as_float((unsigned)(e >> 32));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    q = warp_sum_d(q);
    if (l == 0) { bcnt[b] = c; bsq[b] = q; }
  }
  if (w == NWS - 1) bin_edges(klo, khi, edge);
  __syncthreads();
}

__device__ __forceinline__ bool better(double s1, long long k1, double s2, long long k2) {
  return s1 < s2 || (s1 == s2 && k1 < k2);
}

__global__ void __launch_bounds__(NT, 3) sure_kernel(const float* __restrict__ coeffs, long long cstride, SubTable tab,
                                                     int count, int keep_ll, int* kstar, float* tstar, double* e_sub,
                                                     RankState* rs, unsigned* surv) {
  extern __shared__ __align__(16) unsigned char smraw[];
  // union: pass accumulators (NBIN x NT packed u64) | sort buffers (2 x CAPL u32)
  unsigned long long* pb = reinterpret_cast<unsigned long long*>(smraw);
  unsigned* skeys = reinterpret_cast<unsigned*>(smraw);
  unsigned* sbuf = skeys + CAPL;
  __shared__ double red[NWS + 2];
  __shared__ double scan[2 * NWS + 1];
  __shared__ unsigned bcnt[NBIN];
  __shared__ double bsq[NBIN];
  __shared__ unsigned edge[NIN + 1];
  // leader-side gather areas (written by the ranks over DSMEM)
  __shared__ unsigned g_cnt[G][NBIN];
  __shared__ double g_sq[G][NBIN];
  __shared__ double g_S[G];
  __shared__ long long g_k[G];
  __shared__ unsigned g_key[G];
  __shared__ double g_e[G];
  // state broadcast by the leader
  __shared__ unsigned s_klo, s_khi, s_m;
  __shared__ unsigned s_go;                  // 1: run another pruning pass
  __shared__ unsigned s_u, s_v, s_mg;        // this rank's sub-range and its key count
  __shared__ long long s_cbw;                // count of keys below the window (cluster)
  __shared__ unsigned s_reg;                 // this rank's slot in the survivor list
  __shared__ unsigned s_t;                   // t* bits
  // leader-only state
  __shared__ double s_ub;
  __shared__ int s_first, s_last, s_pass;
  __shared__ int s_J;
  __shared__ unsigned pt_u[G], pt_v[G], pt_m[G], pt_reg[G];
  __shared__ int s_wc[NWS];
  __shared__ double bestS[NWS];
  __shared__ long long bestK[NWS];
  __shared__ unsigned bestT[NWS];

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int cid = blockIdx.x / G;
  const int myrank = (int)tc::cluster_ctarank();
  const int nbig_items = count * tab.nbig;
  int comp, s, nr, rank;
  if (cid < nbig_items) {
    comp = cid / tab.nbig;
    s = tab.big[cid % tab.nbig];
    nr = G;
    rank = myrank;
  } else {
    const int it = (cid - nbig_items) * G + myrank;
    if (it >= count * tab.nsmall) return;    // idle CTA of the last small cluster
    comp = it / tab.nsmall;
    s = tab.small[it % tab.nsmall];
    nr = 1;
    rank = 0;
  }
  const int leader = nr == 1 ? myrank : 0;   // cluster rank of the leader
  const bool is_leader = rank == 0;
  auto rk = [&](int r) { return nr == 1 ? myrank : r; };   // item rank -> cluster rank
  auto gsync = [&]() {
    if (nr > 1) tc::cluster_sync(); else __syncthreads();
  };
  auto put_u32 = [&](unsigned& var, int r, unsigned v) { st_dsm_u32(tc::mapa(tc::smem_u32(&var), rk(r)), v); };
  const int n = tab.n[s];
  const float* xs = coeffs + (long long)comp * cstride + tab.off[s];
  const int lo_i = (int)((long long)n * rank / nr), hi_i = (int)((long long)n * (rank + 1) / nr);
  const float* x = xs + lo_i;                // this rank's slice
  const unsigned* xu = reinterpret_cast<const unsigned*>(x);
  const int ns = hi_i - lo_i;
  unsigned* sl = surv + (long long)comp * cstride + tab.off[s];
  const int ks = comp * tab.nsub + s;
  const double dn = (double)n;
  const bool skip = keep_ll && s == tab.nsub - 1;   // LL kept: t = 0
#ifdef HYDE_SURE_DEBUG
  const long long dbg_t0 = clock64();
  long long dbg_t1 = 0, dbg_t2 = 0, dbg_t3 = 0;
  int dbg_chunks = 0, dbg_pass = 0;
  long long dbg_g = 0, dbg_s = 0, dbg_e = 0, dbg_p = 0, dbg_sc = 0;
#endif

  // ---------------- starting window: exact min / max key ----------------
  {
    unsigned kmn = 0xFFFFFFFFu, kmx = 0u;
    stream_u32<false>(xu, ns, [&](int, unsigned v, bool valid) {
      if (valid) { const unsigned k = v & 0x7FFFFFFFu; kmn = min(kmn, k); kmx = max(kmx, k); }
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
      kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
    }
    if (l == 0) { bcnt[w] = kmn; bcnt[NWS + w] = kmx; }
    __syncthreads();
    if (tid == 0) {
      unsigned a0 = 0xFFFFFFFFu, a1 = 0u;
      for (int q = 0; q < NWS; ++q) { a0 = min(a0, bcnt[q]); a1 = max(a1, bcnt[NWS + q]); }
      st_dsm_u32(tc::mapa(tc::smem_u32(&g_cnt[rank][0]), leader), a0);
      st_dsm_u32(tc::mapa(tc::smem_u32(&g_cnt[rank][1]), leader), a1);
    }
    gsync();
    if (is_leader && tid == 0) {
      unsigned a0 = 0xFFFFFFFFu, a1 = 0u;
      for (int r = 0; r < nr; ++r) { a0 = min(a0, g_cnt[r][0]); a1 = max(a1, g_cnt[r][1]); }
      a1 = min(a1, 0x7F800000u);
      s_m = skip ? 0u : (unsigned)n;
      s_ub = dn;
      s_first = -1;
      s_pass = 0;
      const unsigned go = (!skip && n > CAPL) ? 1u : 0u;   // clusters always prune once (partition)
      for (int r = 0; r < nr; ++r) {
        put_u32(s_klo, r, a0);
        put_u32(s_khi, r, a1);
        put_u32(s_go, r, go);
      }
    }
    gsync();
  }
#ifdef HYDE_SURE_DEBUG
  dbg_t1 = clock64();
#endif

  // ---------------- pruning passes ----------------
  for (int pass = 0; pass < MAXPASS && s_go; ++pass) {
#ifdef HYDE_SURE_DEBUG
    ++dbg_pass;
#endif
    const unsigned klo = s_klo, khi = s_khi;
    bin_pass<false>(x, ns, klo, khi, pb, bcnt, bsq, edge);
    if (w == 0) {                            // push this rank's bins to the leader
      st_dsm_u32(tc::mapa(tc::smem_u32(&g_cnt[rank][l]), leader), bcnt[l]);
      st_dsm_f64(tc::mapa(tc::smem_u32(&g_sq[rank][l]), leader), bsq[l]);
    }
    gsync();
    if (is_leader && w == 0) {
      // lane b: cluster totals of bin b (fixed rank order), then exclusive
      // prefix counts / sums over the bins, one inner bin per lane
      unsigned cb = 0;
      double qb = 0.0;
      for (int r = 0; r < nr; ++r) { cb += g_cnt[r][l]; qb += g_sq[r][l]; }
      bcnt[l] = cb;                          // the leader's bcnt / bsq now hold totals
      bsq[l] = qb;
      long long cincl = cb;
      double qincl = qb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long tc_ = __shfl_up_sync(0xffffffffu, cincl, o);
        const double tq = __shfl_up_sync(0xffffffffu, qincl, o);
        if (l >= o) { cincl += tc_; qincl += tq; }
      }
      const double tot_q = __shfl_sync(0xffffffffu, qincl, 31);
      const long long c = cincl - cb;        // keys below bin l
      const double q = qincl - qb;
      const bool inner = l >= 1 && l <= NIN && cb > 0u;
      double lbv = INFINITY, ubv = INFINITY;
      if (inner) {
        const double m = (double)cb;
        const double lo = kval(edge[l - 1]), hi = kval(edge[l] - 1u);
        lbv = dn - 2.0 * ((double)c + m) + q + (dn - (double)c) * lo * lo;
        ubv = dn - 2.0 * ((double)c + m) + q + qb + (dn - (double)c - m) * hi * hi;
      }
      double ub = ubv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ub = fmin(ub, __shfl_xor_sync(0xffffffffu, ub, o));
      ub = fmin(ub, s_ub);
      const double ept = (double)((n / nr + NT) / NT);   // fp32 terms per thread partial
      const double tol = 1e-9 * dn + 1e-12 * (dn + tot_q) + 4.0 * ept * 5.9604644775390625e-8 * tot_q;
      const unsigned surv_mask = __ballot_sync(0xffffffffu, inner && lbv <= ub + tol);
      unsigned go = 0, nlo = 1u, nhi = 0u, msum = 0;
      int first = -1, last = -1;
      if (surv_mask) {
        first = __ffs(surv_mask) - 2;        // inner bin index = lane - 1
        last = 30 - __clz(surv_mask);
        unsigned part = (l >= first + 1 && l <= last + 1) ? cb : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        msum = part;
        nlo = edge[first];
        nhi = edge[last + 1] - 1u;
        const bool progress = !(nlo == klo && nhi == khi);
        // keep pruning while it makes progress and the survivors exceed a
        // small exact-evaluation set: a streaming pass over the slice is far
        // cheaper than sorting tens of thousands of survivors
        go = (progress && msum > (unsigned)SURV_GOAL) ? 1u : 0u;
      }
      if (l == 0) {
        s_ub = ub;
        s_pass = 1;
        s_first = first;
        s_last = last;
        s_m = msum;                          // 0: only t = 0 (k = 0) can win
      }
      if (l < nr) {
        put_u32(s_klo, l, nlo);
        put_u32(s_khi, l, nhi);
        put_u32(s_go, l, go);
      }
    }
    gsync();
  }
#ifdef HYDE_SURE_DEBUG
  dbg_t2 = clock64();
#endif

  // ---------------- partition the window into one sub-range per rank ----------------
  // (leader) the last pass's bin counts split the window at bin edges into nr
  // owners of ~M/nr keys and give each rank its slot in the survivor list and
  // the exact count below the window; without a pass (single CTA) the window is
  // the whole subband.
  if (is_leader && w == 0) {
    const unsigned klo = s_klo, khi = s_khi;
    const unsigned M = s_m;
    long long cbw = 0;
    if (l == 0) {                            // greedy split (serial, on local smem)
      for (int g = 0; g < nr; ++g) { pt_u[g] = 1u; pt_v[g] = 0u; pt_m[g] = 0u; pt_reg[g] = 0u; }
      if (M == 0u || klo > khi) {
      } else if (!s_pass) {                  // single CTA, whole subband
        pt_u[0] = klo;
        pt_v[0] = khi;
        pt_m[0] = (unsigned)n;
      } else {
        const int first = s_first, last = s_last;
        unsigned woff = 0;
        for (int r = 0; r < nr; ++r) {       // each rank's slot in the survivor list
          pt_reg[r] = woff;
          for (int jj = first; jj <= last; ++jj) woff += g_cnt[r][1 + jj];
        }
        cbw = bcnt[0];
        for (int j = 0; j < first; ++j) cbw += bcnt[1 + j];
        const long long target = ((long long)M + nr - 1) / nr;
        int j = first;
        for (int g = 0; g < nr; ++g) {       // bins first..last -> nr owners of ~M/nr keys
          const int j0 = j;
          long long mg = 0;
          while (j <= last && (mg < target || g == nr - 1)) { mg += bcnt[1 + j]; ++j; }
          if (j > j0) { pt_u[g] = edge[j0]; pt_v[g] = edge[j] - 1u; }
          pt_m[g] = (unsigned)mg;
        }
      }
    }
    cbw = __shfl_sync(0xffffffffu, cbw, 0);
    __syncwarp();
    if (l < nr) {                            // lane g -> rank g
      put_u32(s_m, l, M);
      put_u32(s_u, l, pt_u[l]);
      put_u32(s_v, l, pt_v[l]);
      put_u32(s_mg, l, pt_m[l]);
      put_u32(s_reg, l, pt_reg[l]);
      st_dsm_s64(tc::mapa(tc::smem_u32(&s_cbw), rk(l)), cbw);
    }
  }
  gsync();

#ifdef HYDE_SURE_DEBUG
  dbg_p = clock64() - dbg_t2;
#endif
  // ---------------- survivors -> this rank's slot of the scratch list (clusters) ----------------
  // The same stream sums x^2 below the window exactly (fp64, fixed order).
  const unsigned klo = s_klo, khi = s_khi;
  const unsigned M = s_m;
  const bool clustered = nr > 1 && M > 0u && klo <= khi;
  if (clustered) {
    const unsigned woff = s_reg;
    double qb = 0.0;
    compact_stream<false>(
        xu, ns, [&](unsigned v) { const unsigned k = v & 0x7FFFFFFFu; return k >= klo && k <= khi; },
        [&](int pos, unsigned v) { sl[woff + pos] = v & 0x7FFFFFFFu; },
        [&](unsigned v) {
          const unsigned k = v & 0x7FFFFFFFu;
          if (k < klo) { const double a = kval(k); qb = fma(a, a, qb); }
        },
        s_wc);
    qb = block_sum_d(qb, red);
    if (tid == 0) st_dsm_f64(tc::mapa(tc::smem_u32(&g_e[rank]), leader), qb);
  }
  gsync();
  double qbw = 0.0;                          // exact sum of x^2 below the window (cluster)
  long long cbw = 0;
  if (clustered) {
    double t = 0.0;
    if (l < nr) t = ld_dsm_f64(tc::mapa(tc::smem_u32(&g_e[l]), leader));
    qbw = warp_sum_d(t);
    cbw = s_cbw;
  }

#ifdef HYDE_SURE_DEBUG
  dbg_sc = clock64() - dbg_t2 - dbg_p;
#endif
  // ---------------- exact evaluation of this rank's sub-range ----------------
  // Chunk [u, v] of <= CAPL keys: one compaction stream over the source gathers
  // its keys and sums (count, x^2) of the source keys below u, so the prefix at
  // u is exact: (cbw, qbw) + those.
  double sbest = dn;          // k = 0 (t = 0): S_0 = n
  long long kbest = 0;
  unsigned tkey = 0u;
  {
    const unsigned v_g = s_v;
    unsigned u = s_u;
    unsigned m_rem = s_mg;
    unsigned whi = v_g;
    // source of this sub-range's keys: the survivor list (cluster) or the
    // subband itself (single CTA)
    const bool from_list = nr > 1;
    const unsigned* srcp = from_list ? sl : reinterpret_cast<const unsigned*>(xs);
    const int nsrc = from_list ? (int)M : n;
    for (int it = 0; it < 4096 && u <= v_g && m_rem > 0u; ++it) {
      unsigned v;
      bool run = false;
      if (m_rem <= (unsigned)CAPL && whi == v_g) {
        v = v_g;
      } else {
        if (from_list) bin_pass<true>(srcp, nsrc, u, whi, pb, bcnt, bsq, edge);
        else bin_pass<false>(srcp, nsrc, u, whi, pb, bcnt, bsq, edge);
        if (tid == 0) {
          long long acc = 0;
          int J = 0;
          while (J < NIN && acc + (long long)bcnt[1 + J] <= (long long)CAPL) { acc += bcnt[1 + J]; ++J; }
          s_J = J;
        }
        __syncthreads();
        const int J = s_J;
        const unsigned e1 = edge[1], eJ = edge[J < NIN ? J : NIN];
        __syncthreads();
        if (J == NIN) {
          v = whi;
        } else if (J > 0) {
          v = eJ - 1u;
        } else if (e1 - 1u == u) {
          v = u;
          run = true;
        } else {              // first bin alone exceeds CAPL: narrow and re-bin
          whi = e1 - 1u;
          continue;
        }
      }
#ifdef HYDE_SURE_DEBUG
      ++dbg_chunks;
      long long dq0 = clock64();
#endif
      double sql = 0.0, cl = 0.0;
      auto inr = [&](unsigned val) { const unsigned k = from_list ? val : (val & 0x7FFFFFFFu); return k >= u && k <= v; };
      auto put = [&](int pos, unsigned val) { if (pos < CAPL) skeys[sw(pos)] = from_list ? val : (val & 0x7FFFFFFFu); };
      auto below = [&](unsigned val) {
        const unsigned k = from_list ? val : (val & 0x7FFFFFFFu);
        if (k < u) { const double a = kval(k); sql = fma(a, a, sql); cl += 1.0; }
      };
      const int mc = from_list ? compact_stream<true>(srcp, nsrc, inr, put, below, s_wc)
                               : compact_stream<false>(srcp, nsrc, inr, put, below, s_wc);
      const long long c_run = cbw + (long long)block_sum_d(cl, red);
      const double q_run = qbw + block_sum_d(sql, red);
#ifdef HYDE_SURE_DEBUG
      dbg_g += clock64() - dq0;
#endif
      if (run) {              // one repeated key: best at the run end
        const double a = kval(u);
        const long long k = c_run + mc;
        const double S = dn - 2.0 * (double)k + q_run + (double)mc * a * a + (dn - (double)k) * a * a;
        if (tid == 0 && better(S, k, sbest, kbest)) { sbest = S; kbest = k; tkey = u; }
        m_rem -= (unsigned)mc;
      } else if (mc > CAPL) {
        if (tid == 0) atomicOr(&rs->sure_overflow, 1);   // unreachable by construction
        break;
      } else if (mc > 0) {
        int P2 = 32;
        while (P2 < mc) P2 <<= 1;
        for (int i = mc + tid; i < P2; i += NT) skeys[sw(i)] = 0xFFFFFFFFu;
        __syncthreads();
#ifdef HYDE_SURE_DEBUG
        long long dq1 = clock64();
#endif
        const unsigned* sk = P2 <= NT * 16 ? block_sort<16>(skeys, sbuf, P2) : block_sort<32>(skeys, sbuf, P2);
#ifdef HYDE_SURE_DEBUG
        dbg_s += clock64() - dq1;
        dq1 = clock64();
#endif
        const int seg = (mc + NT - 1) / NT;
        const int b0 = min(mc, tid * seg), b1 = min(mc, b0 + seg);
        double tsum = 0.0;
        for (int i = b0; i < b1; ++i) { const double aa = kval(sk[sw(i)]); tsum = fma(aa, aa, tsum); }
        double tot;
        double Q = q_run + block_excl_scan(tsum, scan, &tot);
        for (int i = b0; i < b1; ++i) {
          const unsigned kk = sk[sw(i)];
          const double aa = kval(kk);
          Q = fma(aa, aa, Q);
          const long long k = c_run + i + 1;
          const double S = dn - 2.0 * (double)k + Q + (dn - (double)k) * aa * aa;
          if (better(S, k, sbest, kbest)) { sbest = S; kbest = k; tkey = kk; }
        }
#ifdef HYDE_SURE_DEBUG
        __syncthreads();
        dbg_e += clock64() - dq1;
#endif
        m_rem -= (unsigned)mc;
      }
      __syncthreads();
      if (v >= v_g) break;
      u = v + 1u;
      whi = v_g;
    }
  }
#ifdef HYDE_SURE_DEBUG
  dbg_t3 = clock64();
#endif
  // block argmin (min S, then min k) -> leader
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, sbest, o);
    const long long ok = __shfl_xor_sync(0xffffffffu, kbest, o);
    const unsigned ot = __shfl_xor_sync(0xffffffffu, tkey, o);
    if (better(os, ok, sbest, kbest)) { sbest = os; kbest = ok; tkey = ot; }
  }
  if (l == 0) { bestS[w] = sbest; bestK[w] = kbest; bestT[w] = tkey; }
  __syncthreads();
  if (tid == 0) {
    double sv = bestS[0];
    long long kv = bestK[0];
    unsigned tv = bestT[0];
    for (int q = 1; q < NWS; ++q)
      if (better(bestS[q], bestK[q], sv, kv)) { sv = bestS[q]; kv = bestK[q]; tv = bestT[q]; }
    st_dsm_f64(tc::mapa(tc::smem_u32(&g_S[rank]), leader), sv);
    st_dsm_s64(tc::mapa(tc::smem_u32(&g_k[rank]), leader), kv);
    st_dsm_u32(tc::mapa(tc::smem_u32(&g_key[rank]), leader), tv);
  }
  gsync();
  if (is_leader && tid == 0) {
    double sv = g_S[0];
    long long kv = g_k[0];
    unsigned tv = g_key[0];
    for (int r = 1; r < nr; ++r)
      if (better(g_S[r], g_k[r], sv, kv)) { sv = g_S[r]; kv = g_k[r]; tv = g_key[r]; }
    g_k[0] = kv;
    for (int r = 0; r < nr; ++r) put_u32(s_t, r, kv > 0 ? tv : 0u);
  }
  gsync();
  // ---------------- E_post = sum (|x| - t)_+^2 over this slice -> leader ----------------
  double e_in = 0.0;
  {
    const double td = kval(s_t);
    stream_u32<false>(xu, ns, [&](int, unsigned v, bool valid) {
      const double aa = kval(v & 0x7FFFFFFFu) - td;
      if (valid && aa > 0.0) e_in = fma(aa, aa, e_in);
    });
  }
  const double e = block_sum_d(e_in, red);
  if (tid == 0) st_dsm_f64(tc::mapa(tc::smem_u32(&g_e[rank]), leader), e);
  gsync();
  if (is_leader && tid == 0) {
    double et = 0.0;
    for (int r = 0; r < nr; ++r) et += g_e[r];
    kstar[ks] = (int)g_k[0];
    tstar[ks] = __uint_as_float(s_t);
    e_sub[ks] = et;
#ifdef HYDE_SURE_DEBUG
    if (n > 40000)
      printf("SUREDBG comp %d sub %d n %d minmax %lld prune %lld (passes %d) eval %lld (chunks %d, M %u: part %lld "
             "scatter %lld gather %lld sort %lld S %lld) epost %lld total %lld\n",
             comp, s, n, dbg_t1 - dbg_t0, dbg_t2 - dbg_t1, dbg_pass, dbg_t3 - dbg_t2, dbg_chunks, M, dbg_p, dbg_sc,
             dbg_g, dbg_s, dbg_e, clock64() - dbg_t3, clock64() - dbg_t0);
#endif
  }
}

// in-place soft threshold of every subband with its tstar (stage API only;
// the hot path thresholds inside the inverse DWT's tile loads)
__global__ void soft_kernel(float* coeffs, long long cstride, SubTable tab, const float* __restrict__ tstar) {
  const int s = blockIdx.y, comp = blockIdx.z;
  const int n = tab.n[s];
  float* x = coeffs + (long long)comp * cstride + tab.off[s];
  const float t = tstar[comp * tab.nsub + s];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float v = x[i];
    const float a = fabsf(v) - t;
    x[i] = a > 0.f ? copysignf(a, v) : 0.f;
  }
}

__global__ void rank_decide_kernel(const double* __restrict__ e_sub, int nsub, int count, int k0, double n_coeffs,
                                   int bands, RankState* rs, double* e_post) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < count; ++k) {
    double e = 0.0;
    for (int s = 0; s < nsub; ++s) e += e_sub[k * nsub + s];
    e_post[k0 + k] = e;
    if (!rs->found) {
      if (e <= n_coeffs) {
        rs->found = 1;
        rs->rank = max(1, k0 + k);
      } else {
        rs->rank = k0 + k + 1;
      }
    }
  }
  if (!rs->found && k0 + count >= bands) {
    rs->found = 1;
    rs->rank = bands;
  }
}

SubTable make_table(const DwtPlan& plan) {
  SubTable tab;
  int s = 0;
  for (int l = 0; l < plan.levels; ++l) {
    const long long nsb = (long long)plan.lv[l].hs * plan.lv[l].ws;
    for (int o = 0; o < 3; ++o) {
      tab.off[s] = plan.sub_off[l] + o * nsb;
      tab.n[s] = (int)nsb;
      ++s;
    }
  }
  tab.off[s] = plan.ll_off;
  tab.n[s] = (int)(plan.n_coeffs - plan.ll_off);
  ++s;
  tab.nsub = s;
  tab.nbig = tab.nsmall = 0;
  for (int i = 0; i < s; ++i) {
    if (tab.n[i] >= BIG_MIN) tab.big[tab.nbig++] = i;
    else tab.small[tab.nsmall++] = i;
  }
  return tab;
}

}  // namespace

cudaError_t launch_sure(float* coeffs, long long cstride, const DwtPlan& plan, int count, int keep_ll, int* kstar,
                        float* tstar, double* e_sub, RankState* rs, unsigned* surv, cudaStream_t st) {
  const SubTable tab = make_table(plan);
  cudaError_t e = cudaFuncSetAttribute(sure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_DYN);
  if (e != cudaSuccess) return e;
  const int nclusters = count * tab.nbig + (count * tab.nsmall + G - 1) / G;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM_DYN;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sure_kernel, (const float*)coeffs, cstride, tab, count, keep_ll, kstar, tstar, e_sub,
                            rs, surv);
}

cudaError_t launch_soft_threshold(float* coeffs, long long cstride, const DwtPlan& plan, int count, const float* tstar,
                                  cudaStream_t st) {
  const SubTable tab = make_table(plan);
  dim3 grid(64, tab.nsub, count);
  soft_kernel<<<grid, 256, 0, st>>>(coeffs, cstride, tab, tstar);
  return cudaGetLastError();
}

cudaError_t launch_rank_decide(const double* e_sub, int nsub, int count, int k0, double n_coeffs, int bands,
                               RankState* rs, double* e_post, cudaStream_t st) {
  rank_decide_kernel<<<1, 32, 0, st>>>(e_sub, nsub, count, k0, n_coeffs, bands, rs, e_post);
  return cudaGetLastError();
}
