// K5 (north_star stage (5)): exact per-subband SURE
// threshold, soft thresholding and post-threshold energy.
//
// For a subband x of n coefficients (whitened units, noise sigma = 1) with
// sorted magnitudes a_(1) <= ... <= a_(n), a_(0) = 0:
//   S_k = n - 2k + sum_{i<=k} a_(i)^2 + (n-k) a_(k)^2,  k = 0..n,
//   k* = smallest argmin S_k,  t* = a_(k*),  x <- sign(x) max(|x| - t*, 0)
// (SURE: Stein's unbiased risk of soft thresholding at t; soft threshold
// SPEC.md:136-137).  E_post = sum of the thresholded squares (rank rule, A5).
//
// Exact argmin without sorting n elements: the fp32 bit pattern of |x| is an
// order-preserving uint32 key.  A 2048-bin histogram over the current key
// range gives, per bin j (count m_j, sum of squares sq_j, c_j elements and
// q_j sum of squares below it, key range [lo_j, hi_j]):
//   S_k >= LB_j = n - 2(c_j+m_j) + q_j + (n - c_j) lo_j^2    for k in bin j,
//   min_k S_k <= UB_j = n - 2(c_j+m_j) + q_j + sq_j + (n-c_j-m_j) hi_j^2.
// Bins with LB_j > min UB cannot hold the argmin; the key range shrinks to
// the hull of the surviving bins and the histogram is refined until at most
// CAP elements remain.  Those are gathered, bitonic-sorted in shared memory,
// and S_k is evaluated exactly with fp64 prefix sums (products of fp32 values
// are exact in fp64).  The count and sum of squares below the range are
// recomputed with a fixed-order reduction, so the result is deterministic.
// One CTA per (component, subband).
#include "common.cuh"

namespace {

constexpr int NT = 512;
constexpr int NWS = NT / 32;
constexpr int NB = 2048;
constexpr int CAP = 16384;
constexpr int MAXPASS = 8;

struct SubTable {
  long long off[3 * HYDE_MAX_LEVELS + 1];
  int n[3 * HYDE_MAX_LEVELS + 1];
  int nsub;
};

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
  if (w == 0) {
    double t = l < NWS ? red[l] : 0.0;
    t = warp_sum_d(t);
    if (l == 0) red[NWS] = t;
  }
  __syncthreads();
  return red[NWS];
}

struct SureState {
  unsigned klo, khi;
  long long cntb;
  double sqb;
  int m_in;
  double best_ub;
};

__global__ void __launch_bounds__(NT) sure_kernel(float* __restrict__ coeffs, long long cstride,
                                                  SubTable tab, int keep_ll, int* kstar, float* tstar,
                                                  double* e_sub, RankState* rs) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned* keys = reinterpret_cast<unsigned*>(smraw);         // CAP
  unsigned* hcnt = keys + CAP;                                   // NB
  double* hsq = reinterpret_cast<double*>(hcnt + NB);            // NB
  double* red = hsq + NB;                                        // NWS + 2
  double* scan = red + NWS + 2;                                  // NT
  __shared__ SureState st;
  __shared__ int nsurv;
  __shared__ double bestS[NWS];
  __shared__ long long bestK[NWS];

  const int s = blockIdx.x, comp = blockIdx.y;
  const int n = tab.n[s];
  float* x = coeffs + (long long)comp * cstride + tab.off[s];
  const int ks = comp * tab.nsub + s;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const double dn = (double)n;

  if (keep_ll && s == tab.nsub - 1) {
    double e = 0.0;
    for (int i = tid; i < n; i += NT) { double v = x[i]; e += v * v; }
    e = block_sum_d(e, red);
    if (tid == 0) { kstar[ks] = 0; tstar[ks] = 0.f; e_sub[ks] = e; }
    return;
  }

  if (tid == 0) {
    st.klo = 0u; st.khi = 0x7F800000u; st.cntb = 0; st.sqb = 0.0; st.m_in = n; st.best_ub = dn;
  }
  __syncthreads();
  double slack = 0.0;
  for (int pass = 0; pass < MAXPASS; ++pass) {
    const SureState cur = st;
    if (cur.m_in <= CAP || cur.khi <= cur.klo) break;
    const unsigned long long span = (unsigned long long)(cur.khi - cur.klo) + 1ull;
    const unsigned long long width = (span + NB - 1) / NB;
    for (int j = tid; j < NB; j += NT) { hcnt[j] = 0u; hsq[j] = 0.0; }
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      const float f = fabsf(x[i]);
      const unsigned u = __float_as_uint(f);
      if (u >= cur.klo && u <= cur.khi) {
        const int b = (int)((unsigned long long)(u - cur.klo) / width);
        atomicAdd(&hcnt[b], 1u);
        atomicAdd(&hsq[b], (double)f * (double)f);
      }
    }
    __syncthreads();
    if (w == 0) {
      constexpr int PER = NB / 32;
      const int j0 = l * PER;
      long long lc = 0;
      double lq = 0.0;
      for (int j = j0; j < j0 + PER; ++j) { lc += hcnt[j]; lq += hsq[j]; }
      // exclusive warp scans
      long long ec = lc;
      double eq = lq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long tc = __shfl_up_sync(0xffffffffu, ec, o);
        double tq = __shfl_up_sync(0xffffffffu, eq, o);
        if (l >= o) { ec += tc; eq += tq; }
      }
      ec -= lc;
      eq -= lq;
      double tot_q = __shfl_sync(0xffffffffu, eq + lq, 31);
      if (pass == 0) slack = 1e-7 * (dn + tot_q + cur.sqb);
      slack = __shfl_sync(0xffffffffu, slack, 0);
      // upper bounds
      long long c = cur.cntb + ec;
      double q = cur.sqb + eq;
      double ub = INFINITY;
      for (int j = j0; j < j0 + PER; ++j) {
        const unsigned m = hcnt[j];
        if (m) {
          unsigned long long hk = (unsigned long long)cur.klo + (unsigned long long)(j + 1) * width - 1ull;
          if (hk > cur.khi) hk = cur.khi;
          const double hv = (double)__uint_as_float((unsigned)hk);
          const double cm = (double)(c + m);
          ub = fmin(ub, dn - 2.0 * cm + q + hsq[j] + (dn - cm) * hv * hv);
        }
        c += m;
        q += hsq[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ub = fmin(ub, __shfl_xor_sync(0xffffffffu, ub, o));
      const double best = fmin(cur.best_ub, ub);
      // survivors: hull [first, last]
      c = cur.cntb + ec;
      q = cur.sqb + eq;
      int first = NB, last = -1;
      long long c_first = 0, c_last_end = 0;
      double q_first = 0.0;
      for (int j = j0; j < j0 + PER; ++j) {
        const unsigned m = hcnt[j];
        if (m) {
          const double lv = (double)__uint_as_float(
              (unsigned)((unsigned long long)cur.klo + (unsigned long long)j * width));
          const double lb = dn - 2.0 * (double)(c + m) + q + (dn - (double)c) * lv * lv;
          if (lb <= best + slack) {
            if (first == NB) { first = j; c_first = c; q_first = q; }
            last = j;
            c_last_end = c + m;
          }
        }
        c += m;
        q += hsq[j];
      }
      // warp-reduce: min first (with its c/q), max last (with its end count)
      int gfirst = first;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gfirst = min(gfirst, __shfl_xor_sync(0xffffffffu, gfirst, o));
      int glast = last;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) glast = max(glast, __shfl_xor_sync(0xffffffffu, glast, o));
      const unsigned fb = __ballot_sync(0xffffffffu, first == gfirst && gfirst < NB);
      const unsigned lb2 = __ballot_sync(0xffffffffu, last == glast && glast >= 0);
      const int fl = fb ? __ffs(fb) - 1 : 0;
      const int ll = lb2 ? __ffs(lb2) - 1 : 0;
      c_first = __shfl_sync(0xffffffffu, c_first, fl);
      q_first = __shfl_sync(0xffffffffu, q_first, fl);
      c_last_end = __shfl_sync(0xffffffffu, c_last_end, ll);
      if (l == 0) {
        st.best_ub = best;
        if (glast < 0) {
          st.m_in = 0;           // only k = 0 can be optimal
          st.khi = 0u; st.klo = 1u;
        } else {
          unsigned long long nlo = (unsigned long long)cur.klo + (unsigned long long)gfirst * width;
          unsigned long long nhi = (unsigned long long)cur.klo + (unsigned long long)(glast + 1) * width - 1ull;
          if (nhi > cur.khi) nhi = cur.khi;
          st.klo = (unsigned)nlo;
          st.khi = (unsigned)nhi;
          st.cntb = c_first;
          st.sqb = q_first;
          st.m_in = (int)(c_last_end - c_first);
        }
      }
    }
    __syncthreads();
  }
  const SureState fin = st;

  // ---- gather the surviving keys; exact count / sum of squares below the range ----
  if (tid == 0) nsurv = 0;
  __syncthreads();
  double part = 0.0;
  long long cbelow = 0;
  for (int i = tid; i < n; i += NT) {
    const float f = fabsf(x[i]);
    const unsigned u = __float_as_uint(f);
    if (u < fin.klo) { part += (double)f * (double)f; ++cbelow; }
    else if (u <= fin.khi) {
      const int pos = atomicAdd(&nsurv, 1);
      if (pos < CAP) keys[pos] = u;
    }
  }
  const double sqb = block_sum_d(part, red);
  const double cb_d = block_sum_d((double)cbelow, red);
  const long long cntb = (long long)cb_d;
  const int M = nsurv;
  long long kbest = 0;
  double sbest = dn;   // k = 0 (t = 0): S_0 = n
  if (M > CAP) {
    if (fin.khi == fin.klo) {   // one repeated magnitude: S falls by 2 per step, best at the run end
      const double a = (double)__uint_as_float(fin.klo);
      const long long k = cntb + M;
      const double S = dn - 2.0 * (double)k + sqb + (double)M * a * a + (dn - (double)k) * a * a;
      if (S < sbest) { sbest = S; kbest = k; }
    } else if (tid == 0) {
      atomicOr(&rs->sure_overflow, 1);
    }
  } else if (M > 0) {
    int P2 = 1;
    while (P2 < M) P2 <<= 1;
    for (int i = M + tid; i < P2; i += NT) keys[i] = 0xFFFFFFFFu;
    __syncthreads();
    for (int k = 2; k <= P2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < P2; i += NT) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const unsigned a = keys[i], b = keys[ixj];
            const bool up = (i & k) == 0;
            if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
          }
        }
        __syncthreads();
      }
    }
    // contiguous segment per thread, fixed-order prefix sums of a^2
    const int seg = (M + NT - 1) / NT;
    const int b0 = tid * seg, b1 = min(M, b0 + seg);
    double tsum = 0.0;
    for (int i = b0; i < b1; ++i) {
      const double a = (double)__uint_as_float(keys[i]);
      tsum += a * a;
    }
    // exclusive block scan of tsum (warp scan + scan of warp totals)
    double incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(0xffffffffu, incl, o);
      if (l >= o) incl += t;
    }
    if (l == 31) scan[w] = incl;
    __syncthreads();
    if (w == 0) {
      double v = l < NWS ? scan[l] : 0.0;
      double iv = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(0xffffffffu, iv, o);
        if (l >= o) iv += t;
      }
      if (l < NWS) scan[NWS + l] = iv - v;   // exclusive warp offsets
    }
    __syncthreads();
    double Q = sqb + scan[NWS + w] + (incl - tsum);
    for (int i = b0; i < b1; ++i) {
      const double a = (double)__uint_as_float(keys[i]);
      Q += a * a;
      const long long k = cntb + i + 1;
      const double S = dn - 2.0 * (double)k + Q + (dn - (double)k) * a * a;
      if (S < sbest) { sbest = S; kbest = k; }   // ascending k: strict < keeps the smallest
    }
  }
  // block argmin (min S, then min k)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, sbest, o);
    const long long ok = __shfl_xor_sync(0xffffffffu, kbest, o);
    if (os < sbest || (os == sbest && ok < kbest)) { sbest = os; kbest = ok; }
  }
  __syncthreads();
  if (l == 0) { bestS[w] = sbest; bestK[w] = kbest; }
  __syncthreads();
  if (w == 0) {
    double sv = l < NWS ? bestS[l] : INFINITY;
    long long kv = l < NWS ? bestK[l] : 0x7fffffffffffffffLL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, sv, o);
      const long long ok = __shfl_xor_sync(0xffffffffu, kv, o);
      if (os < sv || (os == sv && ok < kv)) { sv = os; kv = ok; }
    }
    if (l == 0) { bestS[0] = sv; bestK[0] = kv; }
  }
  __syncthreads();
  const long long kopt = bestK[0];
  float t = 0.f;
  if (kopt > 0) {
    if (M > CAP) t = __uint_as_float(fin.klo);
    else t = __uint_as_float(keys[kopt - cntb - 1]);
  }
  // ---- soft threshold in place + post-threshold energy ----
  double e = 0.0;
  for (int i = tid; i < n; i += NT) {
    const float v = x[i];
    const float a = fabsf(v) - t;
    const float r = a > 0.f ? copysignf(a, v) : 0.f;
    x[i] = r;
    e += (double)r * (double)r;
  }
  e = block_sum_d(e, red);
  if (tid == 0) {
    kstar[ks] = (int)kopt;
    tstar[ks] = t;
    e_sub[ks] = e;
  }
}

__global__ void rank_decide_kernel(const double* __restrict__ e_sub, int nsub, int count, int k0,
                                   double n_coeffs, int bands, RankState* rs, double* e_post) {
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

}  // namespace

cudaError_t launch_sure(float* coeffs, long long cstride, const DwtPlan& plan, int count,
                        int keep_ll, int* kstar, float* tstar, double* e_sub, RankState* rs,
                        cudaStream_t st) {
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
  const size_t smem = (size_t)CAP * 4 + (size_t)NB * 4 + (size_t)NB * 8 + (size_t)(NWS + 2) * 8 +
                      (size_t)NT * 8;
  cudaError_t e = cudaFuncSetAttribute(sure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(tab.nsub, count);
  sure_kernel<<<grid, NT, smem, st>>>(coeffs, cstride, tab, keep_ll, kstar, tstar, e_sub, rs);
  return cudaGetLastError();
}

cudaError_t launch_rank_decide(const double* e_sub, int nsub, int count, int k0, double n_coeffs,
                               int bands, RankState* rs, double* e_post, cudaStream_t st) {
  rank_decide_kernel<<<1, 32, 0, st>>>(e_sub, nsub, count, k0, n_coeffs, bands, rs, e_post);
  return cudaGetLastError();
}
