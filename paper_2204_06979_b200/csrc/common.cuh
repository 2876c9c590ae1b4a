// Shared definitions for libhyde's sm_100a kernels (not shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hyde.h"

#define HYDE_MAX_TAPS 16
#define HYDE_MAX_LEVELS 12
#define HYDE_MAX_CHUNK 32

// Analysis filters (fp32) passed by value as a kernel argument (lives in the
// constant bank).  g_k = (-1)^k h_{T-1-k}.
struct FilterBank {
  float h[HYDE_MAX_TAPS];
  float g[HYDE_MAX_TAPS];
  float2 hg[HYDE_MAX_TAPS];   // {h_m, g_m}: the operand pair of one packed fp32x2 FMA
  int taps;
};

// Geometry of one level of the 2-D DWT: input extent (h_in x w_in), padded
// even extent (H x W), subband extent (H/2 x W/2).
struct LevelGeom {
  int h_in, w_in;   // input image of this level
  int hs, ws;       // subband rows/cols = ceil(h_in/2), ceil(w_in/2)
};

struct DwtPlan {
  int levels;
  int rows, cols;
  LevelGeom lv[HYDE_MAX_LEVELS];
  long long sub_off[HYDE_MAX_LEVELS];  // offset of level l's LH within one coefficient set
  long long ll_off;                    // offset of LL_L
  long long n_coeffs;                  // N_c
};

// host helpers (filters.cpp / plan.cpp)
int hyde_build_filters(int taps, FilterBank* fb, double* h64);
void hyde_make_plan(int rows, int cols, int levels, DwtPlan* p);

// device workspace pieces used by several kernels
// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor drains and waits at pdl_wait() (griddepcontrol.wait, a no-op
// without the attribute) before touching any global data -- hides the launch
// latency of the short dependent kernels of the chunk loop.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

struct RankState {
  int found;        // 1 once a failing component has been seen
  int rank;         // r* once found (else running count of passing components)
  int nonfinite;    // non-finite input flag (set by the Gram kernel)
  int sure_overflow;// SURE survivor set exceeded its capacity (method failure)
  unsigned sure_done; // subbands finished in the current K5 launch (the last one decides the rank)
};

#define HYDE_CUDA_OK(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::hyde_cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)

hyde_status hyde_cuda_fail(cudaError_t e, const char* what, const char* file, int line);

// kernel launchers (each returns cudaGetLastError() of its launch)
cudaError_t launch_gram(const float* Y, long long n, int B, double* partial, int nsplit,
                        double* G, int* nonfinite, cudaStream_t st);
int gram_nsplit(long long n, int B);
cudaError_t launch_gram_reduce(const double* partial, int nsplit, int B, double* G, cudaStream_t st, int sym = 0);
bool gram_tc_supported(int B);
int gram_tc_npairs(long long n, int min_px = 0);
// K1 quantisation of one band (k_gram_tc.cu): y ~ s (q + c), q = rint(y inv_s) - c
struct GramQScale {
  float inv_s;   // fp32 1 / step
  float kf;      // fma addend 1.5 * 2^23 - c (exact)
  int c;         // integer centre, |c| <= 2^21
  int pad;
  double s;      // 1 / (double)inv_s
};
// workspace of launch_gram_tc (scales, clip bitmap, int64 pair partials, fix partials)
size_t gram_tc_ws_bytes(long long n, int B, int npairs);
int gram_tc_launches();   // kernels launch_gram_tc enqueues (4; 5 with HYDE_GRAM_REDUCE)
cudaError_t launch_gram_tc(const float* Y, long long n, int B, void* ws, int npairs, double* G, int* nonfinite,
                           cudaStream_t st, int* state4 = nullptr);
size_t gram_job_bytes();
cudaError_t launch_gram_tc_batched(int nb, const float* const* Y, void* const* ws, double* const* G,
                                   int* const* nonfinite, int* const* state4, double* const* zero8, long long n,
                                   int B, int npairs, void* hjobs, void* djobs, cudaStream_t st);
void gram_tc_debug_ptrs(void* ws, long long n, int B, int npairs, const GramQScale** qs, const int** cnt);
int gram_tc_fix_splits(long long n);
size_t eig_workspace_doubles(int B);
cudaError_t launch_noise_eig(const double* G, long long n, int B, double ridge, int ncomp, int all_lam,
                             double* sigma, double* lam, double* V, double* house,
                             double* tri, float* W, float* U, int ldwu, cudaStream_t st, int cl_pref = 0,
                             int mode = 0);
// launch_noise_eig modes: the first chunk by Lanczos when it converges (T and Q
// then absent); the tridiagonal rerun (sigma given, W/U of the first ncomp kept)
enum { EIG_HOUSEHOLDER = 0, EIG_LANCZOS = 1, EIG_RETRI = 2 };
constexpr int EIG_LANCZOS_MAX_K = 6;   // phase 2L serves at most this many pairs (k_eig.cu LZK)
bool eig_lanczos_enabled();
size_t eig_args_bytes();
double* eig_flags_ptr(double* house, int B);
cudaError_t launch_noise_eig_batched(int nb, const double* const* G, long long n, int B, double ridge, int ncomp,
                                     double* const* sigma, double* const* house, double* const* tri,
                                     float* const* W, float* const* U, int ldwu, void* hargs, void* dargs,
                                     cudaStream_t st, int cl_pref = 0);
// F3: HyMiNoR second stage (k_hyminor.cu)
size_t l1spec_ws_bytes(long long n);
cudaError_t launch_l1spec(const float* M, float* X, long long n, int B, float lam, float mu, int max_iters, float tol,
                          int* iters, void* todo_ws, cudaStream_t st);
// F4: WSRRR (k_wsrrr.cu)
cudaError_t launch_wsrrr_lambda(const double* sigma, int B, long long nc, double* lam, cudaStream_t st);
cudaError_t launch_sumsq(const float* x, long long n, double* partial, double* out, cudaStream_t st);
cudaError_t launch_soft_stats(float* c, long long n, const double* lam, double* partial, double* c2, double* c1,
                              cudaStream_t st);
int wtc_chunks(long long nc, int r);
cudaError_t launch_wtc(const float* W, const float* C, long long nc, int B, int r, double* partial, double* M,
                       cudaStream_t st);
cudaError_t launch_procrustes(const double* M, int B, int r, double* V, float* V32, int ldv32, const double* w2,
                              const double* c2, const double* c1, const double* lam, double* f, cudaStream_t st);
cudaError_t launch_v32(const double* V, int B, int r, float* V32, int ld, cudaStream_t st);
// F2: FORPDN (k_forpdn.cu)
cudaError_t launch_forpdn_lambda(const double* M, const double* Gw, int B, long long n, double ridge, double* npow,
                                 double* rp, double* lam_out, double* Zs, cudaStream_t st);
cudaError_t launch_forpdn_solve(float* C, long long ldc, long long nc, int B, double lam, const double* lam_dev,
                                float* coef, cudaStream_t st);
// F1: HySime (k_hysime.cu)
cudaError_t launch_hysime_prep(const double* G, const double* M, int B, long long n, double ridge, double* Ry,
                               double* Rn, double* Rx, cudaStream_t st);
cudaError_t launch_hysime_delta(const double* V, int ldv, const double* Ry, const double* Rn, int B, double* p,
                                double* s2, double* delta, cudaStream_t st, int ncols = 0);
cudaError_t launch_hysime_bound(const double* lam_n, const double* mu, int B, double* lb, int* m_out, cudaStream_t st);
cudaError_t launch_hysime_fill(const double* mu, const double* lb, int m, int B, double* p, double* delta,
                               cudaStream_t st);
cudaError_t launch_eig_values(const double* tri, const double* house, int B, double* lam, cudaStream_t st);
cudaError_t launch_hysime_select(const double* delta, const double* p, int B, double tol_rel, const double* V,
                                 int ldv, double* basis, int* k_out, cudaStream_t st);
cudaError_t launch_eig_more_raw(const double* tri, const double* house, const double* ones, int B, int k0, int K,
                                double* lam, double* V, int ldv, float* W, float* U, int ldwu, cudaStream_t st);
cudaError_t launch_eig_raw(const double* Amat, int B, int ncomp, double* ones, double* lam, double* V, int ldv,
                           double* house, double* tri, float* W, float* U, int ldwu, cudaStream_t st,
                           int mode = 0);   // EIG_LANCZOS: the top ncomp pairs only (no T / Q afterwards)
cudaError_t launch_eigvec_more(const double* tri, const double* house, const double* sigma, int B,
                               int k0, int ncomp, double* lam_top, double* V, float* W, float* U,
                               int ldwu, cudaStream_t st);
cudaError_t launch_noise_residual(const float* Y, long long n, int B, const double* G, double ridge,
                                  double* work, float* out, cudaStream_t st);
cudaError_t launch_project(const float* Y, long long n, int B, const float* W, int ldw, int ncomp,
                           float* E, long long ldE, cudaStream_t st);
cudaError_t launch_dwt_level(const float* in, long long in_stride, int h_in, int w_in,
                             float* ll, long long ll_stride, float* sub, long long sub_stride,
                             int count, const FilterBank& fb, cudaStream_t st);
cudaError_t launch_idwt_level(const float* ll, long long ll_stride, const float* sub,
                              long long sub_stride, int h_out, int w_out, float* out,
                              long long out_stride, int count, const FilterBank& fb,
                              const float* tstar, int nsub, int s_lh, int s_ll, const RankState* rs, int k0, cudaStream_t st);
cudaError_t launch_soft_threshold(float* coeffs, long long cstride, const DwtPlan& plan, int count, const float* tstar,
                                  cudaStream_t st);
// surv: scratch of count * cstride keys (the survivor lists of the clustered subbands)
cudaError_t launch_sure(float* coeffs, long long cstride, const DwtPlan& plan, int count,
                        int keep_ll, int* kstar, float* tstar, double* e_sub,
                        RankState* rs, unsigned* surv, cudaStream_t st,
                        int k0 = 0, double n_coeffs = 0.0, int bands = 0, double* e_post = nullptr,
                        RankState* rs_mirror = nullptr);
int sure_prof_read(unsigned long long* out16);   // K5 phase cycles (HYDE_SURE_PROF builds), 0 otherwise
cudaError_t launch_rank_decide(const double* e_sub, int nsub, int count, int k0, double n_coeffs,
                               int bands, RankState* rs, double* e_post, cudaStream_t st);
// E1 helpers (k_util.cu)
cudaError_t launch_check_finite(const double* x, long long n, int* flag, cudaStream_t st);
cudaError_t launch_check_finite_f32(const float* x, long long n, int* flag, cudaStream_t st);
cudaError_t launch_scatter_rows(const double* src, int nrows, int ncols, const int* to, double* dst, int dst_rows,
                                const int* flag_in, cudaStream_t st);
cudaError_t launch_flag_from_sum(const double* x, int* flag, cudaStream_t st);
cudaError_t launch_reconstruct(const float* E, long long ldE, long long n, int B, const float* U,
                               int ldu, int rank, float* out, cudaStream_t st, const RankState* rs = nullptr);
