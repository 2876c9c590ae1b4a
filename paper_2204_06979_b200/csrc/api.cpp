// libhyde C-ABI (include/hyde.h): validation, workspace planning, stream
// ordering of the K1-K6 kernels, and the per-chunk rank decision.
//
// Orchestration of hyde_hyres_ex:
//   K1 gram -> K2 noise+eig (first chunk of eigenvectors) ->
//   for each chunk of r_c candidate components:
//       [K2b more eigenvectors] -> K3 project -> K4 DWT levels -> K5 SURE ->
//       rank decision (device) -> one D2H read of the 16-byte rank state ->
//       K6a IDWT of the chunk's kept components
//   -> K6b reconstruct (single write of the BSQ output).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "nccl_shim.h"

namespace {
thread_local std::string g_err;

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int kFirstChunk = 4;   // components in the first chunk of the rank loop

struct Layout {
  int B, chunk, nsplit, nsub, ldwu, taps, levels;
  long long n, ldE;
  DwtPlan plan;
  size_t G, partial, sigma, lam, tri, house, W, U, C, surv, S1, S2, kstar, tstar, esub, epost, rs, total;
  int use_tc, npairs;
  size_t s1_img, s2_img;  // per-image strides (floats) of the LL scratch
};

// gram_min_px > 0: at least that many pixels per K1 SM pair (throughput mode of
// the batched lanes: fewer, longer CTAs leave SMs to the other lanes and keep
// the per-pair partial Grams few); 0 = as many pairs as the GPU has (latency)
void make_layout(int rows, int cols, int B, int chunk, int levels, int taps, Layout* L, int gram_min_px = 0) {
  L->B = B;
  L->chunk = chunk;
  L->taps = taps;
  L->levels = levels;
  L->n = (long long)rows * cols;
  L->ldE = (L->n + 63) / 64 * 64;
  L->nsplit = gram_nsplit(L->n, B);
  L->use_tc = gram_tc_supported(B) ? 1 : 0;
  L->npairs = gram_tc_npairs(L->n, gram_min_px);
  L->ldwu = B;
  hyde_make_plan(rows, cols, levels, &L->plan);
  L->nsub = 3 * levels + 1;
  const size_t P = (size_t)B * (B + 1) / 2;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += al(bytes); return o; };
  L->G = take((size_t)B * B * 8);
  {
    // K1 workspace: the fp64 SIMT partials, or the tensor-core path's pieces
    const size_t simt = (size_t)L->nsplit * B * B * 8;
    const size_t tcw = L->use_tc ? gram_tc_ws_bytes(L->n, B, L->npairs) : 0;
    L->partial = take(simt > tcw ? simt : tcw);
  }
  L->sigma = take((size_t)B * 8);
  L->lam = take((size_t)B * 8);
  L->tri = take((size_t)(3 * B + 8) * 8);
  L->house = take(eig_workspace_doubles(B) * 8);
  L->W = take((size_t)B * L->ldwu * 4);
  L->U = take((size_t)B * L->ldwu * 4);
  L->C = take((size_t)chunk * L->plan.n_coeffs * 4);
  L->surv = take((size_t)chunk * L->plan.n_coeffs * 4);
  L->s1_img = (size_t)L->plan.lv[0].hs * L->plan.lv[0].ws;
  L->s2_img = levels > 1 ? (size_t)L->plan.lv[1].hs * L->plan.lv[1].ws : 1;
  L->S1 = take((size_t)chunk * L->s1_img * 4);
  L->S2 = take((size_t)chunk * L->s2_img * 4);
  L->kstar = take((size_t)chunk * L->nsub * 4);
  L->tstar = take((size_t)chunk * L->nsub * 4);
  L->esub = take((size_t)chunk * L->nsub * 8);
  L->epost = take((size_t)B * 8);
  L->rs = take(sizeof(RankState));
  L->total = off;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};
}  // namespace

struct hyde_ctx {
  int device = 0;
  std::string err;
  char* ws = nullptr;
  size_t ws_cap = 0;
  float* ebuf = nullptr;
  size_t ebuf_cap = 0;   // bytes
  RankState* rs_host = nullptr;      // pinned, mapped host mirror of the rank state
  RankState* rs_host_dev = nullptr;  // its device address
  float* dev_in = nullptr;
  float* dev_out = nullptr;
  size_t dev_io_cap = 0;
  // streaming host path: two cube slots (in, out) and its copy streams / events
  float* pipe_buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t pipe_cap = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  // batched path: lanes (own workspace, stream and host thread) so that
  // independent cubes overlap on the GPU
  std::vector<hyde_ctx*> lanes;
  std::vector<cudaStream_t> lane_st;
  std::vector<cudaEvent_t> lane_ev;
  cudaEvent_t ev_batch = nullptr;
  RankState* last_rs = nullptr;  // device rank/flag state of the last enqueued call
  char* shard_buf = nullptr;     // E1 exchange buffers (grow only)
  size_t shard_cap = 0;
  // phased batched path: per-cube workspaces, pinned mapped rank states, K2 args
  char* bws = nullptr;
  size_t bws_cap = 0;
  float* cubebuf = nullptr;      // F3: the l1 stage's input when it would alias its output
  size_t cubebuf_cap = 0;
  RankState* b_rs_host = nullptr;
  RankState* b_rs_dev = nullptr;
  void* b_args_host = nullptr;
  void* b_jobs_host = nullptr;
  int b_cap = 0;
  cudaEvent_t ev_rank = nullptr; // recorded after the per-chunk D2H copy of the rank state
  int gram_min_px = 0;           // K1 pixels per SM pair, at least (0: latency mode; lanes: throughput)
  int eig_cl = 0;                // K2 cluster size preference (0: largest; 8: throughput lanes)
  // stage profiling
  int prof = 0;
  struct Rec { int stage; int launches; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  long long launch_total = 0;
  long long launch_by_stage[HYDE_NSTAGES] = {0};
  cudaEvent_t ev() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {
// Marks one stage on `st`: counts its kernel launches and, when profiling is
// on, brackets it with CUDA events.
struct Stage {
  hyde_ctx* h;
  int stage, launches;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Stage(hyde_ctx* h_, int s, int nl, cudaStream_t st_) : h(h_), stage(s), launches(nl), st(st_) {
    if (h->prof) { a = h->ev(); cudaEventRecord(a, st); }
  }
  void end() {
    h->launch_total += launches;
    h->launch_by_stage[stage] += launches;
    if (h->prof) {
      cudaEvent_t b = h->ev();
      cudaEventRecord(b, st);
      h->recs.push_back({stage, launches, a, b});
    }
  }
};
}  // namespace

hyde_status hyde_cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  g_err = buf;
  return e == cudaErrorMemoryAllocation ? HYDE_ENOMEM : HYDE_ECUDA;
}

static hyde_status fail(hyde_handle h, hyde_status s, const std::string& msg) {
  g_err = msg;
  if (h) h->err = msg;
  return s;
}

#define CK(expr)                                                              \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      hyde_status _s = hyde_cuda_fail(_e, #expr, __FILE__, __LINE__);         \
      if (h) h->err = g_err;                                                  \
      return _s;                                                              \
    }                                                                         \
  } while (0)

static hyde_status ensure_ws(hyde_handle h, size_t bytes, cudaStream_t st) {
  if (bytes <= h->ws_cap) return HYDE_OK;
  if (h->ws) CK(cudaFreeAsync(h->ws, st));
  h->ws = nullptr;
  h->ws_cap = 0;
  size_t cap = bytes + bytes / 8;
  CK(cudaMallocAsync((void**)&h->ws, cap, st));
  h->ws_cap = cap;
  return HYDE_OK;
}

// grow the eigen-image buffer to `bytes`, preserving the first `keep` bytes
static hyde_status ensure_ebuf(hyde_handle h, size_t bytes, size_t keep, cudaStream_t st) {
  if (bytes <= h->ebuf_cap) return HYDE_OK;
  float* nb = nullptr;
  CK(cudaMallocAsync((void**)&nb, bytes, st));
  if (h->ebuf && keep) CK(cudaMemcpyAsync(nb, h->ebuf, keep, cudaMemcpyDeviceToDevice, st));
  if (h->ebuf) CK(cudaFreeAsync(h->ebuf, st));
  h->ebuf = nb;
  h->ebuf_cap = bytes;
  return HYDE_OK;
}

static void defaults(const hyde_hyres_params* in, hyde_hyres_params* p) {
  hyde_hyres_params_default(p);
  if (!in) return;
  if (in->wavelet_taps) p->wavelet_taps = in->wavelet_taps;
  p->levels = in->levels;
  if (in->chunk) p->chunk = in->chunk;
  if (in->ridge != 0.0) p->ridge = in->ridge;
  p->flags = in->flags;
}

static bool overlap(const void* a, size_t an, const void* b, size_t bn) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bn && y < x + an;
}

static hyde_status validate_shape(hyde_handle h, int rows, int cols, int bands) {
  if (!h) return HYDE_EPARAM;
  if (rows < 1 || cols < 1) return fail(h, HYDE_EPARAM, "rows and cols must be >= 1");
  if (bands < 3) return fail(h, HYDE_EPARAM, "bands must be >= 3 (SPEC.md:363)");
  if (bands > 256) return fail(h, HYDE_EPARAM, "bands must be <= 256");
  if ((long long)rows * cols <= bands) return fail(h, HYDE_EPARAM, "rows*cols must exceed bands (SPEC.md:365)");
  if ((long long)rows * cols > (1LL << 31) / 4) return fail(h, HYDE_EPARAM, "cube too large for one call");
  return HYDE_OK;
}

static hyde_status resolve_params(hyde_handle h, int rows, int cols, const hyde_hyres_params* in,
                                  hyde_hyres_params* p, int* levels) {
  defaults(in, p);
  if (p->wavelet_taps != 2 && p->wavelet_taps != 8 && p->wavelet_taps != 16)
    return fail(h, HYDE_EPARAM, "wavelet_taps must be 2, 8 or 16 (SPEC.md:179 D4)");
  if (p->chunk < 1 || p->chunk > HYDE_MAX_CHUNK) return fail(h, HYDE_EPARAM, "chunk must be in [1, 32]");
  if (p->ridge < 0.0) return fail(h, HYDE_EPARAM, "ridge must be >= 0");
  int lv = p->levels > 0 ? p->levels : hyde_auto_levels(rows, cols, p->wavelet_taps);
  if (lv > HYDE_MAX_LEVELS || (long long)(rows < cols ? rows : cols) < (1LL << lv))
    return fail(h, HYDE_EPARAM, "levels impossible for this image size (SPEC.md:122)");
  *levels = lv;
  return HYDE_OK;
}

// K1: exact int8 tensor-core Gram (B <= 224) or the fp64 SIMT fallback
static cudaError_t run_gram(const Layout& L, char* ws, const float* cube, double* G, int* nonfinite,
                            cudaStream_t st, int* state4 = nullptr) {
  if (L.use_tc) return launch_gram_tc(cube, L.n, L.B, ws + L.partial, L.npairs, G, nonfinite, st, state4);
  return launch_gram(cube, L.n, L.B, (double*)(ws + L.partial), L.nsplit, G, nonfinite, st);
}

// forward DWT of `count` images at E (stride ldE) into C (stride N_c)
static cudaError_t dwt_forward(const Layout& L, char* ws, const float* E, long long ldE, int count,
                               const FilterBank& fb, cudaStream_t st) {
  const long long nc = L.plan.n_coeffs;
  float* C = (float*)(ws + L.C);
  long long sstr[2] = {(long long)L.s1_img, (long long)L.s2_img};
  float* S[2] = {(float*)(ws + L.S1), (float*)(ws + L.S2)};
  for (int l = 0; l < L.levels; ++l) {
    const float* in = l == 0 ? E : S[(l - 1) & 1];
    long long in_str = l == 0 ? ldE : sstr[(l - 1) & 1];
    float* llo = (l == L.levels - 1) ? C + L.plan.ll_off : S[l & 1];
    long long ll_str = (l == L.levels - 1) ? nc : sstr[l & 1];
    cudaError_t e = launch_dwt_level(in, in_str, L.plan.lv[l].h_in, L.plan.lv[l].w_in, llo, ll_str,
                                     C + L.plan.sub_off[l], nc, count, fb, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// inverse DWT of `count` coefficient sets; when tstar != NULL each subband is
// soft-thresholded with its t* as it is loaded (K5 -> K6a fusion)
static cudaError_t dwt_inverse(const Layout& L, char* ws, const float* Cin, float* Eout, long long ldE,
                               int count, const FilterBank& fb, const float* tstar, cudaStream_t st,
                               const RankState* rs = nullptr, int k0 = 0) {
  long long sstr[2] = {(long long)L.s1_img, (long long)L.s2_img};
  float* S[2] = {(float*)(ws + L.S1), (float*)(ws + L.S2)};
  const long long nc = L.plan.n_coeffs;
  for (int l = L.levels - 1; l >= 0; --l) {
    const float* llin = (l == L.levels - 1) ? Cin + L.plan.ll_off : S[l & 1];
    long long ll_str = (l == L.levels - 1) ? nc : sstr[l & 1];
    float* out = l == 0 ? Eout : S[(l - 1) & 1];
    long long out_str = l == 0 ? ldE : sstr[(l - 1) & 1];
    const int s_ll = (l == L.levels - 1) ? 3 * L.levels : -1;   // only LL_L comes from K5
    cudaError_t e = launch_idwt_level(llin, ll_str, Cin + L.plan.sub_off[l], nc, L.plan.lv[l].h_in,
                                      L.plan.lv[l].w_in, out, out_str, count, fb, tstar, L.nsub, 3 * l, s_ll, rs, k0, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

extern "C" {

const char* hyde_version(void) { return "hyde-b200 0.1 (sm_100a)"; }
int hyde_target_sm(void) { return 100; }

const char* hyde_status_string(hyde_status s) {
  switch (s) {
    case HYDE_OK: return "ok";
    case HYDE_EPARAM: return "parameter error";
    case HYDE_EDATA: return "data error (non-finite input)";
    case HYDE_EMETHOD: return "method failure";
    case HYDE_ECUDA: return "CUDA error";
    case HYDE_ENCCL: return "NCCL error";
    case HYDE_ENOMEM: return "out of device memory";
  }
  return "unknown status";
}

const char* hyde_last_error(hyde_handle h) {
  if (h && !h->err.empty()) return h->err.c_str();
  return g_err.c_str();
}

void hyde_hyres_params_default(hyde_hyres_params* p) {
  if (!p) return;
  memset(p, 0, sizeof(*p));
  p->wavelet_taps = 16;
  p->levels = 0;
  p->chunk = 16;
  p->ridge = 1e-6;
  p->flags = 0;
}

hyde_status hyde_create(hyde_handle* out, int device) {
  if (!out) return HYDE_EPARAM;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return hyde_cuda_fail(e, "cudaGetDeviceCount", __FILE__, __LINE__);
  if (device < 0 || device >= ndev) {
    g_err = "no such CUDA device";
    return HYDE_EPARAM;
  }
  hyde_ctx* h = new hyde_ctx();
  h->device = device;
  DeviceGuard g(device);
  // pinned + mapped: the SURE kernel writes each chunk's rank decision here
  e = cudaHostAlloc((void**)&h->rs_host, sizeof(RankState), cudaHostAllocMapped | cudaHostAllocPortable);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&h->rs_host_dev, h->rs_host, 0);
  if (e != cudaSuccess) {
    delete h;
    return hyde_cuda_fail(e, "cudaHostAlloc", __FILE__, __LINE__);
  }
  *out = h;
  return HYDE_OK;
}

hyde_status hyde_destroy(hyde_handle h) {
  if (!h) return HYDE_OK;
  {
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();
    if (h->ws) cudaFree(h->ws);
    if (h->ebuf) cudaFree(h->ebuf);
    if (h->shard_buf) cudaFree(h->shard_buf);
    if (h->bws) cudaFree(h->bws);
    if (h->cubebuf) cudaFree(h->cubebuf);
    if (h->b_rs_host) cudaFreeHost(h->b_rs_host);
    if (h->b_args_host) cudaFreeHost(h->b_args_host);
    if (h->b_jobs_host) cudaFreeHost(h->b_jobs_host);
    if (h->dev_in) cudaFree(h->dev_in);
    if (h->dev_out) cudaFree(h->dev_out);
    for (auto b : h->pipe_buf)
      if (b) cudaFree(b);
    if (h->s_in) cudaStreamDestroy(h->s_in);
    if (h->s_out) cudaStreamDestroy(h->s_out);
    for (int i = 0; i < 2; ++i) {
      if (h->ev_in[i]) cudaEventDestroy(h->ev_in[i]);
      if (h->ev_done[i]) cudaEventDestroy(h->ev_done[i]);
      if (h->ev_out[i]) cudaEventDestroy(h->ev_out[i]);
    }
    for (auto l : h->lanes) hyde_destroy(l);
    for (auto st : h->lane_st) cudaStreamDestroy(st);
    for (auto e : h->lane_ev) cudaEventDestroy(e);
    if (h->ev_batch) cudaEventDestroy(h->ev_batch);
    if (h->ev_rank) cudaEventDestroy(h->ev_rank);
    if (h->rs_host) cudaFreeHost(h->rs_host);
    for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : h->pool) cudaEventDestroy(e);
  }
  delete h;
  return HYDE_OK;
}

size_t hyde_hyres_workspace_size(int rows, int cols, int bands, int batch, const hyde_hyres_params* params) {
  hyde_hyres_params p;
  int lv = 0;
  if (rows < 1 || cols < 1 || bands < 3 || bands > 256) return 0;
  defaults(params, &p);
  if (p.wavelet_taps != 2 && p.wavelet_taps != 8 && p.wavelet_taps != 16) return 0;
  lv = p.levels > 0 ? p.levels : hyde_auto_levels(rows, cols, p.wavelet_taps);
  if (lv > HYDE_MAX_LEVELS) return 0;
  (void)batch;
  Layout L;
  make_layout(rows, cols, bands, p.chunk, lv, p.wavelet_taps, &L);
  return L.total + (size_t)p.chunk * L.ldE * 4;
}

hyde_status hyde_sync_status(hyde_handle h, hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaStreamSynchronize(st));
  if (!h->last_rs) return HYDE_OK;
  CK(cudaMemcpy(h->rs_host, h->last_rs, sizeof(RankState), cudaMemcpyDeviceToHost));
  if (h->rs_host->nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
  if (h->rs_host->sure_overflow) return fail(h, HYDE_EMETHOD, "SURE survivor set exceeded its capacity");
  return HYDE_OK;
}

hyde_status hyde_hyres_ex(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out,
                          const hyde_hyres_params* params, hyde_hyres_info* info, hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!cube || !out) return fail(h, HYDE_EPARAM, "NULL cube/out");
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (cube != out && overlap(cube, bytes, out, bytes)) return fail(h, HYDE_EPARAM, "cube and out partially overlap");
  hyde_hyres_params p;
  int levels = 0;
  s = resolve_params(h, rows, cols, params, &p, &levels);
  if (s != HYDE_OK) return s;
  FilterBank fb;
  if (hyde_build_filters(p.wavelet_taps, &fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "filter derivation failed");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  const int B = bands;
  make_layout(rows, cols, B, p.chunk, levels, p.wavelet_taps, &L, h->gram_min_px);
  s = ensure_ws(h, L.total, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  const long long n = L.n;
  s = ensure_ebuf(h, (size_t)p.chunk * L.ldE * 4, 0, st);
  if (s != HYDE_OK) return s;
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  if (p.flags & HYDE_VALIDATE) {
    CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
    CK(launch_check_finite_f32(cube, n * B, &rs->nonfinite, st));
    CK(cudaMemcpyAsync(&h->rs_host->nonfinite, &rs->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h->rs_host->nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
  }
  if (!L.use_tc) CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  double* G = (double*)(ws + L.G);
  double* sigma = (double*)(ws + L.sigma);
  double* house = (double*)(ws + L.house);
  double* tri = (double*)(ws + L.tri);
  float* W = (float*)(ws + L.W);
  float* U = (float*)(ws + L.U);
  float* C = (float*)(ws + L.C);
  {
    Stage sg(h, HYDE_STAGE_GRAM, L.use_tc ? gram_tc_launches() : 2, st);
    // tensor-core path: the state words are zeroed by the Gram's first (zero) kernel
    CK(run_gram(L, ws, cube, G, &rs->nonfinite, st, L.use_tc ? (int*)rs : nullptr));
    sg.end();
  }
  // Geometric chunk schedule: 4, 8, 16, ... components (capped at p.chunk).
  // The rank rule stops at the first failing component, so small ranks never
  // pay for a full chunk; results do not depend on the schedule.
  auto chunk_len = [&](int c) {
    long long want = (long long)kFirstChunk << (c < 20 ? c : 20);
    if (want > p.chunk) want = p.chunk;
    return (int)want;
  };
  const int first = chunk_len(0) < B ? chunk_len(0) : B;
  {
    Stage sg(h, HYDE_STAGE_EIG, 1, st);
    CK(launch_noise_eig(G, n, B, p.ridge, first, 0, sigma, nullptr, nullptr, house, tri, W, U, L.ldwu, st,
                        h->eig_cl, EIG_LANCZOS));
    sg.end();
  }
  const bool lanczos = first < B && eig_lanczos_enabled();
  int rank = 0, chunks = 0;
  int k0 = 0, comps = 0;
  for (int c = 0;; ++c) {
    const int cl = chunk_len(c);
    const int cnt = (B - k0) < cl ? (B - k0) : cl;
    if (c > 0) {
      s = ensure_ebuf(h, (size_t)(k0 + cnt) * L.ldE * 4, (size_t)k0 * L.ldE * 4, st);
      if (s != HYDE_OK) return s;
      Stage sg(h, HYDE_STAGE_EIG, 1, st);
      // the first chunk may have come from Lanczos (no T, Q): form them now,
      // keeping the first chunk's W / U
      if (c == 1 && lanczos)
        CK(launch_noise_eig(G, n, B, p.ridge, first, 0, sigma, nullptr, nullptr, house, tri, W, U, L.ldwu, st,
                            h->eig_cl, EIG_RETRI));
      CK(launch_eigvec_more(tri, house, sigma, B, k0, cnt, nullptr, nullptr, W, U, L.ldwu, st));
      sg.end();
    }
    float* E = h->ebuf + (size_t)k0 * L.ldE;
    {
      Stage sg(h, HYDE_STAGE_PROJECT, 1, st);
      CK(launch_project(cube, n, B, W + k0, L.ldwu, cnt, E, L.ldE, st));
      sg.end();
    }
    {
      Stage sg(h, HYDE_STAGE_DWT, levels, st);
      CK(dwt_forward(L, ws, E, L.ldE, cnt, fb, st));
      sg.end();
    }
    {
      Stage sg(h, HYDE_STAGE_SURE, 1, st);
      // the rank decision of the chunk is made by the last SURE subband to finish
      CK(launch_sure(C, L.plan.n_coeffs, L.plan, cnt, p.flags & HYDE_KEEP_LL, (int*)(ws + L.kstar),
                     (float*)(ws + L.tstar), (double*)(ws + L.esub), rs, (unsigned*)(ws + L.surv), st, k0,
                     (double)L.plan.n_coeffs, B, (double*)(ws + L.epost), h->rs_host_dev));
      sg.end();
    }
    {
      // the deciding SURE thread also wrote the decision into the pinned host
      // mirror (mapped memory): an event after the kernel is all the host needs
      Stage sg(h, HYDE_STAGE_RANK, 0, st);
      if (!h->ev_rank) CK(cudaEventCreateWithFlags(&h->ev_rank, cudaEventDisableTiming));
      CK(cudaEventRecord(h->ev_rank, st));
      sg.end();
    }
    // The inverse DWT of the kept components and the reconstruction are
    // enqueued BEFORE the host reads the rank: both read r* from the device
    // rank state (no-ops while no failing component has been seen), so the GPU
    // never idles while the host round-trips the 16-byte decision.
    {
      Stage sg(h, HYDE_STAGE_IDWT, levels, st);
      CK(dwt_inverse(L, ws, C, E, L.ldE, cnt, fb, (const float*)(ws + L.tstar), st, rs, k0));
      sg.end();
    }
    {
      Stage sg(h, HYDE_STAGE_RECON, (k0 + cnt + 7) / 8, st);
      CK(launch_reconstruct(h->ebuf, L.ldE, n, B, U, L.ldwu, k0 + cnt, out, st, rs));
      sg.end();
    }
    CK(cudaEventSynchronize(h->ev_rank));
    ++chunks;
    comps += cnt;
    const RankState r = *h->rs_host;
    if (r.nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
    if (r.sure_overflow) return fail(h, HYDE_EMETHOD, "SURE survivor set exceeded its capacity");
    if (r.found) {
      rank = r.rank;
      break;
    }
    k0 += cnt;
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->rank = rank;
    info->levels = levels;
    info->chunks_run = chunks;
    info->nonfinite_input = 0;
    info->n_coeffs = (int)L.plan.n_coeffs;
    info->comps = comps;
  }
  return HYDE_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ E1
// Pixel-sharded single cube (BASELINE.json north_star: "the
// pixel-sharded Gram matrix is all-reduced (B x B); eigen-images or row tiles
// are distributed for the wavelet stage").  The collectives go through
// CommOps: NCCL (hyde_hyres_sharded) or caller callbacks
// (hyde_hyres_sharded_cb, used to emulate ranks on one GPU in the tests).
namespace {
struct P2p {
  int peer;
  void* buf;
  size_t bytes;
};
struct CommOps {
  int rank = 0, world = 1;
  virtual ~CommOps() {}
  virtual hyde_status allreduce_sum_f64(hyde_handle h, double* buf, size_t n, cudaStream_t st) = 0;
  // remote pairs only; between two ranks the i-th send matches the i-th recv
  virtual hyde_status sendrecv(hyde_handle h, const std::vector<P2p>& sends, const std::vector<P2p>& recvs,
                               cudaStream_t st) = 0;
};

struct NcclOps : CommOps {
  const NcclApi* api = nullptr;
  ncclComm_t comm = nullptr;
  hyde_status chk(hyde_handle h, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return HYDE_OK;
    return fail(h, HYDE_ENCCL, std::string(what) + ": " + api->GetErrorString(r));
  }
  hyde_status allreduce_sum_f64(hyde_handle h, double* buf, size_t n, cudaStream_t st) override {
    return chk(h, api->AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  hyde_status sendrecv(hyde_handle h, const std::vector<P2p>& sends, const std::vector<P2p>& recvs,
                       cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return HYDE_OK;
    hyde_status s = chk(h, api->GroupStart(), "ncclGroupStart");
    if (s != HYDE_OK) return s;
    for (const P2p& x : sends)
      if ((s = chk(h, api->Send(x.buf, x.bytes, ncclUint8, x.peer, comm, st), "ncclSend")) != HYDE_OK) break;
    if (s == HYDE_OK)
      for (const P2p& x : recvs)
        if ((s = chk(h, api->Recv(x.buf, x.bytes, ncclUint8, x.peer, comm, st), "ncclRecv")) != HYDE_OK) break;
    const hyde_status e = chk(h, api->GroupEnd(), "ncclGroupEnd");
    return s != HYDE_OK ? s : e;
  }
};

struct CbOps : CommOps {
  const hyde_comm* cb = nullptr;
  hyde_status allreduce_sum_f64(hyde_handle h, double* buf, size_t n, cudaStream_t st) override {
    return cb->allreduce_sum_f64(cb->user, buf, n, (hyde_stream_t)st) == 0
               ? HYDE_OK
               : fail(h, HYDE_ENCCL, "allreduce callback failed");
  }
  hyde_status sendrecv(hyde_handle h, const std::vector<P2p>& sends, const std::vector<P2p>& recvs,
                       cudaStream_t st) override {
    std::vector<hyde_p2p> a(sends.size()), b(recvs.size());
    for (size_t i = 0; i < sends.size(); ++i) a[i] = {sends[i].peer, sends[i].buf, sends[i].bytes};
    for (size_t i = 0; i < recvs.size(); ++i) b[i] = {recvs[i].peer, recvs[i].buf, recvs[i].bytes};
    return cb->sendrecv(cb->user, (int)a.size(), a.data(), (int)b.size(), b.data(), (hyde_stream_t)st) == 0
               ? HYDE_OK
               : fail(h, HYDE_ENCCL, "sendrecv callback failed");
  }
};

// one all-to-all step: self pairs become device copies (matched in order),
// the rest goes to the communicator as one group
hyde_status exchange(hyde_handle h, CommOps& cm, const std::vector<P2p>& sends, const std::vector<P2p>& recvs,
                     cudaStream_t st) {
  std::vector<P2p> rs, rr, ss, sr;
  for (const P2p& x : sends) (x.peer == cm.rank ? ss : rs).push_back(x);
  for (const P2p& x : recvs) (x.peer == cm.rank ? sr : rr).push_back(x);
  if (ss.size() != sr.size()) return fail(h, HYDE_EPARAM, "internal: unmatched self transfers");
  for (size_t i = 0; i < ss.size(); ++i) {
    if (ss[i].bytes != sr[i].bytes) return fail(h, HYDE_EPARAM, "internal: self transfer size");
    CK(cudaMemcpyAsync(sr[i].buf, ss[i].buf, ss[i].bytes, cudaMemcpyDeviceToDevice, st));
  }
  return cm.sendrecv(h, rs, rr, st);
}

hyde_status ensure_shard_buf(hyde_handle h, size_t bytes, cudaStream_t st) {
  if (bytes <= h->shard_cap) return HYDE_OK;
  if (h->shard_buf) CK(cudaFreeAsync(h->shard_buf, st));
  h->shard_buf = nullptr;
  h->shard_cap = 0;
  CK(cudaMallocAsync((void**)&h->shard_buf, bytes, st));
  h->shard_cap = bytes;
  return HYDE_OK;
}

hyde_status sharded_impl(hyde_handle h, CommOps& cm, const float* local, int local_rows, int row0, int rows, int cols,
                         int bands, float* local_out, const hyde_hyres_params* params, hyde_hyres_info* info,
                         cudaStream_t st) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!local || !local_out) return fail(h, HYDE_EPARAM, "NULL slab / output");
  const int G = cm.world, gr = cm.rank;
  if (G < 1 || gr < 0 || gr >= G || rows < G) return fail(h, HYDE_EPARAM, "bad rank / world");
  int r0c = 0, nrc = 0;
  hyde_shard_rows(rows, G, gr, &r0c, &nrc);
  if (row0 != r0c || local_rows != nrc)
    return fail(h, HYDE_EPARAM, "slab must be rows [rank*rows/world, (rank+1)*rows/world)");
  hyde_hyres_params p;
  int levels = 0;
  s = resolve_params(h, rows, cols, params, &p, &levels);
  if (s != HYDE_OK) return s;
  FilterBank fb;
  if (hyde_build_filters(p.wavelet_taps, &fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "filter derivation failed");
  DeviceGuard dg(h->device);
  const int B = bands;
  auto rbeg = [&](int g) {
    int a = 0, c = 0;
    hyde_shard_rows(rows, G, g, &a, &c);
    return a;
  };
  // chunk schedule: first max(4, G) components (every rank owns one), doubling
  const int first_len = std::min(p.chunk, std::max(kFirstChunk, G));
  auto chunk_len = [&](int c) {
    long long want = (long long)first_len << (c < 20 ? c : 20);
    if (want > p.chunk) want = p.chunk;
    return (int)want;
  };
  const int mycap = (p.chunk + G - 1) / G;   // components one rank owns in a chunk, at most
  Layout L;                                  // full-image geometry: this rank's DWT / SURE / IDWT
  make_layout(rows, cols, B, mycap, levels, p.wavelet_taps, &L);
  const long long n_loc = (long long)local_rows * cols;
  Layout Ll;                                 // slab geometry: the local Gram
  make_layout(local_rows, cols, B, 1, 1, 2, &Ll);
  s = ensure_ws(h, L.total + Ll.total, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  char* wl = h->ws + L.total;
  const long long n = L.n;
  // persistent exchange buffers (handle-owned, grow only): the projected slab
  // of every chunk component, this rank's whole eigen-images, the chunk's
  // per-subband SURE statistics (+ one overflow slot)
  const size_t b_slab = al((size_t)p.chunk * n_loc * 4), b_full = al((size_t)mycap * L.ldE * 4),
               b_esub = al(((size_t)p.chunk * L.nsub + 1) * 8);
  s = ensure_shard_buf(h, b_slab + b_full + b_esub, st);
  if (s != HYDE_OK) return s;
  float* slab_e = (float*)h->shard_buf;
  float* full_e = (float*)(h->shard_buf + b_slab);
  double* esub_all = (double*)(h->shard_buf + b_slab + b_full);
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  double* Gm = (double*)(ws + L.G);
  double* sigma = (double*)(ws + L.sigma);
  double* house = (double*)(ws + L.house);
  double* tri = (double*)(ws + L.tri);
  float* W = (float*)(ws + L.W);
  float* U = (float*)(ws + L.U);
  float* C = (float*)(ws + L.C);
  // ---- A1: local Gram of the slab, all-reduced; a global finiteness check ----
  {
    Stage sg(h, HYDE_STAGE_GRAM, Ll.use_tc ? gram_tc_launches() + 1 : 3, st);
    if (Ll.use_tc)
      CK(launch_gram_tc(local, n_loc, B, wl + Ll.partial, Ll.npairs, Gm, &rs->nonfinite, st));
    else
      CK(launch_gram(local, n_loc, B, (double*)(wl + Ll.partial), Ll.nsplit, Gm, &rs->nonfinite, st));
    s = cm.allreduce_sum_f64(h, Gm, (size_t)B * B, st);
    if (s != HYDE_OK) return s;
    CK(launch_check_finite(Gm, (long long)B * B, &rs->nonfinite, st));
    sg.end();
  }
  // ---- A2 (replicated: identical G, code and GPU type give identical V) ----
  const int first = chunk_len(0) < B ? chunk_len(0) : B;
  {
    Stage sg(h, HYDE_STAGE_EIG, 1, st);
    CK(launch_noise_eig(Gm, n, B, p.ridge, first, 0, sigma, nullptr, nullptr, house, tri, W, U, L.ldwu, st,
                        h->eig_cl, EIG_LANCZOS));
    sg.end();
  }
  const bool lanczos = first < B && eig_lanczos_enabled();
  int rank = 0, chunks = 0, k0 = 0, comps = 0;
  for (int c = 0;; ++c) {
    const int cl = chunk_len(c);
    const int cnt = (B - k0) < cl ? (B - k0) : cl;
    if (c > 0) {
      Stage sg(h, HYDE_STAGE_EIG, 1, st);
      if (c == 1 && lanczos)   // T and Q for the later chunks (the first chunk's W / U kept)
        CK(launch_noise_eig(Gm, n, B, p.ridge, first, 0, sigma, nullptr, nullptr, house, tri, W, U, L.ldwu, st,
                            h->eig_cl, EIG_RETRI));
      CK(launch_eigvec_more(tri, house, sigma, B, k0, cnt, nullptr, nullptr, W, U, L.ldwu, st));
      sg.end();
    }
    std::vector<int> mine;   // chunk positions of the components this rank owns (global k % G == rank)
    for (int k = 0; k < cnt; ++k)
      if (hyde_shard_owner(k0 + k, G) == gr) mine.push_back(k);
    const int my = (int)mine.size();
    {
      // A3 on the local slab, then slab -> whole eigen-images of the owned components
      Stage sg(h, HYDE_STAGE_PROJECT, 1, st);
      CK(launch_project(local, n_loc, B, W + k0, L.ldwu, cnt, slab_e, n_loc, st));
      std::vector<P2p> snd, rcv;
      for (int k = 0; k < cnt; ++k)
        snd.push_back({hyde_shard_owner(k0 + k, G), slab_e + (size_t)k * n_loc, (size_t)n_loc * 4});
      for (int j = 0; j < my; ++j)
        for (int g = 0; g < G; ++g)
          rcv.push_back({g, full_e + (size_t)j * L.ldE + (size_t)rbeg(g) * cols,
                         (size_t)(rbeg(g + 1) - rbeg(g)) * cols * 4});
      s = exchange(h, cm, snd, rcv, st);
      if (s != HYDE_OK) return s;
      sg.end();
    }
    if (my > 0) {
      Stage sg(h, HYDE_STAGE_DWT, levels, st);
      CK(dwt_forward(L, ws, full_e, L.ldE, my, fb, st));
      sg.end();
      Stage sg2(h, HYDE_STAGE_SURE, 1, st);
      CK(launch_sure(C, L.plan.n_coeffs, L.plan, my, p.flags & HYDE_KEEP_LL, (int*)(ws + L.kstar),
                     (float*)(ws + L.tstar), (double*)(ws + L.esub), rs, (unsigned*)(ws + L.surv), st));
      sg2.end();
    }
    {
      // every rank gets every component's subband statistics (its own rows,
      // zeros elsewhere, summed) and makes the same first-failure decision
      Stage sg(h, HYDE_STAGE_RANK, 3, st);
      CK(launch_scatter_rows((const double*)(ws + L.esub), my, L.nsub, mine.data(), esub_all, cnt,
                             &rs->sure_overflow, st));
      s = cm.allreduce_sum_f64(h, esub_all, (size_t)cnt * L.nsub + 1, st);
      if (s != HYDE_OK) return s;
      CK(launch_flag_from_sum(esub_all + (size_t)cnt * L.nsub, &rs->sure_overflow, st));
      CK(launch_rank_decide(esub_all, L.nsub, cnt, k0, (double)L.plan.n_coeffs, B, rs, (double*)(ws + L.epost), st));
      CK(cudaMemcpyAsync(h->rs_host, rs, sizeof(RankState), cudaMemcpyDeviceToHost, st));
      sg.end();
    }
    CK(cudaStreamSynchronize(st));
    ++chunks;
    comps += cnt;
    const RankState r = *h->rs_host;
    if (r.nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
    if (r.sure_overflow) return fail(h, HYDE_EMETHOD, "SURE survivor set exceeded its capacity");
    const int kept = r.found ? (r.rank - k0) : cnt;
    int my_kept = 0;
    while (my_kept < my && mine[my_kept] < kept) ++my_kept;
    if (my_kept > 0) {
      Stage sg(h, HYDE_STAGE_IDWT, levels, st);
      CK(dwt_inverse(L, ws, C, full_e, L.ldE, my_kept, fb, (const float*)(ws + L.tstar), st));
      sg.end();
    }
    s = ensure_ebuf(h, (size_t)(k0 + cnt) * n_loc * 4, (size_t)k0 * n_loc * 4, st);
    if (s != HYDE_OK) return s;
    if (kept > 0) {
      // whole denoised images -> the rows of every rank's slab
      Stage sg(h, HYDE_STAGE_IDWT, 0, st);
      std::vector<P2p> snd, rcv;
      for (int j = 0; j < my_kept; ++j)
        for (int g = 0; g < G; ++g)
          snd.push_back({g, full_e + (size_t)j * L.ldE + (size_t)rbeg(g) * cols,
                         (size_t)(rbeg(g + 1) - rbeg(g)) * cols * 4});
      for (int k = 0; k < kept; ++k)
        rcv.push_back({hyde_shard_owner(k0 + k, G), h->ebuf + (size_t)(k0 + k) * n_loc, (size_t)n_loc * 4});
      s = exchange(h, cm, snd, rcv, st);
      if (s != HYDE_OK) return s;
      sg.end();
    }
    if (r.found) {
      rank = r.rank;
      break;
    }
    k0 += cnt;
  }
  {
    // A6 on the local rows only
    Stage sg(h, HYDE_STAGE_RECON, (rank + 7) / 8, st);
    CK(launch_reconstruct(h->ebuf, n_loc, n_loc, B, U, L.ldwu, rank, local_out, st));
    sg.end();
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->rank = rank;
    info->levels = levels;
    info->chunks_run = chunks;
    info->n_coeffs = (int)L.plan.n_coeffs;
    info->comps = comps;
  }
  return HYDE_OK;
}
}  // namespace

extern "C" {

int hyde_shard_rows(int rows, int world, int rank, int* row0, int* nrows) {
  if (world < 1 || rank < 0 || rank > world || rows < 0) return -1;
  const long long a = (long long)rank * rows / world;
  const long long b = rank < world ? (long long)(rank + 1) * rows / world : rows;
  if (row0) *row0 = (int)a;
  if (nrows) *nrows = (int)(b - a);
  return 0;
}

int hyde_shard_owner(int component, int world) { return world < 1 || component < 0 ? -1 : component % world; }

int hyde_nccl_version(void) {
  const NcclApi* a = nccl_api();
  int v = 0;
  if (!a || a->GetVersion(&v) != ncclSuccess) return 0;
  return v;
}

hyde_status hyde_nccl_unique_id(void* id_out) {
  const NcclApi* a = nccl_api();
  if (!id_out) return HYDE_EPARAM;
  if (!a) {
    g_err = "libnccl.so.2 not found";
    return HYDE_ENCCL;
  }
  ncclUniqueId id;
  const ncclResult_t r = a->GetUniqueId(&id);
  if (r != ncclSuccess) {
    g_err = std::string("ncclGetUniqueId: ") + a->GetErrorString(r);
    return HYDE_ENCCL;
  }
  memcpy(id_out, &id, sizeof(id));
  return HYDE_OK;
}

hyde_status hyde_nccl_comm_init(ncclComm_t* comm, int world, int rank, const void* id, int device) {
  const NcclApi* a = nccl_api();
  if (!comm || !id || world < 1 || rank < 0 || rank >= world) return HYDE_EPARAM;
  if (!a) {
    g_err = "libnccl.so.2 not found";
    return HYDE_ENCCL;
  }
  DeviceGuard g(device);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  const ncclResult_t r = a->CommInitRank(comm, world, uid, rank);
  if (r != ncclSuccess) {
    g_err = std::string("ncclCommInitRank: ") + a->GetErrorString(r);
    return HYDE_ENCCL;
  }
  return HYDE_OK;
}

hyde_status hyde_nccl_comm_destroy(ncclComm_t comm) {
  const NcclApi* a = nccl_api();
  if (!comm) return HYDE_OK;
  if (!a) return HYDE_ENCCL;
  return a->CommDestroy(comm) == ncclSuccess ? HYDE_OK : HYDE_ENCCL;
}

hyde_status hyde_hyres_sharded(hyde_handle h, ncclComm_t comm, const float* local, int local_rows, int row0, int rows,
                               int cols, int bands, float* local_out, const hyde_hyres_params* params,
                               hyde_hyres_info* info, hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  if (!comm) return fail(h, HYDE_EPARAM, "NULL communicator");
  NcclOps ops;
  ops.api = nccl_api();
  if (!ops.api) return fail(h, HYDE_ENCCL, "libnccl.so.2 not found");
  ops.comm = comm;
  if (ops.api->CommCount(comm, &ops.world) != ncclSuccess || ops.api->CommUserRank(comm, &ops.rank) != ncclSuccess)
    return fail(h, HYDE_ENCCL, "bad communicator");
  return sharded_impl(h, ops, local, local_rows, row0, rows, cols, bands, local_out, params, info,
                      (cudaStream_t)stream);
}

hyde_status hyde_hyres_sharded_cb(hyde_handle h, const hyde_comm* comm, const float* local, int local_rows, int row0,
                                  int rows, int cols, int bands, float* local_out, const hyde_hyres_params* params,
                                  hyde_hyres_info* info, hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  if (!comm || !comm->allreduce_sum_f64 || !comm->sendrecv) return fail(h, HYDE_EPARAM, "NULL collective callbacks");
  CbOps ops;
  ops.cb = comm;
  ops.rank = comm->rank;
  ops.world = comm->world;
  return sharded_impl(h, ops, local, local_rows, row0, rows, cols, bands, local_out, params, info,
                      (cudaStream_t)stream);
}

hyde_status hyde_profile_enable(hyde_handle h, int on) {
  if (!h) return HYDE_EPARAM;
  DeviceGuard g(h->device);
  CK(cudaDeviceSynchronize());
  for (auto& r : h->recs) { h->pool.push_back(r.a); h->pool.push_back(r.b); }
  h->recs.clear();
  h->prof = on ? 1 : 0;
  return HYDE_OK;
}

hyde_status hyde_profile_read(hyde_handle h, double* ms, long long* launches) {
  if (!h || !ms) return HYDE_EPARAM;
  DeviceGuard g(h->device);
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < HYDE_NSTAGES; ++i) { ms[i] = 0.0; if (launches) launches[i] = 0; }
  for (auto& r : h->recs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.stage] += t;
    if (launches) launches[r.stage] += r.launches;
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
  return HYDE_OK;
}

long long hyde_launch_count(hyde_handle h) { return h ? h->launch_total : 0; }

hyde_status hyde_hyres(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out,
                       hyde_stream_t stream) {
  return hyde_hyres_ex(h, cube, rows, cols, bands, out, nullptr, nullptr, stream);
}

constexpr int kLanesDefault = 16;  // concurrent cubes in hyde_hyres_batched (8-CTA K2 clusters: 5.9 vs 7.3 ms for 64 x 256x256x191 with 8 lanes of 16-CTA K2)
constexpr int kLaneGramMinPx = 8192;   // K1 pixels per SM pair in the lanes (64 K1 stages)
static int lanes_wanted() {
  if (const char* ev = getenv("HYDE_LANES")) {   // experiments
    const int v = atoi(ev);
    if (v >= 1 && v <= 32) return v;
  }
  return kLanesDefault;
}

// Phased batched HyRes (the default of hyde_hyres_batched): the cubes go
// through the stages TOGETHER -- every Gram (on the lane streams), then ONE
// launch of the K2 eigensolver for all cubes (cluster b = cube b: the hardware
// packs the latency-bound solvers back to back on the GPU), then the first
// chunk of every cube (projection, DWT, SURE with the in-kernel rank decision,
// gated IDWT and reconstruction) -- with a single host synchronisation for the
// whole batch.  A cube whose rank rule needs a second chunk (r* >= the first
// chunk) is redone on its own through hyde_hyres_ex.  Every output equals the
// single-cube result (the Gram is exact in integers whatever the pixel split,
// and K2 does not depend on its cluster size).
static hyde_status batched_phased(hyde_handle h, const float* cubes, int batch, int rows, int cols, int bands,
                                  float* outs, const hyde_hyres_params* params, hyde_hyres_info* info,
                                  cudaStream_t st) {
  hyde_hyres_params p;
  int levels = 0;
  hyde_status s = resolve_params(h, rows, cols, params, &p, &levels);
  if (s != HYDE_OK) return s;
  FilterBank fb;
  if (hyde_build_filters(p.wavelet_taps, &fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "filter derivation failed");
  const int B = bands;
  Layout L;
  static const int lane_px = [] {
    const char* ev = getenv("HYDE_LANE_GRAM_PX");   // experiments
    return ev ? atoi(ev) : kLaneGramMinPx;
  }();
  make_layout(rows, cols, B, p.chunk, levels, p.wavelet_taps, &L, lane_px);
  const long long n = L.n;
  const size_t per = (size_t)rows * cols * bands;
  const int first = std::min(std::min(kFirstChunk, p.chunk), B);
  const size_t per_ws = al(L.total), per_e = al((size_t)first * L.ldE * 4);
  const size_t args_b = al((size_t)batch * eig_args_bytes());
  const size_t jobs_b = al((size_t)batch * gram_job_bytes());
  const size_t need = (size_t)batch * (per_ws + per_e) + args_b + jobs_b;
  if (need > h->bws_cap) {
    if (h->bws) CK(cudaFreeAsync(h->bws, st));
    h->bws = nullptr;
    h->bws_cap = 0;
    CK(cudaMallocAsync((void**)&h->bws, need, st));
    h->bws_cap = need;
  }
  if (batch > h->b_cap) {
    CK(cudaStreamSynchronize(st));
    if (h->b_rs_host) CK(cudaFreeHost(h->b_rs_host));
    if (h->b_args_host) CK(cudaFreeHost(h->b_args_host));
    if (h->b_jobs_host) CK(cudaFreeHost(h->b_jobs_host));
    h->b_rs_host = nullptr;
    h->b_args_host = nullptr;
    h->b_jobs_host = nullptr;
    h->b_cap = 0;
    CK(cudaHostAlloc((void**)&h->b_rs_host, sizeof(RankState) * batch, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer((void**)&h->b_rs_dev, h->b_rs_host, 0));
    CK(cudaHostAlloc(&h->b_args_host, (size_t)batch * eig_args_bytes(), cudaHostAllocPortable));
    CK(cudaHostAlloc(&h->b_jobs_host, (size_t)batch * gram_job_bytes(), cudaHostAllocPortable));
    h->b_cap = batch;
  }
  const int NS = std::min(batch, lanes_wanted());
  while ((int)h->lane_st.size() < NS) {
    cudaStream_t ls = nullptr;
    CK(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
    h->lane_st.push_back(ls);
    cudaEvent_t le = nullptr;
    CK(cudaEventCreateWithFlags(&le, cudaEventDisableTiming));
    h->lane_ev.push_back(le);
  }
  if (!h->ev_batch) CK(cudaEventCreateWithFlags(&h->ev_batch, cudaEventDisableTiming));
  auto ws_of = [&](int i) { return h->bws + (size_t)i * (per_ws + per_e); };
  auto e_of = [&](int i) { return (float*)(ws_of(i) + per_ws); };
  auto join_lanes = [&]() -> hyde_status {   // st waits for every lane stream
    for (int j = 0; j < NS; ++j) {
      CK(cudaEventRecord(h->lane_ev[j], h->lane_st[j]));
      CK(cudaStreamWaitEvent(st, h->lane_ev[j], 0));
    }
    return HYDE_OK;
  };
  auto fork_lanes = [&]() -> hyde_status {   // every lane stream waits for st
    CK(cudaEventRecord(h->ev_batch, st));
    for (int j = 0; j < NS; ++j) CK(cudaStreamWaitEvent(h->lane_st[j], h->ev_batch, 0));
    return HYDE_OK;
  };
  memset(h->b_rs_host, 0, sizeof(RankState) * batch);
  if (p.flags & HYDE_VALIDATE) {
    RankState* rs0 = (RankState*)(ws_of(0) + L.rs);
    CK(cudaMemsetAsync(rs0, 0, sizeof(RankState), st));
    CK(launch_check_finite_f32(cubes, (long long)per * batch, &rs0->nonfinite, st));
    CK(cudaMemcpyAsync(&h->rs_host->nonfinite, &rs0->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h->rs_host->nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
  }
  s = fork_lanes();
  if (s != HYDE_OK) return s;
  // ---- A1 for every cube: five launches for the whole batch ----
  if (L.use_tc) {
    Stage sg(h, HYDE_STAGE_GRAM, gram_tc_launches(), st);
    std::vector<const float*> Y(batch);
    std::vector<void*> W(batch);
    std::vector<double*> G(batch), Z(batch);
    std::vector<int*> NF(batch), S4(batch);
    for (int i = 0; i < batch; ++i) {
      char* ws = ws_of(i);
      RankState* rs = (RankState*)(ws + L.rs);
      Y[i] = cubes + per * i;
      W[i] = ws + L.partial;
      G[i] = (double*)(ws + L.G);
      NF[i] = &rs->nonfinite;
      S4[i] = (int*)rs;
      Z[i] = eig_flags_ptr((double*)(ws + L.house), B);
    }
    CK(launch_gram_tc_batched(batch, Y.data(), W.data(), G.data(), NF.data(), S4.data(), Z.data(), n, B, L.npairs,
                              h->b_jobs_host, h->bws + (size_t)batch * (per_ws + per_e) + args_b, st));
    sg.end();
  } else {
    Stage sg(h, HYDE_STAGE_GRAM, batch * 2, st);
    for (int i = 0; i < batch; ++i) {
      cudaStream_t ls = h->lane_st[i % NS];
      char* ws = ws_of(i);
      RankState* rs = (RankState*)(ws + L.rs);
      if (!L.use_tc) CK(cudaMemsetAsync(rs, 0, sizeof(RankState), ls));
      CK(run_gram(L, ws, cubes + per * i, (double*)(ws + L.G), &rs->nonfinite, ls, L.use_tc ? (int*)rs : nullptr));
      CK(cudaMemsetAsync(eig_flags_ptr((double*)(ws + L.house), B), 0, 8 * sizeof(double), ls));
    }
    s = join_lanes();
    if (s != HYDE_OK) return s;
    sg.end();
  }
  // ---- A1 tail + A2: the eigensolvers, one launch per group of cubes ----
  // The solves are latency-bound 8-SM clusters (up to 18 at once): the last,
  // partial wave of one launch for the whole batch leaves SMs idle.  With two
  // groups the second group's solves overlap the first group's chunk phase on
  // the lane streams.  HYDE_BATCH_SPLIT = cubes in the first group (0: one launch;
  // experiments).
  static const int split_env = [] {
    const char* ev = getenv("HYDE_BATCH_SPLIT");
    return ev ? atoi(ev) : -1;
  }();
  // default: two full waves of 8-SM clusters in the first launch (36 on a
  // 148-SM B200: 64 cubes 4.99 -> 4.92 ms; 18 or 27 measured no better)
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device);
  const int two_waves = 2 * (nsm / 8);
  const int sA = split_env >= 0 ? (split_env == 0 || split_env >= batch ? batch : split_env)
                                : (batch > two_waves ? two_waves : batch);
  auto eig_group = [&](int i0, int i1) -> hyde_status {
    const int nbg = i1 - i0;
    std::vector<const double*> G(nbg);
    std::vector<double*> sig(nbg), house(nbg), tri(nbg);
    std::vector<float*> W(nbg), U(nbg);
    for (int i = i0; i < i1; ++i) {
      char* ws = ws_of(i);
      G[i - i0] = (const double*)(ws + L.G);
      sig[i - i0] = (double*)(ws + L.sigma);
      house[i - i0] = (double*)(ws + L.house);
      tri[i - i0] = (double*)(ws + L.tri);
      W[i - i0] = (float*)(ws + L.W);
      U[i - i0] = (float*)(ws + L.U);
    }
    char* hargs = (char*)h->b_args_host + (size_t)i0 * eig_args_bytes();
    char* dargs = h->bws + (size_t)batch * (per_ws + per_e) + (size_t)i0 * eig_args_bytes();
    CK(launch_noise_eig_batched(nbg, G.data(), n, B, p.ridge, first, sig.data(), house.data(), tri.data(),
                                W.data(), U.data(), L.ldwu, hargs, dargs, st, h->eig_cl ? h->eig_cl : 8));
    return HYDE_OK;
  };
  // ---- A3..A6, first chunk of every cube (decision and gating on the device) ----
  auto chunk_group = [&](int i0, int i1) -> hyde_status {
    for (int i = i0; i < i1; ++i) {
      cudaStream_t ls = h->lane_st[i % NS];
      char* ws = ws_of(i);
      RankState* rs = (RankState*)(ws + L.rs);
      float* E = e_of(i);
      float* C = (float*)(ws + L.C);
      CK(launch_project(cubes + per * i, n, B, (float*)(ws + L.W), L.ldwu, first, E, L.ldE, ls));
      CK(dwt_forward(L, ws, E, L.ldE, first, fb, ls));
      CK(launch_sure(C, L.plan.n_coeffs, L.plan, first, p.flags & HYDE_KEEP_LL, (int*)(ws + L.kstar),
                     (float*)(ws + L.tstar), (double*)(ws + L.esub), rs, (unsigned*)(ws + L.surv), ls, 0,
                     (double)L.plan.n_coeffs, B, (double*)(ws + L.epost), h->b_rs_dev + i));
      CK(dwt_inverse(L, ws, C, E, L.ldE, first, fb, (const float*)(ws + L.tstar), ls, rs, 0));
      CK(launch_reconstruct(E, L.ldE, n, B, (float*)(ws + L.U), L.ldwu, first, outs + per * i, ls, rs));
    }
    return HYDE_OK;
  };
  {
    Stage sg(h, HYDE_STAGE_EIG, sA < batch ? 2 : 1, st);
    s = eig_group(0, sA);
    if (s != HYDE_OK) return s;
    s = fork_lanes();                       // the first group's chunks may start
    if (s != HYDE_OK) return s;
    if (sA < batch) {
      s = eig_group(sA, batch);
      if (s != HYDE_OK) return s;
    }
    sg.end();
  }
  {
    Stage sg(h, HYDE_STAGE_SURE, batch * (3 + 2 * levels), st);
    s = chunk_group(0, sA);
    if (s != HYDE_OK) return s;
    if (sA < batch) {
      s = fork_lanes();                     // after the second group's solves
      if (s != HYDE_OK) return s;
      s = chunk_group(sA, batch);
      if (s != HYDE_OK) return s;
    }
    s = join_lanes();
    if (s != HYDE_OK) return s;
    sg.end();
  }
  CK(cudaStreamSynchronize(st));
  hyde_hyres_info* inf = info;
  for (int i = 0; i < batch; ++i) {
    const RankState r = h->b_rs_host[i];
    if (r.nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
    if (r.sure_overflow) return fail(h, HYDE_EMETHOD, "SURE survivor set exceeded its capacity");
    if (!r.found) {
      // r* >= the first chunk: this cube alone through the chunked rank walk
      s = hyde_hyres_ex(h, cubes + per * i, rows, cols, bands, outs + per * i, params, inf ? inf + i : nullptr,
                        (hyde_stream_t)st);
      if (s != HYDE_OK) return s;
      continue;
    }
    if (inf) {
      memset(inf + i, 0, sizeof(*inf));
      inf[i].rank = r.rank;
      inf[i].levels = levels;
      inf[i].chunks_run = 1;
      inf[i].n_coeffs = (int)L.plan.n_coeffs;
      inf[i].comps = first;
    }
  }
  return HYDE_OK;
}

hyde_status hyde_hyres_batched(hyde_handle h, const float* cubes, int batch, int rows, int cols, int bands,
                               float* outs, const hyde_hyres_params* params, hyde_hyres_info* info,
                               hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  if (batch < 0 || (batch > 0 && (!cubes || !outs))) return fail(h, HYDE_EPARAM, "bad batch arguments");
  const size_t per = (size_t)rows * cols * bands;
  if (batch <= 1) {
    for (int i = 0; i < batch; ++i) {
      hyde_status s = hyde_hyres_ex(h, cubes + per * i, rows, cols, bands, outs + per * i, params,
                                    info ? info + i : nullptr, stream);
      if (s != HYDE_OK) return s;
    }
    return HYDE_OK;
  }
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!getenv("HYDE_BATCH_LANES")) {   // HYDE_BATCH_LANES=1: the older per-lane path (experiments)
    DeviceGuard g(h->device);
    return batched_phased(h, cubes, batch, rows, cols, bands, outs, params, info, (cudaStream_t)stream);
  }
  // Independent cubes run on kLanes lanes -- each its own workspace, stream and
  // host thread (hyres_ex synchronises its stream once per rank-loop chunk) --
  // so that, e.g., one cube's K2 cluster (16 SMs) overlaps another cube's
  // HBM-bound stages.  Cube i runs on lane i % kLanes; every output is the one
  // hyde_hyres_ex gives for that cube alone.
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int kLanes = lanes_wanted();
  const int L = batch < kLanes ? batch : kLanes;
  while ((int)h->lanes.size() < L) {
    hyde_handle l = nullptr;
    s = hyde_create(&l, h->device);
    if (s != HYDE_OK) return s;
    l->gram_min_px = kLaneGramMinPx;   // throughput mode: concurrent cubes share the SMs
    if (const char* ev = getenv("HYDE_LANE_GRAM_PX")) l->gram_min_px = atoi(ev);   // experiments
    l->eig_cl = 8;                     // more concurrent eigensolvers (fewer SMs each)
    if (const char* ev = getenv("HYDE_LANE_EIG_CL")) l->eig_cl = atoi(ev);        // experiments (16 = latency)
    h->lanes.push_back(l);
    cudaStream_t ls = nullptr;
    CK(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
    h->lane_st.push_back(ls);
    cudaEvent_t le = nullptr;
    CK(cudaEventCreateWithFlags(&le, cudaEventDisableTiming));
    h->lane_ev.push_back(le);
  }
  if (!h->ev_batch) CK(cudaEventCreateWithFlags(&h->ev_batch, cudaEventDisableTiming));
  CK(cudaEventRecord(h->ev_batch, st));   // the cubes are ready on the caller's stream
  std::vector<hyde_status> res(L, HYDE_OK);
  std::vector<std::thread> th;
  for (int j = 0; j < L; ++j) {
    hyde_ctx* lh = h->lanes[j];
    lh->prof = h->prof;
    th.emplace_back([&, j, lh]() {
      cudaSetDevice(h->device);
      cudaStream_t ls = h->lane_st[j];
      if (cudaStreamWaitEvent(ls, h->ev_batch, 0) != cudaSuccess) {
        res[j] = HYDE_ECUDA;
        return;
      }
      for (int i = j; i < batch; i += L) {
        const hyde_status r = hyde_hyres_ex(lh, cubes + per * i, rows, cols, bands, outs + per * i, params,
                                            info ? info + i : nullptr, (hyde_stream_t)ls);
        if (r != HYDE_OK) {
          res[j] = r;
          return;
        }
      }
      if (cudaEventRecord(h->lane_ev[j], ls) != cudaSuccess) res[j] = HYDE_ECUDA;
    });
  }
  for (auto& t : th) t.join();
  // Every lane is ordered before the caller's stream moves on -- also when one
  // failed: a failed lane (no event recorded) is drained on the host, so no
  // lane kernel can still write `outs` after this call returns an error.
  int first_bad = -1;
  for (int j = 0; j < L; ++j) {
    hyde_ctx* lh = h->lanes[j];
    h->launch_total += lh->launch_total;
    for (int k = 0; k < HYDE_NSTAGES; ++k) h->launch_by_stage[k] += lh->launch_by_stage[k];
    lh->launch_total = 0;
    for (int k = 0; k < HYDE_NSTAGES; ++k) lh->launch_by_stage[k] = 0;
    for (auto& r : lh->recs) h->recs.push_back(r);   // stage time summed over lanes (busy time)
    lh->recs.clear();
    if (res[j] != HYDE_OK) {
      cudaStreamSynchronize(h->lane_st[j]);
      if (first_bad < 0) first_bad = j;
    } else {
      CK(cudaStreamWaitEvent(st, h->lane_ev[j], 0));
    }
  }
  if (first_bad >= 0) {
    hyde_ctx* lh = h->lanes[first_bad];
    return fail(h, res[first_bad], lh->err.empty() ? "batched lane failed" : lh->err);
  }
  return HYDE_OK;
}

hyde_status hyde_hyres_host(hyde_handle h, const float* cube_host, int rows, int cols, int bands,
                            float* out_host, const hyde_hyres_params* params, hyde_hyres_info* info,
                            hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!cube_host || !out_host) return fail(h, HYDE_EPARAM, "NULL host buffers");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (bytes > h->dev_io_cap) {
    if (h->dev_in) CK(cudaFreeAsync(h->dev_in, st));
    if (h->dev_out) CK(cudaFreeAsync(h->dev_out, st));
    h->dev_in = h->dev_out = nullptr;
    h->dev_io_cap = 0;
    CK(cudaMallocAsync((void**)&h->dev_in, bytes, st));
    CK(cudaMallocAsync((void**)&h->dev_out, bytes, st));
    h->dev_io_cap = bytes;
  }
  CK(cudaMemcpyAsync(h->dev_in, cube_host, bytes, cudaMemcpyHostToDevice, st));
  s = hyde_hyres_ex(h, h->dev_in, rows, cols, bands, h->dev_out, params, info, stream);
  if (s != HYDE_OK) return s;
  CK(cudaMemcpyAsync(out_host, h->dev_out, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return HYDE_OK;
}

hyde_status hyde_hyres_host_stream(hyde_handle h, const float* const* cubes_host, float* const* outs_host, int n,
                                   int rows, int cols, int bands, const hyde_hyres_params* params,
                                   hyde_hyres_info* info, hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (n < 0 || (n > 0 && (!cubes_host || !outs_host))) return fail(h, HYDE_EPARAM, "bad stream arguments");
  for (int i = 0; i < n; ++i)
    if (!cubes_host[i] || !outs_host[i]) return fail(h, HYDE_EPARAM, "NULL host buffer");
  if (n == 0) return HYDE_OK;
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (!h->s_in) {
    CK(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming));
    }
  }
  if (bytes > h->pipe_cap) {
    CK(cudaDeviceSynchronize());
    for (auto& b : h->pipe_buf) {
      if (b) CK(cudaFree(b));
      b = nullptr;
    }
    h->pipe_cap = 0;
    for (auto& b : h->pipe_buf) CK(cudaMalloc((void**)&b, bytes));
    h->pipe_cap = bytes;
  }
  // slot j: input pipe_buf[j], output pipe_buf[2 + j].  Order per cube i (slot j = i & 1):
  //   s_in : wait ev_done[j] (cube i-2 consumed slot j's input) -> H2D -> ev_in[j]
  //   st   : wait ev_in[j], wait ev_out[j] (cube i-2's result copied out) -> hyres -> ev_done[j]
  //   s_out: wait ev_done[j] -> D2H -> ev_out[j]
  auto h2d = [&](int i) -> hyde_status {
    const int j = i & 1;
    if (i >= 2) CK(cudaStreamWaitEvent(h->s_in, h->ev_done[j], 0));
    CK(cudaMemcpyAsync(h->pipe_buf[j], cubes_host[i], bytes, cudaMemcpyHostToDevice, h->s_in));
    CK(cudaEventRecord(h->ev_in[j], h->s_in));
    return HYDE_OK;
  };
  s = h2d(0);
  if (s != HYDE_OK) return s;
  for (int i = 0; i < n; ++i) {
    const int j = i & 1;
    if (i + 1 < n) {
      s = h2d(i + 1);   // next cube's copy overlaps this cube's compute
      if (s != HYDE_OK) return s;
    }
    CK(cudaStreamWaitEvent(st, h->ev_in[j], 0));
    if (i >= 2) CK(cudaStreamWaitEvent(st, h->ev_out[j], 0));
    s = hyde_hyres_ex(h, h->pipe_buf[j], rows, cols, bands, h->pipe_buf[2 + j], params, info ? info + i : nullptr,
                      stream);
    if (s != HYDE_OK) return s;
    CK(cudaEventRecord(h->ev_done[j], st));
    CK(cudaStreamWaitEvent(h->s_out, h->ev_done[j], 0));
    CK(cudaMemcpyAsync(outs_host[i], h->pipe_buf[2 + j], bytes, cudaMemcpyDeviceToHost, h->s_out));
    CK(cudaEventRecord(h->ev_out[j], h->s_out));
  }
  CK(cudaStreamSynchronize(h->s_out));
  CK(cudaStreamSynchronize(st));
  return HYDE_OK;
}

hyde_status hyde_estimate_noise(hyde_handle h, const float* cube, int rows, int cols, int bands,
                                double* sigma_out, double* gram_out, float* noise_out,
                                hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!cube || !sigma_out) return fail(h, HYDE_EPARAM, "NULL cube/sigma_out");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  make_layout(rows, cols, bands, 1, 1, 2, &L);
  s = ensure_ws(h, L.total, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  double* G = gram_out ? gram_out : (double*)(ws + L.G);
  CK(run_gram(L, ws, cube, G, &rs->nonfinite, st));
  CK(launch_noise_eig(G, L.n, bands, 1e-6, -1, 0, sigma_out, nullptr, nullptr, (double*)(ws + L.house),
                      (double*)(ws + L.tri), (float*)(ws + L.W), (float*)(ws + L.U), L.ldwu, st));
  if (noise_out)
    CK(launch_noise_residual(cube, L.n, bands, G, 1e-6, (double*)(ws + L.house), noise_out, st));
  return HYDE_OK;
}

// ---------------------------------------------------------------- stages
hyde_status hyde_l1_spectral(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out, double lambda,
                             double mu, int max_iters, double tol, int* iters, hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  if (!cube || !out) return fail(h, HYDE_EPARAM, "NULL cube/out");
  if (bands < 2 || bands > 256 || rows < 1 || cols < 1) return fail(h, HYDE_EPARAM, "bands in [2, 256]");
  if (!(lambda > 0.0) || !(mu > 0.0)) return fail(h, HYDE_EPARAM, "lambda, mu > 0 required (SPEC.md:420)");
  if (max_iters < 1 || !(tol >= 0.0)) return fail(h, HYDE_EPARAM, "max_iters >= 1, tol >= 0");
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (cube != out && overlap(cube, bytes, out, bytes)) return fail(h, HYDE_EPARAM, "cube and out partially overlap");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = (long long)rows * cols;
  hyde_status s = ensure_ws(h, l1spec_ws_bytes(n), st);   // per-tile continue masks
  if (s != HYDE_OK) return s;
  const float* M = cube;
  if (cube == out) {   // in place: the stage streams its output over its input, so keep m aside
    if (bytes > h->cubebuf_cap) {
      if (h->cubebuf) CK(cudaFreeAsync(h->cubebuf, st));
      h->cubebuf = nullptr;
      h->cubebuf_cap = 0;
      CK(cudaMallocAsync((void**)&h->cubebuf, bytes, st));
      h->cubebuf_cap = bytes;
    }
    if (h->cubebuf != cube) CK(cudaMemcpyAsync(h->cubebuf, cube, bytes, cudaMemcpyDeviceToDevice, st));
    M = h->cubebuf;
  }
  CK(launch_l1spec(M, out, n, bands, (float)lambda, (float)mu, max_iters, (float)tol, iters, h->ws, st));
  return HYDE_OK;
}

hyde_status hyde_hyminor(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out, double lambda,
                         double mu, int max_iters, double tol, hyde_hyres_info* info, hyde_stream_t stream) {
  if (lambda == 0.0) lambda = 10.0;   // D19 defaults
  if (mu == 0.0) mu = 5.0;
  if (max_iters <= 0) max_iters = 50;
  if (tol < 0.0) tol = 1e-3;
  if (!(lambda > 0.0) || !(mu > 0.0)) return fail(h, HYDE_EPARAM, "lambda, mu > 0 required (SPEC.md:420)");
  // HyRes into the handle's cube buffer, then the l1 stage from it into out
  // (no in-place pass: the l1 stage reads its input once more than it writes)
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (validate_shape(h, rows, cols, bands) == HYDE_OK && bytes > h->cubebuf_cap) {
    DeviceGuard g(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (h->cubebuf) CK(cudaFreeAsync(h->cubebuf, st));
    h->cubebuf = nullptr;
    h->cubebuf_cap = 0;
    CK(cudaMallocAsync((void**)&h->cubebuf, bytes, st));
    h->cubebuf_cap = bytes;
  }
  hyde_status s = hyde_hyres_ex(h, cube, rows, cols, bands, h->cubebuf, nullptr, info, stream);
  if (s != HYDE_OK) return s;
  return hyde_l1_spectral(h, h->cubebuf, rows, cols, bands, out, lambda, mu, max_iters, tol, nullptr, stream);
}

hyde_status hyde_wsrrr(hyde_handle h, const float* cube, int rows, int cols, int bands, int rank, double lambda,
                       int taps, int levels, int max_iters, double tol, float* out, float* components,
                       int* rank_out, double* lambda_out, int* sweeps_out, double* objective_out,
                       hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!cube || !out) return fail(h, HYDE_EPARAM, "NULL cube/out");
  if (rank < 0 || rank > bands || rank > HYDE_MAX_CHUNK) return fail(h, HYDE_EPARAM, "rank must be in [0, min(bands, 32)] (SPEC.md:401)");
  if (max_iters < 1) max_iters = 20;
  if (!(tol >= 0.0)) tol = 1e-4;
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (cube != out && overlap(cube, bytes, out, bytes)) return fail(h, HYDE_EPARAM, "cube and out partially overlap");
  if (rank == 0) {   // D17: default rank = HySime's k (at least 1)
    int k = 0;
    s = hyde_hysime(h, cube, rows, cols, bands, &k, nullptr, nullptr, nullptr, nullptr, stream);
    if (s != HYDE_OK) return s;
    rank = k < 1 ? 1 : (k > HYDE_MAX_CHUNK ? HYDE_MAX_CHUNK : k);
  }
  hyde_hyres_params pin;
  hyde_hyres_params_default(&pin);
  pin.wavelet_taps = taps;
  pin.levels = levels;
  hyde_hyres_params p;
  int lv = 0;
  s = resolve_params(h, rows, cols, &pin, &p, &lv);
  if (s != HYDE_OK) return s;
  FilterBank fb;
  if (hyde_build_filters(p.wavelet_taps, &fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "filter derivation failed");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int B = bands, r = rank;
  Layout L;
  make_layout(rows, cols, B, B, lv, p.wavelet_taps, &L);
  const size_t BB = (size_t)B * B;
  const long long nc = L.plan.n_coeffs, n = L.n;
  size_t off = L.total;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  const size_t oGw = take(BB * 8), oV = take(BB * 8), oM = take(BB * 8), oLam = take((size_t)B * 8),
               oOnes = take((size_t)B * 8), oScal = take(16 * 8), oPart = take(2048 * 8),
               oWtc = take((size_t)wtc_chunks(nc, r) * B * r * 8), oObj = take((size_t)max_iters * 8);
  const int np2 = gram_tc_npairs(nc);
  const int ns2 = gram_nsplit(nc, B);
  const size_t oGp = take(std::max((size_t)ns2 * BB * 8, gram_tc_supported(B) ? gram_tc_ws_bytes(nc, B, np2) : 0));
  s = ensure_ws(h, off, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  float* Cw = (float*)(ws + L.C);          // W: B x N_c (band-major)
  float* Cc = (float*)(ws + L.surv);       // C: r x N_c
  double* V = (double*)(ws + oV);
  double* M = (double*)(ws + oM);
  double* sc = (double*)(ws + oScal);      // [0] lam [1] ||W||^2 [2] ||C||^2 [3] ||C||_1
  double* obj = (double*)(ws + oObj);
  float* V32 = (float*)(ws + L.W);         // B x B fp32, ld = B
  double* G = (double*)(ws + L.G);
  double* house = (double*)(ws + L.house);
  double* tri = (double*)(ws + L.tri);
  CK(dwt_forward(L, ws, cube, n, B, fb, st));
  // V_0: top-r eigenvectors of W^T W (K1 Gram of the coefficients, K2 raw mode)
  double* Gw = G;
  if (nc == n) {
    CK(run_gram(L, ws, cube, G, &rs->nonfinite, st));
  } else {
    Gw = (double*)(ws + oGw);
    if (gram_tc_supported(B))
      CK(launch_gram_tc(Cw, nc, B, ws + oGp, np2, Gw, &rs->nonfinite, st));
    else
      CK(launch_gram(Cw, nc, B, (double*)(ws + oGp), ns2, Gw, &rs->nonfinite, st));
  }
  if (lambda < 0.0) {   // D17: sigma^ sqrt(2 ln N_c), sigma^ from the regression noise estimate
    double* Gy = G;
    if (nc != n) CK(run_gram(L, ws, cube, Gy, &rs->nonfinite, st));
    CK(launch_noise_eig(Gy, n, B, 1e-6, -1, 0, (double*)(ws + L.sigma), nullptr, nullptr, house, tri, nullptr,
                        nullptr, B, st));
    CK(launch_wsrrr_lambda((double*)(ws + L.sigma), B, nc, sc, st));
  } else {
    CK(cudaMemcpyAsync(sc, &lambda, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  // V0: only the top r eigenpairs of W^T W (phase 2L when it converges)
  CK(launch_eig_raw(Gw, B, r, (double*)(ws + oOnes), (double*)(ws + oLam), V, r, house, tri, (float*)(ws + L.U),
                    (float*)(ws + L.U), B, st, EIG_LANCZOS));
  CK(launch_v32(V, B, r, V32, B, st));
  CK(launch_sumsq(Cw, (long long)B * nc, (double*)(ws + oPart), sc + 1, st));
  int sweeps = 0;
  std::vector<double> fh;
  for (int it = 0; it < max_iters; ++it) {
    CK(launch_project(Cw, nc, B, V32, B, r, Cc, nc, st));                             // W V
    CK(launch_soft_stats(Cc, (long long)r * nc, sc, (double*)(ws + oPart), sc + 2, sc + 3, st));   // C-step
    CK(launch_wtc(Cw, Cc, nc, B, r, (double*)(ws + oWtc), M, st));                      // W^T C
    CK(launch_procrustes(M, B, r, V, V32, B, sc + 1, sc + 2, sc + 3, sc, obj + it, st));   // V-step + objective
    double f = 0.0;
    CK(cudaMemcpyAsync(&f, obj + it, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fh.push_back(f);
    ++sweeps;
    if (it > 0 && std::fabs(fh[it - 1] - f) <= tol * fh[it - 1]) break;
  }
  // X = C V^T (band-major B x N_c over W), per-band inverse DWT; components = IDWT of C's rows
  CK(launch_reconstruct(Cc, nc, nc, B, V32, B, r, Cw, st));
  CK(dwt_inverse(L, ws, Cw, out, n, B, fb, nullptr, st));
  if (components) CK(dwt_inverse(L, ws, Cc, components, n, r, fb, nullptr, st));
  if (rank_out) *rank_out = r;
  if (sweeps_out) *sweeps_out = sweeps;
  if (objective_out)
    for (int i = 0; i < sweeps; ++i) objective_out[i] = fh[i];
  if (lambda_out) {
    double lh = 0.0;
    CK(cudaMemcpyAsync(&lh, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *lambda_out = lh;
  }
  return HYDE_OK;
}

hyde_status hyde_forpdn(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out, double lambda,
                        int taps, int levels, double* lambda_out, hyde_stream_t stream) {
  if (!h) return HYDE_EPARAM;
  if (!cube || !out) return fail(h, HYDE_EPARAM, "NULL cube/out");
  if (bands < 2 || rows < 1 || cols < 1) return fail(h, HYDE_EPARAM, "bands >= 2 required (SPEC.md:392)");
  if (bands > 256) return fail(h, HYDE_EPARAM, "bands <= 256");
  if (lambda < 0.0) return fail(h, HYDE_EPARAM, "lambda > 0 required (SPEC.md:392); 0 = D16 default");
  const bool autolam = lambda == 0.0;
  if (autolam && (bands < 3 || (long long)rows * cols <= bands))
    return fail(h, HYDE_EPARAM, "the default lambda needs HySime's noise estimate: bands >= 3, pixels > bands");
  const size_t bytes = (size_t)rows * cols * bands * sizeof(float);
  if (cube != out && overlap(cube, bytes, out, bytes)) return fail(h, HYDE_EPARAM, "cube and out partially overlap");
  hyde_hyres_params pin;
  hyde_hyres_params_default(&pin);
  pin.wavelet_taps = taps;
  pin.levels = levels;
  hyde_hyres_params p;
  int lv = 0;
  hyde_status s = resolve_params(h, rows, cols, &pin, &p, &lv);
  if (s != HYDE_OK) return s;
  FilterBank fb;
  if (hyde_build_filters(p.wavelet_taps, &fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "filter derivation failed");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int B = bands;
  Layout L;
  make_layout(rows, cols, B, B, lv, p.wavelet_taps, &L);
  const size_t BB = (size_t)B * B;
  const long long nc = L.plan.n_coeffs;
  size_t off = L.total;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
  const size_t oZ = take(4 * BB * 8), oRp = take(4 * 8), oNp = take(8), oLam = take(8), oGw = take(BB * 8),
               oCoef = take(520 * 4);
  const int np2 = gram_tc_npairs(nc);
  const int ns2 = gram_nsplit(nc, B);
  const size_t oPart = take(std::max((size_t)ns2 * BB * 8, gram_tc_supported(B) ? gram_tc_ws_bytes(nc, B, np2) : 0));
  s = ensure_ws(h, off, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  float* C = (float*)(ws + L.C);
  double* lam_dev = (double*)(ws + oLam);
  const long long n = L.n;
  if (autolam) {
    // D16: residual power of each grid lambda vs HySime's noise power (F1)
    double* G = (double*)(ws + L.G);
    double* house = (double*)(ws + L.house);
    CK(run_gram(L, ws, cube, G, &rs->nonfinite, st));
    CK(launch_noise_eig(G, n, B, 1e-6, -1, 0, (double*)(ws + L.sigma), nullptr, nullptr, house,
                        (double*)(ws + L.tri), nullptr, nullptr, B, st));
    CK(dwt_forward(L, ws, cube, n, B, fb, st));
    const double* Gw = G;   // = W^T W when the DWT is orthonormal on the image (N_c == N)
    if (nc != n) {          // padded levels: the band Gram of the coefficients themselves
      double* Gc = (double*)(ws + oGw);
      if (gram_tc_supported(B))
        CK(launch_gram_tc(C, nc, B, ws + oPart, np2, Gc, &rs->nonfinite, st));
      else
        CK(launch_gram(C, nc, B, (double*)(ws + oPart), ns2, Gc, &rs->nonfinite, st));
      Gw = Gc;
    }
    CK(launch_forpdn_lambda(house + 3 * BB, Gw, B, n, 1e-6, (double*)(ws + oNp), (double*)(ws + oRp), lam_dev,
                            (double*)(ws + oZ), st));
  } else {
    CK(dwt_forward(L, ws, cube, n, B, fb, st));
  }
  // X = W (I + lam D^T D)^-1: one Thomas solve along the bands per coefficient, in place
  CK(launch_forpdn_solve(C, nc, nc, B, lambda, autolam ? lam_dev : nullptr, (float*)(ws + oCoef), st));
  CK(dwt_inverse(L, ws, C, out, n, B, fb, nullptr, st));
  if (lambda_out) {
    if (autolam) {
      double lv_host = 0.0;
      CK(cudaMemcpyAsync(&lv_host, lam_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      *lambda_out = lv_host;
    } else {
      *lambda_out = lambda;
    }
  }
  return HYDE_OK;
}

hyde_status hyde_hysime(hyde_handle h, const float* cube, int rows, int cols, int bands, int* k_out, double* basis,
                        double* delta, double* mu, double* noise_cov, hyde_stream_t stream) {
  hyde_status s = validate_shape(h, rows, cols, bands);
  if (s != HYDE_OK) return s;
  if (!cube || !k_out) return fail(h, HYDE_EPARAM, "NULL cube/k_out");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int B = bands;
  Layout L;
  make_layout(rows, cols, B, 1, 1, 2, &L);
  // HySime buffers past the HyRes layout
  const size_t BB = (size_t)B * B;
  size_t off = L.total;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t oRy = take(BB * 8), oRn = take(BB * 8), oRx = take(BB * 8), oV = take(BB * 8), oB = take(BB * 8);
  const size_t oLam = take((size_t)B * 8), oP = take((size_t)B * 8), oS2 = take((size_t)B * 8),
               oD = take((size_t)B * 8), oOnes = take((size_t)B * 8), oK = take(sizeof(int)), oScal = take(8),
               oLamN = take((size_t)B * 8), oW = take(BB * 4),
               oU = take(BB * 4);
  s = ensure_ws(h, off, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  RankState* rs = (RankState*)(ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  double* G = (double*)(ws + L.G);
  double* house = (double*)(ws + L.house);
  double* tri = (double*)(ws + L.tri);
  double* Ry = (double*)(ws + oRy);
  double* Rn = (double*)(ws + oRn);
  double* Rx = (double*)(ws + oRx);
  double* V = (double*)(ws + oV);
  double* lam = (double*)(ws + oLam);
  double* dl = (double*)(ws + oD);
  double* ones = (double*)(ws + oOnes);
  float* W = (float*)(ws + oW);
  float* U = (float*)(ws + oU);
  CK(run_gram(L, ws, cube, G, &rs->nonfinite, st));
  // M = (G + delta I)^-1 (K2 sweep only): R_n without another pass over the cube
  CK(launch_noise_eig(G, L.n, B, 1e-6, -1, 0, (double*)(ws + L.sigma), nullptr, nullptr, house, tri, nullptr,
                      nullptr, B, st));
  const double* M = house + 3 * BB;   // EigWs::M of the K2 workspace
  CK(launch_hysime_prep(G, M, B, L.n, 1e-6, Ry, Rn, Rx, st));
  // the spectrum of R_n first (its smallest eigenvalue bounds which eigenvectors
  // of R_x can be selected), then the eigenpairs of R_x that can
  const int k1 = B < HYDE_MAX_CHUNK ? B : HYDE_MAX_CHUNK;
  double* lam_n = (double*)(ws + oLamN);
  if (k1 < B) {
    CK(launch_eig_raw(Rn, B, 1, ones, lam_n, V, B, house, tri, W, U, B, st));
    CK(launch_eig_values(tri, house, B, lam_n, st));
  }
  CK(launch_eig_raw(Rx, B, k1, ones, lam, V, B, house, tri, W, U, B, st));
  // only eigenvectors that can be selected: mu_i above a lower bound of R_n's
  // spectrum (the rest have delta_i >= 0 whatever the vector -- k_hysime.cu)
  int m = k1;
  if (k1 < B) {
    CK(launch_eig_values(tri, house, B, lam, st));
    CK(launch_hysime_bound(lam_n, lam, B, (double*)(ws + oScal), (int*)(ws + oK), st));
    CK(cudaMemcpyAsync(&h->rs_host->sure_done, ws + oK, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    m = (int)h->rs_host->sure_done;
    if (m < k1) m = k1;
    if (m > k1) CK(launch_eig_more_raw(tri, house, ones, B, k1, m - k1, lam, V, B, W, U, B, st));
  }
  CK(launch_hysime_delta(V, B, Ry, Rn, B, (double*)(ws + oP), (double*)(ws + oS2), dl, st, m));
  if (m < B) CK(launch_hysime_fill(lam, (double*)(ws + oScal), m, B, (double*)(ws + oP), dl, st));
  CK(launch_hysime_select(dl, (double*)(ws + oP), B, 1e-9, V, B, basis ? (double*)(ws + oB) : nullptr,
                          (int*)(ws + oK), st));
  if (basis) CK(cudaMemcpyAsync(basis, ws + oB, BB * 8, cudaMemcpyDeviceToDevice, st));
  if (delta) CK(cudaMemcpyAsync(delta, dl, (size_t)B * 8, cudaMemcpyDeviceToDevice, st));
  if (mu) CK(cudaMemcpyAsync(mu, lam, (size_t)B * 8, cudaMemcpyDeviceToDevice, st));
  if (noise_cov) CK(cudaMemcpyAsync(noise_cov, Rn, BB * 8, cudaMemcpyDeviceToDevice, st));
  int k = 0;
  CK(cudaMemcpyAsync(&h->rs_host->sure_done, ws + oK, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h->rs_host->nonfinite, &rs->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  k = (int)h->rs_host->sure_done;
  if (h->rs_host->nonfinite) return fail(h, HYDE_EDATA, "non-finite value in the input cube (SPEC.md:26)");
  *k_out = k;
  return HYDE_OK;
}

hyde_status hyde_k_gram(hyde_handle h, const float* cube, int n_pixels, int bands, double* gram,
                        hyde_stream_t stream) {
  if (!h || !cube || !gram || n_pixels < 1 || bands < 1 || bands > 256) return fail(h, HYDE_EPARAM, "bad arguments");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  make_layout(n_pixels, 1, bands, 1, 1, 2, &L);
  hyde_status s = ensure_ws(h, L.total, st);
  if (s != HYDE_OK) return s;
  RankState* rs = (RankState*)(h->ws + L.rs);
  h->last_rs = rs;
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  CK(run_gram(L, h->ws, cube, gram, &rs->nonfinite, st));
  return HYDE_OK;
}

hyde_status hyde_debug_gram_quant(hyde_handle h, int n_pixels, int bands, float* inv_s, int* centre,
                                  long long* n_flagged) {
  if (!h || !h->ws || bands < 1 || bands > 256 || n_pixels < 1) return HYDE_EPARAM;
  DeviceGuard g(h->device);
  Layout L;
  make_layout(n_pixels, 1, bands, 1, 1, 2, &L);   // the layout hyde_k_gram used
  if (!L.use_tc) {
    if (n_flagged) *n_flagged = -1;
    return HYDE_OK;
  }
  const GramQScale* qs = nullptr;
  const int* cnt = nullptr;
  gram_tc_debug_ptrs(h->ws + L.partial, L.n, bands, L.npairs, &qs, &cnt);
  std::vector<GramQScale> q(bands);
  std::vector<int> c(gram_tc_fix_splits(L.n));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(q.data(), qs, sizeof(GramQScale) * bands, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(c.data(), cnt, sizeof(int) * c.size(), cudaMemcpyDeviceToHost));
  long long nf = 0;
  for (int v : c) nf += v;
  for (int b = 0; b < bands; ++b) {
    if (inv_s) inv_s[b] = q[b].inv_s;
    if (centre) centre[b] = q[b].c;
  }
  if (n_flagged) *n_flagged = nf;
  return HYDE_OK;
}

hyde_status hyde_k_eig(hyde_handle h, const double* gram, int n_pixels, int bands, double ridge, int ncomp,
                       double* sigma, double* lam, double* V, hyde_stream_t stream) {
  if (!h || !gram || !sigma || n_pixels < 1 || bands < 3 || bands > 256 || ncomp < 0 || ncomp > bands ||
      ncomp > HYDE_MAX_CHUNK)
    return fail(h, HYDE_EPARAM, "bad arguments");
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  make_layout(n_pixels, 1, bands, 1, 1, 2, &L);
  hyde_status s = ensure_ws(h, L.total, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  // without eigenvalues requested, a first chunk of <= EIG_LANCZOS_MAX_K pairs
  // takes the hot path's phase 2L (the stage test of the Lanczos pairs)
  const int mode = (!lam && ncomp > 0 && ncomp <= EIG_LANCZOS_MAX_K) ? EIG_LANCZOS : EIG_HOUSEHOLDER;
  CK(launch_noise_eig(gram, n_pixels, bands, ridge, ncomp, lam ? 1 : 0, sigma, lam, V,
                      (double*)(ws + L.house), (double*)(ws + L.tri), (float*)(ws + L.W),
                      (float*)(ws + L.U), L.ldwu, st, 0, mode));
  return HYDE_OK;
}

int hyde_debug_sure_prof(unsigned long long* out16) { return out16 ? sure_prof_read(out16) : -1; }

hyde_status hyde_debug_eig_state(hyde_handle h, int n_pixels, int bands, double* tri_out, double* house_out) {
  if (!h || !h->ws || !tri_out || !house_out || bands < 3) return HYDE_EPARAM;
  DeviceGuard g(h->device);
  Layout L;
  make_layout(n_pixels, 1, bands, 1, 1, 2, &L);   // the layout hyde_k_eig used
  CK(cudaMemcpy(tri_out, h->ws + L.tri, (size_t)(3 * bands + 2) * 8, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(house_out, h->ws + L.house, ((size_t)bands * bands * 2 + bands) * 8, cudaMemcpyDeviceToDevice));
  return HYDE_OK;
}

hyde_status hyde_k_project(hyde_handle h, const float* cube, int n_pixels, int bands, const float* W, int ncomp,
                           float* E, hyde_stream_t stream) {
  if (!h || !cube || !W || !E || n_pixels < 1 || bands < 1 || ncomp < 1 || ncomp > HYDE_MAX_CHUNK)
    return fail(h, HYDE_EPARAM, "bad arguments");
  DeviceGuard g(h->device);
  CK(launch_project(cube, n_pixels, bands, W, ncomp, ncomp, E, n_pixels, (cudaStream_t)stream));
  return HYDE_OK;
}

static hyde_status stage_layout(hyde_handle h, int count, int rows, int cols, int levels, int taps,
                                Layout* L, FilterBank* fb, cudaStream_t st) {
  if (!h || count < 1 || rows < 1 || cols < 1) return fail(h, HYDE_EPARAM, "bad arguments");
  if (levels < 1 || levels > HYDE_MAX_LEVELS || (long long)(rows < cols ? rows : cols) < (1LL << levels))
    return fail(h, HYDE_EPARAM, "levels impossible for this image size (SPEC.md:122)");
  if (fb && hyde_build_filters(taps, fb, nullptr) != 0) return fail(h, HYDE_EPARAM, "taps must be 2, 8 or 16");
  make_layout(rows, cols, 3, count, levels, taps, L);
  return ensure_ws(h, L->total, st);
}

hyde_status hyde_k_dwt_fwd(hyde_handle h, const float* images, int count, int rows, int cols, int levels,
                           int taps, float* coeffs, hyde_stream_t stream) {
  if (!images || !coeffs) return fail(h, HYDE_EPARAM, "NULL pointer");
  DeviceGuard g(h ? h->device : 0);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  FilterBank fb;
  hyde_status s = stage_layout(h, count, rows, cols, levels, taps, &L, &fb, st);
  if (s != HYDE_OK) return s;
  CK(dwt_forward(L, h->ws, images, (long long)rows * cols, count, fb, st));
  CK(cudaMemcpyAsync(coeffs, h->ws + L.C, (size_t)count * L.plan.n_coeffs * 4, cudaMemcpyDeviceToDevice, st));
  return HYDE_OK;
}

hyde_status hyde_k_idwt(hyde_handle h, const float* coeffs, int count, int rows, int cols, int levels, int taps,
                        float* images, hyde_stream_t stream) {
  if (!images || !coeffs) return fail(h, HYDE_EPARAM, "NULL pointer");
  DeviceGuard g(h ? h->device : 0);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  FilterBank fb;
  hyde_status s = stage_layout(h, count, rows, cols, levels, taps, &L, &fb, st);
  if (s != HYDE_OK) return s;
  CK(dwt_inverse(L, h->ws, coeffs, images, (long long)rows * cols, count, fb, nullptr, st));
  return HYDE_OK;
}

hyde_status hyde_k_sure(hyde_handle h, float* coeffs, int count, int rows, int cols, int levels, int keep_ll,
                        int* kstar, float* tstar, double* e_post, hyde_stream_t stream) {
  if (!coeffs || !kstar || !tstar || !e_post) return fail(h, HYDE_EPARAM, "NULL pointer");
  DeviceGuard g(h ? h->device : 0);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  hyde_status s = stage_layout(h, count, rows, cols, levels, 2, &L, nullptr, st);
  if (s != HYDE_OK) return s;
  RankState* rs = (RankState*)(h->ws + L.rs);
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  CK(launch_sure(coeffs, L.plan.n_coeffs, L.plan, count, keep_ll, kstar, tstar, (double*)(h->ws + L.esub), rs,
                 (unsigned*)(h->ws + L.surv), st));
  CK(launch_soft_threshold(coeffs, L.plan.n_coeffs, L.plan, count, tstar, st));
  CK(launch_rank_decide((double*)(h->ws + L.esub), L.nsub, count, 0, (double)L.plan.n_coeffs, 1 << 30, rs,
                        e_post, st));
  CK(cudaMemcpyAsync(h->rs_host, rs, sizeof(RankState), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h->rs_host->sure_overflow) return fail(h, HYDE_EMETHOD, "SURE survivor set exceeded its capacity");
  return HYDE_OK;
}

hyde_status hyde_wavelet_shrink(hyde_handle h, const float* images, int count, int rows, int cols, int levels,
                                int taps, int keep_ll, float* out, int* kstar, float* tstar, double* e_post,
                                hyde_stream_t stream) {
  if (!images) return fail(h, HYDE_EPARAM, "NULL pointer");
  const size_t ib = (size_t)count * rows * cols * sizeof(float);
  if (out && images != out && overlap(images, ib, out, ib)) return fail(h, HYDE_EPARAM, "images and out partially overlap");
  DeviceGuard g(h ? h->device : 0);
  cudaStream_t st = (cudaStream_t)stream;
  Layout L;
  FilterBank fb;
  hyde_status s = stage_layout(h, count, rows, cols, levels, taps, &L, &fb, st);
  if (s != HYDE_OK) return s;
  char* ws = h->ws;
  RankState* rs = (RankState*)(ws + L.rs);
  CK(cudaMemsetAsync(rs, 0, sizeof(RankState), st));
  float* C = (float*)(ws + L.C);
  int* ks = (int*)(ws + L.kstar);
  float* ts = (float*)(ws + L.tstar);
  double* es = (double*)(ws + L.esub);
  const long long ld = (long long)rows * cols;
  const long long nc = L.plan.n_coeffs;
  // One launch per stage over every image.  (A pipeline of 32-image groups
  // over three streams -- the DWT of one group beside the SURE and IDWT of the
  // previous ones -- measured slower, 1.79 vs 1.41 ms for DWT + SURE on the 224
  // eigen-images of `large`: SURE needs many subbands in flight, and the
  // overlapping stages contend for the SMs.)  out == NULL: DWT + SURE only.
  {
    Stage sg(h, HYDE_STAGE_DWT, levels, st);
    CK(dwt_forward(L, ws, images, ld, count, fb, st));
    sg.end();
  }
  {
    Stage sg(h, HYDE_STAGE_SURE, 1, st);
    CK(launch_sure(C, nc, L.plan, count, keep_ll, ks, ts, es, rs, (unsigned*)(ws + L.surv), st));
    sg.end();
  }
  if (out) {
    Stage sg(h, HYDE_STAGE_IDWT, levels, st);
    CK(dwt_inverse(L, ws, C, out, ld, count, fb, ts, st));
    sg.end();
  }
  if (e_post) {
    Stage sg(h, HYDE_STAGE_RANK, 1, st);
    CK(launch_rank_decide(es, L.nsub, count, 0, (double)L.plan.n_coeffs, 1 << 30, rs, e_post, st));
    sg.end();
  }
  const size_t nk = (size_t)count * L.nsub;
  if (kstar) CK(cudaMemcpyAsync(kstar, ks, nk * sizeof(int), cudaMemcpyDeviceToDevice, st));
  if (tstar) CK(cudaMemcpyAsync(tstar, ts, nk * sizeof(float), cudaMemcpyDeviceToDevice, st));
  h->last_rs = rs;
  return HYDE_OK;
}

hyde_status hyde_k_reconstruct(hyde_handle h, const float* E, int n_pixels, int bands, const float* U, int ldu,
                               int rank, float* out, hyde_stream_t stream) {
  if (!h || !E || !U || !out || n_pixels < 1 || bands < 1 || rank < 1 || ldu < rank)
    return fail(h, HYDE_EPARAM, "bad arguments");
  DeviceGuard g(h->device);
  CK(launch_reconstruct(E, n_pixels, n_pixels, bands, U, ldu, rank, out, (cudaStream_t)stream));
  return HYDE_OK;
}

}  // extern "C"
