/*
 * hyde.h -- C-ABI of the B200-native HyRes hot path (libhyde.so).
 *
 * HyRes is HyDe's parameter-free, low-rank, wavelet-based Gaussian denoiser
 * (Sec. 2.1 "High Level Conventional Methods"); its six
 * stages are BASELINE.json north_star (1)-(6) and SURVEY.md §8(a) rows A1-A6.
 * This header is the boundary of SURVEY.md §8(b): plain pointers and sizes,
 * no torch types.  Every stage runs in this library's sm_100a kernels.
 *
 * Conventions (all entry points):
 *  - Cube layout: band-sequential (BSQ) float32, C-contiguous
 *    float[bands][rows][cols] (SPEC.md:22-27 HsiCube; BSQ order SPEC.md:23).
 *    The BSQ cube is Y^T: a bands x N row-major matrix, N = rows*cols.
 *  - Pointers are DEVICE pointers unless the name ends in _host.
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and is asynchronous unless stated.  Exceptions: argument
 *    validation is synchronous; hyde_hyres / _ex / _batched read the device
 *    rank-decision flag once per component chunk (one stream sync per
 *    chunk) and therefore return after the GPU has finished
 *    the rank decision (the output write may still be in flight).
 *  - Ownership: the caller owns every buffer it passes; the library never
 *    frees caller memory.  Workspace is owned by the handle (grown on demand
 *    with cudaMallocAsync on `stream`, freed by hyde_destroy).
 *  - In-place (out == cube) is allowed: every read of the cube (A1, A3)
 *    precedes the only write (A6).  Partial overlap -> HYDE_EPARAM.
 *  - Errors: no exceptions cross the ABI.  Status codes mirror the SPEC exit
 *    codes: parameter errors -> HYDE_EPARAM (bands < 3 or
 *    rows*cols <= bands: SPEC.md:363, :365, :381; taps not in {2,8,16} or
 *    levels impossible: SPEC.md:122); non-finite input -> HYDE_EDATA
 *    (SPEC.md:26), detected on the device during A1 and reported through
 *    info->nonfinite_input and the return value of the call that synced.
 *    CUDA failures -> HYDE_ECUDA (hyde_last_error() holds the message).
 *  - A handle is not thread-safe; use one handle per host thread.
 */
#ifndef HYDE_H_
#define HYDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hyde_stream_t;   /* == cudaStream_t */

typedef enum {
  HYDE_OK = 0,
  HYDE_EPARAM = 2,   /* SPEC.md:545 exit code 2: usage/parameter error  */
  HYDE_EDATA = 3,    /* SPEC.md:545 exit code 3: data error (non-finite) */
  HYDE_EMETHOD = 4,  /* SPEC.md:545 exit code 4: method failure          */
  HYDE_ECUDA = 5,
  HYDE_ENCCL = 6,
  HYDE_ENOMEM = 7
} hyde_status;

typedef struct hyde_ctx* hyde_handle;

/* Create a handle bound to CUDA device `device` (the caller's current device
 * is restored on return).  Errors: HYDE_EPARAM (NULL out), HYDE_ECUDA. */
hyde_status hyde_create(hyde_handle* out, int device);
/* Synchronizes the handle's device, frees its workspace.  NULL is a no-op. */
hyde_status hyde_destroy(hyde_handle h);
const char* hyde_status_string(hyde_status s);
/* Last error message recorded on this handle (never NULL). */
const char* hyde_last_error(hyde_handle h);
/* Library version string, and the sm architecture the kernels target (100 = sm_100a). */
const char* hyde_version(void);
int hyde_target_sm(void);

/* HyRes parameters.  HyRes is parameter-free:
 * zero-initialised params (or NULL) give the defaults of SURVEY.md §8(c). */
typedef struct {
  int wavelet_taps;  /* 2 (Haar) | 8 (db4) | 16 (db8, default)  -- SPEC.md:179 D4; 0 = 16 */
  int levels;        /* 0 = auto: max(1, min(5, floor(log2(min(R,C)/(taps-1)))))         */
  int chunk;         /* max candidate components per chunk; 0 = 16; max 32. Chunks   */
                     /* grow 4, 8, 16, ... up to this cap (results are independent)  */
  double ridge;      /* delta of (G + delta I)^-1; 0 = 1e-6                */
  int flags;         /* bit0 HYDE_KEEP_LL: leave LL_L unthresholded (variant, Z7)       */
                     /* bit1 HYDE_VALIDATE: before any work, one pass over the input  */
                     /* checks finiteness and the call returns HYDE_EDATA at once     */
                     /* (synchronous; costs one extra read of the cube).  Without it, */
                     /* non-finite input is caught inside K1 (HYDE_EDATA at the first */
                     /* rank decision, or from hyde_sync_status).                     */
} hyde_hyres_params;
#define HYDE_KEEP_LL 1
#define HYDE_VALIDATE 2

/* Diagnostics of one HyRes call (host memory). */
typedef struct {
  int rank;             /* r*: components kept          */
  int levels;           /* DWT levels used                                   */
  int chunks_run;       /* projection chunks processed                       */
  int nonfinite_input;  /* 1 if a NaN/Inf was seen in the cube (A1)          */
  int n_coeffs;         /* N_c: coefficients per eigen-image                  */
  int comps;            /* candidate components projected / transformed       */
  int reserved[2];
} hyde_hyres_info;

void hyde_hyres_params_default(hyde_hyres_params* p);

/* --- A1: noise estimate (north_star stage (1); PAPER.md:105-106 HySime's
 * regression estimator).  sigma_out[b] = sqrt(1/(N M_bb)),
 * M = (G + ridge I)^-1, G = Y Y^T (bands x bands, uncentered, fp64) -- the
 * residual standard deviation of the least-squares regression of band b on
 * all other bands.  gram_out (bands*bands fp64, row-major) and noise_out
 * (BSQ float32 like the cube: residual_b = (M Y)_b / M_bb) may be NULL.
 * Asynchronous; non-finite input is reported by the return value of a later
 * hyde_sync_status(h) (HYDE_EDATA). */
hyde_status hyde_estimate_noise(hyde_handle h, const float* cube, int rows, int cols, int bands,
                                double* sigma_out, double* gram_out, float* noise_out,
                                hyde_stream_t stream);

/* --- Full HyRes (stages (1)-(6)).  hyde_hyres == hyde_hyres_ex(.., NULL, NULL, ..). */
hyde_status hyde_hyres(hyde_handle h, const float* cube, int rows, int cols, int bands,
                       float* out, hyde_stream_t stream);
hyde_status hyde_hyres_ex(hyde_handle h, const float* cube, int rows, int cols, int bands,
                          float* out, const hyde_hyres_params* params, hyde_hyres_info* info,
                          hyde_stream_t stream);
/* Same computation with HOST buffers (pageable or pinned): copies the cube
 * in, runs hyde_hyres_ex, copies the result out; returns after the result is
 * in out_host (synchronous). */
hyde_status hyde_hyres_host(hyde_handle h, const float* cube_host, int rows, int cols, int bands,
                            float* out_host, const hyde_hyres_params* params,
                            hyde_hyres_info* info, hyde_stream_t stream);
/* Streaming end-to-end path for a sequence of same-shape HOST cubes:
 * cubes_host[i] -> outs_host[i] for i < n.  The host->device copy of cube
 * i+1 and the device->host copy of cube i-1 run on the library's own copy
 * streams while cube i is denoised on `stream` (full-duplex PCIe / C2C), with
 * two device-resident cube slots double-buffered.  Host buffers should be
 * pinned for the copies to overlap; info may be NULL or hold n records.
 * Returns after every result is in its host buffer. */
hyde_status hyde_hyres_host_stream(hyde_handle h, const float* const* cubes_host, float* const* outs_host, int n,
                                   int rows, int cols, int bands, const hyde_hyres_params* params,
                                   hyde_hyres_info* info, hyde_stream_t stream);
/* --- E1: pixel-sharded single cube (BASELINE.json
 * north_star: "the pixel-sharded Gram matrix is all-reduced (B x B); eigen-
 * images or row tiles are distributed for the wavelet stage").  Rank g of G
 * holds pixel rows [g*rows/G, (g+1)*rows/G) of every band (a BSQ slab, floor
 * division: hyde_shard_rows).  Per call:
 *   A1  the slab's Gram (K1), ncclAllReduce(sum, fp64, B x B), then a
 *       finiteness check of the summed G (every rank sees the same G, so a
 *       non-finite value on any slab stops every rank at the same point);
 *   A2  replicated (identical input, code and GPU type: identical V);
 *   per chunk of candidate components (first max(4, G), doubling):
 *   A3  projection of the local slab; all-to-all (grouped ncclSend/ncclRecv)
 *       slab -> component: rank g owns component k iff k % G == g
 *       (hyde_shard_owner) and receives every rank's rows of it into a whole
 *       eigen-image (the periodised DWT couples the first and last rows);
 *   A4/A5 DWT + SURE of the owned images only; the per-subband statistics are
 *       all-reduced so every rank makes the same first-failure rank decision;
 *   A6  IDWT of the owned kept images, all-to-all component -> slab rows,
 *       reconstruction of the local rows.
 * Self transfers are device copies.  The result equals hyde_hyres_ex on the
 * whole cube up to the summation order of the Gram partials (each rank's G is
 * the exact Gram of its own 16-bit quantisation, K1).  The exchange buffers
 * live in the handle.  Errors: HYDE_EPARAM (shape, split, NULL), HYDE_ENCCL
 * (no libnccl.so.2, a failed NCCL call or callback), and those of
 * hyde_hyres_ex; non-finite input returns HYDE_EDATA on every rank.
 *
 * NCCL is resolved at run time (the libnccl.so.2 already loaded by the caller,
 * e.g. PyTorch's, is reused).  comm: a communicator from hyde_nccl_comm_init
 * (or any ncclComm_t of the same NCCL); all collectives are enqueued on
 * `stream`. */
#ifndef NCCL_H_
typedef struct ncclComm* ncclComm_t;
#endif
int hyde_nccl_version(void);   /* NCCL_VERSION_CODE of the run-time library, 0 if none */
/* id_out: 128 bytes (ncclUniqueId) to broadcast to every rank (HOST). */
hyde_status hyde_nccl_unique_id(void* id_out);
hyde_status hyde_nccl_comm_init(ncclComm_t* comm, int world, int rank, const void* id, int device);
hyde_status hyde_nccl_comm_destroy(ncclComm_t comm);
hyde_status hyde_hyres_sharded(hyde_handle h, ncclComm_t comm, const float* local, int local_rows, int row0,
                               int rows, int cols, int bands, float* local_out, const hyde_hyres_params* params,
                               hyde_hyres_info* info, hyde_stream_t stream);
/* Slab of `rank` (host, no GPU): rows [*row0, *row0 + *nrows); rank == world
 * gives *row0 = rows.  Returns 0, or -1 for bad arguments. */
int hyde_shard_rows(int rows, int world, int rank, int* row0, int* nrows);
/* Owner rank of candidate component `component` (0-based) in the wavelet stage. */
int hyde_shard_owner(int component, int world);

/* The same path with caller-supplied collectives (tests: ranks emulated as
 * host threads on one GPU).  Callbacks get DEVICE pointers produced by work
 * enqueued on `stream`; they must run after that work, make their results
 * visible to later work on `stream`, and return 0 on success.
 *   allreduce_sum_f64: element-wise sum over ranks, in place;
 *   sendrecv: one group of point-to-point transfers to / from OTHER ranks;
 *             between two ranks the i-th send matches the i-th receive. */
typedef struct {
  int peer;
  void* buf;
  size_t bytes;
} hyde_p2p;
typedef struct {
  int rank, world;
  void* user;
  int (*allreduce_sum_f64)(void* user, double* buf, size_t count, hyde_stream_t stream);
  int (*sendrecv)(void* user, int nsend, const hyde_p2p* sends, int nrecv, const hyde_p2p* recvs,
                  hyde_stream_t stream);
} hyde_comm;
hyde_status hyde_hyres_sharded_cb(hyde_handle h, const hyde_comm* comm, const float* local, int local_rows,
                                  int row0, int rows, int cols, int bands, float* local_out,
                                  const hyde_hyres_params* params, hyde_hyres_info* info, hyde_stream_t stream);

/* --- F1: HySime signal-subspace identification
 * ("HySime ... implemented in HyDe") on the
 * same A1/A2 data: R_y = Y Y^T / N, R_n = N~ N~^T / N with N~ the regression
 * residual of every band on all others (ridge 1e-6, as A1), computed without a
 * second pass as D^-1 (M - delta M^2) D^-1 / N, M = (G + delta I)^-1,
 * D = diag(M); R_x = R_y - R_n = E diag(mu) E^T; delta_i = -e_i^T R_y e_i +
 * 2 e_i^T R_n e_i; *k_out (HOST) = #{delta_i < -1e-9 max_j |p_j|} (DESIGN.md
 * R13).  Optional DEVICE outputs (NULL = skip): basis (bands x bands row-major;
 * columns 0..k-1 = the selected eigenvectors in ascending-delta order, D6 signs),
 * delta and mu ([bands], in descending-mu order), noise_cov (R_n, bands x
 * bands).  Eigenvectors are computed only where mu_i exceeds the smallest
 * eigenvalue l of R_n: elsewhere delta_i = s_i^2 - mu_i >= l - mu_i >= 0 for any
 * vector (never selected) and delta holds that lower bound l - mu_i.
 * Synchronous (returns after k is known).  Errors: as hyde_hyres. */
hyde_status hyde_hysime(hyde_handle h, const float* cube, int rows, int cols, int bands, int* k_out,
                        double* basis, double* delta, double* mu, double* noise_cov, hyde_stream_t stream);

/* --- F2: FORPDN ("full-rank,
 * wavelet-based"): W = per-band 2-D DWT of every band (the A4 transform: taps
 * 0 = 16, levels 0 = auto), X = W (I + lambda D^T D)^-1 with D the first-order
 * spectral difference (A = I + lambda D^T D is tridiagonal: one Thomas solve
 * along the bands per coefficient), out = per-band inverse DWT of X.  lambda <= 0
 * -> HYDE_EPARAM except 0 = the D16 default: the grid value {0.1, 1, 10, 100}
 * whose residual power ||W - X||^2 / (N B) (coefficient domain) is closest to
 * HySime's noise power trace(R_n) / B (R14).  cube / out: DEVICE BSQ
 * (out == cube allowed).  lambda_out (HOST, may be NULL) receives the lambda
 * used; when it is non-NULL and lambda == 0 the call synchronizes.  bands in
 * [2, 256] ([3, 256] and pixels > bands for the default lambda). */
hyde_status hyde_forpdn(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out,
                        double lambda, int taps, int levels, double* lambda_out, hyde_stream_t stream);

/* --- F3: HyMiNoR (SPEC.md:415-423 D19; §2.1
 * "After the Gaussian noise is removed by HyRes, the remaining sparse noise is
 * removed by solving an l1-l1 optimization problem with a modified
 * split-Bregman technique").  hyde_l1_spectral: per pixel spectrum m of cube,
 * min_x ||m - x||_1 + lambda ||D x||_1 (D the first-order spectral difference)
 * by split Bregman with penalty mu, from x = m (R16); a pixel stops
 * when ||x_new - x_old|| <= tol ||x_old|| or after max_iters; iters (DEVICE
 * int[rows*cols], may be NULL) receives the iterations per pixel.  The first
 * iteration runs one thread per pixel (a sequential Thomas sweep along the
 * bands, HBM-bound); pixels that continue run one warp per pixel, state in
 * registers; bands in [2, 256]; out == cube allowed (a pixel continued past
 * the first iteration then uses m = (I + D^T D) x_1, equal to its input up to
 * fp32 rounding).  Uses the handle's workspace (n/32 words).
 * hyde_hyminor: hyde_hyres_ex (defaults; info may be NULL) into out, then
 * hyde_l1_spectral in place; lambda 0 -> 10, mu 0 -> 5, max_iters <= 0 -> 50,
 * tol < 0 -> 1e-3 (D19).  Errors: lambda or mu negative -> HYDE_EPARAM; those of
 * hyde_hyres_ex. */
hyde_status hyde_l1_spectral(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out,
                             double lambda, double mu, int max_iters, double tol, int* iters,
                             hyde_stream_t stream);
hyde_status hyde_hyminor(hyde_handle h, const float* cube, int rows, int cols, int bands, float* out,
                         double lambda, double mu, int max_iters, double tol, hyde_hyres_info* info,
                         hyde_stream_t stream);

/* --- F4: WSRRR (SPEC.md:397-405, :433 D17; §2.1
 * "Wavelet-Based Sparse Reduced-Rank Regression"): min_{C,V} ||W - C V^T||_F^2 +
 * lambda ||C||_1 s.t. V^T V = I, W = per-band DWT coefficients (taps 0 = 16,
 * levels 0 = auto).  V_0 = top-rank eigenvectors of W^T W; per sweep C =
 * soft(W V, lambda/2), V = polar factor of W^T C (orthogonal Procrustes); stop
 * when the objective changes by <= tol (relative; < 0 -> 1e-4) or after
 * max_iters sweeps (<= 0 -> 20) (R15).  rank 0 = HySime's k (at
 * least 1), else 1..min(bands, 32); lambda < 0 = the D17 default
 * sigma^ sqrt(2 ln N_c), sigma^ = RMS of the A1 noise estimate; lambda >= 0 is
 * used as given.  out: DEVICE BSQ denoised cube (inverse DWT of C V^T per
 * band); components: DEVICE (rank x rows x cols) inverse DWT of the columns of
 * C, or NULL.  HOST outputs (may be NULL): rank_out, lambda_out, sweeps_out,
 * objective_out[max_iters] (objective after each sweep).  Synchronous (one
 * host read of the objective per sweep). */
hyde_status hyde_wsrrr(hyde_handle h, const float* cube, int rows, int cols, int bands, int rank,
                       double lambda, int taps, int levels, int max_iters, double tol, float* out,
                       float* components, int* rank_out, double* lambda_out, int* sweeps_out,
                       double* objective_out, hyde_stream_t stream);

/* Bytes of device workspace hyde_hyres_ex / _batched will hold for this shape. */
size_t hyde_hyres_workspace_size(int rows, int cols, int bands, int batch,
                                 const hyde_hyres_params* params);
/* `batch` independent same-shape cubes, cubes[batch][bands][rows][cols] ->
 * outs (same layout); info may be NULL or point to `batch` records. */
hyde_status hyde_hyres_batched(hyde_handle h, const float* cubes, int batch, int rows, int cols,
                               int bands, float* outs, const hyde_hyres_params* params,
                               hyde_hyres_info* info, hyde_stream_t stream);
/* Status of asynchronous device-side checks (non-finite input) of the work
 * enqueued so far; synchronizes `stream`. */
hyde_status hyde_sync_status(hyde_handle h, hyde_stream_t stream);

/* --- Stage entry points (test/diagnostic; same conventions).  Each consumes
 * and produces the oracle's intermediate layout (oracle/hyres_ref.py). ---- */

/* A1: G = Y Y^T, fp64 row-major bands x bands (north_star
 * stage (1)).  bands <= 224: the exact integer tensor-core Gram of the cube
 * with every value rounded to its band's 16-bit grid s_b (q + c_b), except the
 * pixels holding a value outside that grid's range (outliers, NaN/Inf), which
 * enter exactly in fp64 -- see k_gram_tc.cu; bands > 224: fp64 SIMT. */
hyde_status hyde_k_gram(hyde_handle h, const float* cube, int n_pixels, int bands, double* gram,
                        hyde_stream_t stream);
/* Diagnostics of the last hyde_k_gram on this handle (synchronizes the
 * device): per band the fp32 1/step inv_s[b] and the integer centre centre[b]
 * (q = rint(y inv_s) - c), and the number of flagged (exactly added) pixels;
 * n_flagged = -1 when the fp64 SIMT path ran.  Any output may be NULL. */
hyde_status hyde_debug_gram_quant(hyde_handle h, int n_pixels, int bands, float* inv_s, int* centre,
                                  long long* n_flagged);
/* A1+A2: from G (fp64, bands x bands) and N: sigma[bands]; lam[bands] (all
 * eigenvalues of G_w = diag(sigma)^-1 G diag(sigma)^-1 / N, descending);
 * V[bands x ncomp] (row-major, eigenvectors of the ncomp largest, sign-fixed:
 * largest-|.| entry positive, SPEC.md:181 D6).  lam may be NULL; then for
 * ncomp <= 6 the pairs come from the hot path's Lanczos phase (Householder
 * when it does not converge), otherwise from the Householder reduction. */
hyde_status hyde_k_eig(hyde_handle h, const double* gram, int n_pixels, int bands, double ridge,
                       int ncomp, double* sigma, double* lam, double* V, hyde_stream_t stream);
/* A3: E[k][p] = sum_b W[b][k] Y[b][p], W = float32 row-major bands x ncomp. */
hyde_status hyde_k_project(hyde_handle h, const float* cube, int n_pixels, int bands,
                           const float* W, int ncomp, float* E, hyde_stream_t stream);
/* A4: forward DWT of `count` images (each rows x cols, contiguous) into the
 * subband layout: per image, level 1..L x (LH, HL, HH) then LL_L, each
 * subband row-major; n_coeffs per image (see hyde_dwt_coeff_count). */
hyde_status hyde_k_dwt_fwd(hyde_handle h, const float* images, int count, int rows, int cols,
                           int levels, int taps, float* coeffs, hyde_stream_t stream);
int hyde_dwt_coeff_count(int rows, int cols, int levels);
int hyde_auto_levels(int rows, int cols, int taps);
/* A5: per subband SURE (noise sigma = 1): kstar[count*(3L+1)] (index into
 * {0} U sorted |x|), tstar[...] (threshold), in-place soft threshold of
 * coeffs, e_post[count] (sum of squares of the thresholded coefficients). */
hyde_status hyde_k_sure(hyde_handle h, float* coeffs, int count, int rows, int cols, int levels,
                        int keep_ll, int* kstar, float* tstar, double* e_post,
                        hyde_stream_t stream);
/* A6a: inverse DWT of `count` coefficient sets -> images (rows x cols each). */
hyde_status hyde_k_idwt(hyde_handle h, const float* coeffs, int count, int rows, int cols,
                        int levels, int taps, float* images, hyde_stream_t stream);
/* A4 -> A5 -> A6a on `count` images exactly as the hot path runs them
 * (BASELINE.json north_star stages (4)-(6): "a batched multi-level orthogonal
 * 2D discrete wavelet transform of every eigen-image; per-subband SURE
 * threshold selection ... with soft-thresholding; inverse DWT"):
 * forward DWT (L launches), one SURE launch over every (image, subband), and
 * the inverse DWT with each subband soft-thresholded by its t* as it is
 * loaded (no rank rule: every image is reconstructed).  images / out: DEVICE,
 * count x rows x cols fp32 (out == images allowed; partial overlap ->
 * HYDE_EPARAM; out == NULL: DWT + SURE only).  kstar / tstar [count*(3L+1)] (DEVICE, subband order of
 * hyde_k_dwt_fwd) and e_post [count] (DEVICE, sum of the thresholded
 * coefficients squared) may each be NULL.  Workspace (about 2.3 x the image
 * bytes) is held by the handle.  Asynchronous; a SURE capacity failure is
 * reported by hyde_sync_status (HYDE_EMETHOD).  This is the stage-isolated
 * measurement of SURVEY.md §8(d) ("a stage-isolated run on all B eigen-images
 * of large") and a standalone wavelet-shrinkage denoiser. */
hyde_status hyde_wavelet_shrink(hyde_handle h, const float* images, int count, int rows, int cols,
                                int levels, int taps, int keep_ll, float* out, int* kstar,
                                float* tstar, double* e_post, hyde_stream_t stream);
/* A6b: out[b][p] = sum_{k<rank} U[b][k] E[k][p], U float32 row-major bands x ldu. */
hyde_status hyde_k_reconstruct(hyde_handle h, const float* E, int n_pixels, int bands,
                               const float* U, int ldu, int rank, float* out,
                               hyde_stream_t stream);
/* --- Stage timing (diagnostics; bench.py's roofline).  When enabled, the
 * library records CUDA events on the call's stream around each stage of every
 * subsequent call.  hyde_profile_read synchronizes the device, adds the
 * elapsed time of every recorded stage to ms[stage] and the number of kernels
 * launched in it to launches[stage] (arrays of HYDE_NSTAGES), and clears the
 * records.  hyde_launch_count: kernels this handle launched since creation. */
enum {
  HYDE_STAGE_GRAM = 0,     /* K1: G = Y Y^T                       (A1)   */
  HYDE_STAGE_EIG = 1,      /* K2: sigma, whitening, eigenpairs   (A1-A2) */
  HYDE_STAGE_PROJECT = 2,  /* K3: eigen-images                   (A3)   */
  HYDE_STAGE_DWT = 3,      /* K4: forward DWT levels             (A4)   */
  HYDE_STAGE_SURE = 4,     /* K5: SURE + soft threshold          (A5)   */
  HYDE_STAGE_RANK = 5,     /* rank decision + 16-byte D2H        (A5)   */
  HYDE_STAGE_IDWT = 6,     /* K6a: inverse DWT                   (A6)   */
  HYDE_STAGE_RECON = 7,    /* K6b: reconstruction to bands       (A6)   */
  HYDE_NSTAGES = 8
};
hyde_status hyde_profile_enable(hyde_handle h, int on);
hyde_status hyde_profile_read(hyde_handle h, double* ms, long long* launches);
long long hyde_launch_count(hyde_handle h);

/* clock64() stamps (SM cycles, CTA 0 of the K2 cluster) of the last K2
 * launch: [0] start, [1] sweep (sigma) done, [2] tridiagonalisation done,
 * [3] eigenpairs done, [4] vectors written.  With -DHYDE_EIG_PROF builds,
 * [5..17] hold per-segment accumulators (sweep gather / exchange / pivot
 * Cholesky / solves / update; column symv+send / Q update / wait / update /
 * reflector; bisection; inverse iteration).  Copies 32 values; synchronizes. */
hyde_status hyde_debug_eig_clocks(long long* out40);
/* Test hook for K2's first chunk: enable = 0 runs the Householder path (phase
 * 2 + 3) instead of the Lanczos phase 2L; max_steps > 0 caps the Lanczos steps
 * (a cap below convergence exercises the in-kernel fallback).  Process-wide;
 * the default is enable = 1 (HYDE_EIG_LANCZOS=0 in the environment: 0),
 * max_steps = 0 (no cap).  Always HYDE_OK. */
hyde_status hyde_debug_eig_lanczos(int enable, int max_steps);

/* K5 phase profile of the SURE launches since the last call (builds with
 * HYDE_SURE_PROF=1 only; returns 0 and zeros otherwise, 1 when filled):
 * out16[c*8 + p] = SM cycles summed over CTAs, class c (0: subbands longer than
 * the 8192-key window capacity, 1: shorter), phase p (0 window search,
 * 1 compaction, 2 sort + exact evaluation, 3 = number of CTAs, 4 histogram
 * streaming, 5 passes, 6-7 cluster-barrier waits); out16[16..20]: largest /
 * summed window size and item count of the long subbands, longest sort +
 * evaluation (long, short subbands); out16[32 + c*8 + p]: the longest CTA of
 * class c in phase p.  Copies 48 values.  Synchronizes. */
int hyde_debug_sure_prof(unsigned long long* out16);

/* CTAs per K2 eigensolver cluster on the current device: 16 (non-portable
 * cluster size) when the GPU can co-schedule it, else 8. */
int hyde_eig_cluster_size(void);

/* Copies the tridiagonal T (d[B], e[B], e^2[B], glo, ghi) and the first
 * 2 B^2 + B doubles of the K2 workspace (Q = H_0 H_1 ... row-major, the
 * sign-fixed eigenvectors, eigenvalues) of the handle's last hyde_k_eig call
 * (same n_pixels and bands) into device buffers. */
hyde_status hyde_debug_eig_state(hyde_handle h, int n_pixels, int bands, double* tri_out, double* house_out);

/* Analysis low-pass filter the kernels use (host, fp64; taps values). */
hyde_status hyde_filter(int taps, double* h_out);

#ifdef __cplusplus
}
#endif
#endif /* HYDE_H_ */
