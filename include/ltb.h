/*
 * ltb.h -- C ABI of the B200-native online hot path of arXiv 2504.16344
 * (libltb.so, built from paper_2504_16344_b200/csrc for sm_100a).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference's proj/ directory).  INTEGRATION.md shows the
 * reference-side binding (a drop-in fft_matvec.cpp over this ABI, and the
 * ctypes stub the Python tests use).
 *
 * Conventions -- identical to the reference's MatvecPlan
 * (include/ltibayes/fft_matvec.hpp:12-28):
 *   - series are SpaceMajorRows: row r's N_t samples contiguous
 *     (core.hpp:53,73-77);
 *   - kernels are [row][col][lag], lag contiguous (core.hpp:114-140);
 *   - padded length exactly 2 N_t, N_f = N_t + 1 frequencies, forward
 *     transform unnormalised, inverse scaled by 1/(2 N_t), first N_t samples
 *     kept;
 *   - F-hat is stored per frequency as a column-major rows x cols complex
 *     block, row fastest (fft_matvec.cpp:44-46): khat[f][c][r].
 *
 * Errors: every call returns an ltb_status; ltb_last_error() gives the
 * thread-local message.  The codes map one-to-one onto the reference's
 * exception taxonomy (core.hpp:12-35): DimensionError, LayoutError,
 * NumericalError, CapacityError, StateError.
 *
 * Threading: a plan is immutable after creation and may be shared; each
 * concurrent caller needs its own scratch (= MatvecPlan::Scratch,
 * fft_matvec.hpp:45-58), which owns a CUDA stream and device workspace.
 * Host-pointer calls are synchronous (the reference's apply_raw semantics);
 * device-pointer calls are asynchronous on the scratch's stream.
 */
#ifndef LTB_H
#define LTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LTB_OK = 0,
  LTB_DIMENSION = 1, /* DimensionError  (core.hpp:12) */
  LTB_LAYOUT = 2,    /* LayoutError     (core.hpp:15) */
  LTB_NUMERICAL = 3, /* NumericalError  (core.hpp:24) */
  LTB_CAPACITY = 4,  /* CapacityError   (core.hpp:27) */
  LTB_STATE = 5,     /* StateError      (core.hpp:30) */
  LTB_CUDA = 6,      /* CUDA runtime failure (no reference analogue) */
  LTB_INVALID = 7,   /* null handle / bad argument */
  LTB_CONFIG = 8,    /* ConfigError     (core.hpp:21) */
  LTB_IO = 9         /* IoError         (core.hpp:33) */
} ltb_status;

typedef enum { LTB_PTR_HOST = 0, LTB_PTR_DEVICE = 1 } ltb_ptr_kind;

/* KernelTag (core.hpp:103) */
typedef enum { LTB_TAG_F = 0, LTB_TAG_FQ = 1, LTB_TAG_GSTAR = 2, LTB_TAG_GQSTAR = 3 } ltb_tag;

/* Layout (core.hpp:53) */
typedef enum { LTB_TIME_MAJOR_BLOCKS = 0, LTB_SPACE_MAJOR_ROWS = 1 } ltb_layout;

typedef struct ltb_plan ltb_plan;
typedef struct ltb_scratch ltb_scratch;
typedef struct ltb_engine ltb_engine;
typedef struct ltb_splan ltb_splan;       /* MatvecPlan sharded over GPUs */
typedef struct ltb_sscratch ltb_sscratch; /* its Scratch */

typedef struct {
  int device;    /* CUDA ordinal; -1 = current device */
  int unit_cols; /* GEMV work-unit width in columns; 0 = automatic */
} ltb_opts;

const char* ltb_last_error(void);
const char* ltb_version(void);
/* number of kernels this library launched since load (all threads) */
uint64_t ltb_kernel_launches(void);

/* ---- MatvecPlan (fft_matvec.hpp:29-78, ctor fft_matvec.cpp:73-111) ---- */

/* Plan from an explicit kernel tensor [rows][cols][nt] (host or device
 * pointer).  Scans for non-finite entries (core.cpp:73-77 -> LTB_NUMERICAL)
 * and builds F-hat on the device. */
ltb_status ltb_plan_create(const double* kernel_rck, int rows, int cols, int nt, int tag,
                           int ptr_kind, const ltb_opts* opts, ltb_plan** out);

/* Plan whose kernel is generated in place on the device by the counter
 * generator: k(r, c, t) = U(seed, stream, (r * nm_total + c0 + c) * nt + t),
 * c in [0, cols) -- a column shard [c0, c0+cols) of an rows x nm_total
 * kernel.  Needed at Cascadia scale, where the 66 GB time-domain kernel
 * cannot round-trip through host memory. */
ltb_status ltb_plan_create_generated(int rows, int cols, int nt, int tag, uint64_t seed,
                                     uint64_t stream, long long nm_total, long long c0,
                                     const ltb_opts* opts, ltb_plan** out);

/* G* plans built on the device from F: the kernel is premultiplied by the
 * prior covariance Gamma_x = A_x^{-2}, A_x = delta I - gamma L (Neumann
 * Laplacian on the n_cols nodes, spacing h_x), along its column axis before
 * the transform -- PriorOp::premultiply_kernel (prior.cpp:108-134; A_x
 * prior.cpp:9-39).  Tag F -> Gstar, Fq -> Gqstar; LTB_CONFIG for an already
 * premultiplied tag or invalid prior parameters.  Built slab by slab (<= 64
 * kernel rows at a time), so the time-domain kernel is never resident. */
ltb_status ltb_plan_create_premultiplied(const double* kernel_rck, int rows, int cols, int nt,
                                         int tag, int ptr_kind, double h_x, double gamma,
                                         double delta, const ltb_opts* opts, ltb_plan** out);
ltb_status ltb_plan_create_generated_premultiplied(int rows, int cols, int nt, int tag,
                                                   uint64_t seed, uint64_t stream, double h_x,
                                                   double gamma, double delta,
                                                   const ltb_opts* opts, ltb_plan** out);

/* Column shard [c0, c0 + cols) of the G* plan of a generated rows x nm_total
 * kernel: every slab is generated and premultiplied over all nm_total
 * columns (Gamma_x couples the columns), only the shard's columns are
 * transformed -- the per-rank G* of the distributed online phase. */
ltb_status ltb_plan_create_generated_premultiplied_shard(int rows, int cols, int nt, int tag, uint64_t seed,
                                                         uint64_t stream, long long nm_total, long long c0,
                                                         double h_x, double gamma, double delta,
                                                         const ltb_opts* opts, ltb_plan** out);

/* Plan from a BTPZ1 kernel archive written by the reference (io.cpp:71-100:
 * "BTPZ1", u64 rows, cols, N_t, tag, [row][col][lag] doubles), streamed
 * slab by slab to the device (LTB_IO on a missing / bad / truncated file).
 * prior3 = {h_x, gamma, delta} premultiplies on the way (NULL: as stored). */
ltb_status ltb_plan_load_btpz(const char* path, const double* prior3, const ltb_opts* opts,
                              ltb_plan** out);

ltb_status ltb_plan_destroy(ltb_plan* plan);

/* rows_out / n_cols / n_time / padded_len / n_freq / tag (fft_matvec.hpp:38-43) */
ltb_status ltb_plan_dims(const ltb_plan* plan, int* rows_out, int* n_cols, int* n_time,
                         int* padded_len, int* n_freq, int* tag);

/* device bytes held by the plan (F-hat + tables) */
ltb_status ltb_plan_bytes(const ltb_plan* plan, size_t* bytes);

/* kernel_hat_sqnorm (fft_matvec.cpp:124-137) */
ltb_status ltb_kernel_hat_sqnorm(const ltb_plan* plan, double* out);

/* copy F-hat frequencies [f0, f0+nfreq) to host, [f][c][r] complex
 * interleaved (test/diagnostic access) */
ltb_status ltb_plan_copy_kernel_hat(const ltb_plan* plan, int f0, int nfreq, double* host_out);

/* ---- Scratch (fft_matvec.hpp:45-58) ---- */
/* cuda_stream: a cudaStream_t to run on, NULL for a private (non-blocking)
 * stream, or (void*)1 (cudaStreamLegacy) for the legacy default stream */
ltb_status ltb_scratch_create(const ltb_plan* plan, void* cuda_stream, ltb_scratch** out);
ltb_status ltb_scratch_destroy(ltb_scratch* s);
ltb_status ltb_scratch_sync(ltb_scratch* s);
/* the scratch's cudaStream_t (for event timing by the caller) */
void* ltb_scratch_stream(ltb_scratch* s);

/* Per-stage device timing of the applies run on this scratch: with timing
 * enabled, CUDA events are recorded on the scratch's stream around each
 * kernel.  enable != 0 clears and starts accumulation, 0 stops it. */
ltb_status ltb_scratch_timing(ltb_scratch* s, int enable);
/* Accumulated milliseconds since timing was enabled (synchronizes):
 * ms[0..2] = F (pad+r2c, GEMV-N, c2r), ms[3..5] = F* (pad+r2c, GEMV-H, c2r);
 * calls[0] / calls[1] = number of F / F* applies timed. */
ltb_status ltb_scratch_stage_ms(ltb_scratch* s, double* ms6, int* calls2);

/* ---- apply_raw / apply_adjoint_raw (fft_matvec.cpp:139-217) ---- */
/* d = F m: in n_cols*N_t, out rows_out*N_t, SpaceMajorRows */
ltb_status ltb_apply(const ltb_plan* plan, ltb_scratch* s, const double* in, double* out,
                     int ptr_kind);
/* m = F* d: in rows_out*N_t, out n_cols*N_t */
ltb_status ltb_apply_adjoint(const ltb_plan* plan, ltb_scratch* s, const double* in,
                             double* out, int ptr_kind);

/* ---- typed apply / apply_adjoint (fft_matvec.cpp:221-265) ----
 * Checks the layout tag (LTB_LAYOUT unless SpaceMajorRows: "no silent
 * reindex") and the series dims (LTB_DIMENSION), then applies. */
ltb_status ltb_apply_series(const ltb_plan* plan, ltb_scratch* s, const double* in,
                            int n_rows, int n_time, int layout, double* out, int ptr_kind);
ltb_status ltb_apply_adjoint_series(const ltb_plan* plan, ltb_scratch* s, const double* in,
                                    int n_rows, int n_time, int layout, double* out,
                                    int ptr_kind);

/* ---- MatvecPlan sharded over the GPUs of one process ----
 * The same MatvecPlan (fft_matvec.hpp:29-78) with its N_m columns cut into
 * ndev contiguous ranges, shard k on device devs[k] (devices may repeat).
 * F m: each shard applies its columns, the home device devs[0] sums the
 * N_d x N_t partials in shard order (one kernel reading the peers' buffers
 * over NVLink); F* d: d reaches every shard, each writes its columns of m.
 * ltb_apply_sharded / ltb_apply_adjoint_sharded have the semantics of
 * ltb_apply / ltb_apply_adjoint (= apply_raw / apply_adjoint_raw,
 * fft_matvec.cpp:139-217): host pointers synchronous; device pointers on the
 * home device, asynchronous on the scratch's home stream.  A multi-GPU
 * replacement for the single-device plan behind the C++ drop-in
 * (cpp/fft_matvec_b200.cpp selects it with LTB_DEVICES=0,1,...). */
ltb_status ltb_plan_create_sharded(const double* kernel_rck, int rows, int cols, int nt, int tag,
                                   int ndev, const int* devs, const ltb_opts* opts, ltb_splan** out);
ltb_status ltb_plan_create_generated_sharded(int rows, int cols, int nt, int tag, uint64_t seed,
                                             uint64_t stream, int ndev, const int* devs,
                                             const ltb_opts* opts, ltb_splan** out);
ltb_status ltb_splan_destroy(ltb_splan* plan);
ltb_status ltb_splan_dims(const ltb_splan* plan, int* rows_out, int* n_cols, int* n_time,
                          int* n_shards);
/* shard k: device, column range [c0, c1), peer = 1 if the home device reads it over P2P */
ltb_status ltb_splan_shard(const ltb_splan* plan, int k, int* device, long long* c0,
                           long long* c1, int* peer);
ltb_status ltb_splan_kernel_hat_sqnorm(const ltb_splan* plan, double* out);
/* home_stream: cudaStream_t on devs[0] for shard 0 (NULL: private); the
 * other shards get private streams on their devices */
ltb_status ltb_sscratch_create(const ltb_splan* plan, void* home_stream, ltb_sscratch** out);
ltb_status ltb_sscratch_destroy(ltb_sscratch* s);
ltb_status ltb_sscratch_sync(ltb_sscratch* s);
void* ltb_sscratch_stream(ltb_sscratch* s);
ltb_status ltb_apply_sharded(const ltb_splan* plan, ltb_sscratch* s, const double* in, double* out,
                             int ptr_kind);
ltb_status ltb_apply_adjoint_sharded(const ltb_splan* plan, ltb_sscratch* s, const double* in,
                                     double* out, int ptr_kind);

/* ---- dense_apply (fft_matvec.hpp:80-87, fft_matvec.cpp:267-315) ----
 * FFT-free time-domain block-Toeplitz product (the reference's test oracle,
 * kept so the drop-in fft_matvec.cpp is link-complete).  Raises
 * LTB_CAPACITY when rows*nt*cols*nt*8 > mem_cap_bytes (0 = no cap). */
ltb_status ltb_dense_apply(const double* kernel_rck, int rows, int cols, int nt, const double* v,
                           int adjoint, unsigned long long mem_cap_bytes, double* out,
                           int ptr_kind);

/* ---- online subset of InferenceEngine (bayes_engine.hpp:83-107) ---- */

/* Engine over the G* plan (prior-premultiplied kernel, bayes_engine.cpp:105,
 * 112) and an optional F_q plan for the forecast.  The plans must outlive
 * the engine. */
ltb_status ltb_engine_create(const ltb_plan* plan_gstar, const ltb_plan* plan_fq,
                             const ltb_opts* opts, ltb_engine** out);
ltb_status ltb_engine_destroy(ltb_engine* e);

/* set_factor (bayes_engine.cpp:211-217): lower Cholesky factor of K,
 * n = N_d * N_t, column-major with leading dimension ld; only the lower
 * triangle is read (the strict upper part may hold K itself,
 * bayes_engine.cpp:180-193).  Repacked on the device into lower tiles. */
ltb_status ltb_engine_set_factor(ltb_engine* e, const double* L, int n, size_t ld,
                                 int ptr_kind);
/* Distributed K^{-1} over `world` ranks (one process per GPU; call before
 * setting the factor).  The factor is split row-cyclically in 64-row blocks
 * (rank r keeps block rows r, r+world, ...), built per rank by
 * ltb_engine_set_factor_generated; the ranks then exchange the 64-byte CUDA
 * IPC handles of their receive buffers (ltb_engine_ipc_handle, gathered in
 * rank order and passed to ltb_engine_connect).  Every rank must call the
 * solve / infer entry points concurrently.  With world > 1 the engine's G*
 * and F_q plans are the rank's column shard: m_map is the rank's shard and
 * q is the rank's partial forecast, to be summed over ranks by the caller
 * (one small all-reduce). */
ltb_status ltb_engine_set_world(ltb_engine* e, int world, int rank);
ltb_status ltb_engine_ipc_handle(ltb_engine* e, void* out64);
ltb_status ltb_engine_connect(ltb_engine* e, const void* handles);

/* synthetic factor generated on the device (oracle orc_gen_factor) */
ltb_status ltb_engine_set_factor_generated(ltb_engine* e, int n, uint64_t seed);

/* ---- offline phase 2 on the device: form_K + factorize ----
 * form_K (bayes_engine.cpp:136-172): K = F G* + sigma2 I over
 * n = N_d N_t, from the time-domain kernels of F and G = F Gamma_x
 * ([rows][cols][lag], host or device; rows = N_d, cols = N_m of the engine's
 * G* plan).  g_kernel NULL: G is premultiplied from F on the device with
 * prior3 = {h_x, gamma, delta} (bayes_engine.cpp:105, prior.cpp:108-134).
 * Formed as the lag Gram contraction A = F_lag G_lag^T on FP64 tensor cores
 * plus a diagonal recurrence (ltb_formk.h); only the lower triangle is
 * formed (K is symmetric; the reference symmetrises, :154-171), straight
 * into the packed tiles.  Single-GPU engines. */
ltb_status ltb_engine_form_k(ltb_engine* e, const double* f_kernel, const double* g_kernel,
                             const double* prior3, int rows, int cols, int nt, double sigma2,
                             int ptr_kind);
/* form_K of the generated kernel k(r, c, t) = U(seed, stream, (r N_m + c) N_t + t)
 * (ltb_plan_create_generated with nm_total = N_m) and its premultiplied G */
ltb_status ltb_engine_form_k_generated(ltb_engine* e, uint64_t seed, uint64_t stream, double h_x,
                                       double gamma, double delta, double sigma2);
/* factorize (bayes_engine.cpp:176-209): K = L L^T in place (tile Cholesky,
 * DMMA trailing updates); LTB_NUMERICAL if K is not positive definite,
 * LTB_STATE without form_K.  Afterwards the engine is ready to solve. */
ltb_status ltb_engine_factorize(ltb_engine* e);
/* form_Q + form_qoi_cov (bayes_engine.cpp:242-285) on the device, after
 * factorize / set_factor: R = F Gq* and the prior QoI covariance P = Fq Gq*
 * (the form_K contraction, rectangular), K^{-1} R by multi-RHS block
 * substitution on the packed factor (FP64 tensor cores),
 * Gamma_post_q = sym(P - R^T K^{-1} R) (as (L^{-1}R)^T (L^{-1}R)), Q = (K^{-1}R)^T;
 * then the Phase-3 operator is installed exactly as by set_phase3.  Kernels
 * [rows][N_m][N_t]: F (rows N_d), F_q and its premultiplied Gq (rows N_q;
 * gq NULL: premultiplied on the device with prior3).  LTB_NUMERICAL for a
 * negative posterior variance beyond -1e-10 ||Gamma_post_q|| (:276-282). */
ltb_status ltb_engine_form_q(ltb_engine* e, const double* f_kernel, const double* fq_kernel,
                             const double* gq_kernel, const double* prior3, int nd, int nq, int nm,
                             int nt, int ptr_kind);
/* generated F (stream_f) and F_q (stream_fq) kernels, Gq premultiplied */
ltb_status ltb_engine_form_q_generated(ltb_engine* e, uint64_t seed, uint64_t stream_f,
                                       uint64_t stream_fq, int nq, double h_x, double gamma,
                                       double delta);
/* Q (N_q N_t x N_d N_t, column-major, ldq) and, after form_Q, the full
 * Gamma_post_q and prior QoI covariance (m x m, ldg); any output nullable
 * (the Q() / gamma_post_q() / prior_qoi_cov() accessors, :287-306) */
ltb_status ltb_engine_export_phase3(const ltb_engine* e, double* Q, size_t ldq, double* gpost,
                                    double* prior_cov, size_t ldg, int ptr_kind);
/* device milliseconds of the last form_K / factorize / form_Q (nullable) */
ltb_status ltb_engine_offline_ms(const ltb_engine* e, double* formk_ms, double* factorize_ms,
                                 double* formq_ms);
/* K (after form_K) or L (after factorize / set_factor) as an n x n
 * column-major matrix with leading dimension ld: lower triangle, zeros
 * above (the reference's K() / chol_lower() accessors) */
ltb_status ltb_engine_export_lower(const ltb_engine* e, double* out, size_t ld, int ptr_kind);

/* solve_k_inplace (bayes_engine.cpp:236-240): y <- L^{-T} L^{-1} y */
ltb_status ltb_engine_solve_k(const ltb_engine* e, ltb_scratch* s, double* y, int ptr_kind);

/* infer_map timed region (bayes_engine.cpp:311-320): m_map = G* K^{-1} d.
 * seconds (nullable) receives the device time of the call. */
ltb_status ltb_engine_infer_map(const ltb_engine* e, ltb_scratch* s, const double* d,
                                double* m_map, double* seconds, int ptr_kind);

/* forecast q = F_q m (acceptance_main.cpp:243-264 route) */
ltb_status ltb_engine_forecast(const ltb_engine* e, ltb_scratch* s, const double* m,
                               double* q, int ptr_kind);

/* ---- Q d forecast with credible intervals (predict_qoi) ---- */

/* set_phase3 (bayes_engine.cpp:218-234), online part: Q (Nq*Nt x Nd*Nt,
 * column-major with leading dimension ldq -- Eigen storage) and the
 * diagonal of Gamma_post_q (Nq*Nt).  Both copied to the device. */
ltb_status ltb_engine_set_phase3(ltb_engine* e, const double* Q, size_t ldq,
                                 const double* gpost_q_diag, int ptr_kind);

/* predict_qoi (bayes_engine.cpp:340-362): q = Q d; lo / hi = q -/+ z
 * sqrt(max(diag Gamma_post_q, 0)) with z = 1.96 at level 0.95, else the
 * normal quantile of (1+level)/2 (Acklam + one Halley step, :39-75).
 * LTB_CONFIG unless 0 < level < 1; LTB_STATE without set_phase3.  lo / hi
 * nullable. */
ltb_status ltb_engine_predict_qoi(const ltb_engine* e, ltb_scratch* s, const double* d,
                                  double level, double* q, double* lo, double* hi,
                                  double* seconds, int ptr_kind);

/* normal_quantile (bayes_engine.cpp:39-75); LTB_CONFIG unless 0 < p < 1 */
ltb_status ltb_normal_quantile(double p, double* out);

/* ---- artifact loaders (io.cpp) ---- */
/* FNV-1a 64-bit hash of a file (io.cpp:198-219), for manifest checks */
ltb_status ltb_fnv1a64_file(const char* path, uint64_t* out);
/* set_factor from a DNSM1 archive (io.cpp:102-136; "DNSM1", u64 rows, cols,
 * symmetric flag, row-major doubles), streamed in 64-row panels straight
 * into the packed tiles; the strict upper part is ignored (chol.dnsm may
 * hold K there, bayes_engine.cpp:180-193).  Single-GPU engines only. */
ltb_status ltb_engine_load_factor_dnsm(ltb_engine* e, const char* path);
/* writers, the inverse of the loaders (io.cpp:40-85 write_kernel, :102-115
 * write_dense), written to a temp name in the target directory and renamed
 * (atomic_write); m is column-major with leading dimension ld (host or
 * device), written row-major as DNSM1 does */
ltb_status ltb_write_btpz(const char* path, const double* kernel_rck, int rows, int cols, int nt, int tag,
                          int ptr_kind);
ltb_status ltb_write_dnsm(const char* path, const double* m, int rows, int cols, size_t ld, int symmetric,
                          int ptr_kind);
/* set_phase3 from Q.dnsm and Gamma_post_q.dnsm (workflow.cpp:325-330) */
ltb_status ltb_engine_load_phase3_dnsm(ltb_engine* e, const char* q_path, const char* gpost_path);

/* diagnostics: enable != 0 makes the TRSV sweeps record globaltimer stamps
 * (forward chain steps, transposed chain steps, forward worker hand-offs,
 * transposed worker hand-offs: 4 nb values, then the launch start); with
 * host_out the last record (up to n values) is copied out.  enable = 0
 * stops recording. */
ltb_status ltb_engine_trsv_trace(ltb_engine* e, int enable, unsigned long long* host_out, int n);

/* diagnostics: the distributed K^{-1} apply emulated on ONE GPU -- P ranks'
 * row-cyclic shards of the synthetic factor (seed) and one cooperative
 * launch playing all P ranks; x_host = rank 0's K^{-1} b, max_rank_diff =
 * largest deviation of the other ranks' replicated results. */
ltb_status ltb_debug_dtrsv_emulated(int n, int P, uint64_t seed, const double* b_host,
                                    double* x_host, double* max_rank_diff, double* seconds);

/* infer_map's untimed normal-equation residual (bayes_engine.cpp:322-336):
 * || (F*F / sigma2 + Gamma_prior^{-1}) m_map - F* d / sigma2 || / || F* d / sigma2 ||,
 * evaluated with three F-plan applies and the prior precision A_x^2 per time
 * slice (prior.cpp:44-47,82-92).  set_residual_model gives the engine the F
 * plan (not only G*), sigma2 and the prior {h_x, gamma, delta}. */
ltb_status ltb_engine_set_residual_model(ltb_engine* e, const ltb_plan* plan_f, double sigma2,
                                         double h_x, double gamma, double delta);
ltb_status ltb_engine_map_residual(const ltb_engine* e, ltb_scratch* s, const double* d,
                                   const double* m_map, double* rel_residual, int ptr_kind);

/* integrate_displacement (bayes_engine.cpp:411-419): out[x] = dt_obs *
 * sum_j m[x][j] of a SpaceMajorRows field (n_rows x n_time) */
/* ---- distributed offline phase 2 (one process per GPU, world > 1) ----
 * form_K (bayes_engine.cpp:136-172) and factorize (:176-209) straight into
 * the row-cyclic layout the distributed K^{-1} reads, so config 5 (n =
 * 252,000, 254 GB) runs on a real factor.  Collective over NCCL: rank 0 gets
 * an id with ltb_nccl_unique_id, every rank passes it to ltb_engine_set_comm
 * (after ltb_engine_set_world).  form_K takes the GLOBAL N_m of the
 * generated F kernel (F and its prior-premultiplied G, full, on every rank);
 * factorize leaves each rank's block rows of L and prepares the K^{-1} apply
 * (IPC connect as after ltb_engine_set_factor_generated).  world == 1 runs
 * the same code without NCCL. */
ltb_status ltb_nccl_unique_id(void* out128);
ltb_status ltb_engine_set_comm(ltb_engine* e, const void* id128);
ltb_status ltb_engine_form_k_generated_dist(ltb_engine* e, long long nm_total, uint64_t seed, uint64_t stream,
                                            double h_x, double gamma, double delta, double sigma2);
ltb_status ltb_engine_factorize_dist(ltb_engine* e);

/* reindex (core.hpp:92-95, core.cpp:40-51): bijective permutation of an
 * n_rows x n_time series between TimeMajorBlocks (j * n_rows + r) and
 * SpaceMajorRows (r * n_time + j) -- bit exact (a pure permutation).  Host
 * pointers: synchronous; device pointers: asynchronous on cuda_stream (NULL =
 * legacy default stream).  from == to copies; in == out only then. */
ltb_status ltb_reindex(const double* in, int n_rows, int n_time, int from_layout, int to_layout,
                       double* out, int ptr_kind, void* cuda_stream);

ltb_status ltb_integrate_displacement(const double* m, int n_rows, int n_time, double dt_obs,
                                      double* out, int ptr_kind);

/* infer_map + forecast in one call: m_map and q (either nullable) */
ltb_status ltb_engine_infer_and_forecast(const ltb_engine* e, ltb_scratch* s,
                                         const double* d, double* m_map, double* q,
                                         double* seconds, int ptr_kind);

#ifdef __cplusplus
}
#endif

#endif /* LTB_H */
