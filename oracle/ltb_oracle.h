/*
 * ltb_oracle.h -- CPU restatement of the reference's online hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path (paper_2504_16344_b200/) never links,
 * imports or calls anything under oracle/.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to the reference's proj/ directory).  Parity of this restatement is pinned
 * against golden vectors produced by the reference's own sources
 * (oracle/_ref, built from /root/reference by oracle/Makefile) -- see
 * tests/golden/make_golden.cpp and tests/test_oracle_golden.py.
 *
 * Conventions (fft_matvec.hpp:12-28):
 *   - vectors are SpaceMajorRows: row r's N_t samples are contiguous;
 *   - kernels are [row][col][lag], lag contiguous (core.hpp:114-140);
 *   - forward DFT unnormalised, inverse scaled by 1/(2 N_t), padded length
 *     exactly 2 N_t, first N_t samples kept.
 */
#ifndef LTB_ORACLE_H
#define LTB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror include/ltb.h) ---- */
enum {
  ORC_OK = 0,
  ORC_DIMENSION = 1,
  ORC_LAYOUT = 2,
  ORC_NUMERICAL = 3,
  ORC_CAPACITY = 4,
  ORC_STATE = 5
};

/* ---- mixed-radix complex FFT (any n >= 1), unnormalised ---- */
typedef struct orc_fft orc_fft;
orc_fft* orc_fft_create(int n);
void orc_fft_destroy(orc_fft* p);
int orc_fft_size(const orc_fft* p);
/* in/out: n interleaved complex (2n doubles); in-place allowed. sign=-1
 * forward (exp(-2 pi i jk/n)), +1 backward. */
void orc_fft_exec(const orc_fft* p, const double* in, double* out, int sign);
/* real -> half complex (n/2+1 bins), FFTW r2c convention */
void orc_rfft(const orc_fft* p, const double* x, double* X);
/* half complex (n/2+1 bins) -> real n, FFTW c2r convention (unnormalised,
 * the imaginary parts of the DC and, for even n, Nyquist bins ignored) */
void orc_irfft(const orc_fft* p, const double* X, double* x);

/* ---- MatvecPlan restatement (fft_matvec.cpp:73-111,139-217,124-137) ---- */
typedef struct orc_plan orc_plan;
int orc_plan_create(const double* kernel_rck, int rows, int cols, int nt,
                    orc_plan** out);
void orc_plan_destroy(orc_plan* p);
void orc_plan_dims(const orc_plan* p, int* rows, int* cols, int* nt,
                   int* npad, int* nf);
/* kernel_hat, [f][c][r] complex interleaved, nf*rows*cols entries */
const double* orc_plan_khat(const orc_plan* p);
void orc_apply_raw(const orc_plan* p, const double* in, double* out);
void orc_apply_adjoint_raw(const orc_plan* p, const double* in, double* out);
double orc_kernel_hat_sqnorm(const orc_plan* p);

/* fft_matvec.cpp:267-315: FFT-free time-domain product.  Returns
 * ORC_CAPACITY when rows*nt*cols*nt*8 > cap (cap 0 = unlimited). */
int orc_dense_apply(const double* kernel_rck, int rows, int cols, int nt,
                    const double* v, int adjoint, uint64_t mem_cap_bytes,
                    double* out);

/* core.cpp:40-51: layout permutation (bit exact). to_time_major=1 converts
 * SpaceMajorRows -> TimeMajorBlocks, 0 the inverse. */
void orc_reindex(const double* in, int rows, int nt, int to_time_major,
                 double* out);

/* ---- counter-based synthetic inputs (shared bit-for-bit with the GPU
 * generator in paper_2504_16344_b200/csrc/ltb_gen.cuh) ---- */
uint64_t orc_gen_hash(uint64_t seed, uint64_t stream, uint64_t index);
double orc_gen_uniform(uint64_t seed, uint64_t stream, uint64_t index);
void orc_gen_fill(uint64_t seed, uint64_t stream, uint64_t index0, size_t n,
                  double* out);
/* kernel shard: rows x [c0, c0+cols) columns of a rows x nm_total x nt
 * generated kernel, written [row][local col][lag]. */
void orc_gen_kernel(uint64_t seed, uint64_t stream, int rows, int nm_total,
                    int c0, int cols, int nt, double* out);
/* synthetic well-conditioned lower Cholesky factor entry L(i,j) */
double orc_gen_factor_entry(uint64_t seed, int n, int i, int j);
/* dense column-major n x n factor (upper part zero) */
void orc_gen_factor(uint64_t seed, int n, double* L);

/* ---- K^{-1} apply (bayes_engine.cpp:236-240) ---- */
/* column-major factor with leading dimension ld; only the lower triangle
 * is read (the strict upper part may hold anything, bayes_engine.cpp:180-193) */
void orc_trsv_lower(const double* L, int n, size_t ld, double* y);
void orc_trsv_lower_t(const double* L, int n, size_t ld, double* y);
void orc_solve_k(const double* L, int n, size_t ld, double* y);
/* same, factor regenerated on the fly from orc_gen_factor_entry */
void orc_solve_k_gen(uint64_t seed, int n, double* y);
/* same, blocked and split over `threads` POSIX threads (config-5 scale) */
int orc_solve_k_gen_mt(uint64_t seed, int n, double* y, int threads);

/* ---- prior (prior.cpp:9-39,45-48,82-92,108-134) ---- */
/* Gamma_x = A_x^{-2}, A_x = delta I - gamma L (Neumann); premultiply each
 * kernel row's [col][lag] slab: g[s][.][k] = Gamma_x f[s][.][k] */
int orc_prior_premultiply(const double* f_rck, int rows, int nm, int nt,
                          double h_x, double gamma, double delta,
                          double* g_rck);
/* Gamma_prior^{-1} v on a TimeMajorBlocks field (nm x nt) */
int orc_prior_apply_precision(const double* v_tm, int nm, int nt, double h_x,
                              double gamma, double delta, double* out_tm);

/* ---- offline phase 2 (bayes_engine.cpp:122-209) ---- */
/* form_K: column i of K (n = rows * nt, column-major, ld n) is
 * plan_F.apply(G* e_i) with G* e_i from plan_G.apply_adjoint(e_i)
 * (mode 0, ColumnByColumn) or read off the G kernel (mode 1, FusedBatched,
 * read_gstar_column :122-134); K(i, i) += sigma2; then the asymmetry
 * measure (*asym) and the symmetrisation (:153-171).  0 on success. */
int orc_form_k(const double* f_rck, const double* g_rck, int rows, int nm, int nt,
               double sigma2, int mode, double* K, double* asym);
/* factorize: in-place lower Cholesky of the column-major n x n A (ld);
 * the strict upper part is zeroed (Eigen LLT matrixL(), :195-208).
 * Returns 0, or j + 1 for a non-positive pivot in column j. */
int orc_cholesky(double* A, int n, size_t ld);

/* form_Q + form_qoi_cov (bayes_engine.cpp:242-285): with n = nd * nt,
 * m = nq * nt, R = F Gq* (column i = plan_F.apply(read_gstar_column(gq, i))),
 * X = K^{-1} R (solve_k per column, factor L column-major ld n),
 * Q = X^T (m x n, column-major ld m); P = Fq Gq* symmetrised (m x m);
 * Gamma_post_q = P - R^T X symmetrised (m x m).  Returns 0, or 2 when a
 * diagonal entry of Gamma_post_q < -1e-10 ||Gamma_post_q||_F. */
int orc_form_q(const double* f_rck, const double* fq_rck, const double* gq_rck, int nd, int nq,
               int nm, int nt, const double* L, double* Q, double* gpost, double* prior_cov);

/* ---- online phase (bayes_engine.cpp:307-338) ---- */
/* m_map = G* K^{-1} d: y = copy(d); solve_k(y); m = plan_g.apply_adjoint(y) */
void orc_infer_map(const double* L, size_t ld, const orc_plan* plan_g,
                   const double* d, double* m_map);

#ifdef __cplusplus
}
#endif

#endif /* LTB_ORACLE_H */
