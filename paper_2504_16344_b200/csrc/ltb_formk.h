// ltb_formk.h -- offline phase 2 on the device: form_K (bayes_engine.cpp:
// 136-172) and the in-place Cholesky factorize (:176-209), writing straight
// into the packed 64x64 lower tiles the K^{-1} apply reads (ltb_trsv.h).
//
// form_K.  Column (s, j) of K is F G* e_(s,j) + sigma2 e_(s,j).  With
// G* e_(s,j) read off the G kernel (read_gstar_column, :122-134) and F
// causal, entry (r, t; s, j) is
//     K = sum_x sum_{tau <= min(t, j)} f[r][x][t - tau] g[s][x][j - tau]
// which satisfies the diagonal recurrence K(t, j) = A(t, j) + K(t-1, j-1)
// inside every (r, s) block, with the lag Gram matrix
//     A[(r, a), (s, b)] = sum_x f[r][x][a] g[s][x][b]       (n x n x N_m).
// A is one dense FP64 contraction -- DMMA (FP64 tensor core) tiles fed by a
// cp.async multi-stage pipeline -- and the recurrence is one O(n^2) pass.
// Only the lower triangle is formed: G = F Gamma_x with Gamma_x symmetric
// makes K symmetric, which is what the reference's symmetrisation restores.
//
// factorize.  Right-looking tile Cholesky on the packed tiles: per block
// column k, one launch factors L_kk (and L_kk^{-1}) in shared memory and
// forms the panel L_ik = A_ik L_kk^{-T} with DMMA; one launch applies the
// trailing update A_ij -= L_ik L_jk^T with DMMA.
#pragma once

#include <cuda_runtime.h>

#include "ltb_nccl.h"
#include "ltb_trsv.h"

namespace ltb {

// t allocated by trsv_alloc(t, n = nd * nt, 1, 0).  f, g: device kernels
// [nd][nm][nt].  Writes the lower tiles of K (identity padding included).
cudaError_t formk_device(TriFactor& t, const double* f, const double* g, int nd, int nm, int nt,
                         double sigma2, cudaStream_t st);
// In place K -> L.  Returns cudaErrorInvalidValue (and leaves *bad_block the
// first failing block column) when K is not positive definite.
cudaError_t cholesky_packed(TriFactor& t, cudaStream_t st, int* bad_block);
// Packed lower tiles -> column-major n x n device matrix (lower triangle
// incl. the diagonal written; the strict upper part is left untouched).
cudaError_t export_lower(const TriFactor& t, double* out, size_t ld, cudaStream_t st);
// launches issued by the last formk_device / cholesky_packed / ... call
int formk_last_launches();

// ---- form_Q / form_qoi_cov (bayes_engine.cpp:242-285) ----
// out (column-major, ld) = the dense (nda N_t) x (ndb N_t) product of the
// block-lower-triangular-Toeplitz map of kernel a with the adjoint of the map
// of kernel b (both [nd][nm][nt]): F_a G_b^* -- R = F Gq* and P = Fq Gq*.
// Same lag-Gram contraction + diagonal recurrence as form_K.
cudaError_t block_toeplitz_product(const double* a, int nda, const double* b, int ndb, int nm, int nt,
                                   double* out, size_t ld, cudaStream_t st);
// K^{-1} R for nrhs_pad (multiple of 64) columns: R, X column-major n_pad x
// nrhs_pad (ld = nb * 64, padding zero).  Forward sweep R -> Y (in X), then
// (optional) YtY = Y^T Y (m x m, = R^T K^{-1} R), then the transposed sweep
// Y -> K^{-1} R (in R).  Both R and X are overwritten.
cudaError_t trsm_solve_k(const TriFactor& t, double* R, double* X, size_t ld, int nrhs_pad, double* YtY,
                         int m, cudaStream_t st);
// gpost = sym(P - YtY) (P already symmetric), diag = its diagonal
cudaError_t qoi_covariance(const double* P, const double* YtY, int m, double* gpost, double* diag,
                           cudaStream_t st);
cudaError_t symmetrize(double* A, int m, cudaStream_t st);
// Q (m x n, column-major, ld m) = X^T
cudaError_t transpose_to(const double* X, size_t ldx, int n, int m, double* Q, cudaStream_t st);

// ---- distributed (t.P ranks, one process per GPU; t from trsv_alloc(t, n, P, rank)) ----
// form_K into this rank's block rows: f, g are the FULL kernels [nd][nm][nt]
// on every rank; collective over comm (the recurrence carries).  P == 1
// runs the same code without NCCL.
cudaError_t formk_device_dist(TriFactor& t, const double* f, const double* g, int nd, int nm, int nt, double sigma2,
                              const Nccl* api, ncclComm_t comm, cudaStream_t st, const char** err);
// in-place K -> L over the ranks (collective); cudaErrorInvalidValue + bad_block
// on every rank when K is not positive definite
cudaError_t cholesky_dist(TriFactor& t, const Nccl* api, ncclComm_t comm, cudaStream_t st, int* bad_block,
                          const char** err);

}  // namespace ltb
