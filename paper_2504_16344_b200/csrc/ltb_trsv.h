// ltb_trsv.h -- K^{-1} application through the dense lower Cholesky factor
// (replaces InferenceEngine::solve_k_inplace, bayes_engine.cpp:236-240:
// Eigen triangularView<Lower>().solveInPlace then its transpose).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ltb {

constexpr int kTB = 64;    // factor tile edge
constexpr int kLook = 3;   // diagonal-chain lookahead depth (tiles per chain step)

// Lower factor packed as 64x64 tiles (I, J), J <= I, tile index
// I (I+1)/2 + J, each tile column-major (row fastest).  The last tile row /
// column is padded with the identity.  Precomputed once at set_factor time:
//   dinv[I]     = L_II^{-1}
//   mf[I][k-1]  = L_II^{-1} L_{I,I-k}          (k = 1..kLook, forward chain)
//   mb[I][k-1]  = L_II^{-T} L_{I+k,I}^T        (k = 1..kLook, transposed chain)
struct TriFactor {
  int n = 0;
  int nb = 0;
  double* tiles = nullptr;
  double* dinv = nullptr;
  double* mf = nullptr;
  double* mb = nullptr;
  double* work = nullptr;  // 4 * nb * 64 hand-off buffers [yf | x | cf | cb]
  int* status = nullptr;   // device error word (spin timeout / bad pivot)
  unsigned long long* trace = nullptr;  // diagnostic timestamps, 4 nb + 1 (optional)
  size_t bytes = 0;
};

cudaError_t trsv_alloc(TriFactor& t, int n);
void trsv_free(TriFactor& t);
// pack from a device column-major matrix (only the lower triangle is read)
cudaError_t trsv_pack_colmajor(TriFactor& t, const double* L, size_t ld, cudaStream_t st);
// pack the synthetic factor (ltb_gen.cuh gen_factor_entry)
cudaError_t trsv_pack_generated(TriFactor& t, uint64_t seed, cudaStream_t st);
// invert the diagonal tiles and build the chain tiles; returns
// cudaErrorInvalidValue on a zero / non-finite pivot
cudaError_t trsv_prepare(TriFactor& t, cudaStream_t st);
// x = L^{-T} L^{-1} b for a device vector b of length nb * 64 (zero padded);
// the result is left in trsv_result(t).  One memset + one cooperative
// launch; a dependency-wait timeout is reported through t.status.
cudaError_t trsv_solve(TriFactor& t, const double* b, cudaStream_t st);
double* trsv_result(TriFactor& t);

}  // namespace ltb
