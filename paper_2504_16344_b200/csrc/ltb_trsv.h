// ltb_trsv.h -- K^{-1} application through the dense lower Cholesky factor
// (replaces InferenceEngine::solve_k_inplace, bayes_engine.cpp:236-240:
// Eigen triangularView<Lower>().solveInPlace then its transpose).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ltb {

constexpr int kTB = 64;  // factor tile edge

// Lower factor packed as 64x64 tiles (I, J), J <= I, tile index
// I (I+1)/2 + J, each tile column-major (row fastest).  The last tile row /
// column is padded with the identity.  dinv[I] holds L_II^{-1}
// (column-major), inverted on the device once at set_factor time.
struct TriFactor {
  int n = 0;
  int nb = 0;
  double* tiles = nullptr;
  double* dinv = nullptr;
  unsigned* flags = nullptr;  // 2 * nb epoch flags (forward, transposed)
  int* status = nullptr;      // device error word (spin timeout)
  unsigned epoch = 0;
  size_t bytes = 0;
};

cudaError_t trsv_alloc(TriFactor& t, int n);
void trsv_free(TriFactor& t);
// pack from a device column-major matrix (only the lower triangle is read)
cudaError_t trsv_pack_colmajor(TriFactor& t, const double* L, size_t ld, cudaStream_t st);
// pack the synthetic factor (ltb_gen.cuh gen_factor_entry)
cudaError_t trsv_pack_generated(TriFactor& t, uint64_t seed, cudaStream_t st);
cudaError_t trsv_invert_diag(TriFactor& t, cudaStream_t st);
// y <- L^{-T} L^{-1} y (device vector of length n); returns cudaErrorLaunchTimeout
// if a dependency wait timed out.  Launches 2 kernels.
cudaError_t trsv_solve(TriFactor& t, double* y, cudaStream_t st);

}  // namespace ltb
