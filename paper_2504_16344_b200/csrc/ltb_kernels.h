// ltb_kernels.h -- host-side launchers for the sm_100a kernels (internal to
// libltb.so; the public surface is include/ltb.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ltb_fft.cuh"

namespace ltb {

// ---- time-axis transforms (K1 / K4, K7 plan build) ----
struct RfftSrc {
  // logical row g reads input row in_row(g) = (g % P) * Q + g / P + c0
  const double* in;  // memory mode (nullptr -> generated mode)
  uint64_t gen_key;  // generated mode: value = gen_uniform_keyed(key, in_row*nt + k)
  int P;
  long long Q;
  long long c0;
  int bulk = 0;  // set by the launcher: contiguous, 16-byte aligned rows
  // output column of logical row g: (g / oP) * oQ + g % oP + o0 (oP = 0: g);
  // lets a slab of kernel rows land in its F-hat columns [f][c][r0 + rr]
  long long oP = 0, oQ = 0, o0 = 0;
};

// Forward: rows [0, nrows) of real length nt, zero padded to N = 2 nt,
// out[f * ld + g] = r2c(row g)[f] for f < nt + 1.
cudaError_t launch_rfft_rows(const FftDesc& d, const RfftSrc& src, int nt, long long nrows,
                             double2* out, long long ld, cudaStream_t st);

// Inverse: spectrum of row g is in[f * ld_f + p * ld_p + g] summed over
// p < nparts (the GEMV-N partial slabs); out[g * nt + j] = c2r(...)[j] * scale
// for j < nt.
cudaError_t launch_irfft_rows(const FftDesc& d, const double2* in, long long ld_f,
                              long long ld_p, int nparts, int nt, long long nrows,
                              double scale, double* out, cudaStream_t st);

// c2r + truncate + scale of the spectra in[f * ld_f + g] into rows mout (as
// launch_irfft_rows), then pad + r2c of those rows into xout[f * ld_x + g]
// (as launch_rfft_rows): one pass for an F* apply feeding an F apply
cudaError_t launch_c2r_r2c_rows(const FftDesc& d, const double2* in, long long ld_f, int nt, long long nrows,
                                double scale, double* mout, double2* xout, long long ld_x, cudaStream_t st);

size_t fft_smem_bytes(int n, int* pairs_per_cta);

// register-resident two-pass path (ltb_fft_reg.cu) for N in {128, 256, 512,
// 840, 1024}; same contracts as the three launchers above
bool reg_fft_supported(int n);
cudaError_t reg_rfft_rows(const FftDesc& d, const RfftSrc& src, int nt, long long nrows, double2* out, long long ld,
                          cudaStream_t st);
cudaError_t reg_irfft_rows(const FftDesc& d, const double2* in, long long ld_f, long long ld_p, int nparts, int nt,
                           long long nrows, double scale, double* out, cudaStream_t st);
cudaError_t reg_c2r_r2c_rows(const FftDesc& d, const double2* in, long long ld_f, int nt, long long nrows,
                             double scale, double* mout, double2* xout, long long ld_x, cudaStream_t st);

// four-step path (ltb_fft_big.cu): N = n1 n2 with both factors <= max_len
bool big_fft_split(int n, int max_len, int* n1, int* n2);
cudaError_t big_rfft_rows(const BigFft& b, const RfftSrc& src, int nt, long long nrows, double2* out, long long ld,
                          cudaStream_t st);
cudaError_t big_irfft_rows(const BigFft& b, const double2* in, long long ld_f, long long ld_p, int nparts, int nt,
                           long long nrows, double scale, double* out, cudaStream_t st);

// ---- per-frequency GEMVs (K2 / K3) ----
struct GemvShape {
  int nd;          // rows of each frequency block
  long long nm;    // columns (the per-frequency stride of F-hat / x-hat)
  int nf;          // frequencies
  int unit_cols;   // columns per work unit
  int units_per_f;
  // column window [c0, c0 + nc) this launch covers (the host-pointer applies
  // pipeline the copies against column chunks); GEMV-N with accumulate != 0
  // adds the window's products into y instead of overwriting it
  long long c0 = 0, nc = 0;
  int accumulate = 0;
};
GemvShape gemv_shape(int nd, long long nm, int nf, int unit_cols_hint);
GemvShape gemv_window(const GemvShape& s, long long c0, long long nc, int accumulate);

// Y[f][r] = sum_c Fhat[f][c][r] * X[f][c]; per-unit partials go to
// `partials` (gemv_n_partials(s) entries), `tickets` holds
// nf * gemv_n_row_tiles(s) counters (zeroed by the launcher).
size_t gemv_n_partials(const GemvShape& s);
int gemv_n_row_tiles(const GemvShape& s);
cudaError_t launch_gemv_n(const GemvShape& s, const double2* fhat, const double2* x,
                          double2* partials, double2* y, unsigned* tickets, cudaStream_t st);
// Xo[f][c] = sum_r conj(Fhat[f][c][r]) * D[f][r]
cudaError_t launch_gemv_h(const GemvShape& s, const double2* fhat, const double2* dhat,
                          double2* xo, cudaStream_t st);

// ---- reductions ----
// sum |z|^2 over z[0, n) into *out (deterministic two-level tree); work must
// hold at least 1024 doubles.
cudaError_t launch_sqnorm(const double2* z, long long n, double* work, double* out,
                          cudaStream_t st);

// ---- generators ----
cudaError_t launch_gen_fill(uint64_t key, uint64_t index0, long long n, double* out,
                            cudaStream_t st);

}  // namespace ltb
