/*
 * Minimal FFTW3 interface shim for compiling the reference's
 * proj/src/fft_matvec.cpp verbatim (TEST INFRASTRUCTURE ONLY).
 *
 * FFTW3 is absent from this image and unpinned by the reference
 * (proj/CMakeLists.txt:15, bare find_library).  The seven entry points the
 * reference calls (fft_matvec.cpp:88-91,101,148,172,189,210 and the
 * malloc/free/destroy trio) are backed by oracle/ltb_oracle.c's mixed-radix
 * FFT with FFTW's conventions: unnormalised, r2c keeps n/2+1 bins, c2r reads
 * Hermitian input.
 */
#ifndef LTB_SHIM_FFTW3_H
#define LTB_SHIM_FFTW3_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef double fftw_complex[2];
typedef struct ltb_shim_fftw_plan_s* fftw_plan;
#define FFTW_ESTIMATE (1U << 6)
void* fftw_malloc(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
