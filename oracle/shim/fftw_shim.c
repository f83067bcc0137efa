#define _POSIX_C_SOURCE 200112L
/* FFTW3 shim implementation over orc_fft (TEST INFRASTRUCTURE ONLY). */
#include "fftw3.h"
#include <stdlib.h>
#include "../ltb_oracle.h"

struct ltb_shim_fftw_plan_s {
  orc_fft* fft;
  int r2c;
};

void* fftw_malloc(size_t n) {
  void* p = NULL;
  if (posix_memalign(&p, 64, n ? n : 1) != 0) return NULL;
  return p;
}
void fftw_free(void* p) { free(p); }

static fftw_plan make(int n, int r2c) {
  if (n < 1) return NULL;
  fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
  p->fft = orc_fft_create(n);
  p->r2c = r2c;
  return p;
}
fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags) {
  (void)in; (void)out; (void)flags;
  return make(n, 1);
}
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags) {
  (void)in; (void)out; (void)flags;
  return make(n, 0);
}
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  orc_rfft(p->fft, in, (double*)out);
}
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  orc_irfft(p->fft, (const double*)in, out);
}
void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  orc_fft_destroy(p->fft);
  free(p);
}
