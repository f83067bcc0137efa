/*
 * ltb_oracle.c -- CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY; see ltb_oracle.h for the rules on who may use it).
 *
 * Built with -O2 -ffp-contract=off so every product/sum is a separately
 * rounded IEEE operation, in the same order as the reference loops it
 * restates.  Reference paths are relative to /root/reference/proj.
 */
#define _POSIX_C_SOURCE 200809L /* pthread barriers under -std=c11 */
#include "ltb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Mixed-radix FFT.  The reference delegates to FFTW3 (fft_matvec.cpp:88-91,
 * unpinned version); FFTW is absent from this image, so this is a plain
 * recursive decimation-in-time Cooley-Tukey for any n (radices 4,2,3,5,7 and
 * a generic O(p^2) combine for any other prime p).  Twiddles are computed in
 * long double and mirrored so W[n-j] == conj(W[j]) exactly.  Its correctness
 * is pinned by the reference's FFT-free dense_apply (golden vectors) and by
 * numpy.fft in tests/test_oracle_golden.py.
 * ------------------------------------------------------------------------ */

#define ORC_MAXFAC 64

struct orc_fft {
  int n;
  int nfac;
  int fac[ORC_MAXFAC];
  double* wr; /* cos(2 pi j / n), j in [0, n) */
  double* wi; /* sin(2 pi j / n) */
};

static void twiddle_table(int n, double* wr, double* wi) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int j = 0; j <= n / 2; ++j) {
    double c, s;
    if ((4L * j) % n == 0) { /* exact quadrant points */
      const int q = (int)((4L * j) / n);
      c = (q == 0) ? 1.0 : (q == 2 ? -1.0 : 0.0);
      s = (q == 1) ? 1.0 : 0.0;
    } else {
      const long double a = two_pi * (long double)j / (long double)n;
      c = (double)cosl(a);
      s = (double)sinl(a);
    }
    wr[j] = c;
    wi[j] = s;
    if (j > 0 && j < n - j) {
      wr[n - j] = c;
      wi[n - j] = -s;
    }
  }
}

orc_fft* orc_fft_create(int n) {
  if (n < 1) return NULL;
  orc_fft* p = (orc_fft*)calloc(1, sizeof(orc_fft));
  p->n = n;
  int m = n;
  static const int pref[] = {4, 2, 3, 5, 7};
  for (int k = 0; k < 5; ++k) {
    while (m % pref[k] == 0 && p->nfac < ORC_MAXFAC) {
      p->fac[p->nfac++] = pref[k];
      m /= pref[k];
    }
  }
  for (int f = 11; m > 1; f += 2) {
    while (m % f == 0) {
      p->fac[p->nfac++] = f;
      m /= f;
    }
    if ((long)f * f > m && m > 1) {
      p->fac[p->nfac++] = m;
      m = 1;
    }
  }
  p->wr = (double*)malloc(sizeof(double) * (size_t)n);
  p->wi = (double*)malloc(sizeof(double) * (size_t)n);
  twiddle_table(n, p->wr, p->wi);
  return p;
}

void orc_fft_destroy(orc_fft* p) {
  if (!p) return;
  free(p->wr);
  free(p->wi);
  free(p);
}

int orc_fft_size(const orc_fft* p) { return p->n; }

/* out[0..n) = DFT_n(in[0], in[is], in[2 is], ...), sign -1 forward. */
static void fft_rec(const orc_fft* p, const double* in, size_t is, double* out,
                    int n, int fi, size_t wstep, int sign, double* tmp) {
  if (n == 1) {
    out[0] = in[0];
    out[1] = in[1];
    return;
  }
  const int r = p->fac[fi];
  const int m = n / r;
  for (int q = 0; q < r; ++q) {
    fft_rec(p, in + 2 * (size_t)q * is, is * (size_t)r, out + 2 * (size_t)q * m,
            m, fi + 1, wstep * (size_t)r, sign, tmp);
  }
  const size_t N = (size_t)p->n;
  const size_t rstep = N / (size_t)r; /* W_r = W_N^(N/r) */
  const double sg = (double)sign;
  double* tr = tmp;
  double* ti = tmp + r;
  for (int k = 0; k < m; ++k) {
    for (int q = 0; q < r; ++q) {
      const double yr = out[2 * ((size_t)q * m + k)];
      const double yi = out[2 * ((size_t)q * m + k) + 1];
      const size_t w = ((size_t)q * (size_t)k * wstep) % N;
      const double c = p->wr[w], s = sg * p->wi[w];
      tr[q] = yr * c - yi * s;
      ti[q] = yr * s + yi * c;
    }
    for (int s_ = 0; s_ < r; ++s_) {
      double ar = 0.0, ai = 0.0;
      for (int q = 0; q < r; ++q) {
        const size_t w = ((size_t)((q * s_) % r)) * rstep;
        const double c = p->wr[w], s = sg * p->wi[w];
        ar += tr[q] * c - ti[q] * s;
        ai += tr[q] * s + ti[q] * c;
      }
      out[2 * ((size_t)k + (size_t)s_ * m)] = ar;
      out[2 * ((size_t)k + (size_t)s_ * m) + 1] = ai;
    }
  }
}

void orc_fft_exec(const orc_fft* p, const double* in, double* out, int sign) {
  const size_t n = (size_t)p->n;
  double stack_src[2 * 2048];
  double* src = (n <= 2048) ? stack_src : (double*)malloc(sizeof(double) * 2 * n);
  memcpy(src, in, sizeof(double) * 2 * n);
  int maxr = 2;
  for (int i = 0; i < p->nfac; ++i) maxr = p->fac[i] > maxr ? p->fac[i] : maxr;
  double stack_tmp[256];
  double* tmp = (2 * maxr <= 256) ? stack_tmp : (double*)malloc(sizeof(double) * 2 * (size_t)maxr);
  fft_rec(p, src, 1, out, p->n, 0, 1, sign, tmp);
  if (tmp != stack_tmp) free(tmp);
  if (src != stack_src) free(src);
}

void orc_rfft(const orc_fft* p, const double* x, double* X) {
  const int n = p->n;
  double stack_buf[2 * 2048];
  double* z = (n <= 2048) ? stack_buf : (double*)malloc(sizeof(double) * 2 * (size_t)n);
  for (int j = 0; j < n; ++j) {
    z[2 * j] = x[j];
    z[2 * j + 1] = 0.0;
  }
  orc_fft_exec(p, z, z, -1);
  memcpy(X, z, sizeof(double) * 2 * (size_t)(n / 2 + 1));
  if (z != stack_buf) free(z);
}

void orc_irfft(const orc_fft* p, const double* X, double* x) {
  const int n = p->n;
  double stack_buf[2 * 2048];
  double* z = (n <= 2048) ? stack_buf : (double*)malloc(sizeof(double) * 2 * (size_t)n);
  const int nh = n / 2;
  for (int k = 0; k <= nh; ++k) {
    z[2 * k] = X[2 * k];
    z[2 * k + 1] = X[2 * k + 1];
  }
  z[1] = 0.0; /* DC imaginary part ignored (Hermitian input) */
  if (n % 2 == 0) z[2 * nh + 1] = 0.0; /* Nyquist imaginary part ignored */
  for (int k = 1; k < n - nh; ++k) { /* mirror: Z[n-k] = conj(Z[k]) */
    z[2 * (n - k)] = X[2 * k];
    z[2 * (n - k) + 1] = -X[2 * k + 1];
  }
  orc_fft_exec(p, z, z, +1);
  for (int j = 0; j < n; ++j) x[j] = z[2 * j];
  if (z != stack_buf) free(z);
}

/* ------------------------------------------------------------------------ */
/* MatvecPlan (fft_matvec.cpp:41-55 Impl, :73-111 ctor)                      */
/* ------------------------------------------------------------------------ */

struct orc_plan {
  int rows, cols, nt, npad, nf;
  double* khat; /* [f][c][r] complex: f*rows*cols + c*rows + r (:44-46) */
  orc_fft* fft;
};

int orc_plan_create(const double* kernel, int rows, int cols, int nt,
                    orc_plan** out) {
  *out = NULL;
  /* core.cpp:67-78 check_consistent: dims >= 1, all entries finite */
  if (rows < 1 || cols < 1 || nt < 1) return ORC_DIMENSION;
  const size_t total = (size_t)rows * cols * nt;
  for (size_t i = 0; i < total; ++i) {
    if (!isfinite(kernel[i])) return ORC_NUMERICAL;
  }
  orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
  p->rows = rows;
  p->cols = cols;
  p->nt = nt;
  p->npad = 2 * nt; /* :80 */
  p->nf = nt + 1;   /* :81 */
  p->fft = orc_fft_create(p->npad);
  const size_t bc = (size_t)rows * cols;
  p->khat = (double*)malloc(sizeof(double) * 2 * bc * (size_t)p->nf);
  double* real = (double*)malloc(sizeof(double) * (size_t)p->npad);
  double* hat = (double*)malloc(sizeof(double) * 2 * (size_t)p->nf);
  /* :96-110 -- per (r,c): pad lag series to 2 N_t, r2c, scatter to [f][c][r] */
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < cols; ++c) {
      const double* lag = kernel + ((size_t)r * cols + c) * nt;
      memcpy(real, lag, sizeof(double) * (size_t)nt);
      memset(real + nt, 0, sizeof(double) * (size_t)nt);
      orc_rfft(p->fft, real, hat);
      for (int f = 0; f < p->nf; ++f) {
        const size_t o = (size_t)f * bc + (size_t)c * rows + r;
        p->khat[2 * o] = hat[2 * f];
        p->khat[2 * o + 1] = hat[2 * f + 1];
      }
    }
  }
  free(real);
  free(hat);
  *out = p;
  return ORC_OK;
}

void orc_plan_destroy(orc_plan* p) {
  if (!p) return;
  orc_fft_destroy(p->fft);
  free(p->khat);
  free(p);
}

void orc_plan_dims(const orc_plan* p, int* rows, int* cols, int* nt,
                   int* npad, int* nf) {
  if (rows) *rows = p->rows;
  if (cols) *cols = p->cols;
  if (nt) *nt = p->nt;
  if (npad) *npad = p->npad;
  if (nf) *nf = p->nf;
}

const double* orc_plan_khat(const orc_plan* p) { return p->khat; }

/* :124-137 -- interior frequencies appear twice in the full spectrum */
double orc_kernel_hat_sqnorm(const orc_plan* p) {
  const size_t bc = (size_t)p->rows * p->cols;
  const size_t n = (size_t)p->nf * bc;
  const double* k = p->khat;
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += k[2 * i] * k[2 * i] + k[2 * i + 1] * k[2 * i + 1];
  double edge = 0;
  const size_t last = (size_t)(p->nf - 1) * bc;
  for (size_t i = 0; i < bc; ++i) {
    edge += (k[2 * i] * k[2 * i] + k[2 * i + 1] * k[2 * i + 1]) +
            (k[2 * (last + i)] * k[2 * (last + i)] +
             k[2 * (last + i) + 1] * k[2 * (last + i) + 1]);
  }
  return 2 * s - edge;
}

/* :139-179 -- d = F m */
void orc_apply_raw(const orc_plan* p, const double* in, double* out) {
  const int rows = p->rows, cols = p->cols, nt = p->nt, nf = p->nf;
  double* real = (double*)malloc(sizeof(double) * (size_t)p->npad);
  double* ih = (double*)malloc(sizeof(double) * 2 * (size_t)nf * cols);
  double* oh = (double*)malloc(sizeof(double) * 2 * (size_t)nf * rows);
  for (int c = 0; c < cols; ++c) { /* :143-150 */
    memcpy(real, in + (size_t)c * nt, sizeof(double) * (size_t)nt);
    memset(real + nt, 0, sizeof(double) * (size_t)nt);
    orc_rfft(p->fft, real, ih + 2 * (size_t)c * nf);
  }
  const size_t bc = (size_t)rows * cols;
  for (int f = 0; f < nf; ++f) { /* :151-168 */
    const double* kf = p->khat + 2 * (size_t)f * bc;
    for (int r = 0; r < rows; ++r) {
      oh[2 * ((size_t)r * nf + f)] = 0.0;
      oh[2 * ((size_t)r * nf + f) + 1] = 0.0;
    }
    for (int c = 0; c < cols; ++c) {
      const double xr = ih[2 * ((size_t)c * nf + f)];
      const double xi = ih[2 * ((size_t)c * nf + f) + 1];
      const double* kc = kf + 2 * (size_t)c * rows;
      for (int r = 0; r < rows; ++r) {
        const double ar = kc[2 * r], ai = kc[2 * r + 1];
        oh[2 * ((size_t)r * nf + f)] += ar * xr - ai * xi;
        oh[2 * ((size_t)r * nf + f) + 1] += ar * xi + ai * xr;
      }
    }
  }
  const double scale = 1.0 / p->npad; /* :169-178 */
  for (int r = 0; r < rows; ++r) {
    orc_irfft(p->fft, oh + 2 * (size_t)r * nf, real);
    for (int j = 0; j < nt; ++j) out[(size_t)r * nt + j] = real[j] * scale;
  }
  free(real);
  free(ih);
  free(oh);
}

/* :181-217 -- m = F* d */
void orc_apply_adjoint_raw(const orc_plan* p, const double* in, double* out) {
  const int rows = p->rows, cols = p->cols, nt = p->nt, nf = p->nf;
  double* real = (double*)malloc(sizeof(double) * (size_t)p->npad);
  double* ih = (double*)malloc(sizeof(double) * 2 * (size_t)nf * cols);
  double* dh = (double*)malloc(sizeof(double) * 2 * (size_t)nf * rows);
  for (int r = 0; r < rows; ++r) { /* :185-191 */
    memcpy(real, in + (size_t)r * nt, sizeof(double) * (size_t)nt);
    memset(real + nt, 0, sizeof(double) * (size_t)nt);
    orc_rfft(p->fft, real, dh + 2 * (size_t)r * nf);
  }
  const size_t bc = (size_t)rows * cols;
  for (int f = 0; f < nf; ++f) { /* :192-207 */
    const double* kf = p->khat + 2 * (size_t)f * bc;
    for (int c = 0; c < cols; ++c) {
      double accr = 0.0, acci = 0.0;
      const double* kc = kf + 2 * (size_t)c * rows;
      for (int r = 0; r < rows; ++r) {
        const double ar = kc[2 * r], ai = -kc[2 * r + 1]; /* conj */
        const double br = dh[2 * ((size_t)r * nf + f)];
        const double bi = dh[2 * ((size_t)r * nf + f) + 1];
        accr += ar * br - ai * bi;
        acci += ar * bi + ai * br;
      }
      ih[2 * ((size_t)c * nf + f)] = accr;
      ih[2 * ((size_t)c * nf + f) + 1] = acci;
    }
  }
  const double scale = 1.0 / p->npad; /* :208-216 */
  for (int c = 0; c < cols; ++c) {
    orc_irfft(p->fft, ih + 2 * (size_t)c * nf, real);
    for (int j = 0; j < nt; ++j) out[(size_t)c * nt + j] = real[j] * scale;
  }
  free(real);
  free(ih);
  free(dh);
}

/* :267-315 */
int orc_dense_apply(const double* kernel, int rows, int cols, int nt,
                    const double* v, int adjoint, uint64_t cap, double* out) {
  if (rows < 1 || cols < 1 || nt < 1) return ORC_DIMENSION;
  const uint64_t implied = (uint64_t)rows * nt * (uint64_t)cols * nt * 8u;
  if (cap != 0 && implied > cap) return ORC_CAPACITY; /* :272-277 */
  const size_t out_len = (size_t)(adjoint ? cols : rows) * nt;
  memset(out, 0, sizeof(double) * out_len);
  if (!adjoint) {
    for (int r = 0; r < rows; ++r) {
      double* yr = out + (size_t)r * nt;
      for (int c = 0; c < cols; ++c) {
        const double* k = kernel + ((size_t)r * cols + c) * nt;
        const double* mc = v + (size_t)c * nt;
        for (int j = 0; j < nt; ++j) {
          const double mj = mc[j];
          if (mj == 0.0) continue;
          for (int l = 0; l + j < nt; ++l) yr[j + l] += k[l] * mj;
        }
      }
    }
  } else {
    for (int r = 0; r < rows; ++r) {
      const double* dr = v + (size_t)r * nt;
      for (int c = 0; c < cols; ++c) {
        const double* k = kernel + ((size_t)r * cols + c) * nt;
        double* yc = out + (size_t)c * nt;
        for (int j = 0; j < nt; ++j) {
          double acc = 0;
          for (int l = 0; l + j < nt; ++l) acc += k[l] * dr[j + l];
          yc[j] += acc;
        }
      }
    }
  }
  return ORC_OK;
}

/* core.cpp:40-51 -- SpaceMajorRows index r*nt+j, TimeMajorBlocks j*rows+r */
void orc_reindex(const double* in, int rows, int nt, int to_time_major,
                 double* out) {
  for (int r = 0; r < rows; ++r) {
    for (int j = 0; j < nt; ++j) {
      const size_t sm = (size_t)r * nt + j, tm = (size_t)j * rows + r;
      if (to_time_major) out[tm] = in[sm];
      else out[sm] = in[tm];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Counter-based generator (not in the reference: the reference draws from
 * mt19937_64 + normal_distribution, which is libstdc++-specific and serial).
 * Bit-identical to ltb_gen.cuh: integer mixing, then an exact conversion to
 * a uniform double in [-1, 1).
 * ------------------------------------------------------------------------ */

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_gen_hash(uint64_t seed, uint64_t stream, uint64_t index) {
  const uint64_t key = splitmix64(seed ^ splitmix64(stream * 0xD1B54A32D192ED03ull));
  return splitmix64(key ^ (index * 0xC2B2AE3D27D4EB4Full));
}

double orc_gen_uniform(uint64_t seed, uint64_t stream, uint64_t index) {
  const uint64_t h = orc_gen_hash(seed, stream, index);
  const double u = (double)(h >> 11) * 0x1.0p-53; /* exact, in [0,1) */
  return 2.0 * u - 1.0;                           /* exact, in [-1,1) */
}

void orc_gen_fill(uint64_t seed, uint64_t stream, uint64_t index0, size_t n,
                  double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_gen_uniform(seed, stream, index0 + i);
}

void orc_gen_kernel(uint64_t seed, uint64_t stream, int rows, int nm_total,
                    int c0, int cols, int nt, double* out) {
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < cols; ++c) {
      const uint64_t base = ((uint64_t)r * nm_total + (uint64_t)(c0 + c)) * nt;
      double* dst = out + ((size_t)r * cols + c) * nt;
      for (int k = 0; k < nt; ++k) dst[k] = orc_gen_uniform(seed, stream, base + k);
    }
  }
}

/* L(i,i) in [1,2); L(i,j), j<i, uniform(-1,1) * 0.5/sqrt(n); upper zero */
double orc_gen_factor_entry(uint64_t seed, int n, int i, int j) {
  if (j > i) return 0.0;
  const double u = orc_gen_uniform(seed, 0x4C4Full, (uint64_t)i * (uint64_t)n + (uint64_t)j);
  if (i == j) return 1.0 + 0.5 * (u + 1.0);
  const double s = 0.5 / sqrt((double)n);
  return u * s;
}

void orc_gen_factor(uint64_t seed, int n, double* L) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      L[(size_t)j * n + i] = orc_gen_factor_entry(seed, n, i, j);
}

/* ------------------------------------------------------------------------ */
/* K^{-1} via the factor pair (bayes_engine.cpp:236-240): Eigen
 * triangularView<Lower>().solveInPlace then its transpose.  Column-oriented
 * substitution; only the lower triangle is read.
 * ------------------------------------------------------------------------ */

void orc_trsv_lower(const double* L, int n, size_t ld, double* y) {
  for (int j = 0; j < n; ++j) {
    const double* col = L + (size_t)j * ld;
    y[j] = y[j] / col[j];
    const double yj = y[j];
    for (int i = j + 1; i < n; ++i) y[i] -= col[i] * yj;
  }
}

void orc_trsv_lower_t(const double* L, int n, size_t ld, double* y) {
  for (int j = n - 1; j >= 0; --j) {
    const double* col = L + (size_t)j * ld;
    double acc = y[j];
    for (int i = j + 1; i < n; ++i) acc -= col[i] * y[i];
    y[j] = acc / col[j];
  }
}

void orc_solve_k(const double* L, int n, size_t ld, double* y) {
  orc_trsv_lower(L, n, ld, y);
  orc_trsv_lower_t(L, n, ld, y);
}

void orc_solve_k_gen(uint64_t seed, int n, double* y) {
  double* col = (double*)malloc(sizeof(double) * (size_t)n);
  for (int j = 0; j < n; ++j) {
    for (int i = j; i < n; ++i) col[i] = orc_gen_factor_entry(seed, n, i, j);
    y[j] = y[j] / col[j];
    const double yj = y[j];
    for (int i = j + 1; i < n; ++i) y[i] -= col[i] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {
    for (int i = j; i < n; ++i) col[i] = orc_gen_factor_entry(seed, n, i, j);
    double acc = y[j];
    for (int i = j + 1; i < n; ++i) acc -= col[i] * y[i];
    y[j] = acc / col[j];
  }
  free(col);
}

/* The same two substitutions for the synthetic factor at config-5 scale
 * (n = 252,000: 3.2e10 regenerated entries per sweep), blocked by 256
 * columns with the off-diagonal updates split over `threads` POSIX threads.
 * Forward: y_J = L_JJ^{-1} y_J (one thread), then y_I -= L_IJ y_J for every
 * row below (rows split over the threads).  Transposed: every thread sums
 * its rows' share L_IJ^T x_I into a private partial, the partials are added
 * in thread order (deterministic), then x_J = L_JJ^{-T} (y_J - sum).  Same
 * algebra as orc_solve_k_gen / bayes_engine.cpp:236-240; only the summation
 * order of the off-diagonal products differs.  Checker for the distributed
 * K^{-1} at full size (bench config 5, tests/dist_online_check.py). */
#include <pthread.h>

#define ORC_SB 256

typedef struct {
  uint64_t key; /* splitmix64(seed ^ splitmix64(stream * ...)) of the factor stream */
  double offs;  /* 0.5 / sqrt(n) */
  int n, threads;
  double* y;
  double* part; /* threads x ORC_SB */
  pthread_barrier_t* bar;
} orc_solve_ctx;

typedef struct {
  orc_solve_ctx* c;
  int t;
} orc_solve_arg;

/* orc_gen_factor_entry for j <= i with the stream key hoisted (bit-identical) */
static inline double fac_entry(const orc_solve_ctx* c, long i, long j) {
  const uint64_t h = splitmix64(c->key ^ (((uint64_t)i * (uint64_t)c->n + (uint64_t)j) * 0xC2B2AE3D27D4EB4Full));
  const double u = 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
  return i == j ? 1.0 + 0.5 * (u + 1.0) : u * c->offs;
}

static void* orc_solve_worker(void* p) {
  orc_solve_arg* a = (orc_solve_arg*)p;
  orc_solve_ctx* c = a->c;
  const int n = c->n, t = a->t, T = c->threads;
  double* y = c->y;
  for (int jb = 0; jb < n; jb += ORC_SB) { /* forward sweep */
    const int je = jb + ORC_SB < n ? jb + ORC_SB : n;
    if (t == 0)
      for (int j = jb; j < je; ++j) {
        y[j] = y[j] / fac_entry(c, j, j);
        const double yj = y[j];
        for (int i = j + 1; i < je; ++i) y[i] -= fac_entry(c, i, j) * yj;
      }
    pthread_barrier_wait(c->bar);
    const long rows = n - je, i0 = je + rows * t / T, i1 = je + rows * (t + 1) / T;
    for (long i = i0; i < i1; ++i) {
      double acc = 0.0;
      for (int j = jb; j < je; ++j) acc += fac_entry(c, i, j) * y[j];
      y[i] -= acc;
    }
    pthread_barrier_wait(c->bar);
  }
  const int nblk = (n + ORC_SB - 1) / ORC_SB;
  for (int b = nblk - 1; b >= 0; --b) { /* transposed sweep */
    const int jb = b * ORC_SB, je = jb + ORC_SB < n ? jb + ORC_SB : n;
    double* part = c->part + (size_t)t * ORC_SB;
    for (int j = 0; j < ORC_SB; ++j) part[j] = 0.0;
    const long rows = n - je, i0 = je + rows * t / T, i1 = je + rows * (t + 1) / T;
    for (long i = i0; i < i1; ++i) {
      const double xi = y[i];
      for (int j = jb; j < je; ++j) part[j - jb] += fac_entry(c, i, j) * xi;
    }
    pthread_barrier_wait(c->bar);
    if (t == 0)
      for (int j = je - 1; j >= jb; --j) {
        double s = 0.0;
        for (int q = 0; q < T; ++q) s += c->part[(size_t)q * ORC_SB + (j - jb)];
        double acc = y[j] - s;
        for (int i = j + 1; i < je; ++i) acc -= fac_entry(c, i, j) * y[i];
        y[j] = acc / fac_entry(c, j, j);
      }
    pthread_barrier_wait(c->bar);
  }
  return NULL;
}

int orc_solve_k_gen_mt(uint64_t seed, int n, double* y, int threads) {
  if (n < 1) return 0;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)threads);
  orc_solve_ctx c = {splitmix64(seed ^ splitmix64(0x4C4Full * 0xD1B54A32D192ED03ull)), 0.5 / sqrt((double)n), n,
                     threads, y, (double*)malloc(sizeof(double) * ORC_SB * (size_t)threads), &bar};
  orc_solve_arg args[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    args[t].c = &c;
    args[t].t = t;
    if (t > 0) pthread_create(&tid[t], NULL, orc_solve_worker, &args[t]);
  }
  orc_solve_worker(&args[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  pthread_barrier_destroy(&bar);
  free(c.part);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Prior (prior.cpp).  A_x = delta I - gamma L with the Neumann Laplacian
 * (:16-31): off-diagonals -w, diagonal delta + w * (#neighbours),
 * w = gamma / h_x^2.  The reference factors A_x with Eigen SimplicialLLT;
 * here the same SPD tridiagonal system is solved with a Cholesky
 * (Thomas-style) sweep.
 * ------------------------------------------------------------------------ */

typedef struct {
  int n;
  double w;
  double* ldiag; /* Cholesky diagonal */
  double* lsub;  /* Cholesky subdiagonal */
} tri_chol;

static int tri_chol_init(tri_chol* t, int n, double h_x, double gamma, double delta) {
  if (n < 1 || !(h_x > 0) || !(delta > 0) || gamma < 0) return ORC_DIMENSION;
  t->n = n;
  t->w = gamma / (h_x * h_x);
  t->ldiag = (double*)malloc(sizeof(double) * (size_t)n);
  t->lsub = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    double diag = delta;
    if (i > 0) diag += t->w;
    if (i + 1 < n) diag += t->w;
    if (i > 0) {
      t->lsub[i] = -t->w / t->ldiag[i - 1];
      diag -= t->lsub[i] * t->lsub[i];
    } else {
      t->lsub[i] = 0.0;
    }
    if (!(diag > 0)) return ORC_NUMERICAL;
    t->ldiag[i] = sqrt(diag);
  }
  return ORC_OK;
}

static void tri_chol_free(tri_chol* t) {
  free(t->ldiag);
  free(t->lsub);
}

/* x <- A^{-1} x, x strided by `stride` */
static void tri_solve(const tri_chol* t, double* x, size_t stride) {
  const int n = t->n;
  for (int i = 0; i < n; ++i) {
    double v = x[(size_t)i * stride];
    if (i > 0) v -= t->lsub[i] * x[(size_t)(i - 1) * stride];
    x[(size_t)i * stride] = v / t->ldiag[i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double v = x[(size_t)i * stride];
    if (i + 1 < n) v -= t->lsub[i + 1] * x[(size_t)(i + 1) * stride];
    x[(size_t)i * stride] = v / t->ldiag[i];
  }
}

/* prior.cpp:108-134: per kernel row s, Gamma_x applied to each lag column */
int orc_prior_premultiply(const double* f, int rows, int nm, int nt, double h_x,
                          double gamma, double delta, double* g) {
  tri_chol t;
  const int st = tri_chol_init(&t, nm, h_x, gamma, delta);
  if (st != ORC_OK) return st;
  const size_t slab = (size_t)nm * nt;
  memcpy(g, f, sizeof(double) * slab * rows);
  for (int s = 0; s < rows; ++s) {
    double* gs = g + (size_t)s * slab; /* [x][k], x stride nt */
    for (int k = 0; k < nt; ++k) {
      tri_solve(&t, gs + k, (size_t)nt);
      tri_solve(&t, gs + k, (size_t)nt);
    }
  }
  tri_chol_free(&t);
  return ORC_OK;
}

/* prior.cpp:45-48,82-92: per time block, A_x (A_x v) */
int orc_prior_apply_precision(const double* v, int nm, int nt, double h_x,
                              double gamma, double delta, double* out) {
  if (nm < 1 || nt < 1 || !(h_x > 0) || !(delta > 0) || gamma < 0) return ORC_DIMENSION;
  const double w = gamma / (h_x * h_x);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)nm);
  for (int j = 0; j < nt; ++j) {
    const double* b = v + (size_t)j * nm;
    double* o = out + (size_t)j * nm;
    for (int pass = 0; pass < 2; ++pass) {
      const double* src = pass == 0 ? b : tmp;
      double* dst = pass == 0 ? tmp : o;
      double* res = (double*)malloc(sizeof(double) * (size_t)nm);
      for (int i = 0; i < nm; ++i) {
        double diag = delta;
        if (i > 0) diag += w;
        if (i + 1 < nm) diag += w;
        double acc = diag * src[i];
        if (i > 0) acc += -w * src[i - 1];
        if (i + 1 < nm) acc += -w * src[i + 1];
        res[i] = acc;
      }
      memcpy(dst, res, sizeof(double) * (size_t)nm);
      free(res);
    }
  }
  free(tmp);
  return ORC_OK;
}

/* bayes_engine.cpp:311-320 (timed region of infer_map) */
void orc_infer_map(const double* L, size_t ld, const orc_plan* plan_g,
                   const double* d, double* m_map) {
  const int n = plan_g->rows * plan_g->nt;
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(y, d, sizeof(double) * (size_t)n);
  orc_solve_k(L, n, ld, y);
  orc_apply_adjoint_raw(plan_g, y, m_map);
  free(y);
}

/* ------------------------------------------------------------------------ */
/* Offline phase 2: form_K (bayes_engine.cpp:136-172) and factorize
 * (:176-209).  Test infrastructure only. */
/* ------------------------------------------------------------------------ */

/* read_gstar_column (bayes_engine.cpp:122-134): entry (x, t) = g[s][x][j-t]
 * for t <= j, column col = s * nt + j */
static void read_gstar_column(const double* g_rck, int nm, int nt, int col, double* out) {
  const int s = col / nt, j = col % nt;
  memset(out, 0, sizeof(double) * (size_t)nm * nt);
  for (int x = 0; x < nm; ++x) {
    const double* lag = g_rck + ((size_t)s * nm + x) * nt;
    for (int t = 0; t <= j; ++t) out[(size_t)x * nt + t] = lag[j - t];
  }
}

int orc_form_k(const double* f_rck, const double* g_rck, int rows, int nm, int nt,
               double sigma2, int mode, double* K, double* asym) {
  const int n = rows * nt;
  orc_plan* pf = NULL;
  orc_plan* pg = NULL;
  if (orc_plan_create(f_rck, rows, nm, nt, &pf) != 0) return 1;
  if (mode == 0 && orc_plan_create(g_rck, rows, nm, nt, &pg) != 0) {
    orc_plan_destroy(pf);
    return 1;
  }
  double* e = (double*)calloc((size_t)n, sizeof(double));
  double* gcol = (double*)malloc(sizeof(double) * (size_t)nm * nt);
  for (int i = 0; i < n; ++i) { /* :139-151 */
    if (mode == 0) {
      e[i] = 1.0;
      orc_apply_adjoint_raw(pg, e, gcol);
      e[i] = 0.0;
    } else {
      read_gstar_column(g_rck, nm, nt, i, gcol);
    }
    orc_apply_raw(pf, gcol, K + (size_t)i * n);
    K[(size_t)i * n + i] += sigma2;
  }
  /* :153-171: asymmetry of the assembled K, then symmetrise */
  double asym2 = 0, norm2 = 0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j) {
      const double d = K[(size_t)j * n + i] - K[(size_t)i * n + j];
      asym2 += 2 * d * d;
      norm2 += K[(size_t)j * n + i] * K[(size_t)j * n + i] + K[(size_t)i * n + j] * K[(size_t)i * n + j];
    }
    norm2 += K[(size_t)i * n + i] * K[(size_t)i * n + i];
  }
  if (asym) *asym = sqrt(asym2) / fmax(sqrt(norm2), 1e-300);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) {
      const double v = 0.5 * (K[(size_t)j * n + i] + K[(size_t)i * n + j]);
      K[(size_t)j * n + i] = v;
      K[(size_t)i * n + j] = v;
    }
  free(e);
  free(gcol);
  orc_plan_destroy(pf);
  if (pg) orc_plan_destroy(pg);
  return 0;
}

/* Column-oriented (left-looking) Cholesky: L(j,j) = sqrt(A(j,j) - sum_k
 * L(j,k)^2), L(i,j) = (A(i,j) - sum_k L(i,k) L(j,k)) / L(j,j) -- the
 * textbook algorithm LLT / dpotrf block; rounding differs from both only in
 * summation order. */
int orc_cholesky(double* A, int n, size_t ld) {
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * ld + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)k * ld + j] * A[(size_t)k * ld + j];
    if (!(d > 0) || !isfinite(d)) return j + 1;
    const double ljj = sqrt(d);
    A[(size_t)j * ld + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double v = A[(size_t)j * ld + i];
      for (int k = 0; k < j; ++k) v -= A[(size_t)k * ld + i] * A[(size_t)k * ld + j];
      A[(size_t)j * ld + i] = v / ljj;
    }
  }
  for (int j = 1; j < n; ++j)
    for (int i = 0; i < j; ++i) A[(size_t)j * ld + i] = 0.0;
  return 0;
}

int orc_form_q(const double* f_rck, const double* fq_rck, const double* gq_rck, int nd, int nq,
               int nm, int nt, const double* L, double* Q, double* gpost, double* prior_cov) {
  const int n = nd * nt, m = nq * nt;
  orc_plan* pf = NULL;
  orc_plan* pfq = NULL;
  if (orc_plan_create(f_rck, nd, nm, nt, &pf) != 0) return 1;
  if (orc_plan_create(fq_rck, nq, nm, nt, &pfq) != 0) {
    orc_plan_destroy(pf);
    return 1;
  }
  double* R = (double*)malloc(sizeof(double) * (size_t)n * m);
  double* X = (double*)malloc(sizeof(double) * (size_t)n * m);
  double* gcol = (double*)malloc(sizeof(double) * (size_t)nm * nt);
  for (int i = 0; i < m; ++i) { /* :244-249 */
    read_gstar_column(gq_rck, nm, nt, i, gcol);
    orc_apply_raw(pf, gcol, R + (size_t)i * n);
  }
  memcpy(X, R, sizeof(double) * (size_t)n * m);
  for (int i = 0; i < m; ++i) orc_solve_k(L, n, (size_t)n, X + (size_t)i * n); /* :250-255 */
  for (int i = 0; i < m; ++i) /* q_ = x_solve_^T (:256) */
    for (int j = 0; j < n; ++j) Q[(size_t)j * m + i] = X[(size_t)i * n + j];
  for (int i = 0; i < m; ++i) { /* :266-270 */
    read_gstar_column(gq_rck, nm, nt, i, gcol);
    orc_apply_raw(pfq, gcol, prior_cov + (size_t)i * m);
  }
  for (int i = 0; i < m; ++i) /* :271 symmetrise */
    for (int j = 0; j < i; ++j) {
      const double v = 0.5 * (prior_cov[(size_t)j * m + i] + prior_cov[(size_t)i * m + j]);
      prior_cov[(size_t)j * m + i] = v;
      prior_cov[(size_t)i * m + j] = v;
    }
  for (int j = 0; j < m; ++j) /* :273 gamma_post_q = prior - R^T X */
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += R[(size_t)i * n + k] * X[(size_t)j * n + k];
      gpost[(size_t)j * m + i] = prior_cov[(size_t)j * m + i] - acc;
    }
  double nrm = 0.0, min_diag = 0.0;
  for (int i = 0; i < m; ++i) /* :274 symmetrise */
    for (int j = 0; j < i; ++j) {
      const double v = 0.5 * (gpost[(size_t)j * m + i] + gpost[(size_t)i * m + j]);
      gpost[(size_t)j * m + i] = v;
      gpost[(size_t)i * m + j] = v;
    }
  for (size_t e = 0; e < (size_t)m * m; ++e) nrm += gpost[e] * gpost[e];
  for (int i = 0; i < m; ++i) min_diag = i == 0 || gpost[(size_t)i * m + i] < min_diag ? gpost[(size_t)i * m + i] : min_diag;
  free(R);
  free(X);
  free(gcol);
  orc_plan_destroy(pf);
  orc_plan_destroy(pfq);
  return min_diag < -1e-10 * sqrt(nrm) ? 2 : 0; /* :276-282 */
}
