// ltb_fft_big.cu -- the time-axis transforms for padded lengths N = 2 N_t too
// long for one CTA's shared memory (N_t above ~3000; the reference's FFTW
// takes any N_t, fft_matvec.cpp:88-91).  Four-step FFT, N = N1 N2:
//   Z[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_N^(n2 k1) sum_n1 W_N1^(n1 k1) z[N2 n1 + n2]
// with both short transforms done by the shared-memory Stockham code
// (fft_batched) and the intermediate in global memory:
//   pack   : two real rows -> complex z (zero padded)            [pair][n]
//   columns: length-N1 FFTs over n1 (stride N2), twiddle W_N      [pair][k1][n2]
//   rows   : length-N2 FFTs over n2                               [pair][k1 + N1 k2]
//   unpack : Z -> the two rows' half spectra, written transposed (r2c), or
//            rows of Re / -Im (c2r, which runs the same steps on conj Z).
// Rows are processed in batches of pairs so the intermediate stays bounded.
// Not on the configured hot path (N <= 840 there); correctness over speed.
#include <algorithm>

#include "ltb_gen.cuh"
#include "ltb_kernels.h"

namespace ltb {

namespace {

constexpr int kBigThreads = 256;
constexpr size_t kBigSmem = 56 * 1024;
constexpr size_t kBigBatchBytes = 256u << 20;  // per intermediate buffer

int seqs_per_cta(int n) {
  const size_t per = 2 * (size_t)padded_len(n) * sizeof(double2);
  return (int)std::max<size_t>(1, std::min<size_t>(16, kBigSmem / per));
}

LTB_DEV long long big_in_row(const RfftSrc& s, long long g) { return (g % s.P) * s.Q + g / s.P + s.c0; }

LTB_DEV double big_row_value(const RfftSrc& s, long long g, int nt, int n) {
  const long long r = big_in_row(s, g);
  return s.in ? __ldg(s.in + r * nt + n) : gen_uniform_keyed(s.gen_key, (uint64_t)(r * nt + n));
}

// z[p][n] = a_{2p}[n] + i a_{2p+1}[n] (n < N_t), zero padded to N
__global__ void big_pack_real_kernel(const RfftSrc src, int nt, long long nrows, long long p0, int np, int N,
                                     double2* __restrict__ T) {
  const long long total = (long long)np * N;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / N;
    const int n = (int)(e - p * N);
    const long long ga = 2 * (p0 + p), gb = ga + 1;
    double va = 0.0, vb = 0.0;
    if (n < nt) {
      if (ga < nrows) va = big_row_value(src, ga, nt, n);
      if (gb < nrows) vb = big_row_value(src, gb, nt, n);
    }
    T[e] = make_double2(va, vb);
  }
}

// conj of the Hermitian spectrum Z = A + i B of pair p (FFTW c2r semantics:
// Im of DC / Nyquist ignored); spectra in[f * ld_f + q * ld_p + g], q < nparts
__global__ void big_pack_spectra_kernel(const double2* __restrict__ in, long long ld_f, long long ld_p,
                                        int nparts, int nt, long long nrows, long long p0, int np, int N,
                                        double2* __restrict__ T) {
  const long long total = (long long)np * N;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / N;
    const int k = (int)(e - p * N);
    const int f = k <= nt ? k : N - k;
    const long long ga = 2 * (p0 + p), gb = ga + 1;
    double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
    for (int q = 0; q < nparts; ++q) {
      const double2* base = in + (long long)f * ld_f + (long long)q * ld_p;
      if (ga < nrows) a = cadd(a, __ldg(base + ga));
      if (gb < nrows) b = cadd(b, __ldg(base + gb));
    }
    if (f == 0 || f == nt) a.y = b.y = 0.0;
    if (k > nt) {
      a = conjg(a);
      b = conjg(b);
    }
    T[e] = make_double2(a.x - b.y, -(a.y + b.x));  // conj(a + i b)
  }
}

// length-N1 transforms of z[N2 n1 + n2] for B2 consecutive n2 of pair
// blockIdx.y; result times W_N^(n2 k1) to T2[pair][k1][n2]
__global__ void __launch_bounds__(kBigThreads)
    big_cols_kernel(const FftDesc d1, const double2* __restrict__ twN, const double2* __restrict__ T, int N,
                    int N1, int N2, int B2, double2* __restrict__ T2) {
  extern __shared__ __align__(16) double2 bsm[];
  const int NP = padded_len(N1);
  double2* b0 = bsm;
  double2* b1 = bsm + (size_t)B2 * NP;
  const long long p = blockIdx.y;
  const int c0 = blockIdx.x * B2;
  const int nq = min(B2, N2 - c0);
  const double2* z = T + p * N;
  for (int e = threadIdx.x; e < B2 * N1; e += blockDim.x) {
    const int n1 = e / B2, q = e - n1 * B2;  // q fastest: contiguous n2
    b0[(size_t)q * NP + pidx(n1)] = q < nq ? z[(size_t)N2 * n1 + c0 + q] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double2* Y = fft_batched(d1, b0, b1, B2);
  double2* out = T2 + p * N;
  for (int e = threadIdx.x; e < B2 * N1; e += blockDim.x) {
    const int k1 = e / B2, q = e - k1 * B2;
    if (q < nq) {
      const int n2 = c0 + q;
      out[(size_t)k1 * N2 + n2] = cmul(Y[(size_t)q * NP + pidx(k1)], __ldg(twN + (size_t)n2 * k1 % N));
    }
  }
}

// length-N2 transforms of T2[pair][k1][.] for B1 consecutive k1; result to
// Z[pair][k1 + N1 k2]
__global__ void __launch_bounds__(kBigThreads)
    big_rows_kernel(const FftDesc d2, const double2* __restrict__ T2, int N, int N1, int N2, int B1,
                    double2* __restrict__ Z) {
  extern __shared__ __align__(16) double2 bsm[];
  const int NP = padded_len(N2);
  double2* b0 = bsm;
  double2* b1 = bsm + (size_t)B1 * NP;
  const long long p = blockIdx.y;
  const int k0 = blockIdx.x * B1;
  const int nq = min(B1, N1 - k0);
  const double2* src = T2 + p * N;
  for (int e = threadIdx.x; e < B1 * N2; e += blockDim.x) {
    const int q = e / N2, m = e - q * N2;
    b0[(size_t)q * NP + pidx(m)] = q < nq ? src[(size_t)(k0 + q) * N2 + m] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double2* Y = fft_batched(d2, b0, b1, B1);
  double2* out = Z + p * N;
  for (int e = threadIdx.x; e < B1 * N2; e += blockDim.x) {
    const int k2 = e / B1, q = e - k2 * B1;  // q fastest: contiguous k1 runs
    if (q < nq) out[(size_t)(k0 + q) + (size_t)N1 * k2] = Y[(size_t)q * NP + pidx(k2)];
  }
}

// r2c unpack: A_f = (Z_f + conj Z_{N-f}) / 2, B_f = -i (Z_f - conj Z_{N-f}) / 2
__global__ void big_unpack_kernel(const double2* __restrict__ Z, int nt, long long nrows, long long p0, int np,
                                  int N, RfftSrc src, double2* __restrict__ out, long long ld) {
  const long long total = (long long)(nt + 1) * np;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(e / np);
    const long long p = e - (long long)f * np;
    const double2* z = Z + p * N;
    const double2 zk = z[f], zn = z[f == 0 ? 0 : N - f];
    for (int h = 0; h < 2; ++h) {
      const long long g = 2 * (p0 + p) + h;
      if (g >= nrows) continue;
      double2 v;
      if (h == 0) {
        v = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
      } else {
        const double dx = zk.x - zn.x, dy = zk.y + zn.y;
        v = make_double2(0.5 * dy, -0.5 * dx);
      }
      const long long col = src.oP ? (g / src.oP) * src.oQ + g % src.oP + src.o0 : g;
      out[(long long)f * ld + col] = v;
    }
  }
}

// c2r output: rows 2p, 2p+1 = Re Y, -Im Y (first N_t samples) times scale
__global__ void big_output_kernel(const double2* __restrict__ Y, int nt, long long nrows, long long p0, int np,
                                  int N, double scale, double* __restrict__ out) {
  const long long total = (long long)np * nt;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long p = e / nt;
    const int n = (int)(e - p * nt);
    const double2 y = Y[p * N + n];
    const long long ga = 2 * (p0 + p);
    out[ga * nt + n] = y.x * scale;
    if (ga + 1 < nrows) out[(ga + 1) * nt + n] = -y.y * scale;
  }
}

unsigned grid_for(long long n) { return (unsigned)std::max(1ll, std::min(148ll * 16, (n + 255) / 256)); }

// the two passes of the four-step transform over np pairs in T -> Z (T2 scratch)
cudaError_t four_step(const BigFft& b, const double2* T, double2* T2, double2* Z, int np, cudaStream_t st) {
  const int B2 = seqs_per_cta(b.n1), B1 = seqs_per_cta(b.n2);
  const size_t s1 = 2 * (size_t)B2 * padded_len(b.n1) * sizeof(double2);
  const size_t s2 = 2 * (size_t)B1 * padded_len(b.n2) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(big_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(big_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  if (e != cudaSuccess) return e;
  big_cols_kernel<<<dim3((unsigned)((b.n2 + B2 - 1) / B2), (unsigned)np), kBigThreads, s1, st>>>(
      b.d1, b.twN, T, b.n, b.n1, b.n2, B2, T2);
  big_rows_kernel<<<dim3((unsigned)((b.n1 + B1 - 1) / B1), (unsigned)np), kBigThreads, s2, st>>>(
      b.d2, T2, b.n, b.n1, b.n2, B1, Z);
  return cudaGetLastError();
}

struct Scratch3 {
  double2* p = nullptr;
  cudaStream_t st;
  ~Scratch3() {
    if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace

bool big_fft_split(int n, int max_len, int* n1, int* n2) {
  // N1 <= N2, both short enough for the shared-memory FFT, N1 closest to sqrt N
  for (int a = (int)std::sqrt((double)n); a >= 2; --a) {
    if (n % a) continue;
    const int b = n / a;
    if (b <= max_len && a <= max_len) {
      *n1 = a;
      *n2 = b;
      return true;
    }
  }
  return false;
}

cudaError_t big_rfft_rows(const BigFft& b, const RfftSrc& src, int nt, long long nrows, double2* out, long long ld,
                          cudaStream_t st) {
  const long long pairs = (nrows + 1) / 2;
  const int batch = (int)std::max<long long>(1, std::min<long long>(pairs, kBigBatchBytes / (16ll * b.n)));
  Scratch3 buf;
  buf.st = st;
  cudaError_t e = cudaMallocAsync(&buf.p, 2 * (size_t)batch * b.n * sizeof(double2), st);
  if (e != cudaSuccess) return e;
  double2* T = buf.p;
  double2* T2 = buf.p + (size_t)batch * b.n;
  for (long long p0 = 0; p0 < pairs; p0 += batch) {
    const int np = (int)std::min<long long>(batch, pairs - p0);
    big_pack_real_kernel<<<grid_for((long long)np * b.n), 256, 0, st>>>(src, nt, nrows, p0, np, b.n, T);
    if ((e = four_step(b, T, T2, T, np, st)) != cudaSuccess) return e;
    big_unpack_kernel<<<grid_for((long long)(nt + 1) * np), 256, 0, st>>>(T, nt, nrows, p0, np, b.n, src, out, ld);
  }
  return cudaGetLastError();
}

cudaError_t big_irfft_rows(const BigFft& b, const double2* in, long long ld_f, long long ld_p, int nparts, int nt,
                           long long nrows, double scale, double* out, cudaStream_t st) {
  const long long pairs = (nrows + 1) / 2;
  const int batch = (int)std::max<long long>(1, std::min<long long>(pairs, kBigBatchBytes / (16ll * b.n)));
  Scratch3 buf;
  buf.st = st;
  cudaError_t e = cudaMallocAsync(&buf.p, 2 * (size_t)batch * b.n * sizeof(double2), st);
  if (e != cudaSuccess) return e;
  double2* T = buf.p;
  double2* T2 = buf.p + (size_t)batch * b.n;
  for (long long p0 = 0; p0 < pairs; p0 += batch) {
    const int np = (int)std::min<long long>(batch, pairs - p0);
    big_pack_spectra_kernel<<<grid_for((long long)np * b.n), 256, 0, st>>>(in, ld_f, ld_p, nparts, nt, nrows, p0,
                                                                          np, b.n, T);
    if ((e = four_step(b, T, T2, T, np, st)) != cudaSuccess) return e;
    // ifft(Z) = conj(fft(conj Z)): a = Re Y, b = -Im Y
    big_output_kernel<<<grid_for((long long)np * nt), 256, 0, st>>>(T, nt, nrows, p0, np, b.n, scale, out);
  }
  return cudaGetLastError();
}

}  // namespace ltb
