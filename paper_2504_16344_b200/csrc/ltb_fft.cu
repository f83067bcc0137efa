// ltb_fft.cu -- batched pad + r2c (K1, and K7 plan build) and c2r +
// truncate + scale (K4) for sm_100a.  See ltb_fft.cuh for the algorithm.
//
// Shared memory per CTA: two padded ping-pong buffers of B sequences
// (B*NP complex each, NP = padded_len(2 Nt)); the c2r kernel also stages the
// 2B half spectra (unpadded, 2B*Nf) in the second buffer before building
// the Hermitian sequences.
#include <algorithm>

#include "ltb_gen.cuh"
#include "ltb_kernels.h"

namespace ltb {

namespace {

constexpr int kFftThreads = 256;
constexpr size_t kFftSmemBudget = 56 * 1024;  // >= 4 CTAs per SM
constexpr size_t kFftSmemMax = 227 * 1024;
constexpr long long kFftTargetCtas = 8 * 148;  // shrink tiles for few rows

// second buffer: the ping-pong partner, also the c2r staging of 2B half spectra
__host__ __device__ inline size_t stage_len(int n, int B) {
  const size_t np = (size_t)padded_len(n);
  const size_t st = (size_t)2 * B * (n / 2 + 1);
  return np * B > st ? np * B : st;
}

LTB_DEV long long in_row_of(const RfftSrc& s, long long g) {
  return (g % s.P) * s.Q + g / s.P + s.c0;
}

template <class Fft>
__global__ void __launch_bounds__(kFftThreads)
    rfft_rows_kernel(const FftDesc d, const RfftSrc src, int nt, long long nrows, double2* out,
                     long long ld, int B) {
  extern __shared__ __align__(16) double2 smem[];
  const int N = Fft::kN ? Fft::kN : d.n;
  const int NP = padded_len(N);
  double2* b0 = smem;
  double2* b1 = smem + (size_t)B * NP;
  double2* tws = b1 + stage_len(N, B);
  for (int j = threadIdx.x; j < N; j += blockDim.x) tws[j] = __ldg(d.tw + j);
  const long long g0 = (long long)blockIdx.x * 2 * B;
  const long long rows_here = min((long long)2 * B, nrows - g0);

  if (src.bulk) {
    // contiguous input rows g0 .. g0+2B-1: ONE bulk async copy (TMA 1-D) into
    // the ping-pong buffer, then pair them up from shared memory
    __shared__ uint64_t bar;
    double* stage = reinterpret_cast<double*>(b1);
    const long long nvals = rows_here * nt;
    const unsigned bulk_bytes = (unsigned)((nvals * 8) & ~15ll);
    const double* gsrc = src.in + g0 * nt;  // 16-byte aligned: g0 even, base checked by host
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&bar, bulk_bytes);
      if (bulk_bytes) bulk_g2s(stage, gsrc, bulk_bytes, &bar, policy_evict_first());
      if (nvals * 8 > bulk_bytes) stage[nvals - 1] = __ldg(gsrc + nvals - 1);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int idx = threadIdx.x; idx < B * N; idx += blockDim.x) {
      const int s = idx / N, n = idx - s * N;
      double va = 0.0, vb = 0.0;
      if (n < nt) {
        if (2 * s < rows_here) va = stage[(size_t)(2 * s) * nt + n];
        if (2 * s + 1 < rows_here) vb = stage[(size_t)(2 * s + 1) * nt + n];
      }
      b0[(size_t)s * NP + pidx(n)] = make_double2(va, vb);
    }
  } else {
    // strided rows (plan build from a host kernel) or generated values
    for (int idx = threadIdx.x; idx < B * N; idx += blockDim.x) {
      const int s = idx / N, n = idx - s * N;
      double va = 0.0, vb = 0.0;
      if (n < nt) {
        const long long ga = g0 + 2 * s, gb = ga + 1;
        if (src.in) {
          if (ga < nrows) va = __ldg(src.in + in_row_of(src, ga) * nt + n);
          if (gb < nrows) vb = __ldg(src.in + in_row_of(src, gb) * nt + n);
        } else {
          if (ga < nrows) va = gen_uniform_keyed(src.gen_key, (uint64_t)(in_row_of(src, ga) * nt + n));
          if (gb < nrows) vb = gen_uniform_keyed(src.gen_key, (uint64_t)(in_row_of(src, gb) * nt + n));
        }
      }
      b0[(size_t)s * NP + pidx(n)] = make_double2(va, vb);
    }
  }
  __syncthreads();
  const double2* Y = Fft::run(d, tws, b0, b1, B);

  // unpack: A[k] = (Z[k] + conj Z[N-k]) / 2, B[k] = -i (Z[k] - conj Z[N-k]) / 2,
  // written transposed: out[k * ld + g]
  const int nf = nt + 1;
  const int tile = 2 * B;
  for (int idx = threadIdx.x; idx < nf * tile; idx += blockDim.x) {
    const int k = idx / tile, j = idx - k * tile;
    const long long g = g0 + j;
    if (g >= nrows) continue;
    const double2* ys = Y + (size_t)(j >> 1) * NP;
    const double2 zk = ys[pidx(k)];
    const double2 zn = ys[pidx(k == 0 ? 0 : N - k)];
    double2 v;
    if ((j & 1) == 0) {
      v = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
    } else {
      // d = zk - conj(zn); B = -i d / 2 = (d.y, -d.x) / 2
      const double dx = zk.x - zn.x, dy = zk.y + zn.y;
      v = make_double2(0.5 * dy, -0.5 * dx);
    }
    const long long col = src.oP ? (g / src.oP) * src.oQ + g % src.oP + src.o0 : g;
    out[(long long)k * ld + col] = v;
  }
}

template <class Fft>
__global__ void __launch_bounds__(kFftThreads)
    irfft_rows_kernel(const FftDesc d, const double2* __restrict__ in, long long ld_f,
                      long long ld_p, int nparts, int nt, long long nrows, double scale,
                      double* __restrict__ out, int B) {
  extern __shared__ __align__(16) double2 smem[];
  const int N = Fft::kN ? Fft::kN : d.n;
  const int NP = padded_len(N);
  const int nf = nt + 1;
  const int tile = 2 * B;
  double2* b0 = smem;
  double2* b1 = smem + (size_t)B * NP;  // also the staging area (2B * nf)
  double2* tws = b1 + stage_len(N, B);
  for (int j = threadIdx.x; j < N; j += blockDim.x) tws[j] = __ldg(d.tw + j);
  const long long g0 = (long long)blockIdx.x * tile;

  // gather the half spectra of the 2B rows (summing partial slabs in a fixed
  // order when nparts > 1); FFTW c2r semantics: Im of DC / Nyquist ignored
#pragma unroll 8
  for (int idx = threadIdx.x; idx < nf * tile; idx += blockDim.x) {
    const int k = idx / tile, j = idx - k * tile;
    const long long g = g0 + j;
    double2 v = make_double2(0.0, 0.0);
    if (g < nrows) {
      const double2* p = in + (long long)k * ld_f + g;
      v = __ldg(p);
      for (int q = 1; q < nparts; ++q) v = cadd(v, __ldg(p + (long long)q * ld_p));
    }
    if (k == 0 || k == nt) v.y = 0.0;
    b1[(size_t)j * nf + k] = v;
  }
  __syncthreads();
  // conj of the full Hermitian spectrum Z = A + i B of each pair
  for (int idx = threadIdx.x; idx < B * N; idx += blockDim.x) {
    const int s = idx / N, k = idx - s * N;
    double2 a, b;
    if (k <= nt) {
      a = b1[(size_t)(2 * s) * nf + k];
      b = b1[(size_t)(2 * s + 1) * nf + k];
    } else {
      a = conjg(b1[(size_t)(2 * s) * nf + (N - k)]);
      b = conjg(b1[(size_t)(2 * s + 1) * nf + (N - k)]);
    }
    // Z = (a.x - b.y) + i (a.y + b.x); store conj(Z)
    b0[(size_t)s * NP + pidx(k)] = make_double2(a.x - b.y, -(a.y + b.x));
  }
  __syncthreads();
  // ifft(Z) = conj(fft(conj Z)): a = Re Y, b = -Im Y
  const double2* Y = Fft::run(d, tws, b0, b1, B);
  for (int idx = threadIdx.x; idx < tile * nt; idx += blockDim.x) {
    const int j = idx / nt, n = idx - j * nt;
    const long long g = g0 + j;
    if (g >= nrows) continue;
    const double2 y = Y[(size_t)(j >> 1) * NP + pidx(n)];
    const double v = (j & 1) ? -y.y : y.x;
    out[g * nt + n] = v * scale;
  }
}

// c2r of 2B rows' spectra (the G* output) -> the rows m (written out) ->
// zero padded -> r2c into the transposed spectra of the next map (F_q):
// the forecast's round trip in one pass, m never read back from HBM.
template <class Fft>
__global__ void __launch_bounds__(kFftThreads)
    c2r_r2c_rows_kernel(const FftDesc d, const double2* __restrict__ in, long long ld_f, int nt, long long nrows,
                        double scale, double* __restrict__ mout, double2* __restrict__ xout, long long ld_x,
                        int B) {
  extern __shared__ __align__(16) double2 smem[];
  const int N = Fft::kN ? Fft::kN : d.n;
  const int NP = padded_len(N);
  const int nf = nt + 1;
  const int tile = 2 * B;
  double2* b0 = smem;
  double2* b1 = smem + (size_t)B * NP;
  double2* tws = b1 + stage_len(N, B);
  for (int j = threadIdx.x; j < N; j += blockDim.x) tws[j] = __ldg(d.tw + j);
  const long long g0 = (long long)blockIdx.x * tile;
#pragma unroll 8
  for (int idx = threadIdx.x; idx < nf * tile; idx += blockDim.x) {
    const int k = idx / tile, j = idx - k * tile;
    const long long g = g0 + j;
    double2 v = g < nrows ? __ldg(in + (long long)k * ld_f + g) : make_double2(0.0, 0.0);
    if (k == 0 || k == nt) v.y = 0.0;
    b1[(size_t)j * nf + k] = v;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < B * N; idx += blockDim.x) {
    const int s = idx / N, k = idx - s * N;
    double2 a, b;
    if (k <= nt) {
      a = b1[(size_t)(2 * s) * nf + k];
      b = b1[(size_t)(2 * s + 1) * nf + k];
    } else {
      a = conjg(b1[(size_t)(2 * s) * nf + (N - k)]);
      b = conjg(b1[(size_t)(2 * s + 1) * nf + (N - k)]);
    }
    b0[(size_t)s * NP + pidx(k)] = make_double2(a.x - b.y, -(a.y + b.x));
  }
  __syncthreads();
  const double2* Y = Fft::run(d, tws, b0, b1, B);
  double2* Z = (Y == b0) ? b1 : b0;
  for (int idx = threadIdx.x; idx < B * N; idx += blockDim.x) {
    const int s = idx / N, n = idx - s * N;
    double va = 0.0, vb = 0.0;
    if (n < nt) {
      const double2 y = Y[(size_t)s * NP + pidx(n)];
      va = y.x * scale;
      vb = -y.y * scale;
      const long long ga = g0 + 2 * s;
      if (ga < nrows) mout[ga * nt + n] = va;
      if (ga + 1 < nrows) mout[(ga + 1) * nt + n] = vb;
    }
    Z[(size_t)s * NP + pidx(n)] = make_double2(va, vb);
  }
  __syncthreads();
  const double2* Y2 = Fft::run(d, tws, Z, const_cast<double2*>(Y), B);
  for (int idx = threadIdx.x; idx < nf * tile; idx += blockDim.x) {
    const int k = idx / tile, j = idx - k * tile;
    const long long g = g0 + j;
    if (g >= nrows) continue;
    const double2* ys = Y2 + (size_t)(j >> 1) * NP;
    const double2 zk = ys[pidx(k)];
    const double2 zn = ys[pidx(k == 0 ? 0 : N - k)];
    double2 v;
    if ((j & 1) == 0) {
      v = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
    } else {
      const double dx = zk.x - zn.x, dy = zk.y + zn.y;
      v = make_double2(0.5 * dy, -0.5 * dx);
    }
    xout[(long long)k * ld_x + g] = v;
  }
}

size_t smem_for(int n, int B) {
  return ((size_t)padded_len(n) * B + stage_len(n, B) + n) * sizeof(double2);  // + the twiddles
}

int pairs_for(int n, long long nrows) {
  int b = 16;
  while (b > 1 && smem_for(n, b) > kFftSmemBudget) --b;
  // few rows: smaller tiles so the grid still covers the machine
  const long long want = (nrows + 2 * kFftTargetCtas - 1) / (2 * kFftTargetCtas);
  return (int)std::max(1ll, std::min((long long)b, want));
}

cudaError_t prep_smem(const void* fn, size_t smem) {
  if (smem > kFftSmemMax) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  return cudaSuccess;
}

// the compile-time schedule for n (any factor order is a valid Stockham
// schedule over the same twiddle table), or the runtime one
template <template <class> class Kern>
struct FftDispatch {
  template <class... Args>
  static cudaError_t go(int n, dim3 grid, size_t smem, cudaStream_t st, Args... args) {
    switch (n) {
      case 128: return launch<FftFixed<128, 8, 8, 2>>(grid, smem, st, args...);
      case 256: return launch<FftFixed<256, 8, 8, 4>>(grid, smem, st, args...);
      case 512: return launch<FftFixed<512, 8, 8, 8>>(grid, smem, st, args...);
      case 840: return launch<FftFixed<840, 8, 3, 5, 7>>(grid, smem, st, args...);
      case 1024: return launch<FftFixed<1024, 8, 8, 8, 2>>(grid, smem, st, args...);
      default: return launch<FftRuntime>(grid, smem, st, args...);
    }
  }
  template <class F, class... Args>
  static cudaError_t launch(dim3 grid, size_t smem, cudaStream_t st, Args... args) {
    auto fn = Kern<F>::fn();
    cudaError_t e = prep_smem((const void*)fn, smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kFftThreads, smem, st>>>(args...);
    return cudaGetLastError();
  }
};
template <class F>
struct RfftKern {
  static auto fn() { return rfft_rows_kernel<F>; }
};
template <class F>
struct IrfftKern {
  static auto fn() { return irfft_rows_kernel<F>; }
};
template <class F>
struct RoundTripKern {
  static auto fn() { return c2r_r2c_rows_kernel<F>; }
};

}  // namespace

size_t fft_smem_bytes(int n, int* pairs_per_cta) {
  const int b = pairs_for(n, 1ll << 40);
  if (pairs_per_cta) *pairs_per_cta = b;
  return smem_for(n, b);
}

cudaError_t launch_rfft_rows(const FftDesc& d, const RfftSrc& src, int nt, long long nrows,
                             double2* out, long long ld, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  if (d.big) return big_rfft_rows(*d.big, src, nt, nrows, out, ld, st);
  if (reg_fft_supported(d.n)) {
    RfftSrc s2 = src;
    s2.bulk = (src.in && src.P == 1 && src.c0 == 0 && ((uintptr_t)src.in & 15) == 0) ? 1 : 0;
    return reg_rfft_rows(d, s2, nt, nrows, out, ld, st);
  }
  const int B = pairs_for(d.n, nrows);
  const size_t smem = smem_for(d.n, B);
  const long long grid = (nrows + 2 * B - 1) / (2 * B);
  RfftSrc s2 = src;
  s2.bulk = (src.in && src.P == 1 && src.c0 == 0 && ((uintptr_t)src.in & 15) == 0) ? 1 : 0;
  return FftDispatch<RfftKern>::go(d.n, dim3((unsigned)grid), smem, st, d, s2, nt, nrows, out, ld, B);
}

cudaError_t launch_irfft_rows(const FftDesc& d, const double2* in, long long ld_f,
                              long long ld_p, int nparts, int nt, long long nrows,
                              double scale, double* out, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  if (d.big) return big_irfft_rows(*d.big, in, ld_f, ld_p, nparts, nt, nrows, scale, out, st);
  if (reg_fft_supported(d.n)) return reg_irfft_rows(d, in, ld_f, ld_p, nparts, nt, nrows, scale, out, st);
  const int B = pairs_for(d.n, nrows);
  const size_t smem = smem_for(d.n, B);
  const long long grid = (nrows + 2 * B - 1) / (2 * B);
  return FftDispatch<IrfftKern>::go(d.n, dim3((unsigned)grid), smem, st, d, in, ld_f, ld_p, nparts, nt, nrows,
                                    scale, out, B);
}

cudaError_t launch_c2r_r2c_rows(const FftDesc& d, const double2* in, long long ld_f, int nt, long long nrows,
                                double scale, double* mout, double2* xout, long long ld_x, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  if (d.big) {  // four-step path: the two transforms separately
    cudaError_t e = big_irfft_rows(*d.big, in, ld_f, 0, 1, nt, nrows, scale, mout, st);
    if (e != cudaSuccess) return e;
    RfftSrc src{mout, 0, 1, 0, 0};
    return big_rfft_rows(*d.big, src, nt, nrows, xout, ld_x, st);
  }
  if (reg_fft_supported(d.n)) return reg_c2r_r2c_rows(d, in, ld_f, nt, nrows, scale, mout, xout, ld_x, st);
  const int B = pairs_for(d.n, nrows);
  const size_t smem = smem_for(d.n, B);
  const long long grid = (nrows + 2 * B - 1) / (2 * B);
  return FftDispatch<RoundTripKern>::go(d.n, dim3((unsigned)grid), smem, st, d, in, ld_f, nt, nrows, scale, mout,
                                        xout, ld_x, B);
}

}  // namespace ltb
