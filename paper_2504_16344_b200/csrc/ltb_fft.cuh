// ltb_fft.cuh -- time-axis transforms for the block-Toeplitz matvec.
//
// Replaces the reference's per-row FFTW calls (fft_matvec.cpp:96-110 plan
// build, :143-150 / :185-191 forward pad+r2c, :169-178 / :208-216 c2r +
// truncate + 1/(2 N_t)) with batched shared-memory Stockham FFTs:
//
//   * a CTA owns a tile of 2B rows; rows are packed in pairs into B complex
//     sequences z = a + i b of length N = 2 N_t (zero padded past N_t), so
//     one complex FFT serves two real rows;
//   * radix-8/4/2/3/5/7 butterflies (generic O(p^2) butterfly for any other
//     prime, so every N_t works), ping-ponging between two shared-memory
//     buffers, twiddles from a per-plan table W[j] = exp(-2 pi i j/N) built on
//     the host in long double;
//   * spectra are written TRANSPOSED, out[f * ld + row], so the per-frequency
//     GEMVs read x-hat / d-hat with unit stride and F-hat comes out directly
//     in the reference's [f][c][r] order (fft_matvec.cpp:44-46,104-108).
#pragma once

#include "ltb_common.cuh"

namespace ltb {

constexpr int kMaxStages = 32;

// Shared-memory sequences are padded by one complex per 8 so the stride-R
// scatter of the first Stockham stage (and the strided unpack) hits distinct
// 16-byte bank groups within each quarter-warp phase.
__host__ __device__ __forceinline__ int pidx(int x) { return x + (x >> 3); }
__host__ __device__ __forceinline__ int padded_len(int n) { return n + (n >> 3) + 1; }

struct BigFft;  // four-step plan for lengths beyond one CTA (ltb_fft_big.cu)

struct FftDesc {
  int n;        // complex transform length N = 2 N_t
  int nstages;
  int radix[kMaxStages];
  const double2* tw;  // W[j] = exp(-2 pi i j / N), j in [0, N)
  const BigFft* big = nullptr;  // host-side: set when N needs the four-step path
};

// N = n1 n2 four-step transform: both factors run through fft_batched
struct BigFft {
  int n = 0, n1 = 0, n2 = 0;
  FftDesc d1{}, d2{};
  const double2* twN = nullptr;  // W_N^j, j in [0, N)
};

// One radix-R Stockham step (Bainville formulation): butterfly i of T = N/R
// reads src[i + r T], applies W^(j r N/(Ns R)) with j = i mod Ns, does a
// length-R DFT and writes dst[(i/Ns) Ns R + j + q Ns].
template <int R>
LTB_DEV void dft_small(double2 (&v)[R]);

template <>
LTB_DEV void dft_small<2>(double2 (&v)[2]) {
  const double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
LTB_DEV void dft_small<4>(double2 (&v)[4]) {
  const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  const double2 b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
  v[0] = cadd(a0, b0);
  v[2] = csub(a0, b0);
  v[1] = make_double2(a1.x + b1.y, a1.y - b1.x);  // a1 - i b1
  v[3] = make_double2(a1.x - b1.y, a1.y + b1.x);  // a1 + i b1
}

template <>
LTB_DEV void dft_small<8>(double2 (&v)[8]) {
  constexpr double c = 0.7071067811865475244008;
  double2 e[4] = {v[0], v[2], v[4], v[6]};
  double2 o[4] = {v[1], v[3], v[5], v[7]};
  dft_small<4>(e);
  dft_small<4>(o);
  // o[k] *= W8^k, W8 = exp(-i pi/4)
  const double2 o1 = make_double2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
  const double2 o2 = make_double2(o[2].y, -o[2].x);
  const double2 o3 = make_double2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// odd prime R: pair r with R-r, V_q = v0 + sum s_r cos - i sum d_r sin.
// cos / sin (2 pi m / R), m in [1, (R-1)/2], to 22 digits (mpmath).
LTB_DEV constexpr double odd_cos(int R, int m) {
  return R == 3 ? -0.5
       : R == 5 ? (m == 1 ? 0.3090169943749474241023 : -0.8090169943749474241023)
                : (m == 1 ? 0.623489801858733530525
                          : m == 2 ? -0.2225209339563144042889 : -0.9009688679024191262361);
}
LTB_DEV constexpr double odd_sin(int R, int m) {
  return R == 3 ? 0.8660254037844386467637
       : R == 5 ? (m == 1 ? 0.9510565162951535721164 : 0.5877852522924731291687)
                : (m == 1 ? 0.7818314824680298087084
                          : m == 2 ? 0.9749279121818236070181 : 0.4338837391175581204758);
}

template <int R>
LTB_DEV void dft_odd(double2 (&v)[R]) {
  constexpr int h = (R - 1) / 2;
  double2 sm[h], df[h];
#pragma unroll
  for (int r = 1; r <= h; ++r) {
    sm[r - 1] = cadd(v[r], v[R - r]);
    df[r - 1] = csub(v[r], v[R - r]);
  }
  double2 out[R];
  out[0] = v[0];
#pragma unroll
  for (int r = 0; r < h; ++r) out[0] = cadd(out[0], sm[r]);
#pragma unroll
  for (int q = 1; q <= h; ++q) {
    double2 a = v[0], b = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 1; r <= h; ++r) {
      const int m = (r * q) % R;              // angle index in [1, R)
      const int mm = m <= h ? m : R - m;      // cos symmetric
      const double sg = m <= h ? 1.0 : -1.0;  // sin antisymmetric
      const double cs = odd_cos(R, mm);
      const double sn = sg * odd_sin(R, mm);
      a.x = fma(sm[r - 1].x, cs, a.x);
      a.y = fma(sm[r - 1].y, cs, a.y);
      b.x = fma(df[r - 1].x, sn, b.x);
      b.y = fma(df[r - 1].y, sn, b.y);
    }
    out[q] = make_double2(a.x + b.y, a.y - b.x);      // a - i b
    out[R - q] = make_double2(a.x - b.y, a.y + b.x);  // a + i b
  }
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = out[q];
}
template <>
LTB_DEV void dft_small<3>(double2 (&v)[3]) { dft_odd<3>(v); }
template <>
LTB_DEV void dft_small<5>(double2 (&v)[5]) { dft_odd<5>(v); }
template <>
LTB_DEV void dft_small<7>(double2 (&v)[7]) { dft_odd<7>(v); }

template <int R>
LTB_DEV void stockham_butterfly(const double2* __restrict__ src, double2* __restrict__ dst,
                                const double2* __restrict__ tw, int N, int Ns, int i) {
  const int T = N / R;
  const int j = i % Ns;
  const int tstep = j * (N / (Ns * R));
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = src[pidx(i + r * T)];
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * tstep]);
  dft_small<R>(v);
  const int o = (i / Ns) * Ns * R + j;
#pragma unroll
  for (int r = 0; r < R; ++r) dst[pidx(o + r * Ns)] = v[r];
}

// any radix (rare lengths): O(R^2) straight from shared memory
LTB_DEV void stockham_butterfly_generic(const double2* __restrict__ src, double2* __restrict__ dst,
                                        const double2* __restrict__ tw, int N, int Ns, int R,
                                        int i) {
  const int T = N / R;
  const int j = i % Ns;
  const int tstep = j * (N / (Ns * R));
  const int rstep = N / R;
  const int o = (i / Ns) * Ns * R + j;
  for (int q = 0; q < R; ++q) {
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      double2 x = src[pidx(i + r * T)];
      if (r) x = cmul(x, tw[r * tstep]);
      cmac(acc, x, tw[((r * q) % R) * rstep]);
    }
    dst[pidx(o + q * Ns)] = acc;
  }
}

// Batched forward FFT of `nseq` sequences laid out back to back (stride
// padded_len(N), element n at pidx(n)) in `a`; `b` is the ping-pong buffer.
// Returns the buffer holding the result.  Must be called by all threads of
// the CTA.
LTB_DEV double2* fft_batched(const FftDesc& d, double2* a, double2* b, int nseq,
                             const double2* tw = nullptr) {
  if (!tw) tw = d.tw;
  const int N = d.n;
  const int NP = padded_len(N);
  int Ns = 1;
  for (int s = 0; s < d.nstages; ++s) {
    const int R = d.radix[s];
    const int T = N / R;
    const int total = nseq * T;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int q = idx / T, i = idx - q * T;
      const double2* src = a + (size_t)q * NP;
      double2* dst = b + (size_t)q * NP;
      switch (R) {
        case 8: stockham_butterfly<8>(src, dst, tw, N, Ns, i); break;
        case 4: stockham_butterfly<4>(src, dst, tw, N, Ns, i); break;
        case 2: stockham_butterfly<2>(src, dst, tw, N, Ns, i); break;
        case 3: stockham_butterfly<3>(src, dst, tw, N, Ns, i); break;
        case 5: stockham_butterfly<5>(src, dst, tw, N, Ns, i); break;
        case 7: stockham_butterfly<7>(src, dst, tw, N, Ns, i); break;
        default: stockham_butterfly_generic(src, dst, tw, N, Ns, R, i); break;
      }
    }
    __syncthreads();
    double2* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

// ---- compile-time schedules for the common lengths ------------------------
// Same Stockham steps with N, the radix sequence and every stride known to
// the compiler: no runtime integer division / radix switch in the butterfly
// loops (the generic path spends most of its instructions there).
template <int R, int N, int Ns>
LTB_DEV void stockham_butterfly_ct(const double2* __restrict__ src, double2* __restrict__ dst,
                                   const double2* __restrict__ tw, int i) {
  constexpr int T = N / R;
  const int j = i % Ns;
  const int tstep = j * (N / (Ns * R));
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = src[pidx(i + r * T)];
  if (Ns > 1) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * tstep]);
  }
  dft_small<R>(v);
  const int o = (i / Ns) * Ns * R + j;
#pragma unroll
  for (int r = 0; r < R; ++r) dst[pidx(o + r * Ns)] = v[r];
}

template <int N, int Ns, int R, int... Rest>
LTB_DEV double2* fft_stages_ct(const double2* tw, double2* a, double2* b, int nseq) {
  constexpr int T = N / R;
  constexpr int NP = N + (N >> 3) + 1;
  const int total = nseq * T;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int q = idx / T, i = idx - q * T;
    stockham_butterfly_ct<R, N, Ns>(a + (size_t)q * NP, b + (size_t)q * NP, tw, i);
  }
  __syncthreads();
  if constexpr (sizeof...(Rest) > 0) {
    return fft_stages_ct<N, Ns * R, Rest...>(tw, b, a, nseq);
  } else {
    return b;
  }
}

// transform policies for the row kernels
// (tw: the twiddle table staged in shared memory by the row kernels -- with
// the shared-memory carve-out of 4 CTAs per SM there is little L1 left, and
// __ldg twiddles stalled the butterflies on L2 round trips)
struct FftRuntime {
  static constexpr int kN = 0;
  static LTB_DEV double2* run(const FftDesc& d, const double2* tw, double2* a, double2* b, int nseq) {
    return fft_batched(d, a, b, nseq, tw);
  }
};
template <int N, int... Rs>
struct FftFixed {
  static constexpr int kN = N;
  static LTB_DEV double2* run(const FftDesc& d, const double2* tw, double2* a, double2* b, int nseq) {
    return fft_stages_ct<N, 1, Rs...>(tw, a, b, nseq);
  }
};

}  // namespace ltb
