// ltb_fft_reg.cu -- register-resident two-pass transforms for the common
// padded lengths (K1 / K4 and the fused forecast round trip, sm_100a).
//
// Same maps as ltb_fft.cu (fft_matvec.cpp:143-150 pad + r2c, :169-178 c2r +
// truncate + 1/(2 N_t)), restructured for bandwidth:
//
//   * N = R1 R2 with R1, R2 <= 32: pass 1 is R2 butterflies of radix R1 over
//     inputs strided by R2, pass 2 is R1 butterflies of radix R2 after the
//     W_N^(r i) twiddles -- each butterfly a fully unrolled DFT in registers
//     (composite radices split again at compile time, constant twiddles
//     folded from ltb_fft_consts.cuh), so a sequence crosses shared memory
//     once between the passes instead of once per radix-8/4/2/3/5/7 stage;
//   * a group of <= 32 lanes owns one complex sequence (two real rows packed
//     as a + i b), groups synchronise with __syncwarp only, and warps loop
//     persistently over row pairs: no CTA barriers in the steady state and
//     the pass-2 twiddle table is staged once per CTA;
//   * pass-1 operands come straight from global memory (row loads
//     coalesced across the lanes; the zero padding is never stored) and the
//     c2r output leaves from registers; only the r2c unpack (Z[k] with
//     Z[N-k]) goes back through shared memory to write the transposed
//     spectra out[f * ld + row].
//
// Shared layout per sequence: R2 rows of R1 complex padded to R1 + 1
// (natural index n at n + n / R1): the pass-1 scatter (stride R1 + 1) and the
// pass-2 gather (unit stride) are both bank-conflict free.
#include <algorithm>

#include "ltb_fft_consts.cuh"
#include "ltb_gen.cuh"
#include "ltb_kernels.h"

namespace ltb {

namespace {

// ---- register DFTs -----------------------------------------------------
template <int R>
LTB_DEV double2 twc(double2 x, int m) {
  // x * W_R^m with the trivial angles special-cased (m is a constant after
  // unrolling, so the branches fold)
  if (m == 0) return x;
  if (4 * m == R) return make_double2(x.y, -x.x);   // -i
  if (2 * m == R) return make_double2(-x.x, -x.y);  // -1
  if (4 * m == 3 * R) return make_double2(-x.y, x.x);  // +i
  const double c = w_re(R, m), s = w_im(R, m);
  return make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
}

constexpr int split_of(int R) {
  return (R % 8 == 0 && R > 8) ? 8 : (R % 4 == 0 && R > 4) ? 4 : (R % 2 == 0 && R > 2) ? 2 : (R % 3 == 0 && R > 3) ? 3 : 5;
}
constexpr bool is_leaf(int R) { return R == 2 || R == 3 || R == 4 || R == 5 || R == 7 || R == 8; }

template <int R>
LTB_DEV void dftr(double2 (&v)[R]);

// X[k1 + P k2] = sum_n2 W_Q^(n2 k2) W_R^(n2 k1) sum_n1 W_P^(n1 k1) x[Q n1 + n2]
template <int P, int Q>
LTB_DEV void dft_comp(double2 (&v)[P * Q]) {
  constexpr int R = P * Q;
  double2 u[R];
#pragma unroll
  for (int n2 = 0; n2 < Q; ++n2) {
    double2 t[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) t[n1] = v[Q * n1 + n2];
    dftr<P>(t);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) u[k1 * Q + n2] = twc<R>(t[k1], (n2 * k1) % R);
  }
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) {
    double2 s[Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) s[n2] = u[k1 * Q + n2];
    dftr<Q>(s);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) v[k1 + P * k2] = s[k2];
  }
}

template <int R>
LTB_DEV void dftr(double2 (&v)[R]) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (is_leaf(R)) {
    dft_small<R>(v);
  } else {
    constexpr int P = split_of(R);
    dft_comp<P, R / P>(v);
  }
}

// ---- plan ----------------------------------------------------------------
template <int R1_, int R2_>
struct RegFft {
  static constexpr int R1 = R1_, R2 = R2_, N = R1 * R2;
  static constexpr int L = R1 > R2 ? R1 : R2;                      // active lanes per sequence
  static constexpr int LP = L <= 8 ? 8 : L <= 16 ? 16 : 32;        // lane group
  static constexpr int S = 32 / LP;                                // sequences per warp
  static constexpr int ROW = R1 + 1;                               // padded row
  static constexpr int SEQ = R2 * ROW;                             // padded sequence (complex)
  static LTB_DEV int addr(int n) { return n + n / R1; }
};

// 8 warps per CTA, one CTA per SM (the register DFTs want ~255 registers;
// capping them at 168 for 12 warps spills)
constexpr int kRegWarps = 8;
constexpr int kRegThreads = 32 * kRegWarps;
constexpr int kRegMinCtas = 1;

template <class F>
constexpr size_t reg_smem() {
  return ((size_t)kRegWarps * F::S * F::SEQ + F::N) * sizeof(double2);
}

// stage the pass-2 twiddles tw2[r R1 + i] = W_N^(r i)
template <class F>
LTB_DEV void stage_tw2(const double2* __restrict__ tw, double2* tw2) {
  for (int j = threadIdx.x; j < F::N; j += blockDim.x) {
    const int r = j / F::R1, i = j - r * F::R1;
    tw2[j] = __ldg(tw + r * i);
  }
  __syncthreads();
}

// pass 1 from registers v (lane li < R2 holds x[li + r R2]) into buf, then
// pass 2 (lane li < R1) leaving X[li + q R1] in v2
template <class F>
LTB_DEV void two_pass(double2 (&v)[F::R1], double2* buf, const double2* tw2, int li, double2 (&v2)[F::R2]) {
  if (li < F::R2) {
    dftr<F::R1>(v);
#pragma unroll
    for (int q = 0; q < F::R1; ++q) buf[li * F::ROW + q] = v[q];
  }
  __syncwarp();
  if (li < F::R1) {
#pragma unroll
    for (int r = 0; r < F::R2; ++r) {
      const double2 x = buf[r * F::ROW + li];
      v2[r] = r == 0 ? x : cmul(x, tw2[r * F::R1 + li]);
    }
    dftr<F::R2>(v2);
  }
  __syncwarp();
}

// X (lane li < R1 holds X[li + q R1] in v2) -> buf, then the two half
// spectra of the pair, transposed: out[k * ld + col(g)], out[k * ld + col(g + 1)]
template <class F>
LTB_DEV void unpack_store(const double2 (&v2)[F::R2], double2* buf, int li, int nt, long long g, long long nrows,
                          const RfftSrc& src, double2* __restrict__ out, long long ld) {
  if (li < F::R1) {
#pragma unroll
    for (int q = 0; q < F::R2; ++q) buf[q * F::ROW + li] = v2[q];
  }
  __syncwarp();
  const bool has_a = g < nrows, has_b = g + 1 < nrows;
  const long long ca = src.oP ? (g / src.oP) * src.oQ + g % src.oP + src.o0 : g;
  const long long cb = src.oP ? ((g + 1) / src.oP) * src.oQ + (g + 1) % src.oP + src.o0 : g + 1;
  for (int k = li; k <= nt; k += F::LP) {
    const double2 zk = buf[F::addr(k)];
    const double2 zn = buf[F::addr(k == 0 ? 0 : F::N - k)];
    if (has_a) out[(long long)k * ld + ca] = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
    if (has_b) out[(long long)k * ld + cb] = make_double2(0.5 * (zk.y + zn.y), -0.5 * (zk.x - zn.x));
  }
  __syncwarp();
}

LTB_DEV long long in_row(const RfftSrc& s, long long g) { return (g % s.P) * s.Q + g / s.P + s.c0; }

template <class F>
__global__ void __launch_bounds__(kRegThreads, kRegMinCtas)
    rfft_reg_kernel(const double2* __restrict__ tw, const RfftSrc src, int nt, long long nrows, double2* out,
                    long long ld) {
  extern __shared__ __align__(16) double2 smem[];
  double2* tw2 = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / F::LP, li = lane % F::LP;
  double2* buf = smem + F::N + (size_t)(warp * F::S + grp) * F::SEQ;
  stage_tw2<F>(tw, tw2);
  const long long npairs = (nrows + 1) / 2;
  const long long tasks = (npairs + F::S - 1) / F::S;
  for (long long t = (long long)blockIdx.x * kRegWarps + warp; t < tasks; t += (long long)gridDim.x * kRegWarps) {
    const long long g = 2 * (t * F::S + grp);
    double2 v[F::R1];
    if (li < F::R2) {
      const bool ha = g < nrows, hb = g + 1 < nrows;
      const long long ra = ha ? in_row(src, g) : 0, rb = hb ? in_row(src, g + 1) : 0;
#pragma unroll
      for (int r = 0; r < F::R1; ++r) {
        const int n = li + r * F::R2;
        double va = 0.0, vb = 0.0;
        if (n < nt) {
          if (src.in) {
            if (ha) va = __ldg(src.in + ra * nt + n);
            if (hb) vb = __ldg(src.in + rb * nt + n);
          } else {
            if (ha) va = gen_uniform_keyed(src.gen_key, (uint64_t)(ra * nt + n));
            if (hb) vb = gen_uniform_keyed(src.gen_key, (uint64_t)(rb * nt + n));
          }
        }
        v[r] = make_double2(va, vb);
      }
    }
    double2 v2[F::R2];
    two_pass<F>(v, buf, tw2, li, v2);
    unpack_store<F>(v2, buf, li, nt, g, nrows, src, out, ld);
  }
}

// the two half spectra of the pair (rows g, g + 1; nparts slabs summed in a
// fixed order) into buf[k] / buf[nf + k] -- every element read once, 32
// contiguous bytes per frequency -- then conj of the Hermitian-extended
// Z = A + i B at the pass-1 indices k = li + r R2 into v (FFTW c2r semantics:
// Im of DC / Nyquist ignored)
template <class F>
LTB_DEV void load_conj_pair(const double2* __restrict__ in, long long ld_f, long long ld_p, int nparts, int nt,
                            long long g, bool ha, bool hb, double2* buf, int li, double2 (&v)[F::R1]) {
  const int nf = nt + 1;
  if (ha) {
#pragma unroll 4
    for (int k = li; k < nf; k += F::LP) {
      const double2* p = in + (long long)k * ld_f + g;
      double2 a = __ldg(p), b = hb ? __ldg(p + 1) : make_double2(0.0, 0.0);
      for (int q = 1; q < nparts; ++q) {
        a = cadd(a, __ldg(p + (long long)q * ld_p));
        if (hb) b = cadd(b, __ldg(p + (long long)q * ld_p + 1));
      }
      if (k == 0 || k == nt) {
        a.y = 0.0;
        b.y = 0.0;
      }
      buf[k] = a;
      buf[nf + k] = b;
    }
  }
  __syncwarp();
  if (li < F::R2) {
#pragma unroll
    for (int r = 0; r < F::R1; ++r) {
      const int k = li + r * F::R2;
      const bool mirror = k > nt;
      const int kk = mirror ? F::N - k : k;
      double2 a = ha ? buf[kk] : make_double2(0.0, 0.0), b = ha ? buf[nf + kk] : make_double2(0.0, 0.0);
      if (mirror) {
        a.y = -a.y;
        b.y = -b.y;
      }
      v[r] = make_double2(a.x - b.y, -(a.y + b.x));
    }
  }
  __syncwarp();
}

template <class F>
__global__ void __launch_bounds__(kRegThreads, kRegMinCtas)
    irfft_reg_kernel(const double2* __restrict__ tw, const double2* __restrict__ in, long long ld_f, long long ld_p,
                     int nparts, int nt, long long nrows, double scale, double* __restrict__ out) {
  extern __shared__ __align__(16) double2 smem[];
  double2* tw2 = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / F::LP, li = lane % F::LP;
  double2* buf = smem + F::N + (size_t)(warp * F::S + grp) * F::SEQ;
  stage_tw2<F>(tw, tw2);
  const long long npairs = (nrows + 1) / 2;
  const long long tasks = (npairs + F::S - 1) / F::S;
  for (long long t = (long long)blockIdx.x * kRegWarps + warp; t < tasks; t += (long long)gridDim.x * kRegWarps) {
    const long long g = 2 * (t * F::S + grp);
    const bool ha = g < nrows, hb = g + 1 < nrows;
    double2 v[F::R1];
    load_conj_pair<F>(in, ld_f, ld_p, nparts, nt, g, ha, hb, buf, li, v);
    double2 v2[F::R2];
    two_pass<F>(v, buf, tw2, li, v2);
    // ifft(Z) = conj(fft(conj Z)): row a = Re Y, row b = -Im Y
    if (li < F::R1) {
#pragma unroll
      for (int q = 0; q < F::R2 / 2; ++q) {  // n = li + q R1 < nt = N / 2 exactly for q < R2 / 2
        const int n = li + q * F::R1;
        {
          if (ha) out[g * nt + n] = v2[q].x * scale;
          if (hb) out[(g + 1) * nt + n] = -v2[q].y * scale;
        }
      }
    }
  }
}

// c2r of a pair (rows written to mout) -> zero padded -> r2c into xout
template <class F>
__global__ void __launch_bounds__(kRegThreads, kRegMinCtas)
    c2r_r2c_reg_kernel(const double2* __restrict__ tw, const double2* __restrict__ in, long long ld_f, int nt,
                       long long nrows, double scale, double* __restrict__ mout, double2* __restrict__ xout,
                       long long ld_x) {
  extern __shared__ __align__(16) double2 smem[];
  double2* tw2 = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / F::LP, li = lane % F::LP;
  double2* buf = smem + F::N + (size_t)(warp * F::S + grp) * F::SEQ;
  stage_tw2<F>(tw, tw2);
  const RfftSrc ident{nullptr, 0, 1, 0, 0};
  const long long npairs = (nrows + 1) / 2;
  const long long tasks = (npairs + F::S - 1) / F::S;
  for (long long t = (long long)blockIdx.x * kRegWarps + warp; t < tasks; t += (long long)gridDim.x * kRegWarps) {
    const long long g = 2 * (t * F::S + grp);
    const bool ha = g < nrows, hb = g + 1 < nrows;
    double2 v[F::R1];
    load_conj_pair<F>(in, ld_f, 0, 1, nt, g, ha, hb, buf, li, v);
    double2 v2[F::R2];
    two_pass<F>(v, buf, tw2, li, v2);
    if (li < F::R1) {
#pragma unroll
      for (int q = 0; q < F::R2; ++q) {
        const int n = li + q * F::R1;
        const double a = v2[q].x * scale, b = -v2[q].y * scale;
        if (n < nt) {
          if (ha) mout[g * nt + n] = a;
          if (hb) mout[(g + 1) * nt + n] = b;
        }
        buf[q * F::ROW + li] = make_double2(n < nt && ha ? a : 0.0, n < nt && hb ? b : 0.0);
      }
    }
    __syncwarp();
    if (li < F::R2) {
#pragma unroll
      for (int r = 0; r < F::R1; ++r) {
        const int n = li + r * F::R2;
        v[r] = n < nt ? buf[F::addr(n)] : make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    two_pass<F>(v, buf, tw2, li, v2);
    unpack_store<F>(v2, buf, li, nt, g, nrows, ident, xout, ld_x);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

template <class F>
unsigned reg_grid(long long nrows) {
  const long long tasks = ((nrows + 1) / 2 + F::S - 1) / F::S;
  const long long ctas = (tasks + kRegWarps - 1) / kRegWarps;
  return (unsigned)std::max(1ll, std::min(ctas, (long long)kRegMinCtas * sm_count()));
}

template <class F, class K, class... Args>
cudaError_t reg_launch(K kern, long long nrows, cudaStream_t st, Args... args) {
  constexpr size_t smem = reg_smem<F>();
  static_assert(smem <= 227 * 1024, "register FFT tile exceeds shared memory");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<reg_grid<F>(nrows), kRegThreads, smem, st>>>(args...);
  return cudaGetLastError();
}

// the lengths with a register schedule (N = R1 R2)
template <class Op>
cudaError_t reg_dispatch(int n, Op op) {
  switch (n) {
    case 128: return op(RegFft<16, 8>{});
    case 256: return op(RegFft<16, 16>{});
    case 512: return op(RegFft<16, 32>{});
    case 840: return op(RegFft<28, 30>{});
    case 1024: return op(RegFft<32, 32>{});
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

bool reg_fft_supported(int n) {
  return n == 128 || n == 256 || n == 512 || n == 840 || n == 1024;
}

cudaError_t reg_rfft_rows(const FftDesc& d, const RfftSrc& src, int nt, long long nrows, double2* out, long long ld,
                          cudaStream_t st) {
  return reg_dispatch(d.n, [&](auto f) {
    using F = decltype(f);
    return reg_launch<F>(rfft_reg_kernel<F>, nrows, st, d.tw, src, nt, nrows, out, ld);
  });
}

cudaError_t reg_irfft_rows(const FftDesc& d, const double2* in, long long ld_f, long long ld_p, int nparts, int nt,
                           long long nrows, double scale, double* out, cudaStream_t st) {
  return reg_dispatch(d.n, [&](auto f) {
    using F = decltype(f);
    return reg_launch<F>(irfft_reg_kernel<F>, nrows, st, d.tw, in, ld_f, ld_p, nparts, nt, nrows, scale, out);
  });
}

cudaError_t reg_c2r_r2c_rows(const FftDesc& d, const double2* in, long long ld_f, int nt, long long nrows,
                             double scale, double* mout, double2* xout, long long ld_x, cudaStream_t st) {
  return reg_dispatch(d.n, [&](auto f) {
    using F = decltype(f);
    return reg_launch<F>(c2r_r2c_reg_kernel<F>, nrows, st, d.tw, in, ld_f, nt, nrows, scale, mout, xout, ld_x);
  });
}

}  // namespace ltb
