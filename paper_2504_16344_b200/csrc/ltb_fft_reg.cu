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
//   * the next pair's operands are prefetched by cp.async into a per-warp
//     staging buffer while the current pair computes (r2c: the two
//     contiguous rows; c2r: the pair's two half spectra, 32 contiguous bytes
//     per frequency, each element read once); strided / generated rows (plan
//     build) and summed partial slabs load directly; the zero padding is
//     never stored;
//   * the c2r rows leave from registers (coalesced across the lanes); the
//     r2c unpack (Z[k] with Z[N-k]) goes back through shared memory and
//     writes the transposed spectra out[f * ld + row] with one 256-bit store
//     per frequency for the pair.
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

// One CTA of W warps per SM (the register DFTs want ~255 registers; capping
// them at 168 for 12 warps spills).  Per warp group: the pass-1/pass-2
// exchange buffer (SEQ complex) and a staging buffer (STG complex) the NEXT
// pair's operands are prefetched into with cp.async while the current pair
// computes.  Staging: r2c rows 2 N_t doubles (N/2 complex); c2r spectra
// 2 (N_t + 1) complex.
constexpr size_t kRegSmemMax = 227 * 1024;

template <class F, bool kSpectra>
struct RegCfg {
  static constexpr int STG = kSpectra ? F::N + 2 : F::N / 2;
  static constexpr size_t per_warp = (size_t)F::S * (F::SEQ + STG) * sizeof(double2);
  static constexpr size_t tw_bytes = (size_t)F::N * sizeof(double2);
  static constexpr int W0 = (int)((kRegSmemMax - tw_bytes) / per_warp);
  static constexpr int W = W0 > 8 ? 8 : W0;
  static constexpr size_t smem = W * per_warp + tw_bytes;
  static_assert(W >= 1, "register FFT tile exceeds shared memory");
};

LTB_DEV void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
LTB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
LTB_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

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
  // both columns adjacent and 32-byte aligned: one 256-bit store per frequency
  const bool wide = has_b && cb == ca + 1 && (((uintptr_t)(out + ca) | (uintptr_t)(ld * 16)) & 31) == 0;
  for (int k = li; k <= nt; k += F::LP) {
    const double2 zk = buf[F::addr(k)];
    const double2 zn = buf[F::addr(k == 0 ? 0 : F::N - k)];
    const double2 A = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
    const double2 B = make_double2(0.5 * (zk.y + zn.y), -0.5 * (zk.x - zn.x));
    double2* p = out + (long long)k * ld + ca;
    if (wide) {
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(A.x), "d"(A.y), "d"(B.x), "d"(B.y)
                   : "memory");
    } else {
      if (has_a) *p = A;
      if (has_b) out[(long long)k * ld + cb] = B;
    }
  }
  __syncwarp();
}

LTB_DEV long long in_row(const RfftSrc& s, long long g) { return (g % s.P) * s.Q + g / s.P + s.c0; }

// r2c operands of the pair at row g into v (lane li < R2: x[li + r R2],
// rows a / b as re / im, zero past N_t): straight from memory or generated
template <class F>
LTB_DEV void direct_rows(const RfftSrc& src, int nt, long long g, long long nrows, int li, double2 (&v)[F::R1]) {
  if (li >= F::R2) return;
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

// contiguous rows g, g + 1 (16-byte aligned) -> stg as doubles [a | b]
template <class F>
LTB_DEV void prefetch_rows(const double* __restrict__ in, int nt, long long g, long long nrows, int li, double2* stg) {
  if (g >= nrows) return;
  const int chunks = (g + 1 < nrows ? 2 * nt : nt) / 2;  // N_t even on every register schedule
  const double* base = in + g * nt;
  for (int c = li; c < chunks; c += F::LP) cp_async16(stg + c, base + 2 * c);
}

template <class F>
LTB_DEV void staged_rows(const double2* stg, int nt, long long g, long long nrows, int li, double2 (&v)[F::R1]) {
  if (li >= F::R2) return;
  const double* sd = reinterpret_cast<const double*>(stg);
  const bool ha = g < nrows, hb = g + 1 < nrows;
#pragma unroll
  for (int r = 0; r < F::R1; ++r) {
    const int n = li + r * F::R2;
    v[r] = make_double2(n < nt && ha ? sd[n] : 0.0, n < nt && hb ? sd[nt + n] : 0.0);
  }
}

// the two half spectra of the pair (rows g, g + 1) -> stg[k] / stg[nf + k]:
// 32 contiguous bytes per frequency, every element read once
template <class F>
LTB_DEV void prefetch_spectra(const double2* __restrict__ in, long long ld_f, int nt, long long g, long long nrows,
                              int li, double2* stg) {
  if (g >= nrows) return;
  const int nf = nt + 1;
  const bool hb = g + 1 < nrows;
  for (int k = li; k < nf; k += F::LP) {
    const double2* p = in + (long long)k * ld_f + g;
    cp_async16(stg + k, p);
    if (hb) cp_async16(stg + nf + k, p + 1);
  }
}

// synchronous variant summing nparts slabs in a fixed order
template <class F>
LTB_DEV void load_spectra(const double2* __restrict__ in, long long ld_f, long long ld_p, int nparts, int nt,
                          long long g, long long nrows, int li, double2* stg) {
  if (g >= nrows) return;
  const int nf = nt + 1;
  const bool hb = g + 1 < nrows;
#pragma unroll 4
  for (int k = li; k < nf; k += F::LP) {
    const double2* p = in + (long long)k * ld_f + g;
    double2 a = __ldg(p), b = hb ? __ldg(p + 1) : make_double2(0.0, 0.0);
    for (int q = 1; q < nparts; ++q) {
      a = cadd(a, __ldg(p + (long long)q * ld_p));
      if (hb) b = cadd(b, __ldg(p + (long long)q * ld_p + 1));
    }
    stg[k] = a;
    stg[nf + k] = b;
  }
}

// conj of the Hermitian-extended pair spectrum Z = A + i B at the pass-1
// indices k = li + r R2 (FFTW c2r semantics: Im of DC / Nyquist ignored)
template <class F>
LTB_DEV void staged_conj_pair(const double2* stg, int nt, long long g, long long nrows, int li, double2 (&v)[F::R1]) {
  if (li >= F::R2) return;
  const int nf = nt + 1;
  const bool ha = g < nrows, hb = g + 1 < nrows;
#pragma unroll
  for (int r = 0; r < F::R1; ++r) {
    const int k = li + r * F::R2;
    const bool mirror = k > nt;
    const int kk = mirror ? F::N - k : k;
    double2 a = ha ? stg[kk] : make_double2(0.0, 0.0), b = hb ? stg[nf + kk] : make_double2(0.0, 0.0);
    if (kk == 0 || kk == nt) {
      a.y = 0.0;
      b.y = 0.0;
    }
    if (mirror) {
      a.y = -a.y;
      b.y = -b.y;
    }
    v[r] = make_double2(a.x - b.y, -(a.y + b.x));
  }
}

// warp-group geometry shared by the kernels
template <class F, int W>
struct Lanes {
  int grp, li;
  double2* buf;  // SEQ exchange buffer
  double2* stg;  // staging
  long long t0, stride, tasks;
  template <int STG>
  LTB_DEV void init(double2* smem, long long nrows) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    grp = lane / F::LP;
    li = lane % F::LP;
    double2* base = smem + F::N + (size_t)(warp * F::S + grp) * (F::SEQ + STG);
    buf = base;
    stg = base + F::SEQ;
    t0 = (long long)blockIdx.x * W + warp;
    stride = (long long)gridDim.x * W;
    tasks = ((nrows + 1) / 2 + F::S - 1) / F::S;
  }
  LTB_DEV long long row(long long t) const { return 2 * (t * F::S + grp); }
};

template <class F, int W>
__global__ void __launch_bounds__(32 * W, 1)
    rfft_reg_kernel(const double2* __restrict__ tw, const RfftSrc src, int nt, long long nrows, double2* out,
                    long long ld) {
  using C = RegCfg<F, false>;
  extern __shared__ __align__(16) double2 smem[];
  Lanes<F, W> L;
  L.template init<C::STG>(smem, nrows);
  stage_tw2<F>(tw, smem);
  const bool staged = src.bulk && !(src.oP);
  if (staged && L.t0 < L.tasks) prefetch_rows<F>(src.in, nt, L.row(L.t0), nrows, L.li, L.stg);
  cp_async_commit();
  for (long long t = L.t0; t < L.tasks; t += L.stride) {
    const long long g = L.row(t);
    double2 v[F::R1];
    if (staged) {
      cp_async_wait_all();
      __syncwarp();
      staged_rows<F>(L.stg, nt, g, nrows, L.li, v);
      __syncwarp();
      if (t + L.stride < L.tasks) prefetch_rows<F>(src.in, nt, L.row(t + L.stride), nrows, L.li, L.stg);
      cp_async_commit();
    } else {
      direct_rows<F>(src, nt, g, nrows, L.li, v);
    }
    double2 v2[F::R2];
    two_pass<F>(v, L.buf, smem, L.li, v2);
    unpack_store<F>(v2, L.buf, L.li, nt, g, nrows, src, out, ld);
  }
  cp_async_wait_all();
}

template <class F, int W>
__global__ void __launch_bounds__(32 * W, 1)
    irfft_reg_kernel(const double2* __restrict__ tw, const double2* __restrict__ in, long long ld_f, long long ld_p,
                     int nparts, int nt, long long nrows, double scale, double* __restrict__ out) {
  using C = RegCfg<F, true>;
  extern __shared__ __align__(16) double2 smem[];
  Lanes<F, W> L;
  L.template init<C::STG>(smem, nrows);
  stage_tw2<F>(tw, smem);
  const bool staged = nparts == 1;
  if (staged && L.t0 < L.tasks) prefetch_spectra<F>(in, ld_f, nt, L.row(L.t0), nrows, L.li, L.stg);
  cp_async_commit();
  for (long long t = L.t0; t < L.tasks; t += L.stride) {
    const long long g = L.row(t);
    const bool ha = g < nrows, hb = g + 1 < nrows;
    if (staged) {
      cp_async_wait_all();
    } else {
      load_spectra<F>(in, ld_f, ld_p, nparts, nt, g, nrows, L.li, L.stg);
    }
    __syncwarp();
    double2 v[F::R1];
    staged_conj_pair<F>(L.stg, nt, g, nrows, L.li, v);
    __syncwarp();
    if (staged && t + L.stride < L.tasks) prefetch_spectra<F>(in, ld_f, nt, L.row(t + L.stride), nrows, L.li, L.stg);
    cp_async_commit();
    double2 v2[F::R2];
    two_pass<F>(v, L.buf, smem, L.li, v2);
    // ifft(Z) = conj(fft(conj Z)): row a = Re Y, row b = -Im Y
    if (L.li < F::R1) {
#pragma unroll
      for (int q = 0; q < F::R2 / 2; ++q) {  // n = li + q R1 < nt = N / 2 exactly for q < R2 / 2
        const int n = L.li + q * F::R1;
        if (ha) out[g * nt + n] = v2[q].x * scale;
        if (hb) out[(g + 1) * nt + n] = -v2[q].y * scale;
      }
    }
  }
  cp_async_wait_all();
}

// c2r of a pair (rows written to mout) -> zero padded -> r2c into xout
template <class F, int W>
__global__ void __launch_bounds__(32 * W, 1)
    c2r_r2c_reg_kernel(const double2* __restrict__ tw, const double2* __restrict__ in, long long ld_f, int nt,
                       long long nrows, double scale, double* __restrict__ mout, double2* __restrict__ xout,
                       long long ld_x) {
  using C = RegCfg<F, true>;
  extern __shared__ __align__(16) double2 smem[];
  Lanes<F, W> L;
  L.template init<C::STG>(smem, nrows);
  stage_tw2<F>(tw, smem);
  const RfftSrc ident{nullptr, 0, 1, 0, 0};
  if (L.t0 < L.tasks) prefetch_spectra<F>(in, ld_f, nt, L.row(L.t0), nrows, L.li, L.stg);
  cp_async_commit();
  for (long long t = L.t0; t < L.tasks; t += L.stride) {
    const long long g = L.row(t);
    const bool ha = g < nrows, hb = g + 1 < nrows;
    const int li = L.li;
    cp_async_wait_all();
    __syncwarp();
    double2 v[F::R1];
    staged_conj_pair<F>(L.stg, nt, g, nrows, li, v);
    __syncwarp();
    if (t + L.stride < L.tasks) prefetch_spectra<F>(in, ld_f, nt, L.row(t + L.stride), nrows, li, L.stg);
    cp_async_commit();
    double2 v2[F::R2];
    two_pass<F>(v, L.buf, smem, li, v2);
    if (li < F::R1) {
#pragma unroll
      for (int q = 0; q < F::R2; ++q) {
        const int n = li + q * F::R1;
        const double a = v2[q].x * scale, b = -v2[q].y * scale;
        if (q < F::R2 / 2) {  // n < nt
          if (ha) mout[g * nt + n] = a;
          if (hb) mout[(g + 1) * nt + n] = b;
        }
        L.buf[q * F::ROW + li] = make_double2(q < F::R2 / 2 && ha ? a : 0.0, q < F::R2 / 2 && hb ? b : 0.0);
      }
    }
    __syncwarp();
    if (li < F::R2) {
#pragma unroll
      for (int r = 0; r < F::R1; ++r) {
        const int n = li + r * F::R2;
        v[r] = n < nt ? L.buf[F::addr(n)] : make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    two_pass<F>(v, L.buf, smem, li, v2);
    unpack_store<F>(v2, L.buf, li, nt, g, nrows, ident, xout, ld_x);
  }
  cp_async_wait_all();
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

template <class F, int W>
unsigned reg_grid(long long nrows) {
  const long long tasks = ((nrows + 1) / 2 + F::S - 1) / F::S;
  const long long ctas = (tasks + W - 1) / W;
  return (unsigned)std::max(1ll, std::min(ctas, (long long)sm_count()));
}

template <class F, bool kSpectra, class K, class... Args>
cudaError_t reg_launch(K kern, long long nrows, cudaStream_t st, Args... args) {
  using C = RegCfg<F, kSpectra>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
  if (e != cudaSuccess) return e;
  kern<<<reg_grid<F, C::W>(nrows), 32 * C::W, C::smem, st>>>(args...);
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
    return reg_launch<F, false>(rfft_reg_kernel<F, RegCfg<F, false>::W>, nrows, st, d.tw, src, nt, nrows, out, ld);
  });
}

cudaError_t reg_irfft_rows(const FftDesc& d, const double2* in, long long ld_f, long long ld_p, int nparts, int nt,
                           long long nrows, double scale, double* out, cudaStream_t st) {
  return reg_dispatch(d.n, [&](auto f) {
    using F = decltype(f);
    return reg_launch<F, true>(irfft_reg_kernel<F, RegCfg<F, true>::W>, nrows, st, d.tw, in, ld_f, ld_p, nparts, nt, nrows, scale, out);
  });
}

cudaError_t reg_c2r_r2c_rows(const FftDesc& d, const double2* in, long long ld_f, int nt, long long nrows,
                             double scale, double* mout, double2* xout, long long ld_x, cudaStream_t st) {
  return reg_dispatch(d.n, [&](auto f) {
    using F = decltype(f);
    return reg_launch<F, true>(c2r_r2c_reg_kernel<F, RegCfg<F, true>::W>, nrows, st, d.tw, in, ld_f, nt, nrows, scale, mout, xout, ld_x);
  });
}

}  // namespace ltb
