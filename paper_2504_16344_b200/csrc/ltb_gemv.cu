// ltb_gemv.cu -- the per-frequency complex FP64 GEMVs that stream F-hat
// (K2 GEMV-N for F m, K3 GEMV-H for F* d), plus the small reductions.
//
// Replaces fft_matvec.cpp:151-168 (out_hat[r][f] += khat_f(r,c) in_hat[c][f])
// and :192-207 (in_hat[c][f] = sum_r conj(khat_f(r,c)) d[r][f]).  F-hat keeps
// the reference layout khat[f][c][r] (r fastest), so for a fixed f a range of
// columns is ONE contiguous block of HBM: a work unit (f, column range) is a
// contiguous stream of unit_cols * Nd complex values read exactly once with
// 128-bit L1-bypassing loads.  The bound is HBM bandwidth (0.5 flop/byte);
// see DESIGN.md for the roofline.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ltb_gen.cuh"
#include "ltb_kernels.h"

namespace ltb {

namespace {

constexpr int kGemvThreads = 256;
constexpr int kGemvNMaxThreads = 512;
constexpr long long kUnitElems = 1ll << 18;  // 4 MB of F-hat per unit
constexpr int kMinUnits = 8 * 148;
constexpr size_t kBulkStage = 24 * 1024;   // target bytes per TMA stage
constexpr size_t kBulkSmem = 100 * 1024;   // stage ring per CTA (2 CTAs / SM)
constexpr int kBulkMaxStages = 8;

// ---------------------------------------------------------------------------
// GEMV-N: thread (rt, cl) owns rows rt + k RT (k < RPT) and columns
// c = c_begin + cl + j CL.  A warp's loads cover contiguous rows of one column
// (or consecutive columns when Nd < 32), so every load instruction is one
// fully coalesced 512-byte segment.  The unit's partial y goes to
// P[f][u][r]; the last unit of frequency f to finish (atomic ticket) sums the
// units_per_f partials in index order into Y[f][r] -- deterministic, and the
// partials are still L2-resident when read.
// ---------------------------------------------------------------------------
template <int RPT, int U>
__global__ void __launch_bounds__(kGemvNMaxThreads)
    gemv_n_kernel(GemvShape s, const double2* __restrict__ fhat, const double2* __restrict__ x,
                  double2* __restrict__ partials, double2* __restrict__ y,
                  unsigned* __restrict__ tickets, int RT, int CL) {
  extern __shared__ double2 red[];  // CL * RT * RPT (only when CL > 1)
  __shared__ bool last;
  const int unit = blockIdx.x;
  const int f = unit / s.units_per_f;
  const int u = unit - f * s.units_per_f;
  const int row0 = blockIdx.y * RT * RPT;  // row tile
  const long long c_begin = s.c0 + (long long)u * s.unit_cols;
  const long long c_end = min(s.c0 + s.nc, c_begin + s.unit_cols);
  const int t = threadIdx.x;
  const int rt = t % RT, cl = t / RT;
  const bool active = cl < CL;

  double2 acc[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) acc[k] = make_double2(0.0, 0.0);

  const double2* Ff = fhat + (long long)f * s.nm * s.nd;
  const double2* Xf = x + (long long)f * s.nm;
  if (active) {
    for (long long c = c_begin + cl; c < c_end; c += (long long)CL * U) {
      double2 a[U][RPT];
      double2 xv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const long long cc = c + (long long)q * CL;
        const bool ok = cc < c_end;
        xv[q] = ok ? __ldg(Xf + cc) : make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int r = row0 + rt + k * RT;
          a[q][k] = (ok && r < s.nd) ? ld_stream(Ff + cc * s.nd + r) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int k = 0; k < RPT; ++k) cmac(acc[k], a[q][k], xv[q]);
    }
  }

  if (CL > 1) {
    if (active) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) red[((size_t)cl * RPT + k) * RT + rt] = acc[k];
    }
    __syncthreads();
    if (cl == 0) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        double2 v = red[(size_t)k * RT + rt];
        for (int q = 1; q < CL; ++q) v = cadd(v, red[((size_t)q * RPT + k) * RT + rt]);
        acc[k] = v;
      }
    }
  }
  double2* P = partials + ((long long)f * s.units_per_f + u) * s.nd;
  if (cl == 0) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = row0 + rt + k * RT;
      if (r < s.nd) P[r] = acc[k];
    }
  }
  // last-unit-of-f reduction
  __threadfence();
  __syncthreads();
  if (t == 0) {
    const unsigned ticket = atomicAdd(tickets + (size_t)f * gridDim.y + blockIdx.y, 1u);
    last = (ticket == (unsigned)s.units_per_f - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double2* Pf = partials + (long long)f * s.units_per_f * s.nd;
  const int rows_here = min(RT * RPT, s.nd - row0);
  for (int i = t; i < rows_here; i += blockDim.x) {
    const int r = row0 + i;
    double2 v = __ldcg(Pf + r);
    for (int q = 1; q < s.units_per_f; ++q) v = cadd(v, __ldcg(Pf + (long long)q * s.nd + r));
    y[(long long)f * s.nd + r] = s.accumulate ? cadd(y[(long long)f * s.nd + r], v) : v;
  }
}

// ---------------------------------------------------------------------------
// GEMV-N, TMA-staged: the unit's contiguous F-hat stream is cut into chunks
// of `cps` whole columns; one thread keeps NS chunks in flight with 1-D bulk
// async copies (cp.async.bulk, L2 evict-first) completing on per-stage
// mbarriers, so the bytes in flight per SM (~2 CTAs x NS-1 stages x ~20 KB)
// cost no registers.  Consumers use the same (rt, cl) mapping as above but
// read the tile from shared memory.
// ---------------------------------------------------------------------------
template <int RPT>
__global__ void __launch_bounds__(kGemvNMaxThreads)
    gemv_n_bulk_kernel(GemvShape s, const double2* __restrict__ fhat, const double2* __restrict__ x,
                       double2* __restrict__ partials, double2* __restrict__ y,
                       unsigned* __restrict__ tickets, int RT, int CL, int cps, int NS) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  __shared__ bool last;
  // stage = [cps columns of F-hat | the cps matching x-hat values]
  const size_t chunk_elems = (size_t)cps * s.nd;
  const size_t stage_elems = chunk_elems + cps;
  double2* stages = reinterpret_cast<double2*>(bulk_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(bulk_smem + NS * stage_elems * sizeof(double2));
  const int unit = blockIdx.x;
  const int f = unit / s.units_per_f;
  const int u = unit - f * s.units_per_f;
  const long long c_begin = s.c0 + (long long)u * s.unit_cols;
  const long long c_end = min(s.c0 + s.nc, c_begin + s.unit_cols);
  const int ncols = (int)(c_end - c_begin);
  const int nchunks = (ncols + cps - 1) / cps;
  const int t = threadIdx.x;
  const int rt = t % RT, cl = t / RT;
  const bool active = cl < CL;
  const double2* src = fhat + ((long long)f * s.nm + c_begin) * s.nd;
  const double2* Xu = x + (long long)f * s.nm + c_begin;
  uint64_t policy = 0;
  if (t == 0) {
    for (int k = 0; k < NS; ++k) mbar_init(full + k, 1);
    fence_mbar_init();
    policy = policy_evict_first();
    for (int i = 0; i < NS && i < nchunks; ++i) {
      const int cols = min(cps, ncols - i * cps);
      const unsigned bytes = (unsigned)(cols * s.nd * sizeof(double2));
      const unsigned xbytes = (unsigned)(cols * sizeof(double2));
      double2* dst = stages + (size_t)i * stage_elems;
      mbar_arrive_expect_tx(full + i, bytes + xbytes);
      bulk_g2s(dst, src + (size_t)i * chunk_elems, bytes, full + i, policy);
      bulk_g2s(dst + chunk_elems, Xu + (size_t)i * cps, xbytes, full + i, policy);
    }
  }
  __syncthreads();

  double2 acc[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int i = 0; i < nchunks; ++i) {
    const int st = i % NS;
    mbar_wait(full + st, (unsigned)((i / NS) & 1));
    const int cols = min(cps, ncols - i * cps);
    const double2* S = stages + (size_t)st * stage_elems;
    const double2* XS = S + chunk_elems;
    if (active) {
      for (int cc = cl; cc < cols; cc += CL) {
        const double2 xv = XS[cc];
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int r = rt + k * RT;
          if (r < s.nd) cmac(acc[k], S[(size_t)cc * s.nd + r], xv);
        }
      }
    }
    __syncthreads();  // stage st fully consumed
    if (t == 0 && i + NS < nchunks) {
      const int j = i + NS;
      const int cols2 = min(cps, ncols - j * cps);
      const unsigned bytes = (unsigned)(cols2 * s.nd * sizeof(double2));
      const unsigned xbytes = (unsigned)(cols2 * sizeof(double2));
      double2* dst = stages + (size_t)st * stage_elems;
      mbar_arrive_expect_tx(full + st, bytes + xbytes);
      bulk_g2s(dst, src + (size_t)j * chunk_elems, bytes, full + st, policy);
      bulk_g2s(dst + chunk_elems, Xu + (size_t)j * cps, xbytes, full + st, policy);
    }
  }

  // cross-lane reduction (reuses stage 0; all copies have completed)
  double2* red = stages;
  if (CL > 1) {
    if (active) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) red[((size_t)cl * RPT + k) * RT + rt] = acc[k];
    }
    __syncthreads();
    if (cl == 0) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        double2 v = red[(size_t)k * RT + rt];
        for (int q = 1; q < CL; ++q) v = cadd(v, red[((size_t)q * RPT + k) * RT + rt]);
        acc[k] = v;
      }
    }
  }
  double2* P = partials + ((long long)f * s.units_per_f + u) * s.nd;
  if (cl == 0) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = rt + k * RT;
      if (r < s.nd) P[r] = acc[k];
    }
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    const unsigned ticket = atomicAdd(tickets + f, 1u);
    last = (ticket == (unsigned)s.units_per_f - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double2* Pf = partials + (long long)f * s.units_per_f * s.nd;
  for (int r = t; r < s.nd; r += blockDim.x) {
    double2 v = __ldcg(Pf + r);
    for (int q = 1; q < s.units_per_f; ++q) v = cadd(v, __ldcg(Pf + (long long)q * s.nd + r));
    y[(long long)f * s.nd + r] = s.accumulate ? cadd(y[(long long)f * s.nd + r], v) : v;
  }
}

// ---------------------------------------------------------------------------
// GEMV-H, TMA-staged: F-hat chunks of `cps` columns arrive by bulk async copy
// as in GEMV-N; a group of GS lanes owns one column at a time, lane l holding
// d-hat_f[l + GS k] (k < RPL) in registers for the whole unit.  With GS >= 8 a
// quarter-warp reads one contiguous 128-byte line per shared load, so the
// reads are conflict-free; 32/GS columns close their dot products in the
// same log2(GS)-level shuffle tree.  Loops are warp-uniform so every lane
// takes part in every shuffle.
// ---------------------------------------------------------------------------
template <int GS, int RPL>
__global__ void __launch_bounds__(kGemvThreads)
    gemv_h_bulk_kernel(GemvShape s, const double2* __restrict__ fhat,
                       const double2* __restrict__ dhat, double2* __restrict__ xo, int cps, int NS) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  const size_t stage_elems = (size_t)cps * s.nd;
  double2* stages = reinterpret_cast<double2*>(bulk_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(bulk_smem + NS * stage_elems * sizeof(double2));
  const int unit = blockIdx.x;
  const int f = unit / s.units_per_f;
  const int u = unit - f * s.units_per_f;
  const long long c_begin = s.c0 + (long long)u * s.unit_cols;
  const long long c_end = min(s.c0 + s.nc, c_begin + s.unit_cols);
  const int ncols = (int)(c_end - c_begin);
  const int nchunks = (ncols + cps - 1) / cps;
  const int t = threadIdx.x;
  const double2* src = fhat + ((long long)f * s.nm + c_begin) * s.nd;
  uint64_t policy = 0;
  if (t == 0) {
    for (int k = 0; k < NS; ++k) mbar_init(full + k, 1);
    fence_mbar_init();
    policy = policy_evict_first();
    for (int i = 0; i < NS && i < nchunks; ++i) {
      const int cols = min(cps, ncols - i * cps);
      const unsigned bytes = (unsigned)(cols * s.nd * sizeof(double2));
      mbar_arrive_expect_tx(full + i, bytes);
      bulk_g2s(stages + (size_t)i * stage_elems, src + (size_t)i * stage_elems, bytes, full + i, policy);
    }
  }
  const int lane = t % GS;
  constexpr int GPW = 32 / GS;  // column groups per warp
  const int warp = t / 32, gw = (t % 32) / GS, nwarps = blockDim.x / 32;
  double2 dv[RPL];
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int r = lane + GS * k;
    dv[k] = r < s.nd ? __ldg(dhat + (long long)f * s.nd + r) : make_double2(0.0, 0.0);
  }
  double2* xout = xo + (long long)f * s.nm + c_begin;
  __syncthreads();
  for (int i = 0; i < nchunks; ++i) {
    const int st = i % NS;
    mbar_wait(full + st, (unsigned)((i / NS) & 1));
    const int cols = min(cps, ncols - i * cps);
    const double2* S = stages + (size_t)st * stage_elems;
    for (int base = warp * GPW; base < cols; base += nwarps * GPW) {
      const int cc = base + gw;
      const bool ok = cc < cols;
      double2 acc = make_double2(0.0, 0.0);
      if (ok) {
        const double2* col = S + (size_t)cc * s.nd;
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const int r = lane + GS * k;
          if (r < s.nd) cmac_conj(acc, col[r], dv[k]);
        }
      }
#pragma unroll
      for (int m = GS / 2; m > 0; m >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m, GS);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m, GS);
      }
      if (ok && lane == 0) xout[(size_t)i * cps + cc] = acc;
    }
    __syncthreads();  // stage st fully consumed
    if (t == 0 && i + NS < nchunks) {
      const int j = i + NS;
      const int cols2 = min(cps, ncols - j * cps);
      const unsigned bytes = (unsigned)(cols2 * s.nd * sizeof(double2));
      mbar_arrive_expect_tx(full + st, bytes);
      bulk_g2s(stages + (size_t)st * stage_elems, src + (size_t)j * stage_elems, bytes, full + st, policy);
    }
  }
}

// ---------------------------------------------------------------------------
// GEMV-H: GS lanes per column (GS = 32 for Nd >= 32), lane l owns rows
// l + j GS; d-hat_f staged once per unit in shared memory; the dot product
// closes with a width-GS shuffle tree.  KU independent 128-bit loads per lane
// per step keep ~KU * 512 B in flight per warp.
// ---------------------------------------------------------------------------
template <int GS, int KU>
__global__ void __launch_bounds__(kGemvThreads)
    gemv_h_kernel(GemvShape s, const double2* __restrict__ fhat, const double2* __restrict__ dhat,
                  double2* __restrict__ xo) {
  extern __shared__ double2 dsm[];  // nd
  const int unit = blockIdx.x;
  const int f = unit / s.units_per_f;
  const int u = unit - f * s.units_per_f;
  const long long c_begin = s.c0 + (long long)u * s.unit_cols;
  const long long c_end = min(s.c0 + s.nc, c_begin + s.unit_cols);
  for (int r = threadIdx.x; r < s.nd; r += blockDim.x) dsm[r] = __ldg(dhat + (long long)f * s.nd + r);
  __syncthreads();
  const int lane = threadIdx.x % GS;
  constexpr int GPW = 32 / GS;
  const int warp = threadIdx.x / 32, gw = (threadIdx.x % 32) / GS, nwarps = blockDim.x / 32;
  const double2* Ff = fhat + (long long)f * s.nm * s.nd;
  // warp-uniform trip count: every lane reaches every shuffle
  for (long long base = c_begin + warp * GPW; base < c_end; base += (long long)nwarps * GPW) {
    const long long c = base + gw;
    const bool ok = c < c_end;
    const double2* col = Ff + c * s.nd;
    double2 acc = make_double2(0.0, 0.0);
    for (int r0 = lane; ok && r0 < s.nd; r0 += GS * KU) {
      double2 a[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int r = r0 + k * GS;
        a[k] = r < s.nd ? ld_stream(col + r) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int r = r0 + k * GS;
        if (r < s.nd) cmac_conj(acc, a[k], dsm[r]);
      }
    }
#pragma unroll
    for (int m = GS / 2; m > 0; m >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m, GS);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m, GS);
    }
    if (ok && lane == 0) xo[(long long)f * s.nm + c] = acc;
  }
}

// ---------------------------------------------------------------------------
// sum |z|^2, deterministic: fixed grid, per-block tree, then one block.
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 1024;

__global__ void __launch_bounds__(256) sqnorm_partial_kernel(const double2* __restrict__ z, long long n,
                                                             double* __restrict__ work) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldg(z + i);
    acc = fma(v.x, v.x, acc);
    acc = fma(v.y, v.y, acc);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int m = 128; m > 0; m >>= 1) {
    if (threadIdx.x < m) sh[threadIdx.x] += sh[threadIdx.x + m];
    __syncthreads();
  }
  if (threadIdx.x == 0) work[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) sum_kernel(const double* __restrict__ work, int n, double* out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += work[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int m = 128; m > 0; m >>= 1) {
    if (threadIdx.x < m) sh[threadIdx.x] += sh[threadIdx.x + m];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void gen_fill_kernel(uint64_t key, uint64_t index0, long long n, double* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = gen_uniform_keyed(key, index0 + (uint64_t)i);
}

struct NConfig {
  int rpt, rt, cl, threads;
};

NConfig n_config(int nd) {
  NConfig c;
  c.rpt = 1;
  while (c.rpt < 8 && (nd + c.rpt - 1) / c.rpt > 512) c.rpt *= 2;
  c.rt = std::min(512, (nd + c.rpt - 1) / c.rpt);
  c.cl = c.rt >= 256 ? 1 : std::max(1, 256 / c.rt);
  c.threads = ((c.rt * c.cl + 31) / 32) * 32;
  return c;
}

}  // namespace

GemvShape gemv_shape(int nd, long long nm, int nf, int unit_cols_hint) {
  GemvShape s;
  s.nd = nd;
  s.nm = nm;
  s.nf = nf;
  long long uc = unit_cols_hint > 0 ? unit_cols_hint : std::max(1ll, kUnitElems / std::max(1, nd));
  // keep enough units to fill the machine on small problems
  if (unit_cols_hint <= 0) {
    const long long upf = (nm + uc - 1) / uc;
    if ((long long)nf * upf < kMinUnits) {
      uc = std::max(1ll, ((long long)nf * nm + kMinUnits - 1) / kMinUnits);
    }
  }
  uc = std::min(uc, nm);
  s.unit_cols = (int)uc;
  s.units_per_f = (int)((nm + uc - 1) / uc);
  s.c0 = 0;
  s.nc = nm;
  s.accumulate = 0;
  return s;
}

GemvShape gemv_window(const GemvShape& s, long long c0, long long nc, int accumulate) {
  GemvShape w = s;
  w.c0 = c0;
  w.nc = nc;
  w.units_per_f = (int)((nc + s.unit_cols - 1) / s.unit_cols);
  w.accumulate = accumulate;
  return w;
}

size_t gemv_n_partials(const GemvShape& s) {
  return (size_t)s.nf * s.units_per_f * s.nd;
}
int gemv_n_row_tiles(const GemvShape& s) {
  const NConfig c = n_config(s.nd);
  return (s.nd + c.rt * c.rpt - 1) / (c.rt * c.rpt);
}

cudaError_t launch_gemv_n(const GemvShape& s_in, const double2* fhat, const double2* x,
                          double2* partials, double2* y, unsigned* tickets,
                          cudaStream_t st) {
  // Small problems: gemv_shape widened the split to fill the machine, but
  // every extra unit per frequency is another partial for GEMV-N's
  // last-unit reduction -- here about one wave of 2 CTAs per SM is faster
  // (tools/gemv_units.py: F_q of config 2, 63.5 -> 52 us).  Fewer units than
  // the plan's shape always fit its partials buffer.
  GemvShape s = s_in;
  {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    if ((long long)s.nf * s.units_per_f <= kMinUnits + s.nf) {
      const int upf = std::max(1, 2 * sms / std::max(1, s.nf));
      if (upf < s.units_per_f) {
        s.unit_cols = (int)((s.nc + upf - 1) / upf);
        s.units_per_f = (int)((s.nc + s.unit_cols - 1) / s.unit_cols);
      }
    }
  }
  const NConfig c = n_config(s.nd);
  const int tiles = (s.nd + c.rt * c.rpt - 1) / (c.rt * c.rpt);
  cudaError_t e = cudaMemsetAsync(tickets, 0, sizeof(unsigned) * (size_t)s.nf * tiles, st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((long long)s.nf * s.units_per_f), (unsigned)tiles);
  // TMA-staged path whenever one row tile covers Nd and >= 2 stages of whole
  // columns fit in ~100 KB (two CTAs per SM); LTB_GEMV_N=ldg forces the
  // register-staged kernel (A/B tuning knob)
  const size_t col_bytes = (size_t)s.nd * sizeof(double2);
  static const char* knob = getenv("LTB_GEMV_N");
  const bool want_bulk = !(knob && strcmp(knob, "ldg") == 0);
  if (want_bulk && tiles == 1 && 2 * col_bytes <= kBulkSmem) {
    const int cps = (int)std::max<size_t>(1, kBulkStage / col_bytes);
    const size_t stage_bytes = (size_t)cps * (col_bytes + sizeof(double2));
    const int ns = (int)std::min<size_t>(kBulkMaxStages, kBulkSmem / stage_bytes);
    const size_t red_bytes = (size_t)c.cl * c.rt * c.rpt * sizeof(double2);
    const size_t smem_al = std::max((size_t)ns * stage_bytes, red_bytes) + 8 * kBulkMaxStages;
#define LTB_NB(R)                                                                              \
  do {                                                                                         \
    cudaFuncSetAttribute(gemv_n_bulk_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                         (int)smem_al);                                                        \
    gemv_n_bulk_kernel<R><<<grid, c.threads, smem_al, st>>>(s, fhat, x, partials, y, tickets,  \
                                                            c.rt, c.cl, cps, ns);              \
  } while (0)
    switch (c.rpt) {
      case 1: LTB_NB(1); break;
      case 2: LTB_NB(2); break;
      case 4: LTB_NB(4); break;
      default: LTB_NB(8); break;
    }
#undef LTB_NB
    return cudaGetLastError();
  }
  const size_t smem = c.cl > 1 ? (size_t)c.cl * c.rt * c.rpt * sizeof(double2) : 0;
  constexpr int U = 4;
  switch (c.rpt) {
    case 1: gemv_n_kernel<1, U><<<grid, c.threads, smem, st>>>(s, fhat, x, partials, y, tickets, c.rt, c.cl); break;
    case 2: gemv_n_kernel<2, U><<<grid, c.threads, smem, st>>>(s, fhat, x, partials, y, tickets, c.rt, c.cl); break;
    case 4: gemv_n_kernel<4, U><<<grid, c.threads, smem, st>>>(s, fhat, x, partials, y, tickets, c.rt, c.cl); break;
    default: gemv_n_kernel<8, U><<<grid, c.threads, smem, st>>>(s, fhat, x, partials, y, tickets, c.rt, c.cl); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_gemv_h(const GemvShape& s, const double2* fhat, const double2* dhat,
                          double2* xo, cudaStream_t st) {
  const dim3 grid((unsigned)((long long)s.nf * s.units_per_f));
  // TMA-staged path for Nd <= 768 (d-hat fits the lanes' registers);
  // LTB_GEMV_H=ldg forces the register-staged kernel (A/B tuning knob)
  static const char* knob = getenv("LTB_GEMV_H");
  const bool want_bulk = !(knob && strcmp(knob, "ldg") == 0);
  const size_t col_bytes = (size_t)s.nd * sizeof(double2);
  if (want_bulk && s.nd <= 768) {
    const int gsb = s.nd <= 64 ? 8 : (s.nd <= 128 ? 16 : 32);
    const int need = (s.nd + gsb - 1) / gsb;
    const int cps = (int)std::max<size_t>(1, kBulkStage / col_bytes);
    const size_t stage_bytes = (size_t)cps * col_bytes;
    const int ns = (int)std::min<size_t>(kBulkMaxStages, kBulkSmem / stage_bytes);
    const size_t smem_b = (size_t)ns * stage_bytes + 8 * kBulkMaxStages;
#define LTB_HB(G, R)                                                                            \
  do {                                                                                          \
    cudaFuncSetAttribute(gemv_h_bulk_kernel<G, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem_b);                                                          \
    gemv_h_bulk_kernel<G, R><<<grid, kGemvThreads, smem_b, st>>>(s, fhat, dhat, xo, cps, ns);   \
  } while (0)
    if (gsb == 8) {
      if (need <= 1) LTB_HB(8, 1);
      else if (need <= 2) LTB_HB(8, 2);
      else if (need <= 4) LTB_HB(8, 4);
      else LTB_HB(8, 8);
    } else if (gsb == 16) {
      LTB_HB(16, 8);
    } else {
      if (need <= 8) LTB_HB(32, 8);
      else if (need <= 12) LTB_HB(32, 12);
      else if (need <= 16) LTB_HB(32, 16);
      else if (need <= 20) LTB_HB(32, 20);
      else LTB_HB(32, 24);
    }
#undef LTB_HB
    return cudaGetLastError();
  }
  const size_t smem = (size_t)s.nd * sizeof(double2);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  constexpr int KU = 8;
  int gs = 1;
  while (gs < 32 && gs < s.nd) gs *= 2;
#define LTB_H(G)                                                                           \
  do {                                                                                     \
    if (smem > 48 * 1024)                                                                  \
      cudaFuncSetAttribute(gemv_h_kernel<G, KU>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                     \
    gemv_h_kernel<G, KU><<<grid, kGemvThreads, smem, st>>>(s, fhat, dhat, xo);             \
  } while (0)
  switch (gs) {
    case 1: LTB_H(1); break;
    case 2: LTB_H(2); break;
    case 4: LTB_H(4); break;
    case 8: LTB_H(8); break;
    case 16: LTB_H(16); break;
    default: LTB_H(32); break;
  }
#undef LTB_H
  return cudaGetLastError();
}

cudaError_t launch_sqnorm(const double2* z, long long n, double* work, double* out,
                          cudaStream_t st) {
  sqnorm_partial_kernel<<<kRedBlocks, 256, 0, st>>>(z, n, work);
  sum_kernel<<<1, 256, 0, st>>>(work, kRedBlocks, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_fill(uint64_t key, uint64_t index0, long long n, double* out,
                            cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((n + 255) / 256, 148 * 64);
  gen_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(key, index0, n, out);
  return cudaGetLastError();
}

}  // namespace ltb
