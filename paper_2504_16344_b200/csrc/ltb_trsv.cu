// ltb_trsv.cu -- blocked triangular solves for K^{-1} = L^{-T} L^{-1}
// (bayes_engine.cpp:236-240) on sm_100a.
//
// Single-RHS TRSV is a GEMV over the packed factor (HBM bound, ~0.25
// flop/byte) plus a sequential dependency chain over the nb = n/64 diagonal
// blocks.  Design:
//   * one persistent cooperative launch per sweep; CTA b owns block rows
//     b, b + G, b + 2G, ... and processes them in sweep order, so every CTA
//     streams its panel tiles while the chain is still far behind and only
//     the last tile + the diagonal block sit on the critical path;
//   * each thread keeps ONE running partial (forward) / sixteen (transposed)
//     in registers across all tiles of its row and prefetches the next tile
//     while waiting; the row is reduced once at the end;
//   * rows complete strictly in chain order, so a single 64-bit progress
//     word (epoch << 32 | rows done) replaces per-row flags: a thread polls
//     it (ld.acquire.gpu) only when it needs a block beyond what it already
//     saw published;
//   * diagonal blocks are applied through their precomputed inverses
//     (L_II^{-1}, inverted once at set_factor time), so the critical path is
//     two 64x64 GEMVs instead of a 64-step substitution.
#include <math.h>

#include "ltb_common.cuh"
#include "ltb_gen.cuh"
#include "ltb_trsv.h"

namespace ltb {

namespace {

constexpr int kThreads = 256;
constexpr int kPad = 65;                      // padded smem tile stride
constexpr unsigned long long kSpinNs = 4000000000ull;  // 4 s dependency-wait timeout

LTB_DEV unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
LTB_DEV void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
LTB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait until the progress word reaches `need`; returns the value seen.  On
// timeout (or once any CTA has timed out) it sets *status and returns `need`
// so the kernel still runs to completion -- the host then reports the error
// instead of the GPU hanging.
LTB_DEV unsigned long long wait_progress(const unsigned long long* prog, unsigned long long need,
                                         int* status) {
  unsigned long long v = ld_acquire(prog);
  if (v >= need) return v;
  const unsigned long long t0 = globaltimer();
  while (true) {
    v = ld_acquire(prog);
    if (v >= need) return v;
    if (*(volatile int*)status) return need;
    if (globaltimer() - t0 > kSpinNs) {
      atomicExch(status, 1);
      return need;
    }
    __nanosleep(64);
  }
}

LTB_DEV size_t tile_off(int I, int J) { return ((size_t)I * (I + 1) / 2 + J) * (kTB * kTB); }

// ---------------------------------------------------------------------------
// forward: y_I = Dinv_II (b_I - sum_{J<I} L_IJ y_J), rows in increasing order
// thread (i = tid & 63, q = tid >> 6) owns row i and columns [16q, 16q+16)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2)
    trsv_fwd_kernel(const double* __restrict__ tiles, const double* __restrict__ dinv,
                    double* y, unsigned long long* prog, unsigned epoch, int nb, int* status) {
  __shared__ double sD[kTB * kPad];
  __shared__ double red[4][kTB];
  __shared__ double rr[kTB];
  const int tid = threadIdx.x, i = tid & 63, q = tid >> 6;
  const unsigned long long base = (unsigned long long)epoch << 32;
  unsigned long long seen = 0;
  for (int I = blockIdx.x; I < nb; I += gridDim.x) {
    const double* D = dinv + (size_t)I * kTB * kTB;
    for (int e = tid; e < kTB * kTB; e += kThreads) sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
    const double* row = tiles + tile_off(I, 0);
    double a[16], an[16];
    double acc = 0.0;
    if (I > 0) {
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = __ldg(row + (16 * q + k) * kTB + i);
    }
    for (int J = 0; J < I; ++J) {
      if (J + 1 < I) {
        const double* nt = row + (size_t)(J + 1) * kTB * kTB;
#pragma unroll
        for (int k = 0; k < 16; ++k) an[k] = __ldg(nt + (16 * q + k) * kTB + i);
      }
      if (seen < base + J + 1) {
        seen = wait_progress(prog, base + J + 1, status);
      }
      const double* yJ = y + (size_t)J * kTB + 16 * q;
#pragma unroll
      for (int k = 0; k < 16; ++k) acc = fma(a[k], __ldcg(yJ + k), acc);
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = an[k];
    }
    red[q][i] = acc;
    __syncthreads();
    if (tid < kTB) rr[tid] = __ldcg(y + (size_t)I * kTB + tid) - ((red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]));
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s = fma(sD[(16 * q + k) * kPad + i], rr[16 * q + k], s);
    red[q][i] = s;
    __syncthreads();
    if (tid < kTB) {
      y[(size_t)I * kTB + tid] = (red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release(prog, base + I + 1);
  }
}

// ---------------------------------------------------------------------------
// transposed: x_I = Dinv_II^T (y_I - sum_{J>I} L_JI^T x_J), rows in decreasing
// order; thread (j = tid & 63, q = tid >> 6) reads row j of tile L_JI,
// columns [16q, 16q+16), keeping 16 partial sums.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    trsv_bwd_kernel(const double* __restrict__ tiles, const double* __restrict__ dinv,
                    double* y, unsigned long long* prog, unsigned epoch, int nb, int* status) {
  __shared__ double sD[kTB * kPad];
  __shared__ double sR[2 * kTB];
  __shared__ double sP[4][kTB];
  __shared__ double rr[kTB];
  const int tid = threadIdx.x, j = tid & 63, q = tid >> 6;
  const unsigned long long base = (unsigned long long)epoch << 32;
  unsigned long long seen = 0;
  const int G = gridDim.x;
  // CTA b owns rows nb-1-b, nb-1-b-G, ...
  for (int I = nb - 1 - (int)blockIdx.x; I >= 0; I -= G) {
    const double* D = dinv + (size_t)I * kTB * kTB;
    for (int e = tid; e < kTB * kTB; e += kThreads) sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    double a[16], an[16];
    if (I + 1 < nb) {
      const double* t = tiles + tile_off(nb - 1, I);
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = __ldg(t + (16 * q + k) * kTB + j);
    }
    for (int J = nb - 1; J > I; --J) {
      if (J - 1 > I) {
        const double* t = tiles + tile_off(J - 1, I);
#pragma unroll
        for (int k = 0; k < 16; ++k) an[k] = __ldg(t + (16 * q + k) * kTB + j);
      }
      const unsigned long long need = base + (unsigned long long)(nb - J);
      if (seen < need) {
        seen = wait_progress(prog, need, status);
      }
      const double xj = __ldcg(y + (size_t)J * kTB + j);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fma(a[k], xj, acc[k]);
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = an[k];
    }
    // reduce over j: 32-lane shuffle tree per partial, then the two warps of
    // each column quarter meet in shared memory
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double v = acc[k];
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
      acc[k] = v;
    }
    if ((j & 31) == 0) {
#pragma unroll
      for (int k = 0; k < 16; ++k) sR[(j >> 5) * kTB + 16 * q + k] = acc[k];
    }
    __syncthreads();
    if (tid < kTB) rr[tid] = __ldcg(y + (size_t)I * kTB + tid) - (sR[tid] + sR[kTB + tid]);
    __syncthreads();
    {
      const int ii = tid & 63, part = tid >> 6;
      double s = 0.0;
      // (Dinv^T)[ii][jj] = Dinv[jj][ii] = sD[ii * kPad + jj]
#pragma unroll
      for (int k = 0; k < 16; ++k) s = fma(sD[ii * kPad + 16 * part + k], rr[16 * part + k], s);
      sP[part][ii] = s;
    }
    __syncthreads();
    if (tid < kTB) {
      y[(size_t)I * kTB + tid] = (sP[0][tid] + sP[1][tid]) + (sP[2][tid] + sP[3][tid]);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release(prog, base + (unsigned long long)(nb - I));
  }
}

// tile (I, J) for tile index t = I (I+1)/2 + J
LTB_DEV void tile_ij(long long t, int* I, int* J) {
  long long r = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (r * (r + 1) / 2 > t) --r;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  *I = (int)r;
  *J = (int)(t - r * (r + 1) / 2);
}

__global__ void pack_colmajor_kernel(const double* __restrict__ L, size_t ld, int n,
                                     double* __restrict__ tiles) {
  int I, J;
  tile_ij(blockIdx.x, &I, &J);
  double* dst = tiles + (size_t)blockIdx.x * kTB * kTB;
  for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
    const int jj = e >> 6, ii = e & 63;
    const int r = I * kTB + ii, c = J * kTB + jj;
    double v;
    if (r < n && c < n) v = (c <= r) ? L[(size_t)c * ld + r] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    dst[e] = v;
  }
}

__global__ void pack_generated_kernel(uint64_t key, int n, double scale, double* __restrict__ tiles) {
  int I, J;
  tile_ij(blockIdx.x, &I, &J);
  double* dst = tiles + (size_t)blockIdx.x * kTB * kTB;
  for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
    const int jj = e >> 6, ii = e & 63;
    const int r = I * kTB + ii, c = J * kTB + jj;
    double v;
    if (r < n && c < n) v = gen_factor_entry(key, n, scale, r, c);
    else v = (r == c) ? 1.0 : 0.0;
    dst[e] = v;
  }
}

// one CTA per diagonal tile, thread c solves L_II x = e_c
__global__ void __launch_bounds__(64) invert_diag_kernel(const double* __restrict__ tiles,
                                                         double* __restrict__ dinv, int* status) {
  extern __shared__ double inv_smem[];
  double* sL = inv_smem;              // kTB * kPad
  double* sX = inv_smem + kTB * kPad;  // kTB * kPad
  const int I = blockIdx.x, c = threadIdx.x;
  const double* T = tiles + tile_off(I, I);
  for (int e = c; e < kTB * kTB; e += kTB) sL[(e >> 6) * kPad + (e & 63)] = T[e];
  __syncthreads();
  for (int i = 0; i < kTB; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
    if (i >= c) {
      for (int k = c; k < i; ++k) s -= sL[k * kPad + i] * sX[c * kPad + k];
      const double d = sL[i * kPad + i];
      if (!(d != 0.0) || !isfinite(d)) atomicExch(status, 2);
      s = s / d;
    } else {
      s = 0.0;
    }
    sX[c * kPad + i] = s;
  }
  __syncthreads();
  double* D = dinv + (size_t)I * kTB * kTB;
  for (int e = c; e < kTB * kTB; e += kTB) D[e] = sX[(e >> 6) * kPad + (e & 63)];
}

int g_coop_grid = -1;

}  // namespace

cudaError_t trsv_alloc(TriFactor& t, int n) {
  trsv_free(t);
  t.n = n;
  t.nb = (n + kTB - 1) / kTB;
  const size_t ntiles = (size_t)t.nb * (t.nb + 1) / 2;
  t.bytes = (ntiles + t.nb) * kTB * kTB * sizeof(double);
  cudaError_t e;
  if ((e = cudaMalloc(&t.tiles, ntiles * kTB * kTB * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.dinv, (size_t)t.nb * kTB * kTB * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.flags, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.status, sizeof(int))) != cudaSuccess) return e;
  cudaMemset(t.flags, 0, 2 * sizeof(unsigned long long));
  cudaMemset(t.status, 0, sizeof(int));
  t.epoch = 0;
  return cudaSuccess;
}

void trsv_free(TriFactor& t) {
  cudaFree(t.tiles);
  cudaFree(t.dinv);
  cudaFree(t.flags);
  cudaFree(t.status);
  t = TriFactor();
}

cudaError_t trsv_pack_colmajor(TriFactor& t, const double* L, size_t ld, cudaStream_t st) {
  const size_t ntiles = (size_t)t.nb * (t.nb + 1) / 2;
  pack_colmajor_kernel<<<(unsigned)ntiles, 256, 0, st>>>(L, ld, t.n, t.tiles);
  return cudaGetLastError();
}

cudaError_t trsv_pack_generated(TriFactor& t, uint64_t seed, cudaStream_t st) {
  const size_t ntiles = (size_t)t.nb * (t.nb + 1) / 2;
  const double scale = 0.5 / sqrt((double)t.n);
  pack_generated_kernel<<<(unsigned)ntiles, 256, 0, st>>>(gen_key(seed, kStreamFactor), t.n, scale,
                                                          t.tiles);
  return cudaGetLastError();
}

cudaError_t trsv_invert_diag(TriFactor& t, cudaStream_t st) {
  const int smem = 2 * kTB * kPad * (int)sizeof(double);
  cudaFuncSetAttribute(invert_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  invert_diag_kernel<<<t.nb, kTB, smem, st>>>(t.tiles, t.dinv, t.status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int h = 0;
  e = cudaMemcpyAsync(&h, t.status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  return h ? cudaErrorInvalidValue : cudaSuccess;
}

cudaError_t trsv_solve(TriFactor& t, double* y, cudaStream_t st) {
  if (g_coop_grid < 0) {
    int dev = 0, sms = 0, per = 0, per2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, trsv_fwd_kernel, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, trsv_bwd_kernel, kThreads, 0);
    g_coop_grid = sms * (per < per2 ? per : per2);
    if (g_coop_grid < 1) g_coop_grid = 1;
  }
  const int grid = t.nb < g_coop_grid ? t.nb : g_coop_grid;
  ++t.epoch;
  unsigned long long* prog_f = reinterpret_cast<unsigned long long*>(t.flags);
  unsigned long long* prog_b = prog_f + 1;
  void* args_f[] = {(void*)&t.tiles, (void*)&t.dinv, (void*)&y, (void*)&prog_f, (void*)&t.epoch,
                    (void*)&t.nb, (void*)&t.status};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)trsv_fwd_kernel, grid, kThreads, args_f, 0, st);
  if (e != cudaSuccess) return e;
  void* args_b[] = {(void*)&t.tiles, (void*)&t.dinv, (void*)&y, (void*)&prog_b, (void*)&t.epoch,
                    (void*)&t.nb, (void*)&t.status};
  return cudaLaunchCooperativeKernel((const void*)trsv_bwd_kernel, grid, kThreads, args_b, 0, st);
}

}  // namespace ltb
