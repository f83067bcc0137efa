// ltb_trsv.cu -- blocked triangular solves for K^{-1} = L^{-T} L^{-1}
// (bayes_engine.cpp:236-240) on sm_100a.
//
// Single-RHS TRSV is a GEMV over the packed factor (HBM bound, ~0.25
// flop/byte) plus a sequential dependency chain over the nb = n/64 diagonal
// blocks.  The design splits the two:
//
//   * one persistent cooperative launch per sweep; CTA 0 is the CHAIN CTA,
//     CTAs 1..G-1 are WORKERS;
//   * worker rows (round robin) stream their panel tiles as soon as the
//     needed solution blocks are published, but stop kLook tiles short of
//     the diagonal and hand the chain c_I = L_II^{-1} (b_I - sum_{J<I-kLook}
//     L_IJ y_J);
//   * the chain finishes y_I = c_I - sum_{k=1..kLook} M_{I,k} y_{I-k} with the
//     precomputed M_{I,k} = L_II^{-1} L_{I,I-k} (prefetched into registers a
//     step ahead) and the last kLook blocks of y kept in shared memory, so
//     the critical path per block is one 64 x (64 kLook) GEMV plus one flag
//     round trip -- the workers' streaming latency is hidden behind kLook
//     chain steps;
//   * rows complete in chain order, so one 64-bit progress word
//     (epoch << 32 | rows done) tells every worker which blocks are final;
//     worker results use per-row epoch flags.
//
// The transposed sweep is the mirror image (rows in decreasing order, panel
// tiles read down the block column, M'_{I,k} = L_II^{-T} L_{I+k,I}^T).
#include <math.h>

#include "ltb_common.cuh"
#include "ltb_gen.cuh"
#include "ltb_trsv.h"

namespace ltb {

namespace {

constexpr int kThreads = 256;
constexpr int kPad = 65;                               // padded smem tile stride
constexpr int kTile = kTB * kTB;
constexpr unsigned long long kSpinNs = 4000000000ull;  // 4 s dependency-wait timeout

LTB_DEV unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
LTB_DEV unsigned ld_acquire32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
LTB_DEV void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
LTB_DEV void st_release32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
LTB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait until the progress word reaches `need`.  On timeout (or once any CTA
// has timed out) set *status and return `need`, so the kernel still runs to
// completion and the host reports the error instead of the GPU hanging.
LTB_DEV unsigned long long wait_progress(const unsigned long long* prog, unsigned long long need,
                                         int* status) {
  unsigned long long v = ld_acquire64(prog);
  if (v >= need) return v;
  const unsigned long long t0 = globaltimer();
  while (true) {
    v = ld_acquire64(prog);
    if (v >= need) return v;
    if (*(volatile int*)status) return need;
    if (globaltimer() - t0 > kSpinNs) {
      atomicExch(status, 1);
      return need;
    }
    __nanosleep(32);
  }
}

LTB_DEV void wait_flag(const unsigned* flag, unsigned epoch, int* status) {
  if (ld_acquire32(flag) == epoch) return;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire32(flag) != epoch) {
    if (*(volatile int*)status) return;
    if (globaltimer() - t0 > kSpinNs) {
      atomicExch(status, 1);
      return;
    }
    __nanosleep(32);
  }
}

LTB_DEV size_t tile_off(int I, int J) { return ((size_t)I * (I + 1) / 2 + J) * kTile; }

// ---------------------------------------------------------------------------
// forward sweep: y <- L^{-1} y
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    trsv_fwd_kernel(const double* __restrict__ tiles, const double* __restrict__ dinv,
                    const double* __restrict__ mf, double* y, double* cbuf, unsigned* cflag,
                    unsigned long long* prog, unsigned epoch, int nb, int* status) {
  __shared__ double sD[kTB * kPad];
  __shared__ double red[4][kTB];
  __shared__ double rr[kTB];
  __shared__ double ys[kLook][kTB];
  const int tid = threadIdx.x, i = tid & 63, q = tid >> 6;
  const unsigned long long base = (unsigned long long)epoch << 32;

  if (blockIdx.x == 0) {
    // ---------------- chain CTA ----------------
    double mreg[kLook][16], mnext[kLook][16];
    for (int I = 0; I < nb; ++I) {
      // prefetch the chain tiles of step I+1 (independent of everything else)
      if (I + 1 < nb) {
#pragma unroll
        for (int k = 0; k < kLook; ++k) {
          if (k + 1 <= I + 1) {
            const double* M = mf + ((size_t)(I + 1) * kLook + k) * kTile;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) mnext[k][kk] = __ldg(M + (16 * q + kk) * kTB + i);
          }
        }
      }
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < kLook; ++k) {
        if (k + 1 <= I) {
          const double* yv = ys[(I - k - 1) % kLook] + 16 * q;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) p = fma(mreg[k][kk], yv[kk], p);
        }
      }
      red[q][i] = p;
      __syncthreads();
      if (tid < kTB) {
        wait_flag(cflag + I, epoch, status);
        const double c = __ldcg(cbuf + (size_t)I * kTB + tid);
        const double v = c - ((red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]));
        y[(size_t)I * kTB + tid] = v;
        ys[I % kLook][tid] = v;
        __threadfence();
      }
      __syncthreads();
      if (tid == 0) st_release64(prog, base + I + 1);
#pragma unroll
      for (int k = 0; k < kLook; ++k)
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) mreg[k][kk] = mnext[k][kk];
    }
    return;
  }

  // ---------------- workers ----------------
  const int W = gridDim.x - 1, w = blockIdx.x - 1;
  unsigned long long seen = 0;
  for (int I = w; I < nb; I += W) {
    const double* D = dinv + (size_t)I * kTile;
    for (int e = tid; e < kTile; e += kThreads) sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
    const int jmax = I - kLook;  // panel tiles J < jmax; the chain does the rest
    const double* row = tiles + tile_off(I, 0);
    double a[16], an[16];
    double acc = 0.0;
    if (jmax > 0) {
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = __ldg(row + (16 * q + k) * kTB + i);
    }
    for (int J = 0; J < jmax; ++J) {
      if (J + 1 < jmax) {
        const double* nt = row + (size_t)(J + 1) * kTile;
#pragma unroll
        for (int k = 0; k < 16; ++k) an[k] = __ldg(nt + (16 * q + k) * kTB + i);
      }
      if (seen < base + J + 1) seen = wait_progress(prog, base + J + 1, status);
      const double* yJ = y + (size_t)J * kTB + 16 * q;
#pragma unroll
      for (int k = 0; k < 16; ++k) acc = fma(a[k], __ldcg(yJ + k), acc);
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = an[k];
    }
    red[q][i] = acc;
    __syncthreads();
    if (tid < kTB)
      rr[tid] = __ldcg(y + (size_t)I * kTB + tid) -
                ((red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]));
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s = fma(sD[(16 * q + k) * kPad + i], rr[16 * q + k], s);
    red[q][i] = s;
    __syncthreads();
    if (tid < kTB) {
      cbuf[(size_t)I * kTB + tid] = (red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release32(cflag + I, epoch);
  }
}

// ---------------------------------------------------------------------------
// transposed sweep: y <- L^{-T} y
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    trsv_bwd_kernel(const double* __restrict__ tiles, const double* __restrict__ dinv,
                    const double* __restrict__ mb, double* y, double* cbuf, unsigned* cflag,
                    unsigned long long* prog, unsigned epoch, int nb, int* status) {
  __shared__ double sD[kTB * kPad];
  __shared__ double sR[2 * kTB];
  __shared__ double sP[4][kTB];
  __shared__ double rr[kTB];
  __shared__ double xs[kLook][kTB];
  const int tid = threadIdx.x;
  const unsigned long long base = (unsigned long long)epoch << 32;

  if (blockIdx.x == 0) {
    // ---------------- chain CTA ----------------
    const int i = tid & 63, q = tid >> 6;
    double mreg[kLook][16], mnext[kLook][16];
    for (int I = nb - 1; I >= 0; --I) {
      if (I - 1 >= 0) {
#pragma unroll
        for (int k = 0; k < kLook; ++k) {
          if (I - 1 + k + 1 < nb) {
            const double* M = mb + ((size_t)(I - 1) * kLook + k) * kTile;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) mnext[k][kk] = __ldg(M + (16 * q + kk) * kTB + i);
          }
        }
      }
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < kLook; ++k) {
        if (I + k + 1 < nb) {
          const double* xv = xs[(I + k + 1) % kLook] + 16 * q;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) p = fma(mreg[k][kk], xv[kk], p);
        }
      }
      sP[q][i] = p;
      __syncthreads();
      if (tid < kTB) {
        wait_flag(cflag + nb + I, epoch, status);
        const double c = __ldcg(cbuf + (size_t)I * kTB + tid);
        const double v = c - ((sP[0][tid] + sP[1][tid]) + (sP[2][tid] + sP[3][tid]));
        y[(size_t)I * kTB + tid] = v;
        xs[I % kLook][tid] = v;
        __threadfence();
      }
      __syncthreads();
      if (tid == 0) st_release64(prog, base + (unsigned long long)(nb - I));
#pragma unroll
      for (int k = 0; k < kLook; ++k)
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) mreg[k][kk] = mnext[k][kk];
    }
    return;
  }

  // ---------------- workers ----------------
  // thread (j = tid & 63, q = tid >> 6) reads row j of tile L_JI, columns
  // [16q, 16q+16), keeping 16 partial sums of (L_JI^T x_J)
  const int j = tid & 63, q = tid >> 6;
  const int W = gridDim.x - 1, w = blockIdx.x - 1;
  unsigned long long seen = 0;
  for (int I = nb - 1 - w; I >= 0; I -= W) {
    const double* D = dinv + (size_t)I * kTile;
    for (int e = tid; e < kTile; e += kThreads) sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    const int jmin = I + kLook;  // panel tiles J > jmin; the chain does the rest
    double a[16], an[16];
    if (nb - 1 > jmin) {
      const double* t = tiles + tile_off(nb - 1, I);
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = __ldg(t + (16 * q + k) * kTB + j);
    }
    for (int J = nb - 1; J > jmin; --J) {
      if (J - 1 > jmin) {
        const double* t = tiles + tile_off(J - 1, I);
#pragma unroll
        for (int k = 0; k < 16; ++k) an[k] = __ldg(t + (16 * q + k) * kTB + j);
      }
      const unsigned long long need = base + (unsigned long long)(nb - J);
      if (seen < need) seen = wait_progress(prog, need, status);
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
      cbuf[(size_t)I * kTB + tid] = (sP[0][tid] + sP[1][tid]) + (sP[2][tid] + sP[3][tid]);
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) st_release32(cflag + nb + I, epoch);
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
  double* dst = tiles + (size_t)blockIdx.x * kTile;
  for (int e = threadIdx.x; e < kTile; e += blockDim.x) {
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
  double* dst = tiles + (size_t)blockIdx.x * kTile;
  for (int e = threadIdx.x; e < kTile; e += blockDim.x) {
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
  for (int e = c; e < kTile; e += kTB) sL[(e >> 6) * kPad + (e & 63)] = T[e];
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
  double* D = dinv + (size_t)I * kTile;
  for (int e = c; e < kTile; e += kTB) D[e] = sX[(e >> 6) * kPad + (e & 63)];
}

// chain tiles: blockIdx = (I, k-1, dir)
//   dir 0: mf[I][k-1] = Dinv_II L_{I,I-k}          C[i][j] = sum_l D[i][l] L[l][j]
//   dir 1: mb[I][k-1] = Dinv_II^T L_{I+k,I}^T      C[i][j] = sum_l D[l][i] L[j][l]
__global__ void __launch_bounds__(256) chain_tiles_kernel(const double* __restrict__ tiles,
                                                          const double* __restrict__ dinv,
                                                          double* __restrict__ mf,
                                                          double* __restrict__ mb, int nb) {
  extern __shared__ double ct_smem[];
  double* sA = ct_smem;               // Dinv_II, sA[col * kPad + row]
  double* sB = ct_smem + kTB * kPad;  // panel tile, same layout
  const int I = blockIdx.x, k = blockIdx.y + 1, dir = blockIdx.z;
  double* C = (dir == 0 ? mf : mb) + ((size_t)I * kLook + k - 1) * kTile;
  const int tid = threadIdx.x, i = tid & 63, q = tid >> 6;
  const int J = dir == 0 ? I - k : I + k;
  if (J < 0 || J >= nb) {
    for (int e = tid; e < kTile; e += blockDim.x) C[e] = 0.0;
    return;
  }
  const double* A = dinv + (size_t)I * kTile;
  const double* B = dir == 0 ? tiles + tile_off(I, J) : tiles + tile_off(J, I);
  for (int e = tid; e < kTile; e += blockDim.x) {
    sA[(e >> 6) * kPad + (e & 63)] = A[e];
    sB[(e >> 6) * kPad + (e & 63)] = B[e];
  }
  __syncthreads();
  for (int jj = 16 * q; jj < 16 * q + 16; ++jj) {
    double s = 0.0;
    if (dir == 0) {
      for (int l = 0; l < kTB; ++l) s = fma(sA[l * kPad + i], sB[jj * kPad + l], s);
    } else {
      for (int l = 0; l < kTB; ++l) s = fma(sA[i * kPad + l], sB[l * kPad + jj], s);
    }
    C[(size_t)jj * kTB + i] = s;
  }
}

int g_coop_grid = -1;

}  // namespace

cudaError_t trsv_alloc(TriFactor& t, int n) {
  trsv_free(t);
  t.n = n;
  t.nb = (n + kTB - 1) / kTB;
  const size_t ntiles = (size_t)t.nb * (t.nb + 1) / 2;
  const size_t chain = (size_t)t.nb * kLook * kTile;
  t.bytes = (ntiles + t.nb + 2 * chain / kTile) * kTile * sizeof(double);
  cudaError_t e;
  if ((e = cudaMalloc(&t.tiles, ntiles * kTile * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.dinv, (size_t)t.nb * kTile * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.mf, chain * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.mb, chain * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.cbuf, (size_t)t.nb * kTB * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.cflag, 2 * (size_t)t.nb * sizeof(unsigned))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.prog, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.status, sizeof(int))) != cudaSuccess) return e;
  cudaMemset(t.cflag, 0, 2 * (size_t)t.nb * sizeof(unsigned));
  cudaMemset(t.prog, 0, 2 * sizeof(unsigned long long));
  cudaMemset(t.status, 0, sizeof(int));
  t.epoch = 0;
  return cudaSuccess;
}

void trsv_free(TriFactor& t) {
  cudaFree(t.tiles);
  cudaFree(t.dinv);
  cudaFree(t.mf);
  cudaFree(t.mb);
  cudaFree(t.cbuf);
  cudaFree(t.cflag);
  cudaFree(t.prog);
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

cudaError_t trsv_prepare(TriFactor& t, cudaStream_t st) {
  const int smem = 2 * kTB * kPad * (int)sizeof(double);
  cudaFuncSetAttribute(invert_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(chain_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  invert_diag_kernel<<<t.nb, kTB, smem, st>>>(t.tiles, t.dinv, t.status);
  chain_tiles_kernel<<<dim3(t.nb, kLook, 2), 256, smem, st>>>(t.tiles, t.dinv, t.mf, t.mb, t.nb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int h = 0;
  e = cudaMemcpyAsync(&h, t.status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  if (h) {
    cudaMemset(t.status, 0, sizeof(int));
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

cudaError_t trsv_solve(TriFactor& t, double* y, cudaStream_t st) {
  if (g_coop_grid < 0) {
    int dev = 0, sms = 0, per = 0, per2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, trsv_fwd_kernel, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, trsv_bwd_kernel, kThreads, 0);
    g_coop_grid = sms * (per < per2 ? per : per2);
    if (g_coop_grid < 2) g_coop_grid = 2;
  }
  // one chain CTA + up to one worker per block row
  const int grid = t.nb + 1 < g_coop_grid ? t.nb + 1 : g_coop_grid;
  ++t.epoch;
  unsigned long long* prog_f = t.prog;
  unsigned long long* prog_b = t.prog + 1;
  void* args_f[] = {(void*)&t.tiles, (void*)&t.dinv, (void*)&t.mf, (void*)&y, (void*)&t.cbuf,
                    (void*)&t.cflag, (void*)&prog_f, (void*)&t.epoch, (void*)&t.nb, (void*)&t.status};
  cudaError_t e =
      cudaLaunchCooperativeKernel((const void*)trsv_fwd_kernel, grid, kThreads, args_f, 0, st);
  if (e != cudaSuccess) return e;
  void* args_b[] = {(void*)&t.tiles, (void*)&t.dinv, (void*)&t.mb, (void*)&y, (void*)&t.cbuf,
                    (void*)&t.cflag, (void*)&prog_b, (void*)&t.epoch, (void*)&t.nb, (void*)&t.status};
  return cudaLaunchCooperativeKernel((const void*)trsv_bwd_kernel, grid, kThreads, args_b, 0, st);
}

}  // namespace ltb
