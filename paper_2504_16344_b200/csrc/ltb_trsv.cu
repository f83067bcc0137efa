// ltb_trsv.cu -- blocked triangular solves for K^{-1} = L^{-T} L^{-1}
// (bayes_engine.cpp:236-240) on sm_100a.
//
// Single-RHS TRSV is a GEMV over the packed factor (HBM bound, ~0.25
// flop/byte) plus a sequential dependency chain over the nb = n/64 diagonal
// blocks.  Design (one cooperative persistent launch for BOTH sweeps):
//
//   * CTA 0 is the CHAIN CTA, CTAs 1..G-1 are WORKERS;
//   * worker rows (round robin) stream their panel tiles as soon as the
//     needed solution blocks exist, but stop kLook tiles short of the
//     diagonal and hand the chain c_I = L_II^{-1} (b_I - sum_{J<I-kLook}
//     L_IJ y_J);
//   * the chain finishes y_I = c_I - sum_{k=1..kLook} M_{I,k} y_{I-k} with the
//     precomputed M_{I,k} = L_II^{-1} L_{I,I-k} (prefetched into registers a
//     step ahead) and the last kLook blocks of y kept in shared memory, so
//     the critical path per 64-block is one 64 x (64 kLook) GEMV plus one
//     L2 round trip;
//   * no flags: every hand-off buffer (c_I, y, x) is pre-filled with a NaN
//     sentinel (all ones, never produced by arithmetic, which yields the
//     canonical NaN) and consumers poll the VALUES themselves with
//     gpu-scope relaxed loads -- one L2 round trip per hand-off instead of
//     flag + data;
//   * the transposed sweep is the mirror image (rows descending, panel tiles
//     down the block column, M'_{I,k} = L_II^{-T} L_{I+k,I}^T) and follows in
//     the same launch: a worker moves on to its transposed rows as soon as its
//     forward rows are done.
#include <math.h>

#include "ltb_common.cuh"
#include "ltb_gen.cuh"
#include "ltb_trsv.h"

namespace ltb {

namespace {

constexpr int kQ = 8;                // column groups per 64-row tile
constexpr int kThreads = 64 * kQ;   // 512: thread (row, group)
constexpr int kCPT = kTB / kQ;      // 8 tile columns per thread
constexpr int kPad = 65;                               // padded smem tile stride
constexpr int kTile = kTB * kTB;
constexpr unsigned long long kSentinel = ~0ull;        // all-ones NaN
constexpr unsigned long long kSpinNs = 4000000000ull;  // 4 s dependency-wait timeout

LTB_DEV unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
LTB_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Poll a hand-off value until it is no longer the sentinel.  On timeout (or
// once any CTA timed out) set *status and return 0.0 so the kernel runs to
// completion and the host reports the error instead of the GPU hanging.
LTB_DEV double poll_value(const double* p, int* status) {
  unsigned long long v = ld_relaxed_u64(p);
  if (v != kSentinel) return __longlong_as_double((long long)v);
  const unsigned long long t0 = globaltimer();
  while (true) {
    __nanosleep(20);
    v = ld_relaxed_u64(p);
    if (v != kSentinel) return __longlong_as_double((long long)v);
    if (*(volatile int*)status) return 0.0;
    if (globaltimer() - t0 > kSpinNs) {
      atomicExch(status, 1);
      return 0.0;
    }
  }
}

LTB_DEV size_t tile_off(int I, int J) { return ((size_t)I * (I + 1) / 2 + J) * kTile; }

struct SweepArgs {
  const double* tiles;
  const double* dinv;
  const double* mf;
  const double* mb;
  const double* b;  // right-hand side (padded)
  double* yf;       // forward result   (sentinel on entry)
  double* xb;       // transposed result (sentinel on entry) = the solution
  double* cf;       // forward worker hand-offs  (sentinel on entry)
  double* cb;       // transposed worker hand-offs (sentinel on entry)
  int nb;
  int* status;
  unsigned long long* trace;  // optional: per-step timestamps (ltb_trsv_trace)
};

// fixed-order sum of the kQ column-group partials of row r
LTB_DEV double red_sum(const double (&red)[kQ][kTB], int r) {
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < kQ; ++g) s += red[g][r];
  return s;
}

struct ChainSmem {
  double ring[kLook][kTB];
  double red[kQ][kTB];
};

struct WorkerSmem {
  double sD[kTB * kPad];
  double red[kQ][kTB];
  double rr[kTB];
  double sR[2 * kTB];
};

// The chain tiles of step I are loaded into registers one step ahead.  The
// two register sets alternate (manual 2x unroll) so a prefetch is first
// consumed one full step after it was issued -- its HBM latency overlaps
// the poll of the previous step instead of stalling a register copy.
LTB_DEV void load_chain_tiles(const double* mtiles, int step, int nvalid, double (&m)[kLook][kCPT]) {
  const int i = threadIdx.x & 63, q = threadIdx.x >> 6;
#pragma unroll
  for (int k = 0; k < kLook; ++k) {
    if (k < nvalid) {
      const double* M = mtiles + ((size_t)step * kLook + k) * kTile;
#pragma unroll
      for (int kk = 0; kk < kCPT; ++kk) m[k][kk] = __ldg(M + (kCPT * q + kk) * kTB + i);
    }
  }
}

// one chain step: out_I = c_I - sum_{k < nvalid} M_{I,k} ring[slot_k]
template <bool kForward>
LTB_DEV void chain_step(const SweepArgs& a, ChainSmem& sm, int I, int nvalid,
                        const double (&m)[kLook][kCPT], unsigned long long cur,
                        unsigned long long& nxt) {
  const int tid = threadIdx.x, i = tid & 63, q = tid >> 6;
  const double* cbuf = kForward ? a.cf : a.cb;
  // speculative prefetch of the next step's hand-off (workers usually run
  // ahead); a sentinel just means "poll it then"
  const int In = kForward ? I + 1 : I - 1;
  if (tid < kTB && In >= 0 && In < a.nb) nxt = ld_relaxed_u64(cbuf + (size_t)In * kTB + tid);
  double p = 0.0;
#pragma unroll
  for (int k = 0; k < kLook; ++k) {
    if (k < nvalid) {
      const int src = kForward ? I - k - 1 : I + k + 1;
      const double* v = sm.ring[src % kLook] + kCPT * q;
#pragma unroll
      for (int kk = 0; kk < kCPT; ++kk) p = fma(m[k][kk], v[kk], p);
    }
  }
  sm.red[q][i] = p;
  __syncthreads();
  if (tid < kTB) {
    const double c = cur != kSentinel ? __longlong_as_double((long long)cur)
                                      : poll_value(cbuf + (size_t)I * kTB + tid, a.status);
    const double v = c - (red_sum(sm.red, tid));
    (kForward ? a.yf : a.xb)[(size_t)I * kTB + tid] = v;
    sm.ring[I % kLook][tid] = v;
  }
  __syncthreads();
  if (a.trace && threadIdx.x == 0) a.trace[(kForward ? 0 : a.nb) + I] = globaltimer();
}

// ---------------- chain, forward: y_I = c_I - sum_k M_{I,k} y_{I-k} ----------
LTB_DEV void chain_forward(const SweepArgs& a, ChainSmem& sm) {
  double mA[kLook][kCPT], mB[kLook][kCPT];
  unsigned long long cA = kSentinel, cB = kSentinel;
  auto nvalid = [&](int I) { return I < kLook ? I : kLook; };
  for (int I = 0; I < a.nb; I += 2) {
    if (I + 1 < a.nb) load_chain_tiles(a.mf, I + 1, nvalid(I + 1), mB);
    chain_step<true>(a, sm, I, nvalid(I), mA, cA, cB);
    if (I + 1 < a.nb) {
      if (I + 2 < a.nb) load_chain_tiles(a.mf, I + 2, nvalid(I + 2), mA);
      chain_step<true>(a, sm, I + 1, nvalid(I + 1), mB, cB, cA);
    }
  }
}

// ---------------- chain, transposed: x_I = c_I - sum_k M'_{I,k} x_{I+k} ------
LTB_DEV void chain_transposed(const SweepArgs& a, ChainSmem& sm) {
  double mA[kLook][kCPT], mB[kLook][kCPT];
  const int nb = a.nb;
  auto nvalid = [&](int I) { return nb - 1 - I < kLook ? nb - 1 - I : kLook; };
  unsigned long long cA = kSentinel, cB = kSentinel;
  for (int I = nb - 1; I >= 0; I -= 2) {
    if (I - 1 >= 0) load_chain_tiles(a.mb, I - 1, nvalid(I - 1), mB);
    chain_step<false>(a, sm, I, nvalid(I), mA, cA, cB);
    if (I - 1 >= 0) {
      if (I - 2 >= 0) load_chain_tiles(a.mb, I - 2, nvalid(I - 2), mA);
      chain_step<false>(a, sm, I - 1, nvalid(I - 1), mB, cB, cA);
    }
  }
}

// ---------------- workers: TMA tile ring ------------------------------------
// Panel tiles stream through a kRing-deep ring of 32 KB shared-memory stages
// filled by 1-D bulk async copies (one elected thread, one mbarrier per
// stage), so a worker keeps ~96 KB of the factor in flight without holding
// it in registers.  A running tile counter carries the stage / phase across
// rows and sweeps.
constexpr int kRing = 4;

struct TileRing {
  double* stage;  // kRing * kTile doubles (dynamic shared memory)
  uint64_t* full; // kRing mbarriers
  unsigned next;  // tiles consumed so far by this CTA
};

LTB_DEV void ring_issue(TileRing& r, unsigned g, const double* src, uint64_t policy) {
  const int s = g % kRing;
  mbar_arrive_expect_tx(r.full + s, kTile * sizeof(double));
  bulk_g2s(r.stage + (size_t)s * kTile, src, kTile * sizeof(double), r.full + s, policy);
}

// forward row I: thread (i = tid & 63, q = tid >> 6) owns row i, columns
// [8q, 8q+8) of each tile L_IJ, J < I - kLook (contiguous in memory)
LTB_DEV void worker_forward_row(const SweepArgs& a, WorkerSmem& sm, TileRing& ring, int I,
                                uint64_t policy) {
  const int tid = threadIdx.x, i = tid & 63, q = tid >> 6;
  const int jmax = I - kLook;  // panel tiles J < jmax; the chain does the rest
  const double* row = a.tiles + tile_off(I, 0);
  const unsigned g0 = ring.next;
  if (tid == 0)
    for (int J = 0; J < jmax && J < kRing; ++J) ring_issue(ring, g0 + J, row + (size_t)J * kTile, policy);
  const double* D = a.dinv + (size_t)I * kTile;
  for (int e = tid; e < kTile; e += kThreads) sm.sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
  double acc = 0.0;
  unsigned long long yraw[kCPT];
  if (jmax > 0) {
#pragma unroll
    for (int k = 0; k < kCPT; ++k) yraw[k] = ld_relaxed_u64(a.yf + kCPT * q + k);
  }
  for (int J = 0; J < jmax; ++J) {
    // resolve this tile's solution block (prefetched one tile ago)
    double yv[kCPT];
#pragma unroll
    for (int k = 0; k < kCPT; ++k)
      yv[k] = yraw[k] != kSentinel ? __longlong_as_double((long long)yraw[k])
                                   : poll_value(a.yf + (size_t)J * kTB + kCPT * q + k, a.status);
    if (J + 1 < jmax) {
#pragma unroll
      for (int k = 0; k < kCPT; ++k) yraw[k] = ld_relaxed_u64(a.yf + (size_t)(J + 1) * kTB + kCPT * q + k);
    }
    const unsigned g = g0 + J;
    mbar_wait(ring.full + g % kRing, (g / kRing) & 1);
    const double* T = ring.stage + (size_t)(g % kRing) * kTile;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) acc = fma(T[(kCPT * q + k) * kTB + i], yv[k], acc);
    __syncthreads();  // stage consumed
    if (tid == 0 && J + kRing < jmax) ring_issue(ring, g + kRing, row + (size_t)(J + kRing) * kTile, policy);
  }
  ring.next = g0 + (jmax > 0 ? jmax : 0);
  sm.red[q][i] = acc;
  __syncthreads();
  if (tid < kTB)
    sm.rr[tid] = __ldg(a.b + (size_t)I * kTB + tid) -
                 (red_sum(sm.red, tid));
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kCPT; ++k) s = fma(sm.sD[(kCPT * q + k) * kPad + i], sm.rr[kCPT * q + k], s);
  sm.red[q][i] = s;
  __syncthreads();
  if (tid < kTB)
    a.cf[(size_t)I * kTB + tid] = red_sum(sm.red, tid);
  __syncthreads();
  if (a.trace && tid == 0) a.trace[2 * a.nb + I] = globaltimer();
}

// transposed row I: thread (j = tid & 63, q = tid >> 6) reads row j of tile
// L_JI (J descending, J > I + kLook), columns [8q, 8q+8), keeping 8
// partial sums of (L_JI^T x_J)
LTB_DEV void worker_transposed_row(const SweepArgs& a, WorkerSmem& sm, TileRing& ring, int I,
                                   uint64_t policy) {
  const int tid = threadIdx.x, j = tid & 63, q = tid >> 6;
  const int nb = a.nb;
  const int jmin = I + kLook;  // panel tiles J > jmin; the chain does the rest
  const int ntile = nb - 1 - jmin > 0 ? nb - 1 - jmin : 0;
  const unsigned g0 = ring.next;
  if (tid == 0)
    for (int t = 0; t < ntile && t < kRing; ++t) ring_issue(ring, g0 + t, a.tiles + tile_off(nb - 1 - t, I), policy);
  const double* D = a.dinv + (size_t)I * kTile;
  for (int e = tid; e < kTile; e += kThreads) sm.sD[(e >> 6) * kPad + (e & 63)] = __ldg(D + e);
  double acc[kCPT];
#pragma unroll
  for (int k = 0; k < kCPT; ++k) acc[k] = 0.0;
  unsigned long long xraw = ntile > 0 ? ld_relaxed_u64(a.xb + (size_t)(nb - 1) * kTB + j) : 0ull;
  for (int t = 0; t < ntile; ++t) {
    const int J = nb - 1 - t;
    const double xj = xraw != kSentinel ? __longlong_as_double((long long)xraw)
                                        : poll_value(a.xb + (size_t)J * kTB + j, a.status);
    if (t + 1 < ntile) xraw = ld_relaxed_u64(a.xb + (size_t)(J - 1) * kTB + j);
    const unsigned g = g0 + t;
    mbar_wait(ring.full + g % kRing, (g / kRing) & 1);
    const double* T = ring.stage + (size_t)(g % kRing) * kTile;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) acc[k] = fma(T[(kCPT * q + k) * kTB + j], xj, acc[k]);
    __syncthreads();  // stage consumed
    if (tid == 0 && t + kRing < ntile) ring_issue(ring, g + kRing, a.tiles + tile_off(J - kRing, I), policy);
  }
  ring.next = g0 + ntile;
  // reduce over j: 32-lane shuffle tree per partial, then the two warps of
  // each column quarter meet in shared memory
#pragma unroll
  for (int k = 0; k < kCPT; ++k) {
    double v = acc[k];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    acc[k] = v;
  }
  if ((j & 31) == 0) {
#pragma unroll
    for (int k = 0; k < kCPT; ++k) sm.sR[(j >> 5) * kTB + kCPT * q + k] = acc[k];
  }
  __syncthreads();
  // y_I is the forward result: final (polled, the forward chain wrote it)
  if (tid < kTB)
    sm.rr[tid] = poll_value(a.yf + (size_t)I * kTB + tid, a.status) - (sm.sR[tid] + sm.sR[kTB + tid]);
  __syncthreads();
  {
    const int ii = tid & 63, part = tid >> 6;
    double s = 0.0;
    // (Dinv^T)[ii][jj] = Dinv[jj][ii] = sD[ii * kPad + jj]
#pragma unroll
    for (int k = 0; k < kCPT; ++k) s = fma(sm.sD[ii * kPad + kCPT * part + k], sm.rr[kCPT * part + k], s);
    sm.red[part][ii] = s;
  }
  __syncthreads();
  if (tid < kTB)
    a.cb[(size_t)I * kTB + tid] = red_sum(sm.red, tid);
  __syncthreads();
  if (a.trace && tid == 0) a.trace[3 * a.nb + I] = globaltimer();
}

__global__ void __launch_bounds__(kThreads, 1) trsv_kernel(const SweepArgs a) {
  __shared__ union {
    ChainSmem chain;
    WorkerSmem worker;
  } sm;
  extern __shared__ __align__(128) unsigned char ring_smem[];
  if (a.trace && threadIdx.x == 0 && blockIdx.x == 0) a.trace[4 * a.nb] = globaltimer();
  if (blockIdx.x == 0) {
    chain_forward(a, sm.chain);
    chain_transposed(a, sm.chain);
    return;
  }
  TileRing ring;
  ring.stage = reinterpret_cast<double*>(ring_smem);
  ring.full = reinterpret_cast<uint64_t*>(ring_smem + (size_t)kRing * kTile * sizeof(double));
  ring.next = 0;
  uint64_t policy = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(ring.full + s, 1);
    fence_mbar_init();
    policy = policy_evict_first();
  }
  __syncthreads();
  const int W = gridDim.x - 1, w = blockIdx.x - 1;
  for (int I = w; I < a.nb; I += W) worker_forward_row(a, sm.worker, ring, I, policy);
  for (int I = a.nb - 1 - w; I >= 0; I -= W) worker_transposed_row(a, sm.worker, ring, I, policy);
}

constexpr size_t kRingSmem = (size_t)kRing * kTile * sizeof(double) + kRing * sizeof(uint64_t);

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
  const size_t vec = (size_t)t.nb * kTB;
  t.bytes = (ntiles + t.nb + 2 * chain / kTile) * kTile * sizeof(double) + 5 * vec * sizeof(double);
  cudaError_t e;
  if ((e = cudaMalloc(&t.tiles, ntiles * kTile * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.dinv, (size_t)t.nb * kTile * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.mf, chain * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.mb, chain * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.work, 4 * vec * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.status, sizeof(int))) != cudaSuccess) return e;
  cudaMemset(t.status, 0, sizeof(int));
  return cudaSuccess;
}

void trsv_free(TriFactor& t) {
  cudaFree(t.tiles);
  cudaFree(t.dinv);
  cudaFree(t.mf);
  cudaFree(t.mb);
  cudaFree(t.work);
  cudaFree(t.status);
  cudaFree(t.trace);
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

double* trsv_result(TriFactor& t) { return t.work + (size_t)t.nb * kTB; }

cudaError_t trsv_solve(TriFactor& t, const double* b, cudaStream_t st) {
  if (g_coop_grid < 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, trsv_kernel, kThreads, kRingSmem);
    g_coop_grid = sms * per;
    if (g_coop_grid < 2) g_coop_grid = 2;
  }
  // one chain CTA + up to one worker per block row
  const int grid = t.nb + 1 < g_coop_grid ? t.nb + 1 : g_coop_grid;
  const size_t vec = (size_t)t.nb * kTB;
  // hand-off buffers [yf | xb | cf | cb] <- sentinel (all-ones bytes)
  cudaError_t e = cudaMemsetAsync(t.work, 0xFF, 4 * vec * sizeof(double), st);
  if (e != cudaSuccess) return e;
  SweepArgs a;
  a.tiles = t.tiles;
  a.dinv = t.dinv;
  a.mf = t.mf;
  a.mb = t.mb;
  a.b = b;
  a.yf = t.work;
  a.xb = t.work + vec;
  a.cf = t.work + 2 * vec;
  a.cb = t.work + 3 * vec;
  a.nb = t.nb;
  a.status = t.status;
  a.trace = t.trace;
  void* args[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((const void*)trsv_kernel, grid, kThreads, args, kRingSmem, st);
}

}  // namespace ltb
