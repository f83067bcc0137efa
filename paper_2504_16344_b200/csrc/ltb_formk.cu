// ltb_formk.cu -- form_K and the tile Cholesky on FP64 tensor cores (DMMA,
// mma.sync m16n8k4 f64 -> SASS DMMA.8x8x4 on sm_100a).  See ltb_formk.h for
// the algebra.  Packed tile layout as in ltb_trsv.h (P = 1): block row I
// starts at tile I (I+1) / 2, tile (I, J) is column-major 64x64.
#include <math.h>

#include <algorithm>
#include <vector>

#include "ltb_common.cuh"
#include "ltb_formk.h"

namespace ltb {

namespace {

constexpr int kT = kTB;          // 64
constexpr int kTile = kT * kT;   // 4096 doubles
int g_last_launches = 0;

__host__ __device__ inline size_t tile_at(int I, int J) { return ((size_t)I * (I + 1) / 2 + J) * kTile; }

// lower-triangular pair (i >= j) of linear index b
LTB_DEV void tri_pair(long long b, int* i, int* j) {
  long long r = (long long)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= b) ++r;
  while (r * (r + 1) / 2 > b) --r;
  *i = (int)r;
  *j = (int)(b - r * (r + 1) / 2);
}

// D += A B for one m16n8k4 FP64 tile.  Fragments (g = lane / 4, q = lane % 4):
// a0 = A[g][q], a1 = A[g+8][q], b0 = B[q][g];
// d = {D[g][2q], D[g][2q+1], D[g+8][2q], D[g+8][2q+1]}
LTB_DEV void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

LTB_DEV void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
LTB_DEV void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
LTB_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LTB_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// (1) lag Gram A = F_lag G_lag^T, lower 128x128 CTA tiles, into the packed
// tiles.  Operand row i = (r, a) = divmod(i, nt) reads f[(r nm + x) nt + a]:
// for a fixed x a run of rows is contiguous, so a stage (kBK values of x,
// 128 rows) is kBK contiguous 1 KB runs.  Shared stages are k-major
// [x][row] with a row stride of 132 doubles (== 4 mod 16: the DMMA fragment
// loads of a half-warp hit 32 distinct banks).
// ---------------------------------------------------------------------------
constexpr int kBM = 128;
constexpr int kBK = 32;
constexpr int kStages = 3;
constexpr int kSS = kBM + 4;
constexpr int kGemmThreads = 256;
constexpr size_t kStageDoubles = (size_t)2 * kBK * kSS;
constexpr size_t kGemmSmem = kStages * kStageDoubles * sizeof(double);

template <bool kPair>
LTB_DEV void gram_load_stage(double* sA, double* sB, const double* f, const double* g,
                             const double* pa, const double* pb, int x0, int nm, int nt) {
  const int tid = threadIdx.x;
  if (kPair) {
    // thread: row pair m = 2 (tid & 63), x rows kr + 4 q
    const int m = 2 * (tid & 63), kr = tid >> 6;
#pragma unroll
    for (int q = 0; q < kBK / 4; ++q) {
      const int k = kr + 4 * q, x = x0 + k;
      const bool okx = x < nm;
      cp_async16(sA + k * kSS + m, (pa && okx) ? pa + (size_t)x * nt : f, (pa && okx) ? 16 : 0);
      cp_async16(sB + k * kSS + m, (pb && okx) ? pb + (size_t)x * nt : g, (pb && okx) ? 16 : 0);
    }
  } else {
    // thread: row m = tid & 127, x rows kr + 2 q
    const int m = tid & 127, kr = tid >> 7;
#pragma unroll
    for (int q = 0; q < kBK / 2; ++q) {
      const int k = kr + 2 * q, x = x0 + k;
      const bool okx = x < nm;
      cp_async8(sA + k * kSS + m, (pa && okx) ? pa + (size_t)x * nt : f, (pa && okx) ? 8 : 0);
      cp_async8(sB + k * kSS + m, (pb && okx) ? pb + (size_t)x * nt : g, (pb && okx) ? 8 : 0);
    }
  }
}

// Output of a lag Gram: the packed lower 64x64 tiles of K (dense == 0), or
// a dense column-major block (dense == 1, rows x cols, leading dim ld).
// dense == 2: the packed lower tiles of ONE rank of a row-cyclic factor
// (block row I on rank I mod P, ltb_trsv.h); CTA row tile bi then covers this
// rank's local block rows 2 bi and 2 bi + 1 (global I = rank + P (2 bi + h)),
// and cum[bi] counts the column tiles of the row tiles before bi.
struct GramOut {
  int dense;
  double* p;
  size_t ld;
  int rows, cols;  // dense extent
  int nb;          // packed: 64-blocks
  int tiles_j;     // dense: 128-wide column tiles
  int P, rank;     // dense == 2
  const long long* cum;
  int npairs;
};

// tile offset of local block row li on rank r of P (ltb_trsv.cu row_off)
__host__ __device__ inline size_t drow_off(long long li, int r, int P) {
  return (size_t)(li * (r + 1) + (long long)P * li * (li - 1) / 2);
}

// global row of row m of CTA row tile bi
LTB_DEV int grow(const GramOut& o, int bi, int m) {
  if (o.dense != 2) return bi * kBM + m;
  return (o.rank + o.P * (2 * bi + (m >> 6))) * kT + (m & 63);
}

LTB_DEV double* out_elem(const GramOut& o, int i, int j) {
  if (o.dense == 2) {
    const int I = i >> 6, J = j >> 6;
    if (I >= o.nb || J > I || I % o.P != o.rank) return nullptr;
    return o.p + (drow_off(I / o.P, o.rank, o.P) + J) * kTile + (size_t)(j & 63) * kT + (i & 63);
  }
  if (o.dense) return (i < o.rows && j < o.cols) ? o.p + (size_t)j * o.ld + i : nullptr;
  const int I = i >> 6, J = j >> 6;
  return (I < o.nb && J <= I) ? o.p + tile_at(I, J) + (size_t)(j & 63) * kT + (i & 63) : nullptr;
}

LTB_DEV void gram_tile(const GramOut& o, long long t, int* bi, int* bj) {
  if (o.dense == 2) {
    int lo = 0, hi = o.npairs - 1;  // largest bi with cum[bi] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (o.cum[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    *bi = lo;
    *bj = (int)(t - o.cum[lo]);
  } else if (o.dense) {
    *bi = (int)(t / o.tiles_j);
    *bj = (int)(t % o.tiles_j);
  } else {
    tri_pair(t, bi, bj);
  }
}

// A[i][j] = sum_x a_row(i)[x] b_row(j)[x] for 128x128 CTA tiles, operand row
// i = (r, lag) of a [rows][nm][nt] kernel.  split == 1: CTA b computes tile
// tile0 + b over all of N_m and writes it out.  split > 1 (the last, partial
// wave): CTA b computes k-slice b % split of tile tile0 + b / split into
// `partial` ([tile][slice][128 x 128]); reduce_partials_kernel sums the
// slices in order (deterministic) and writes them out.
template <bool kPair>
__global__ void __launch_bounds__(kGemmThreads, 1)
    lag_gram_kernel(const double* __restrict__ f, const double* __restrict__ g, int nm, int nt,
                    int na, int nbr, const GramOut o, long long tile0, int split,
                    double* __restrict__ partial) {
  extern __shared__ __align__(16) double gsm[];
  const long long tile = tile0 + blockIdx.x / split;
  const int slice = blockIdx.x % split;
  int bi, bj;
  gram_tile(o, tile, &bi, &bj);
  const int j0 = bj * kBM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile 64 (rows) x 32 (cols)

  // this thread's operand row base pointers (nullptr = padding row)
  const double* rowA;
  const double* rowB;
  {
    const int m = kPair ? 2 * (tid & 63) : (tid & 127);
    const int ia = grow(o, bi, m), ib = j0 + m;
    rowA = ia < na ? f + (size_t)(ia / nt) * nm * nt + ia % nt : nullptr;
    rowB = ib < nbr ? g + (size_t)(ib / nt) * nm * nt + ib % nt : nullptr;
  }

  double acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  const int nk_all = (nm + kBK - 1) / kBK;
  const int kb = (int)((long long)slice * nk_all / split);
  const int nk = (int)((long long)(slice + 1) * nk_all / split) - kb;  // this CTA's k-chunks
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) {
      double* st = gsm + s * kStageDoubles;
      gram_load_stage<kPair>(st, st + kBK * kSS, f, g, rowA, rowB, (kb + s) * kBK, nm, nt);
    }
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();
    {
      const int nx = kt + kStages - 1;
      if (nx < nk) {
        double* st = gsm + (nx % kStages) * kStageDoubles;
        gram_load_stage<kPair>(st, st + kBK * kSS, f, g, rowA, rowB, (kb + nx) * kBK, nm, nt);
      }
      cp_commit();
    }
    const double* sA = gsm + (kt % kStages) * kStageDoubles;
    const double* sB = sA + kBK * kSS;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const int kr = (kk * 4 + tq) * kSS;
      double a[4][2], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        a[mt][0] = sA[kr + wm * 64 + mt * 16 + gq];
        a[mt][1] = sA[kr + wm * 64 + mt * 16 + gq + 8];
      }
#pragma unroll
      for (int nt8 = 0; nt8 < 4; ++nt8) b[nt8] = sB[kr + wn * 32 + nt8 * 8 + gq];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt8 = 0; nt8 < 4; ++nt8) dmma(acc[mt][nt8], a[mt][0], a[mt][1], b[nt8]);
    }
  }
  cp_wait<0>();

  if (split > 1) {
    // partial 128x128 block, row-major [m][n]
    double* P = partial + ((size_t)(blockIdx.x / split) * split + slice) * kBM * kBM;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt8 = 0; nt8 < 4; ++nt8)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = wm * 64 + mt * 16 + gq + 8 * h, c = wn * 32 + nt8 * 8 + 2 * tq;
          *reinterpret_cast<double2*>(P + (size_t)m * kBM + c) =
              make_double2(acc[mt][nt8][2 * h], acc[mt][nt8][2 * h + 1]);
        }
    return;
  }
  // epilogue: packed tiles (skip J > I and I >= nb) or the dense block
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 4; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int i = grow(o, bi, wm * 64 + mt * 16 + gq + 8 * h);
          const int j = j0 + wn * 32 + nt8 * 8 + 2 * tq + c;
          double* dst = out_elem(o, i, j);
          if (dst) *dst = acc[mt][nt8][2 * h + c];
        }
}

// sum the k-slices of the split tiles in slice order, write like the
// data-parallel epilogue
__global__ void reduce_partials_kernel(const double* __restrict__ partial, long long tile0, int split,
                                       const GramOut o) {
  const long long t = blockIdx.y;
  int bi, bj;
  gram_tile(o, tile0 + t, &bi, &bj);
  const double* P = partial + (size_t)t * split * kBM * kBM;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kBM * kBM; e += gridDim.x * blockDim.x) {
    const int m = e / kBM, c = e % kBM;
    double v = 0.0;
    for (int s = 0; s < split; ++s) v += P[(size_t)s * kBM * kBM + e];
    double* dst = out_elem(o, grow(o, bi, m), bj * kBM + c);
    if (dst) *dst = v;
  }
}

// ---------------------------------------------------------------------------
// (2) the diagonal recurrence C(t, j) = A(t, j) + C(t-1, j-1) inside each
// (r, s) block of N_t x N_t (packed K: r >= s and only the lower diagonals of
// r == s, plus sigma2 on the diagonal; dense: every block, every diagonal).
// One thread per diagonal; consecutive threads take consecutive diagonal
// starts (coalesced on the left-edge diagonals).  Loads of a diagonal are
// batched 8 at a time so the walk is not latency-serial.
// ---------------------------------------------------------------------------
__global__ void diag_prefix_kernel(const GramOut o, int nda, int ndb, int nt, double sigma2) {
  const long long per = 2ll * nt - 1;
  const long long pairs = o.dense ? (long long)nda * ndb : (long long)nda * (nda + 1) / 2;
  const long long total = pairs * per;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const long long p = id / per;
    const int d = (int)(id - p * per);
    int r, s;
    if (o.dense) {
      r = (int)(p / ndb);
      s = (int)(p % ndb);
    } else {
      tri_pair(p, &r, &s);
    }
    int t0, j0;
    if (d < nt) {
      t0 = d;
      j0 = 0;
    } else {
      if (!o.dense && r == s) continue;  // strict upper of a diagonal block: not stored
      t0 = 0;
      j0 = d - nt + 1;
    }
    const bool diag = !o.dense && r == s && t0 == 0;
    const int len = nt - max(t0, j0);
    const int ib = r * nt + t0, jb = s * nt + j0;
    double run = 0.0;
    for (int k0 = 0; k0 < len; k0 += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (k0 + q < len) v[q] = *out_elem(o, ib + k0 + q, jb + k0 + q);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (k0 + q < len) {
          run += v[q];
          *out_elem(o, ib + k0 + q, jb + k0 + q) = diag ? run + sigma2 : run;
        }
    }
  }
}

LTB_DEV double* elem(double* tiles, int i, int j) {
  return tiles + tile_at(i >> 6, j >> 6) + (size_t)(j & 63) * kT + (i & 63);
}

// identity on the padding diagonal (rows / columns >= n of the last block)
__global__ void pad_identity_kernel(double* tiles, int n, int nb) {
  const int i = n + threadIdx.x;
  if (i < nb * kT) *elem(tiles, i, i) = 1.0;
}

// ---------------------------------------------------------------------------
// (3) tile Cholesky.  Panel step k: one CTA per panel tile row holds
// X = [A_kk; A_ik] (128 rows x 64, column-major in shared memory, column
// stride 132 == 4 mod 16) and factors it blocked by 16 columns: for column
// block b,
//   (1) warp 0 factors the 16 x 16 diagonal block in registers (lane l owns
//       row 16 b + l; column broadcasts by shuffle, no CTA barrier),
//   (2) the rows below it (in A_kk and A_ik) solve against it, one thread
//       per row (forward substitution, the diagonal block read as shared
//       broadcasts),
//   (3) the trailing columns are updated with DMMA (m16n8k4, k = 16).
// 3 barriers per column block instead of one per column.  CTA 0 writes L_kk
// (strict upper zeroed), every CTA its panel tile L_ik = A_ik L_kk^{-T}.
// ---------------------------------------------------------------------------
constexpr int kPanelRows = 2 * kT;
constexpr int kPanelThreads = 256;
constexpr int kXS = kPanelRows + 4;  // 132
constexpr int kPB = 16;              // column block
constexpr size_t kPanelSmem = (size_t)kT * kXS * sizeof(double) + kT * sizeof(double);
#ifdef LTB_PANEL_STAMPS  // tools/probes/panel_probe.cu only
__device__ long long g_pstamp[32];
#define PSTAMP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_pstamp[i] = clock64()
#else
#define PSTAMP(i)
#endif

// one CTA: diagonal block from diag_in (rows 0-63), panel tile `panel`
// (rows 64-127, nullptr = none); L_kk to diag_out (nullptr = not this CTA),
// L_ik back into `panel` and, if given, a copy into panel_copy
LTB_DEV void chol_panel_cta(const double* diag_in, double* diag_out, double* panel, double* panel_copy, int k,
                            bool report, int* status) {
  extern __shared__ __align__(16) double psm[];
  double* X = psm;              // X[c * kXS + r]
  double* rinv = psm + kT * kXS;  // 1 / L_cc
  __shared__ int bad_any;
  __shared__ double cbuf[2 * kPB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad_any = 0;
  PSTAMP(0);
  {
    // thread: rows r, r + 1 (r = 2 (tid & 63)) of columns tid / 64 + 4 q; all
    // 16 loads in flight before the shared stores
    const int r = 2 * (tid & 63), c0 = tid >> 6;
    const double* src = r < kT ? diag_in + r : (panel ? panel + r - kT : nullptr);
    double2 v[kT / 4];
#pragma unroll
    for (int q = 0; q < kT / 4; ++q)
      v[q] = src ? *reinterpret_cast<const double2*>(src + (c0 + 4 * q) * kT) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < kT / 4; ++q) *reinterpret_cast<double2*>(X + (c0 + 4 * q) * kXS + r) = v[q];
  }
  __syncthreads();
  PSTAMP(1);
#pragma unroll 1
  for (int cb = 0; cb < kT; cb += kPB) {
    // (1) the diagonal block, rows / columns cb .. cb + 15: unscaled
    // elimination a_rj -= a_rc (a_jc / a_cc) (the column's shuffles do not
    // wait for this step's reciprocal), then L_rc = a_rc / sqrt(a_cc)
    if (warp == 0) {
      const int l = lane & 15, r = cb + l;
      double d[kPB];
#pragma unroll
      for (int j = 0; j < kPB; ++j) d[j] = X[(cb + j) * kXS + r];
      bool bad = false;
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        // column c (a_jc, unscaled) through a per-step shared slot: one
        // store per lane, then broadcast loads (fewer instructions on the
        // dependent chain than 16 double shuffles)
        double* cs = cbuf + (c & 1) * kPB;
        cs[l] = d[c];
        __syncwarp();
        double col[kPB];
#pragma unroll
        for (int j = 0; j < kPB; ++j)
          if (j >= c) col[j] = cs[j];
        double piv = col[c];
        if (!(piv > 0.0) || !isfinite(piv)) {
          bad = true;
          piv = 1.0;
        }
        const double f = l > c ? d[c] * (1.0 / piv) : 0.0;
#pragma unroll
        for (int j = 1; j < kPB; ++j)
          if (j > c && l >= j) d[j] = fma(-f, col[j], d[j]);
      }
      // pivots: lane l's a_ll; rs_c = 1 / sqrt(a_cc) to every lane
      double dl = 1.0;
#pragma unroll
      for (int j = 0; j < kPB; ++j)
        if (j == l) dl = d[j];
      if (!(dl > 0.0) || !isfinite(dl)) dl = 1.0;
      const double sq = sqrt(dl), rs = 1.0 / sq;
      if (lane < kPB) {
#pragma unroll
        for (int j = 0; j < kPB; ++j) {
          const double rsj = __shfl_sync(0x0000ffffu, rs, j);
          if (j < l) X[(cb + j) * kXS + r] = d[j] * rsj;
        }
        X[(cb + l) * kXS + r] = sq;
        rinv[r] = rs;
      }
      if (bad && lane == 0) bad_any = 1;
    }
    __syncthreads();
    PSTAMP(2 + 3 * (cb / kPB));
    // (2) rows below the diagonal block: x D^T = a
    const int r0 = cb + kPB;
    if (tid < kPanelRows - r0) {
      const int r = r0 + tid;
      double x[kPB];
#pragma unroll
      for (int j = 0; j < kPB; ++j) x[j] = X[(cb + j) * kXS + r];
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        x[c] *= rinv[cb + c];
#pragma unroll
        for (int j = 1; j < kPB; ++j)
          if (j > c) x[j] = fma(-x[c], X[(cb + c) * kXS + cb + j], x[j]);
      }
#pragma unroll
      for (int j = 0; j < kPB; ++j) X[(cb + j) * kXS + r] = x[j];
    }
    __syncthreads();
    PSTAMP(3 + 3 * (cb / kPB));
    if (r0 >= kT) break;
    // (3) X(r, j) -= sum_l X(r, cb + l) X(j, cb + l), r >= r0, r0 <= j < 64:
    // 16 x 8 DMMA tiles, rows in groups of 16 from r0, columns in 8s from r0
    {
      const int gq = lane >> 2, tq = lane & 3;
      const int nR = (kPanelRows - r0) / 16, nC = (kT - r0) / 8;
      for (int t = warp; t < nR * nC; t += kPanelThreads / 32) {
        const int rt = r0 + 16 * (t / nC), ct = r0 + 8 * (t % nC);
        if (rt + 15 < ct) continue;  // strictly upper part of the diagonal block
        double acc[4];
        acc[0] = X[(ct + 2 * tq) * kXS + rt + gq];
        acc[1] = X[(ct + 2 * tq + 1) * kXS + rt + gq];
        acc[2] = X[(ct + 2 * tq) * kXS + rt + gq + 8];
        acc[3] = X[(ct + 2 * tq + 1) * kXS + rt + gq + 8];
#pragma unroll
        for (int kk = 0; kk < kPB / 4; ++kk) {
          const double* col = X + (cb + 4 * kk + tq) * kXS;
          dmma(acc, -col[rt + gq], -col[rt + gq + 8], col[ct + gq]);
        }
        X[(ct + 2 * tq) * kXS + rt + gq] = acc[0];
        X[(ct + 2 * tq + 1) * kXS + rt + gq] = acc[1];
        X[(ct + 2 * tq) * kXS + rt + gq + 8] = acc[2];
        X[(ct + 2 * tq + 1) * kXS + rt + gq + 8] = acc[3];
      }
    }
    __syncthreads();
    PSTAMP(4 + 3 * (cb / kPB));
  }
  PSTAMP(14);
  if (bad_any && report && tid == 0) atomicCAS(status, 0, k + 1);
  for (int e = tid; e < kT * kPanelRows / 2; e += kPanelThreads) {
    const int c = e >> 6, r = 2 * (e & 63);
    double2 v = *reinterpret_cast<const double2*>(X + c * kXS + r);
    if (r < kT) {
      if (diag_out) {
        if (c > r) v.x = 0.0;
        if (c > r + 1) v.y = 0.0;
        *reinterpret_cast<double2*>(diag_out + c * kT + r) = v;
      }
    } else if (panel) {
      *reinterpret_cast<double2*>(panel + c * kT + r - kT) = v;
      if (panel_copy) *reinterpret_cast<double2*>(panel_copy + c * kT + r - kT) = v;
    }
  }
  PSTAMP(15);
}

__global__ void __launch_bounds__(kPanelThreads)
    chol_panel_kernel(double* __restrict__ tiles, int nb, int k, int* status) {
  const int ip = k + 1 + blockIdx.x;  // panel tile row (none when ip >= nb)
  double* dkk = tiles + tile_at(k, k);
  chol_panel_cta(dkk, blockIdx.x == 0 ? dkk : nullptr, ip < nb ? tiles + tile_at(ip, k) : nullptr, nullptr, k,
                 blockIdx.x == 0, status);
}

// ---------------------------------------------------------------------------
// (4) trailing update A_ij -= L_ik L_jk^T (+ L_i,k+1 L_j,k+1^T): one CTA per
// 64x64 tile, 8 warps (warp tile 32 x 16), accumulators seeded from A_ij
// and stored back.  Block columns are updated in pairs (K = 128), so a
// trailing tile is read and written once per two columns -- half the tile
// traffic per flop of a K = 64 update.  Operands stream through a ring of S
// cp.async stages of KS k columns (k-major = the column-major tile).
// ---------------------------------------------------------------------------
constexpr int kUS = kT + 4;  // 68 == 4 mod 16
constexpr int kUpdThreads = 256;

// A_ij -= sum_{c < kc} Li[c] Lj[c]^T for one tile, Li[c] / Lj[c] the operand
// tiles of block column c of the update (kc <= 2)
template <int KS, int S>
LTB_DEV void tile_update_ring(const double* const (&Li)[2], const double* const (&Lj)[2], int kc,
                              double* __restrict__ Aij) {
  extern __shared__ __align__(16) double usm[];
  constexpr int kStage = 2 * KS * kUS, kPer = kT / KS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  const int nch = kPer * kc;
  // chunk q (k columns [KS (q % kPer), +KS) of block column k + q / kPer)
  // into ring stage q % S by bulk copies (TMA, 1-D): lane c of warp 0 moves
  // one 512-byte tile column into its padded shared row (stride kUS keeps
  // the DMMA fragment loads conflict free); they complete on full[q % S]
  uint64_t* full = reinterpret_cast<uint64_t*>(usm + S * kStage);
  auto load = [&](int q) {
    if (q >= nch) return;
    const size_t off = (size_t)(q % kPer) * KS * kT;
    const double* a = (q >= kPer ? Li[1] : Li[0]) + off;  // (not indexed: would go to local memory)
    const double* bb = (q >= kPer ? Lj[1] : Lj[0]) + off;
    double* sa = usm + (q % S) * kStage;
    if (lane == 0) mbar_arrive_expect_tx(full + q % S, 2 * KS * kT * sizeof(double));
    __syncwarp();
    if (lane < 2 * KS) {
      const int c = lane % KS;
      // the stage was last read by generic loads: order them before the async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t pol;  // the L tiles are re-read by the whole block row / column: normal L2 priority
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      bulk_g2s(sa + (lane < KS ? 0 : KS * kUS) + c * kUS, (lane < KS ? a : bb) + (size_t)c * kT,
               kT * sizeof(double), full + q % S, pol);
    }
  };
  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(full + st, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < S - 1; ++q) load(q);
  }
  double acc[2][2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = wm * 32 + mt * 16 + gq + 8 * h, col = wn * 16 + nt8 * 8 + 2 * tq + c;
          acc[mt][nt8][2 * h + c] = Aij[col * kT + r];
        }
  for (int q = 0; q < nch; ++q) {
    __syncthreads();  // every thread is done with stage (q - 1) % S
    if (warp == 0) load(q + S - 1);
    mbar_wait(full + q % S, (q / S) & 1);
    const double* sA = usm + (q % S) * kStage;
    const double* sB = sA + KS * kUS;
#pragma unroll
    for (int kk = 0; kk < KS / 4; ++kk) {
      const int kr = (kk * 4 + tq) * kUS;
      double a[2][2], bf[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        a[mt][0] = -sA[kr + wm * 32 + mt * 16 + gq];
        a[mt][1] = -sA[kr + wm * 32 + mt * 16 + gq + 8];
      }
#pragma unroll
      for (int nt8 = 0; nt8 < 2; ++nt8) bf[nt8] = sB[kr + wn * 16 + nt8 * 8 + gq];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt8 = 0; nt8 < 2; ++nt8) dmma(acc[mt][nt8], a[mt][0], a[mt][1], bf[nt8]);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = wm * 32 + mt * 16 + gq + 8 * h, col = wn * 16 + nt8 * 8 + 2 * tq + c;
          Aij[col * kT + r] = acc[mt][nt8][2 * h + c];
        }
}

template <int KS, int S>
constexpr size_t upd_smem() { return (size_t)S * 2 * KS * kUS * sizeof(double) + S * sizeof(uint64_t); }

// 16-column k stages, double buffered: 35 KB of shared memory and 62
// registers -> 4 CTAs per SM (32-column stages / deeper rings measured
// slower: 3 CTAs per SM hide the tile loads and stores less well)
constexpr int kUpdKS = 16, kUpdStages = 2;
constexpr size_t kUpdSmem = upd_smem<kUpdKS, kUpdStages>();

// tiles: mode 0, the lower triangle from (base, base); mode 1, block columns
// base and base + 1 (i >= j); mode 2, block column base
__global__ void __launch_bounds__(kUpdThreads, 4)
    chol_update_kernel(double* __restrict__ tiles, int nb, int k, int kc, int base, int mode) {
  int i, j;
  const int b = (int)blockIdx.x, m0 = nb - base;
  if (mode == 0) {
    int li, lj;
    tri_pair(b, &li, &lj);
    i = base + li;
    j = base + lj;
  } else if (mode == 2 || b < m0) {
    i = base + b;
    j = base;
  } else {
    i = base + 1 + (b - m0);
    j = base + 1;
  }
  const double* const Li[2] = {tiles + tile_at(i, k), tiles + tile_at(i, k + kc - 1)};
  const double* const Lj[2] = {tiles + tile_at(j, k), tiles + tile_at(j, k + kc - 1)};
  tile_update_ring<kUpdKS, kUpdStages>(Li, Lj, kc, tiles + tile_at(i, j));
}

// packed lower tiles -> column-major lower triangle
__global__ void export_lower_kernel(const double* __restrict__ tiles, int n, double* __restrict__ out,
                                    size_t ld) {
  int I, J;
  tri_pair(blockIdx.x, &I, &J);
  const double* T = tiles + tile_at(I, J);
  for (int e = threadIdx.x; e < kTile; e += blockDim.x) {
    const int jj = e >> 6, ii = e & 63;
    const int i = I * kT + ii, j = J * kT + jj;
    if (i < n && j < n && i >= j) out[(size_t)j * ld + i] = T[e];
  }
}

// ---------------------------------------------------------------------------
// (5) multi-RHS block substitution (form_Q's K^{-1} R, bayes_engine.cpp:250-255)
// on the packed factor, 64 right-hand sides per CTA, DMMA for every product.
// Forward (kTrans = false), step I (-1 <= I <= nb-2), CTA (chunk, J = I+1+y):
//   R_J -= L_JI X_I                   (I >= 0)
//   J == I+1:  X_J = L_JJ^{-1} R_J    (into X; R_J is dead afterwards)
// Transposed, step I (nb >= I >= 1), CTA (chunk, J = I-1-y):
//   R_J -= L_IJ^T X_I                 (I < nb)
//   J == I-1:  X_J = L_JJ^{-T} R_J
// R, X column-major with ld = nb * 64 rows (padding rows zero).  8 warps, warp
// tile 32 rows x 16 columns; shared tiles with stride 68 (== 4 mod 16) read
// either way round conflict-free.
// ---------------------------------------------------------------------------
constexpr int kRC = 64;
constexpr int kTS = kT + 4;
constexpr size_t kTrsmSmem = (size_t)2 * kT * kTS * sizeof(double);

template <bool kTrans>
__global__ void __launch_bounds__(256)
    trsm_step_kernel(const double* __restrict__ tiles, const double* __restrict__ dinv, int nb, int I,
                     double* __restrict__ R, double* __restrict__ X, size_t ld) {
  extern __shared__ __align__(16) double tsm[];
  double* sA = tsm;             // [col][row] of a 64x64 tile
  double* sB = tsm + kT * kTS;  // [rhs][k]
  const int c0 = blockIdx.x * kRC;
  const int J = kTrans ? I - 1 - (int)blockIdx.y : I + 1 + (int)blockIdx.y;
  const bool upd = kTrans ? (I < nb) : (I >= 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  double* RJ = R + (size_t)c0 * ld + (size_t)J * kT;
  double acc[2][2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          acc[mt][nt8][2 * h + c] =
              RJ[(size_t)(wn * 16 + nt8 * 8 + 2 * tq + c) * ld + wm * 32 + mt * 16 + gq + 8 * h];
  auto tile_mma = [&](double (&d)[2][2][4], bool trans_a, double sign) {
#pragma unroll
    for (int kk = 0; kk < kT / 4; ++kk) {
      const int k = kk * 4 + tq;
      double a[2][2], b[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + mt * 16 + gq + 8 * h;
          a[mt][h] = sign * (trans_a ? sA[r * kTS + k] : sA[k * kTS + r]);
        }
#pragma unroll
      for (int nt8 = 0; nt8 < 2; ++nt8) b[nt8] = sB[(wn * 16 + nt8 * 8 + gq) * kTS + k];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt8 = 0; nt8 < 2; ++nt8) dmma(d[mt][nt8], a[mt][0], a[mt][1], b[nt8]);
    }
  };
  if (upd) {
    const double* T = tiles + (kTrans ? tile_at(I, J) : tile_at(J, I));
    const double* XI = X + (size_t)c0 * ld + (size_t)I * kT;
    for (int c = tid; c < kTile / 2; c += 256) {
      const int col = c >> 5, r2 = 2 * (c & 31);
      cp_async16(sA + col * kTS + r2, T + col * kT + r2, 16);
      cp_async16(sB + col * kTS + r2, XI + (size_t)col * ld + r2, 16);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    tile_mma(acc, kTrans, -1.0);
  }
  const bool last = J == (kTrans ? I - 1 : I + 1);
  if (!last) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            RJ[(size_t)(wn * 16 + nt8 * 8 + 2 * tq + c) * ld + wm * 32 + mt * 16 + gq + 8 * h] =
                acc[mt][nt8][2 * h + c];
    return;
  }
  // X_J = L_JJ^{-1} R_J (or L_JJ^{-T} R_J): R_J becomes the B operand
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          sB[(wn * 16 + nt8 * 8 + 2 * tq + c) * kTS + wm * 32 + mt * 16 + gq + 8 * h] = acc[mt][nt8][2 * h + c];
  const double* D = dinv + (size_t)J * kTile;
  for (int c = tid; c < kTile / 2; c += 256) {
    const int col = c >> 5, r2 = 2 * (c & 31);
    cp_async16(sA + col * kTS + r2, D + col * kT + r2, 16);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  double out[2][2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int e = 0; e < 4; ++e) out[mt][nt8][e] = 0.0;
  tile_mma(out, kTrans, 1.0);
  double* XJ = X + (size_t)c0 * ld + (size_t)J * kT;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt8 = 0; nt8 < 2; ++nt8)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          XJ[(size_t)(wn * 16 + nt8 * 8 + 2 * tq + c) * ld + wm * 32 + mt * 16 + gq + 8 * h] =
              out[mt][nt8][2 * h + c];
}

// out = 0.5 ((P - G) + (P - G)^T), m x m column-major (form_qoi_cov :271-274
// with P symmetrised first: identical in exact arithmetic)
__global__ void gpost_kernel(const double* __restrict__ P, const double* __restrict__ G, int m,
                             double* __restrict__ out, double* __restrict__ diag) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)m * m;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const double a = P[(size_t)j * m + i] - G[(size_t)j * m + i];
    const double b = P[(size_t)i * m + j] - G[(size_t)i * m + j];
    const double v = 0.5 * (a + b);
    out[e] = v;
    if (i == j) diag[i] = v;
  }
}

__global__ void symmetrize_kernel(double* __restrict__ A, int m) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)m * m;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    if (i > j) {
      const double v = 0.5 * (A[(size_t)j * m + i] + A[(size_t)i * m + j]);
      A[(size_t)j * m + i] = v;
      A[(size_t)i * m + j] = v;
    }
  }
}

// Q (m x n, ld m) = X^T, X column-major (n rows used, ld ldx)
__global__ void transpose_kernel(const double* __restrict__ X, size_t ldx, int n, int m,
                                 double* __restrict__ Q) {
  __shared__ double t[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;  // i: row of X (< n), j: column (< m)
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + threadIdx.x, j = j0 + r;
    t[r][threadIdx.x] = (i < n && j < m) ? X[(size_t)j * ldx + i] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + threadIdx.x, i = i0 + r;
    if (i < n && j < m) Q[(size_t)i * m + j] = t[threadIdx.x][r];
  }
}

}  // namespace

int formk_last_launches() { return g_last_launches; }

namespace {

// lag Gram of kernel rows (a: na rows, b: nbr rows, contraction N_m) into o,
// then the diagonal recurrence over (nda x ndb) blocks
cudaError_t lag_gram(const double* a, int na, const double* b, int nbr, int nm, int nt, const GramOut& o,
                     long long ctas, cudaStream_t st) {
  const bool pair = (nt % 2 == 0) && ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0);
  auto kern = pair ? lag_gram_kernel<true> : lag_gram_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
  if (e != cudaSuccess) return e;
  // one CTA per SM: full waves data-parallel; a short last wave (<= half the
  // SMs) is split along N_m instead so it does not cost a whole wave
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long rem = ctas % sms;
  int split = rem > 0 && rem <= sms / 2 && ctas > sms ? (int)std::min<long long>(sms / rem, (nm + kBK - 1) / kBK) : 1;
  if (split < 2) rem = 0;
  double* partial = nullptr;
  if (rem) {
    e = cudaMallocAsync(&partial, (size_t)rem * split * kBM * kBM * sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  if (ctas - rem > 0) {
    kern<<<(unsigned)(ctas - rem), kGemmThreads, kGemmSmem, st>>>(a, b, nm, nt, na, nbr, o, 0, 1, nullptr);
    ++g_last_launches;
  }
  if (rem) {
    kern<<<(unsigned)(rem * split), kGemmThreads, kGemmSmem, st>>>(a, b, nm, nt, na, nbr, o, ctas - rem, split,
                                                                    partial);
    reduce_partials_kernel<<<dim3(16, (unsigned)rem), 256, 0, st>>>(partial, ctas - rem, split, o);
    cudaFreeAsync(partial, st);
    g_last_launches += 2;
  }
  return cudaGetLastError();
}

cudaError_t diag_recurrence(const GramOut& o, int nda, int ndb, int nt, double sigma2, cudaStream_t st) {
  const long long pairs = o.dense ? (long long)nda * ndb : (long long)nda * (nda + 1) / 2;
  const long long diags = pairs * (2ll * nt - 1);
  const unsigned pblocks = (unsigned)std::max(1ll, std::min(148ll * 32, (diags + 255) / 256));
  diag_prefix_kernel<<<pblocks, 256, 0, st>>>(o, nda, ndb, nt, sigma2);
  ++g_last_launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t formk_device(TriFactor& t, const double* f, const double* g, int nd, int nm, int nt,
                         double sigma2, cudaStream_t st) {
  if (t.P != 1 || t.n != nd * nt || nm < 1) return cudaErrorInvalidValue;
  const int n = t.n, nb = t.nb;
  const long long nbm = (n + kBM - 1) / kBM;
  GramOut o{};
  o.dense = 0;
  o.p = t.tiles;
  o.nb = nb;
  g_last_launches = 0;
  cudaError_t e = lag_gram(f, n, g, n, nm, nt, o, nbm * (nbm + 1) / 2, st);
  if (e == cudaSuccess) e = diag_recurrence(o, nd, nd, nt, sigma2, st);
  if (e != cudaSuccess) return e;
  pad_identity_kernel<<<1, kT, 0, st>>>(t.tiles, n, nb);
  ++g_last_launches;
  return cudaGetLastError();
}

cudaError_t block_toeplitz_product(const double* a, int nda, const double* b, int ndb, int nm, int nt,
                                   double* out, size_t ld, cudaStream_t st) {
  GramOut o{};
  o.dense = 1;
  o.p = out;
  o.ld = ld;
  o.rows = nda * nt;
  o.cols = ndb * nt;
  o.tiles_j = (o.cols + kBM - 1) / kBM;
  const long long ctas = (long long)((o.rows + kBM - 1) / kBM) * o.tiles_j;
  g_last_launches = 0;
  cudaError_t e = lag_gram(a, o.rows, b, o.cols, nm, nt, o, ctas, st);
  if (e == cudaSuccess) e = diag_recurrence(o, nda, ndb, nt, 0.0, st);
  return e;
}

cudaError_t cholesky_packed(TriFactor& t, cudaStream_t st, int* bad_block) {
  if (t.P != 1) return cudaErrorInvalidValue;
  const int nb = t.nb;
  cudaError_t e = cudaFuncSetAttribute(chol_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kUpdSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(chol_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmem);
  if (e != cudaSuccess) return e;
  // Lookahead over two streams: the high-priority stream runs panel(k) and
  // the update of block column k+1 only (U1), so panel(k+1) can start while
  // the low-priority stream applies the rest of update k (U2) -- the
  // latency-bound panel hides under the DMMA / bandwidth-bound trailing
  // update.  U2(k) waits for panel(k); U1(k) waits for U2(k-1) (column k+1 is
  // in it).
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  cudaStream_t main_s = nullptr, side = nullptr;
  if ((e = cudaStreamCreateWithPriority(&main_s, cudaStreamNonBlocking, greatest)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, least)) != cudaSuccess) {
    cudaStreamDestroy(main_s);
    return e;
  }
  cudaEvent_t ev_panel = nullptr, ev_u2 = nullptr, ev_fork = nullptr, ev_join = nullptr;
  cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_u2, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
  cudaMemsetAsync(t.status, 0, sizeof(int), st);
  cudaEventRecord(ev_fork, st);
  cudaStreamWaitEvent(main_s, ev_fork, 0);
  cudaStreamWaitEvent(side, ev_fork, 0);
  int launches = 0;
  bool u2_pending = false;
  const auto panel = [&](int k) {
    chol_panel_kernel<<<std::max(1, nb - k - 1), kPanelThreads, kPanelSmem, main_s>>>(t.tiles, nb, k, t.status);
    ++launches;
  };
  // block columns in pairs (k, k + 1): panel k, column k + 1 -= L_k L_k+1,k^T,
  // panel k + 1, then the pair's K = 128 update of everything to the right
  for (int k = 0; k < nb; k += 2) {
    panel(k);
    if (k + 1 >= nb) break;
    chol_update_kernel<<<(unsigned)(nb - k - 1), kUpdThreads, kUpdSmem, main_s>>>(t.tiles, nb, k, 1, k + 1, 2);
    panel(k + 1);
    launches += 1;
    if (k + 2 >= nb) break;
    // U2(k): tiles (i, j), k + 4 <= j <= i
    const int m2 = nb - k - 4;
    if (m2 > 0) {
      cudaEventRecord(ev_panel, main_s);
      cudaStreamWaitEvent(side, ev_panel, 0);
      chol_update_kernel<<<(unsigned)((long long)m2 * (m2 + 1) / 2), kUpdThreads, kUpdSmem, side>>>(
          t.tiles, nb, k, 2, k + 4, 0);
      ++launches;
    }
    // U1(k): block columns k + 2, k + 3, after U2(k - 2) updated them
    if (u2_pending) cudaStreamWaitEvent(main_s, ev_u2, 0);
    const int m1 = nb - k - 2;
    chol_update_kernel<<<(unsigned)(m1 + std::max(0, m1 - 1)), kUpdThreads, kUpdSmem, main_s>>>(t.tiles, nb, k, 2,
                                                                                               k + 2, 1);
    ++launches;
    u2_pending = m2 > 0;
    if (u2_pending) cudaEventRecord(ev_u2, side);
  }
  cudaEventRecord(ev_join, side);
  cudaStreamWaitEvent(main_s, ev_join, 0);
  cudaEventRecord(ev_join, main_s);
  cudaStreamWaitEvent(st, ev_join, 0);
  g_last_launches = launches;
  e = cudaGetLastError();
  int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, t.status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamSynchronize(main_s);
  cudaStreamSynchronize(side);
  cudaStreamDestroy(main_s);
  cudaStreamDestroy(side);
  cudaEventDestroy(ev_panel);
  cudaEventDestroy(ev_u2);
  cudaEventDestroy(ev_fork);
  cudaEventDestroy(ev_join);
  if (e != cudaSuccess) return e;
  if (h) {
    cudaMemset(t.status, 0, sizeof(int));
    if (bad_block) *bad_block = h - 1;
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

cudaError_t export_lower(const TriFactor& t, double* out, size_t ld, cudaStream_t st) {
  const long long ntiles = (long long)t.nb * (t.nb + 1) / 2;
  export_lower_kernel<<<(unsigned)ntiles, 256, 0, st>>>(t.tiles, t.n, out, ld);
  return cudaGetLastError();
}

cudaError_t trsm_solve_k(const TriFactor& t, double* R, double* X, size_t ld, int nrhs_pad, double* YtY,
                         int m, cudaStream_t st) {
  if (t.P != 1 || nrhs_pad % kRC) return cudaErrorInvalidValue;
  const int nb = t.nb;
  cudaError_t e = cudaFuncSetAttribute(trsm_step_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kTrsmSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(trsm_step_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kTrsmSmem);
  if (e != cudaSuccess) return e;
  const unsigned chunks = (unsigned)(nrhs_pad / kRC);
  g_last_launches = 0;
  // forward: Y = L^{-1} R into X (R is scratch)
  for (int I = -1; I <= nb - 2; ++I) {
    trsm_step_kernel<false><<<dim3(chunks, (unsigned)(nb - 1 - I)), 256, kTrsmSmem, st>>>(t.tiles, t.dinv, nb, I,
                                                                                       R, X, ld);
    ++g_last_launches;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // R^T K^{-1} R = Y^T Y (m x m), before the transposed sweep consumes Y
  if (YtY) {
    const int keep = g_last_launches;
    e = block_toeplitz_product(X, m, X, m, (int)ld, 1, YtY, (size_t)m, st);
    g_last_launches += keep;
    if (e != cudaSuccess) return e;
  }
  // transposed: K^{-1} R = L^{-T} Y into R (Y is scratch)
  for (int I = nb; I >= 1; --I) {
    trsm_step_kernel<true><<<dim3(chunks, (unsigned)I), 256, kTrsmSmem, st>>>(t.tiles, t.dinv, nb, I, X, R, ld);
    ++g_last_launches;
  }
  return cudaGetLastError();
}

cudaError_t qoi_covariance(const double* P, const double* YtY, int m, double* gpost, double* diag,
                           cudaStream_t st) {
  const long long mm = (long long)m * m;
  const unsigned blocks = (unsigned)std::max(1ll, std::min(148ll * 8, (mm + 255) / 256));
  gpost_kernel<<<blocks, 256, 0, st>>>(P, YtY, m, gpost, diag);
  return cudaGetLastError();
}

cudaError_t symmetrize(double* A, int m, cudaStream_t st) {
  const long long mm = (long long)m * m;
  symmetrize_kernel<<<(unsigned)std::max(1ll, std::min(148ll * 8, (mm + 255) / 256)), 256, 0, st>>>(A, m);
  return cudaGetLastError();
}

cudaError_t transpose_to(const double* X, size_t ldx, int n, int m, double* Q, cudaStream_t st) {
  transpose_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32)), dim3(32, 8), 0, st>>>(X, ldx, n, m,
                                                                                                     Q);
  return cudaGetLastError();
}


// ===========================================================================
// Distributed offline phase 2 (one process per GPU, P ranks): form_K and the
// tile Cholesky straight into the row-cyclic layout the distributed K^{-1}
// reads (block row I on rank I mod P, ltb_trsv.h), NCCL for the exchanges.
//  * form_K: each rank computes the lag Gram for its own block rows (CTA row
//    tiles = pairs of its block rows, all columns of the lower triangle);
//    the diagonal recurrence K(t, j) = A(t, j) + K(t-1, j-1) then runs block
//    row by block row in order, the last row of block row I handed to the
//    owner of I + 1 (2 MB at n = 252,000, NCCL send / recv) as the carry;
//  * Cholesky, block column k: the owner broadcasts A_kk (32 KB); every rank
//    forms its panel tiles L_ik = A_ik L_kk^{-T} (the one-GPU panel CTA) and
//    all-gathers the column; every rank applies A_ij -= L_ik L_jk^T to its
//    own rows (the one-GPU DMMA tile update).
// Per-tile arithmetic is the one-GPU kernels', in the same order, so the
// distributed factor equals the one-GPU factor (up to the split-k tail of
// the lag Gram, which sums k-slices in order either way).
// ===========================================================================
namespace {

// recurrence over block row I with carry_in = row 64 I - 1 (columns
// 0 .. 64 I - 1) and carry_out = row 64 I + 63 (columns 0 .. 64 I + 63) of
// F G* (sigma2 is added to the stored diagonal only, as diag_prefix_kernel);
// thread per diagonal delta = i - j
__global__ void dist_recur_kernel(const GramOut o, int I, int n, int nt, double sigma2,
                                  const double* __restrict__ carry_in, double* __restrict__ carry_out) {
  const int r0 = I * kT, rend = min(r0 + kT, n);
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < r0 + kT; d += gridDim.x * blockDim.x) {
    int i = max(r0, d);
    if (i >= rend) continue;
    double prev = (i == r0 && i - d - 1 >= 0 && r0 > 0) ? carry_in[i - d - 1] : 0.0;
    for (; i < rend; i += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (i + q < rend) v[q] = *out_elem(o, i + q, i + q - d);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (i + q < rend) {
          const int ii = i + q, jj = ii - d;
          double x = v[q];
          if (ii % nt != 0 && jj % nt != 0) x += prev;  // the recurrence runs on F G* alone
          *out_elem(o, ii, jj) = d == 0 ? x + sigma2 : x;
          prev = x;
          if (ii == r0 + kT - 1 && carry_out) carry_out[jj] = x;
        }
    }
  }
}

// identity on the padding diagonal of the last block row (its owner)
__global__ void dist_pad_identity_kernel(double* tiles, int n, int nb, int r, int P) {
  const int i = n + threadIdx.x, I = nb - 1;
  if (i < nb * kT) tiles[(drow_off(I / P, r, P) + I) * kTile + (size_t)(i & 63) * kT + (i & 63)] = 1.0;
}

// first block row > k owned by rank q, and how many there are
__host__ __device__ inline int dist_first(int k, int q, int P) { return k + 1 + ((q - (k + 1)) % P + P) % P; }
__host__ __device__ inline int dist_count(int first, int nb, int P) { return first < nb ? (nb - 1 - first) / P + 1 : 0; }

__global__ void __launch_bounds__(kPanelThreads)
    dist_panel_kernel(double* __restrict__ tiles, int r, int P, int k, int nb, const double* __restrict__ akk,
                      int owner, double* __restrict__ sendbuf, int* status) {
  const int first = dist_first(k, r, P), cnt = dist_count(first, nb, P);
  const int b = blockIdx.x, i = first + P * b;
  double* dkk = owner && b == 0 ? tiles + (drow_off(k / P, r, P) + k) * kTile : nullptr;
  double* pt = b < cnt ? tiles + (drow_off(i / P, r, P) + k) * kTile : nullptr;
  chol_panel_cta(akk, dkk, pt, b < cnt ? sendbuf + (size_t)b * kTile : nullptr, k, owner && b == 0, status);
}

// Gathered block column c of the factor: rank q's rows > c at
// recv[q * cntmax + (j - dist_first(c, q, P)) / P]
struct DistCol {
  const double* recv;
  int cntmax;
};

LTB_DEV const double* dist_gathered(const DistCol& g, int c, int j, int P) {
  const int q = j % P;
  return g.recv + ((size_t)q * g.cntmax + (j - dist_first(c, q, P)) / P) * kTile;
}

// own rows i > kl (kl = k + kc - 1), tiles j in (kl, i]:
// A_ij -= sum_{c < kc} L_i,k+c L_j,k+c^T (column_only: just j = kl + 1, kc = 1)
__global__ void __launch_bounds__(kUpdThreads, 4)
    dist_update_kernel(double* __restrict__ tiles, int r, int P, int k, int kc, int nb, const DistCol g0,
                       const DistCol g1, int column_only) {
  const int kl = k + kc - 1;
  const int first = dist_first(kl, r, P), cnt = dist_count(first, nb, P);
  const long long b = blockIdx.x;
  int a, j;
  if (column_only) {
    a = (int)b;
    j = kl + 1;
  } else {
    int lo = 0, hi = cnt - 1;  // row a: tiles before it a (first - kl) + P a (a - 1) / 2
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if ((long long)mid * (first - kl) + (long long)P * mid * (mid - 1) / 2 <= b) lo = mid;
      else hi = mid - 1;
    }
    a = lo;
    j = kl + 1 + (int)(b - ((long long)a * (first - kl) + (long long)P * a * (a - 1) / 2));
  }
  const int i = first + P * a;
  const size_t row = drow_off(i / P, r, P);
  const double* const Li[2] = {tiles + (row + k) * kTile, tiles + (row + kl) * kTile};
  const double* const Lj[2] = {dist_gathered(g0, k, j, P), dist_gathered(kc == 2 ? g1 : g0, kl, j, P)};
  tile_update_ring<kUpdKS, kUpdStages>(Li, Lj, kc, tiles + (row + j) * kTile);
}

#define NCCL_TRY(expr)                                                            \
  do {                                                                            \
    ncclResult_t r_ = (expr);                                                     \
    if (r_ != ncclSuccess) {                                                      \
      if (err) *err = api->GetErrorString(r_);                                    \
      return cudaErrorUnknown;                                                    \
    }                                                                             \
  } while (0)

struct DevMem {
  void* p = nullptr;
  ~DevMem() { cudaFree(p); }
};

}  // namespace

cudaError_t formk_device_dist(TriFactor& t, const double* f, const double* g, int nd, int nm, int nt, double sigma2,
                              const Nccl* api, ncclComm_t comm, cudaStream_t st, const char** err) {
  const int n = t.n, nb = t.nb, P = t.P, r = t.rank;
  if (n != nd * nt || nm < 1 || (P > 1 && (!api || !comm))) return cudaErrorInvalidValue;
  const int nloc = r < nb ? (nb - 1 - r) / P + 1 : 0, npairs = (nloc + 1) / 2;
  g_last_launches = 0;
  GramOut o{};
  o.dense = 2;
  o.p = t.tiles;
  o.nb = nb;
  o.P = P;
  o.rank = r;
  o.npairs = npairs;
  std::vector<long long> cum(npairs + 1, 0);
  for (int bi = 0; bi < npairs; ++bi) {
    const int I1 = r + P * (2 * bi + 1), Imax = I1 < nb ? I1 : r + P * 2 * bi;
    cum[bi + 1] = cum[bi] + ((long long)kT * Imax + kT - 1) / kBM + 1;
  }
  DevMem dcum, cin, cout;
  cudaError_t e;
  if ((e = cudaMalloc(&dcum.p, sizeof(long long) * (npairs + 1))) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(dcum.p, cum.data(), sizeof(long long) * (npairs + 1), cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return e;
  o.cum = static_cast<const long long*>(dcum.p);
  if (npairs > 0 && (e = lag_gram(f, n, g, n, nm, nt, o, cum[npairs], st)) != cudaSuccess) return e;
  // the recurrence, block row by block row, carries handed to the next owner
  if ((e = cudaMalloc(&cin.p, sizeof(double) * (size_t)nb * kT)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&cout.p, sizeof(double) * (size_t)nb * kT)) != cudaSuccess) return e;
  double* ci = static_cast<double*>(cin.p);
  double* co = static_cast<double*>(cout.p);
  for (int li = 0; li < nloc; ++li) {
    const int I = r + P * li;
    if (I > 0 && P > 1) NCCL_TRY(api->Recv(ci, (size_t)kT * I, ncclDouble, (I - 1) % P, comm, st));
    const int diags = kT * I + kT;
    dist_recur_kernel<<<(unsigned)std::max(1, std::min(148 * 4, (diags + 255) / 256)), 256, 0, st>>>(
        o, I, n, nt, sigma2, ci, co);
    ++g_last_launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (I + 1 < nb) {
      if (P > 1) NCCL_TRY(api->Send(co, (size_t)kT * I + kT, ncclDouble, (I + 1) % P, comm, st));
      else std::swap(ci, co);
    }
  }
  if ((nb - 1) % P == r && nb * kT > n) {
    dist_pad_identity_kernel<<<1, kT, 0, st>>>(t.tiles, n, nb, r, P);
    ++g_last_launches;
  }
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the temporaries above are freed on return
  return e;
}

cudaError_t cholesky_dist(TriFactor& t, const Nccl* api, ncclComm_t comm, cudaStream_t st, int* bad_block,
                          const char** err) {
  const int nb = t.nb, P = t.P, r = t.rank;
  if (P > 1 && (!api || !comm)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dist_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kUpdSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dist_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmem);
  if (e != cudaSuccess) return e;
  const int cnt0 = (nb + P - 1) / P;  // bound on any rank's rows > k
  DevMem akk, sendb, recvb, stat;
  if ((e = cudaMalloc(&akk.p, sizeof(double) * kTile)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&sendb.p, sizeof(double) * kTile * (size_t)cnt0 * 2)) != cudaSuccess) return e;
  if (P > 1 && (e = cudaMalloc(&recvb.p, sizeof(double) * kTile * (size_t)cnt0 * P * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&stat.p, sizeof(int) * P)) != cudaSuccess) return e;
  double* a = static_cast<double*>(akk.p);
  cudaMemsetAsync(t.status, 0, sizeof(int), st);
  g_last_launches = 0;
  // block column c: owner broadcasts A_cc, every rank factors its panel tiles
  // (copies into send buffer c & 1), all-gather -> the gathered column
  const auto panel_step = [&](int c, DistCol* g) -> cudaError_t {
    const int owner = c % P;
    double* sb = static_cast<double*>(sendb.p) + (size_t)(c & 1) * cnt0 * kTile;
    double* rb = P > 1 ? static_cast<double*>(recvb.p) + (size_t)(c & 1) * cnt0 * P * kTile : sb;
    cudaError_t e2;
    if (r == owner &&
        (e2 = cudaMemcpyAsync(a, t.tiles + (drow_off(c / P, r, P) + c) * kTile, sizeof(double) * kTile,
                              cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      return e2;
    if (P > 1) NCCL_TRY(api->Broadcast(a, a, kTile, ncclDouble, owner, comm, st));
    const int cnt = dist_count(dist_first(c, r, P), nb, P);
    const int grid = cnt > 0 ? cnt : (r == owner ? 1 : 0);
    if (grid) {
      dist_panel_kernel<<<grid, kPanelThreads, kPanelSmem, st>>>(t.tiles, r, P, c, nb, a, r == owner, sb, t.status);
      ++g_last_launches;
    }
    int cntmax = 0;
    for (int q = 0; q < P; ++q) cntmax = std::max(cntmax, dist_count(dist_first(c, q, P), nb, P));
    if (P > 1 && c < nb - 1) NCCL_TRY(api->AllGather(sb, rb, (size_t)cntmax * kTile, ncclDouble, comm, st));
    g->recv = rb;
    g->cntmax = P > 1 ? cntmax : cnt0;
    return cudaGetLastError();
  };
  // block columns in pairs (as cholesky_packed): panel k, column k + 1 -= its
  // L_k part, panel k + 1, then the K = 128 update of the rest
  for (int k = 0; k < nb; k += 2) {
    DistCol g0{}, g1{};
    if ((e = panel_step(k, &g0)) != cudaSuccess) return e;
    if (k == nb - 1) break;
    const int cnt_c = dist_count(dist_first(k, r, P), nb, P);  // own rows >= k + 1
    if (cnt_c > 0) {
      dist_update_kernel<<<(unsigned)cnt_c, kUpdThreads, kUpdSmem, st>>>(t.tiles, r, P, k, 1, nb, g0, g0, 1);
      ++g_last_launches;
    }
    if ((e = panel_step(k + 1, &g1)) != cudaSuccess) return e;
    if (k + 1 == nb - 1) break;
    const int first = dist_first(k + 1, r, P), cnt = dist_count(first, nb, P);
    const long long tiles = (long long)cnt * (first - k - 1) + (long long)P * cnt * (cnt - 1) / 2;
    if (tiles > 0) {
      dist_update_kernel<<<(unsigned)tiles, kUpdThreads, kUpdSmem, st>>>(t.tiles, r, P, k, 2, nb, g0, g1, 0);
      ++g_last_launches;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // every rank learns of a failed pivot (only the owner's CTA reports it)
  int* sp = static_cast<int*>(stat.p);
  if (P > 1) NCCL_TRY(api->AllGather(t.status, sp, 1, ncclInt, comm, st));
  else if ((e = cudaMemcpyAsync(sp, t.status, sizeof(int), cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  std::vector<int> h(P, 0);
  if ((e = cudaMemcpyAsync(h.data(), sp, sizeof(int) * P, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  int bad = 0;
  for (int v : h) bad = (v && (!bad || v < bad)) ? v : bad;
  cudaMemsetAsync(t.status, 0, sizeof(int), st);
  if (bad) {
    if (bad_block) *bad_block = bad - 1;
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

#undef NCCL_TRY

}  // namespace ltb
