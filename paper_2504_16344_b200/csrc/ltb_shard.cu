// ltb_shard.cu -- one MatvecPlan sharded over several GPUs of one process
// (SURVEY 8(b) "ltb_plan_create_sharded(..., ndev, devs)", 8(e)).
//
// Column c of F-hat only meets x-hat_c (F m) or produces x-hat_c (F* d), so
// the plan is cut into contiguous column ranges, one ltb_plan per device
// (devices may repeat: two shards on one GPU exercise the same code path on a
// one-GPU box).  The exchange per matvec is small and fixed:
//   F m : every shard computes its partial d_k (N_d x N_t, 2 MB at Cascadia)
//         from its own slice of m; the home device (devs[0]) sums the
//         partials in shard order with one kernel that reads the other
//         devices' buffers straight through NVLink peer mappings
//         (deterministic; a staged peer copy where P2P is unavailable);
//   F* d: d goes to every shard (host pointers: one H2D per device; device
//         pointers: peer copies from the home device over NVLink), every
//         shard writes its own column range of m (host: pipelined D2H per
//         shard; device: peer copy into the home device's m).
// The streaming GEMVs (~20 ms per Cascadia shard) dwarf the 2-4 MB
// exchanges (~us over NVLink), so the shards run concurrently and the
// exchange is one small kernel, not a collective library call.
//
// Semantics follow ltb_apply: host pointers are synchronous (the reference's
// apply_raw); device pointers live on the home device and the call is
// asynchronous on the scratch's home stream (shard 0's stream).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ltb.h"

namespace ltb_internal {
ltb_status set_error(ltb_status st, const char* msg);
ltb_status apply_device(const ltb_plan* p, ltb_scratch* s, const double* in, double* out, bool adjoint);
ltb_status fm_from_host(const ltb_plan* p, ltb_scratch* s, const double* in_host, double* d_dev);
ltb_status fstar_to_host(const ltb_plan* p, ltb_scratch* s, const double* d_dev, double* m_host);
cudaStream_t scratch_stream(ltb_scratch* s);
double* scratch_stage_in(ltb_scratch* s, size_t n);
double* scratch_stage_out(ltb_scratch* s, size_t n);
void count_launches(uint64_t n);
}  // namespace ltb_internal

using namespace ltb_internal;

namespace {

constexpr int kMaxShards = 16;

ltb_status sfail(ltb_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return set_error(st, buf);
}

#define SH_CUDA(expr)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return sfail(LTB_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (d >= 0 && d != prev) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct PartPtrs {
  const double* p[kMaxShards];
};

// out[i] = (((d_0[i] + d_1[i]) + d_2[i]) + ...) -- shard order, so the sum is
// deterministic; d_k may live on another GPU (peer mapping over NVLink)
__global__ void sum_shards_kernel(PartPtrs parts, int n, long long len, double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    double s = __ldcv(parts.p[0] + i);
    for (int k = 1; k < n; ++k) s += __ldcv(parts.p[k] + i);
    out[i] = s;
  }
}

}  // namespace

struct ltb_splan {
  int rows = 0, cols = 0, nt = 0, tag = 0, n = 0;
  int dev[kMaxShards] = {};
  long long c0[kMaxShards + 1] = {};
  bool peer[kMaxShards] = {};  // shard k's memory is readable from the home device
  ltb_plan* sh[kMaxShards] = {};
};

struct ltb_sscratch {
  const ltb_splan* p = nullptr;
  ltb_scratch* s[kMaxShards] = {};
  double* part[kMaxShards] = {};   // partial d of shard k, on its device (rows * nt)
  double* din[kMaxShards] = {};    // d on shard k's device (rows * nt), k > 0
  double* staged = nullptr;        // home: peer copies of non-P2P partials
  double* dout = nullptr;          // home: reduced d (host-pointer path)
  cudaEvent_t ev[kMaxShards] = {};
  cudaEvent_t start = nullptr;
};

namespace {

ltb_status split(ltb_splan* p, int cols, int ndev, const int* devs) {
  if (ndev < 1 || ndev > kMaxShards || !devs) return sfail(LTB_INVALID, "sharded plan: 1 <= ndev <= %d", kMaxShards);
  if (cols < ndev) return sfail(LTB_DIMENSION, "sharded plan: %d columns over %d shards", cols, ndev);
  int count = 0;
  cudaGetDeviceCount(&count);
  p->n = ndev;
  const long long base = cols / ndev, extra = cols % ndev;
  for (int k = 0; k < ndev; ++k) {
    if (devs[k] < 0 || devs[k] >= count) return sfail(LTB_INVALID, "sharded plan: device %d of %d", devs[k], count);
    p->dev[k] = devs[k];
    p->c0[k + 1] = p->c0[k] + base + (k < extra ? 1 : 0);
  }
  // peer mappings from the home device (NVLink on a B200 box)
  p->peer[0] = true;
  for (int k = 1; k < ndev; ++k) {
    if (devs[k] == devs[0]) {
      p->peer[k] = true;
      continue;
    }
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, devs[0], devs[k]);
    if (ok) {
      DevGuard g(devs[0]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devs[k], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      ok = (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled);
    }
    p->peer[k] = ok != 0;
  }
  return LTB_OK;
}

void splan_free(ltb_splan* p) {
  if (!p) return;
  for (int k = 0; k < p->n; ++k)
    if (p->sh[k]) ltb_plan_destroy(p->sh[k]);
  delete p;
}

ltb_status check_pair(const ltb_splan* p, const ltb_sscratch* s) {
  if (!p || !s) return sfail(LTB_INVALID, "sharded apply: null plan or scratch");
  if (s->p != p) return sfail(LTB_INVALID, "sharded apply: scratch was created for another plan");
  return LTB_OK;
}

// home stream waits for everything queued so far on shard k's stream
ltb_status join(ltb_sscratch* s, int k, cudaStream_t home) {
  {
    DevGuard g(s->p->dev[k]);
    SH_CUDA(cudaEventRecord(s->ev[k], scratch_stream(s->s[k])));
  }
  DevGuard g(s->p->dev[0]);
  SH_CUDA(cudaStreamWaitEvent(home, s->ev[k], 0));
  return LTB_OK;
}

// shard k's stream waits for the work queued so far on the home stream
ltb_status fork(ltb_sscratch* s, int k, cudaStream_t home) {
  if (k == 0) return LTB_OK;
  SH_CUDA(cudaStreamWaitEvent(scratch_stream(s->s[k]), s->start, 0));
  return LTB_OK;
}

// sum the partials into `out` (home device) on the home stream
ltb_status reduce(const ltb_splan* p, ltb_sscratch* s, double* out) {
  const cudaStream_t home = scratch_stream(s->s[0]);
  const long long len = (long long)p->rows * p->nt;
  PartPtrs pp = {};
  for (int k = 0; k < p->n; ++k) {
    if (k > 0) {
      ltb_status st = join(s, k, home);
      if (st != LTB_OK) return st;
    }
    if (p->peer[k]) {
      pp.p[k] = s->part[k];
    } else {
      double* dst = s->staged + (size_t)k * len;
      SH_CUDA(cudaMemcpyPeerAsync(dst, p->dev[0], s->part[k], p->dev[k], sizeof(double) * len, home));
      pp.p[k] = dst;
    }
  }
  DevGuard g(p->dev[0]);
  const unsigned blocks = (unsigned)std::max(1ll, std::min(148ll * 4, (len + 255) / 256));
  sum_shards_kernel<<<blocks, 256, 0, home>>>(pp, p->n, len, out);
  SH_CUDA(cudaGetLastError());
  count_launches(1);
  return LTB_OK;
}

ltb_status sync_all(const ltb_splan* p, ltb_sscratch* s) {
  for (int k = 0; k < p->n; ++k) {
    DevGuard g(p->dev[k]);
    SH_CUDA(cudaStreamSynchronize(scratch_stream(s->s[k])));
  }
  return LTB_OK;
}

}  // namespace

extern "C" {

ltb_status ltb_plan_create_sharded(const double* kernel_rck, int rows, int cols, int nt, int tag, int ndev,
                                   const int* devs, const ltb_opts* opts, ltb_splan** out) {
  if (!out || !kernel_rck) return sfail(LTB_INVALID, "ltb_plan_create_sharded: null argument");
  *out = nullptr;
  if (rows < 1 || cols < 1 || nt < 1) return sfail(LTB_DIMENSION, "MatvecPlan: kernel dims must be >= 1");
  ltb_splan* p = new ltb_splan();
  p->rows = rows;
  p->cols = cols;
  p->nt = nt;
  p->tag = tag;
  ltb_status st = split(p, cols, ndev, devs);
  if (st != LTB_OK) {
    splan_free(p);
    return st;
  }
  // [rows][c0, c1)[nt] of the host kernel, one shard at a time
  std::vector<double> slab;
  for (int k = 0; k < p->n; ++k) {
    const long long c0 = p->c0[k], nc = p->c0[k + 1] - c0;
    slab.resize((size_t)rows * nc * nt);
    for (int r = 0; r < rows; ++r)
      std::copy(kernel_rck + ((size_t)r * cols + c0) * nt, kernel_rck + ((size_t)r * cols + c0 + nc) * nt,
                slab.begin() + (size_t)r * nc * nt);
    ltb_opts o = opts ? *opts : ltb_opts{-1, 0};
    o.device = p->dev[k];
    if ((st = ltb_plan_create(slab.data(), rows, (int)nc, nt, tag, LTB_PTR_HOST, &o, &p->sh[k])) != LTB_OK) {
      splan_free(p);
      return st;
    }
  }
  *out = p;
  return LTB_OK;
}

ltb_status ltb_plan_create_generated_sharded(int rows, int cols, int nt, int tag, uint64_t seed, uint64_t stream,
                                             int ndev, const int* devs, const ltb_opts* opts, ltb_splan** out) {
  if (!out) return sfail(LTB_INVALID, "ltb_plan_create_generated_sharded: null out");
  *out = nullptr;
  if (rows < 1 || cols < 1 || nt < 1) return sfail(LTB_DIMENSION, "MatvecPlan: kernel dims must be >= 1");
  ltb_splan* p = new ltb_splan();
  p->rows = rows;
  p->cols = cols;
  p->nt = nt;
  p->tag = tag;
  ltb_status st = split(p, cols, ndev, devs);
  if (st != LTB_OK) {
    splan_free(p);
    return st;
  }
  for (int k = 0; k < p->n; ++k) {
    ltb_opts o = opts ? *opts : ltb_opts{-1, 0};
    o.device = p->dev[k];
    st = ltb_plan_create_generated(rows, (int)(p->c0[k + 1] - p->c0[k]), nt, tag, seed, stream, cols, p->c0[k], &o,
                                   &p->sh[k]);
    if (st != LTB_OK) {
      splan_free(p);
      return st;
    }
  }
  *out = p;
  return LTB_OK;
}

ltb_status ltb_splan_destroy(ltb_splan* p) {
  splan_free(p);
  return LTB_OK;
}

ltb_status ltb_splan_dims(const ltb_splan* p, int* rows_out, int* n_cols, int* n_time, int* n_shards) {
  if (!p) return sfail(LTB_INVALID, "ltb_splan_dims: null plan");
  if (rows_out) *rows_out = p->rows;
  if (n_cols) *n_cols = p->cols;
  if (n_time) *n_time = p->nt;
  if (n_shards) *n_shards = p->n;
  return LTB_OK;
}

ltb_status ltb_splan_shard(const ltb_splan* p, int k, int* device, long long* c0, long long* c1, int* peer) {
  if (!p) return sfail(LTB_INVALID, "ltb_splan_shard: null plan");
  if (k < 0 || k >= p->n) return sfail(LTB_DIMENSION, "ltb_splan_shard: shard %d of %d", k, p->n);
  if (device) *device = p->dev[k];
  if (c0) *c0 = p->c0[k];
  if (c1) *c1 = p->c0[k + 1];
  if (peer) *peer = p->peer[k] ? 1 : 0;
  return LTB_OK;
}

ltb_status ltb_splan_kernel_hat_sqnorm(const ltb_splan* p, double* out) {
  if (!p || !out) return sfail(LTB_INVALID, "ltb_splan_kernel_hat_sqnorm: null argument");
  double sum = 0.0;
  for (int k = 0; k < p->n; ++k) {
    double v = 0.0;
    ltb_status st = ltb_kernel_hat_sqnorm(p->sh[k], &v);
    if (st != LTB_OK) return st;
    sum += v;
  }
  *out = sum;
  return LTB_OK;
}

ltb_status ltb_sscratch_destroy(ltb_sscratch* s) {
  if (!s) return LTB_OK;
  const ltb_splan* p = s->p;
  for (int k = 0; k < (p ? p->n : 0); ++k) {
    DevGuard g(p->dev[k]);
    if (s->s[k]) cudaStreamSynchronize(scratch_stream(s->s[k]));
    cudaFree(s->part[k]);
    cudaFree(s->din[k]);
    if (s->ev[k]) cudaEventDestroy(s->ev[k]);
    if (s->s[k]) ltb_scratch_destroy(s->s[k]);
  }
  if (p) {
    DevGuard g(p->dev[0]);
    cudaFree(s->staged);
    cudaFree(s->dout);
    if (s->start) cudaEventDestroy(s->start);
  }
  delete s;
  return LTB_OK;
}

ltb_status ltb_sscratch_create(const ltb_splan* p, void* home_stream, ltb_sscratch** out) {
  if (!p || !out) return sfail(LTB_INVALID, "ltb_sscratch_create: null argument");
  *out = nullptr;
  ltb_sscratch* s = new ltb_sscratch();
  s->p = p;
  const size_t len = (size_t)p->rows * p->nt;
  auto bail = [&](ltb_status st) {
    ltb_sscratch_destroy(s);
    return st;
  };
  for (int k = 0; k < p->n; ++k) {
    ltb_status st = ltb_scratch_create(p->sh[k], k == 0 ? home_stream : nullptr, &s->s[k]);
    if (st != LTB_OK) return bail(st);
    DevGuard g(p->dev[k]);
    if (cudaMalloc(&s->part[k], sizeof(double) * len) != cudaSuccess ||
        (k > 0 && cudaMalloc(&s->din[k], sizeof(double) * len) != cudaSuccess) ||
        cudaEventCreateWithFlags(&s->ev[k], cudaEventDisableTiming) != cudaSuccess)
      return bail(sfail(LTB_CUDA, "ltb_sscratch_create: %s", cudaGetErrorString(cudaGetLastError())));
  }
  DevGuard g(p->dev[0]);
  if (cudaMalloc(&s->dout, sizeof(double) * len) != cudaSuccess ||
      cudaMalloc(&s->staged, sizeof(double) * len * p->n) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->start, cudaEventDisableTiming) != cudaSuccess)
    return bail(sfail(LTB_CUDA, "ltb_sscratch_create: %s", cudaGetErrorString(cudaGetLastError())));
  *out = s;
  return LTB_OK;
}

void* ltb_sscratch_stream(ltb_sscratch* s) { return s && s->s[0] ? scratch_stream(s->s[0]) : nullptr; }

// d = F m (fft_matvec.cpp:139-179) over the shards
ltb_status ltb_apply_sharded(const ltb_splan* p, ltb_sscratch* s, const double* in, double* out, int ptr_kind) {
  ltb_status st = check_pair(p, s);
  if (st != LTB_OK) return st;
  if (!in || !out) return sfail(LTB_INVALID, "sharded apply: null input/output");
  const cudaStream_t home = scratch_stream(s->s[0]);
  const long long nt = p->nt;
  if (ptr_kind == LTB_PTR_HOST) {
    for (int k = 0; k < p->n; ++k) {  // every shard streams its own slice of m
      DevGuard g(p->dev[k]);
      if ((st = fm_from_host(p->sh[k], s->s[k], in + p->c0[k] * nt, s->part[k])) != LTB_OK) return st;
    }
    {
      DevGuard g(p->dev[0]);
      if ((st = reduce(p, s, s->dout)) != LTB_OK) return st;
      SH_CUDA(cudaMemcpyAsync(out, s->dout, sizeof(double) * p->rows * nt, cudaMemcpyDeviceToHost, home));
    }
    return sync_all(p, s);
  }
  if (ptr_kind != LTB_PTR_DEVICE) return sfail(LTB_INVALID, "sharded apply: bad ptr_kind %d", ptr_kind);
  {
    DevGuard g(p->dev[0]);
    SH_CUDA(cudaEventRecord(s->start, home));
  }
  for (int k = 0; k < p->n; ++k) {
    DevGuard g(p->dev[k]);
    const long long nc = p->c0[k + 1] - p->c0[k];
    const double* src = in + p->c0[k] * nt;
    if (k > 0) {  // this shard's slice of m from the home device over NVLink
      if ((st = fork(s, k, home)) != LTB_OK) return st;
      double* dst = scratch_stage_in(s->s[k], (size_t)std::max<long long>(nc, p->rows) * nt);
      if (!dst) return sfail(LTB_CUDA, "sharded apply: staging alloc failed");
      SH_CUDA(cudaMemcpyPeerAsync(dst, p->dev[k], src, p->dev[0], sizeof(double) * nc * nt,
                                  scratch_stream(s->s[k])));
      src = dst;
    }
    if ((st = apply_device(p->sh[k], s->s[k], src, s->part[k], false)) != LTB_OK) return st;
  }
  DevGuard g(p->dev[0]);
  return reduce(p, s, out);
}

// m = F* d (fft_matvec.cpp:181-217) over the shards
ltb_status ltb_apply_adjoint_sharded(const ltb_splan* p, ltb_sscratch* s, const double* in, double* out,
                                     int ptr_kind) {
  ltb_status st = check_pair(p, s);
  if (st != LTB_OK) return st;
  if (!in || !out) return sfail(LTB_INVALID, "sharded apply_adjoint: null input/output");
  const cudaStream_t home = scratch_stream(s->s[0]);
  const long long nt = p->nt, len = (long long)p->rows * nt;
  if (ptr_kind == LTB_PTR_HOST) {
    for (int k = 0; k < p->n; ++k) {  // d to every device, each writes its m columns to the host
      DevGuard g(p->dev[k]);
      const cudaStream_t sk = scratch_stream(s->s[k]);
      double* dk = k == 0 ? s->part[0] : s->din[k];
      SH_CUDA(cudaMemcpyAsync(dk, in, sizeof(double) * len, cudaMemcpyHostToDevice, sk));
      if ((st = fstar_to_host(p->sh[k], s->s[k], dk, out + p->c0[k] * nt)) != LTB_OK) return st;
    }
    return sync_all(p, s);
  }
  if (ptr_kind != LTB_PTR_DEVICE) return sfail(LTB_INVALID, "sharded apply_adjoint: bad ptr_kind %d", ptr_kind);
  {
    DevGuard g(p->dev[0]);
    SH_CUDA(cudaEventRecord(s->start, home));
  }
  for (int k = 0; k < p->n; ++k) {
    DevGuard g(p->dev[k]);
    const long long nc = p->c0[k + 1] - p->c0[k];
    if (k == 0) {
      if ((st = apply_device(p->sh[0], s->s[0], in, out, true)) != LTB_OK) return st;
      continue;
    }
    const cudaStream_t sk = scratch_stream(s->s[k]);
    if ((st = fork(s, k, home)) != LTB_OK) return st;
    // broadcast of d over NVLink, the shard's F*, its m columns back
    SH_CUDA(cudaMemcpyPeerAsync(s->din[k], p->dev[k], in, p->dev[0], sizeof(double) * len, sk));
    double* mk = scratch_stage_out(s->s[k], (size_t)std::max<long long>(nc, p->rows) * nt);
    if (!mk) return sfail(LTB_CUDA, "sharded apply_adjoint: staging alloc failed");
    if ((st = apply_device(p->sh[k], s->s[k], s->din[k], mk, true)) != LTB_OK) return st;
    SH_CUDA(cudaMemcpyPeerAsync(out + p->c0[k] * nt, p->dev[0], mk, p->dev[k], sizeof(double) * nc * nt, sk));
  }
  DevGuard g(p->dev[0]);
  for (int k = 1; k < p->n; ++k)
    if ((st = join(s, k, home)) != LTB_OK) return st;
  return LTB_OK;
}

ltb_status ltb_sscratch_sync(ltb_sscratch* s) {
  if (!s) return sfail(LTB_INVALID, "ltb_sscratch_sync: null scratch");
  return sync_all(s->p, s);
}

}  // extern "C"
