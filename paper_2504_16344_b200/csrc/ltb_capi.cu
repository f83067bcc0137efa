// ltb_capi.cu -- the C ABI (include/ltb.h) over the sm_100a kernels.
//
// Object model mirrors the reference's MatvecPlan (fft_matvec.cpp:41-69):
//   ltb_plan    <-> MatvecPlan::Impl   (owns F-hat, now in HBM, plus the
//                                       FFT descriptor / twiddle table)
//   ltb_scratch <-> MatvecPlan::Scratch (owns x-hat / d-hat workspaces, a
//                                       CUDA stream, host staging buffers)
//   ltb_engine  <-> online subset of InferenceEngine (bayes_engine.cpp)
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>

#include "../../include/ltb.h"
#include "ltb_gen.cuh"
#include "ltb_kernels.h"
#include "ltb_trsv.h"

using namespace ltb;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

ltb_status fail(ltb_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define LTB_CUDA_TRY(expr)                                                            \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(LTB_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                          \
  } while (0)

#define LTB_LAUNCH(expr, nkernels)  \
  do {                              \
    LTB_CUDA_TRY(expr);             \
    g_launches += (nkernels);       \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// radix schedule for the Stockham FFT: 8s, then 4 / 2, then 3, 5, 7, then
// any remaining primes (generic butterfly)
bool fft_radices(int n, int* radix, int* nstages) {
  int m = n, k = 0;
  auto push = [&](int r) {
    if (k >= kMaxStages) return false;
    radix[k++] = r;
    return true;
  };
  while (m % 8 == 0) { if (!push(8)) return false; m /= 8; }
  while (m % 4 == 0) { if (!push(4)) return false; m /= 4; }
  while (m % 2 == 0) { if (!push(2)) return false; m /= 2; }
  for (int p : {3, 5, 7}) while (m % p == 0) { if (!push(p)) return false; m /= p; }
  for (int p = 11; m > 1; p += 2) {
    while (m % p == 0) { if (!push(p)) return false; m /= p; }
    if ((long long)p * p > m && m > 1) { if (!push(m)) return false; m = 1; }
  }
  *nstages = k;
  return true;
}

// W[j] = exp(-2 pi i j / n) in long double, exact at quadrant points and
// mirrored so W[n-j] = conj(W[j])
std::vector<double2> twiddles(int n) {
  std::vector<double2> w(n);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int j = 0; j <= n / 2; ++j) {
    double c, s;
    if ((4LL * j) % n == 0) {
      const int q = (int)((4LL * j) / n);
      c = q == 0 ? 1.0 : (q == 2 ? -1.0 : 0.0);
      s = q == 1 ? 1.0 : 0.0;
    } else {
      const long double a = two_pi * (long double)j / (long double)n;
      c = (double)cosl(a);
      s = (double)sinl(a);
    }
    w[j] = make_double2(c, -s);
    if (j > 0 && j < n - j) w[n - j] = make_double2(c, s);
  }
  return w;
}

}  // namespace

struct ScratchPool {
  std::mutex mu;
  std::vector<ltb_scratch*> free;
  bool plan_alive = true;
};
constexpr size_t kScratchPoolMax = 8;

struct ltb_plan {
  int device = 0;
  int rows = 0, cols = 0, nt = 0, npad = 0, nf = 0, tag = 0;
  double2* fhat = nullptr;
  double2* tw = nullptr;
  FftDesc fft{};
  BigFft big{};                 // four-step tables when 2 N_t is too long for one CTA
  double2* big_tw = nullptr;    // [W_n1 | W_n2 | W_N]
  GemvShape shape{};
  size_t bytes = 0;
  // Scratch pool: the reference builds a fresh Scratch for every apply(m)
  // (fft_matvec.cpp:232-235), every infer_map (bayes_engine.cpp:317) and
  // every form_K column (:144).  Released scratches park here with their
  // workspaces and private stream, so such a Scratch costs a pointer swap
  // instead of ~0.5 GB of cudaMalloc + a device-synchronizing cudaFree.
  // Shared with the scratches, so a Scratch may outlive its plan (as in the
  // reference, where a Scratch owns its buffers outright).
  std::shared_ptr<struct ScratchPool> pool = std::make_shared<ScratchPool>();
};

struct ltb_scratch {
  const ltb_plan* plan = nullptr;
  std::shared_ptr<ScratchPool> pool;
  int device = 0;
  cudaStream_t stream = nullptr;  // the stream applies run on (caller's or priv)
  cudaStream_t priv = nullptr;    // private stream (created when no stream is given; kept by the pool)
  cudaEvent_t released = nullptr; // recorded on release: the next owner's stream waits on it
  double2* xhat = nullptr;      // nf * cols
  double2* dhat = nullptr;      // nf * rows
  double2* partials = nullptr;  // GEMV-N unit partials
  unsigned* tickets = nullptr;
  double* red = nullptr;        // 1024 + 4 doubles
  double* stage_in = nullptr;   // host-pointer staging (lazily allocated)
  double* stage_out = nullptr;
  size_t stage_in_n = 0, stage_out_n = 0;
  // host-pointer pipelining: a copy stream and per-chunk events
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t pipe_ev[17] = {};
  // per-stage timing (ltb_scratch_timing): 4 events per timed apply
  bool timing = false;
  std::vector<cudaEvent_t> events;
  std::vector<int> event_dir;  // 0 = F, 1 = F*, per quadruple
  size_t next_quad = 0;
};

namespace {
cudaEvent_t* timing_quad(ltb_scratch* s, int dir) {
  if (!s->timing) return nullptr;
  const size_t q = s->next_quad++;
  if (4 * (q + 1) > s->events.size()) {
    for (int k = 0; k < 4; ++k) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      s->events.push_back(e);
    }
    s->event_dir.push_back(dir);
  }
  s->event_dir[q] = dir;
  return &s->events[4 * q];
}
}  // namespace

extern "C" {

const char* ltb_last_error(void) { return g_err.c_str(); }
const char* ltb_version(void) { return "ltb 0.1 (sm_100a)"; }
uint64_t ltb_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"

namespace {

ltb_status plan_init(ltb_plan* p, int rows, int cols, int nt, int tag, const ltb_opts* opts) {
  if (rows < 1 || cols < 1 || nt < 1)
    return fail(LTB_DIMENSION, "MatvecPlan: kernel dims must be >= 1 (rows=%d cols=%d nt=%d)", rows,
                cols, nt);
  if (tag < 0 || tag > 3) return fail(LTB_INVALID, "MatvecPlan: bad kernel tag %d", tag);
  p->device = (opts && opts->device >= 0) ? opts->device : -1;
  if (p->device < 0) cudaGetDevice(&p->device);
  DeviceGuard g(p->device);  // F-hat and the twiddles live on the plan's device
  p->rows = rows;
  p->cols = cols;
  p->nt = nt;
  p->npad = 2 * nt;
  p->nf = nt + 1;
  p->tag = tag;
  int B = 0;
  const bool big = fft_smem_bytes(p->npad, &B) > 227 * 1024;
  if (!big && !fft_radices(p->npad, p->fft.radix, &p->fft.nstages))
    return fail(LTB_CAPACITY, "MatvecPlan: too many FFT stages for 2*N_t=%d", p->npad);
  p->fft.n = p->npad;
  if (big) {
    // four-step: 2 N_t = n1 n2, both within the shared-memory FFT
    int max_len = 2;
    while (fft_smem_bytes(2 * max_len, &B) <= 227 * 1024) max_len *= 2;
    while (fft_smem_bytes(max_len + 1, &B) <= 227 * 1024) ++max_len;
    int n1 = 0, n2 = 0;
    if (!big_fft_split(p->npad, max_len, &n1, &n2) || !fft_radices(n1, p->big.d1.radix, &p->big.d1.nstages) ||
        !fft_radices(n2, p->big.d2.radix, &p->big.d2.nstages))
      return fail(LTB_CAPACITY, "MatvecPlan: 2*N_t=%d has no factorisation into two transforms of <= %d", p->npad,
                  max_len);
    const auto w1 = twiddles(n1), w2 = twiddles(n2), wn = twiddles(p->npad);
    LTB_CUDA_TRY(cudaMalloc(&p->big_tw, sizeof(double2) * (w1.size() + w2.size() + wn.size())));
    LTB_CUDA_TRY(cudaMemcpy(p->big_tw, w1.data(), sizeof(double2) * w1.size(), cudaMemcpyHostToDevice));
    LTB_CUDA_TRY(cudaMemcpy(p->big_tw + w1.size(), w2.data(), sizeof(double2) * w2.size(), cudaMemcpyHostToDevice));
    LTB_CUDA_TRY(cudaMemcpy(p->big_tw + w1.size() + w2.size(), wn.data(), sizeof(double2) * wn.size(),
                            cudaMemcpyHostToDevice));
    p->big.n = p->npad;
    p->big.n1 = n1;
    p->big.n2 = n2;
    p->big.d1.n = n1;
    p->big.d1.tw = p->big_tw;
    p->big.d2.n = n2;
    p->big.d2.tw = p->big_tw + w1.size();
    p->big.twN = p->big_tw + w1.size() + w2.size();
    p->fft.big = &p->big;
  }
  p->shape = gemv_shape(rows, cols, p->nf, opts ? opts->unit_cols : 0);
  const size_t fhat_bytes = sizeof(double2) * (size_t)p->nf * rows * cols;
  size_t free_b = 0, total_b = 0;
  LTB_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  if (fhat_bytes + (64u << 20) > free_b)
    return fail(LTB_CAPACITY, "MatvecPlan: F-hat needs %zu bytes, %zu free on device %d", fhat_bytes,
                free_b, p->device);
  LTB_CUDA_TRY(cudaMalloc(&p->fhat, fhat_bytes));
  const auto w = twiddles(p->npad);
  LTB_CUDA_TRY(cudaMalloc(&p->tw, sizeof(double2) * w.size()));
  LTB_CUDA_TRY(cudaMemcpy(p->tw, w.data(), sizeof(double2) * w.size(), cudaMemcpyHostToDevice));
  p->fft.tw = p->tw;
  p->bytes = fhat_bytes + sizeof(double2) * w.size();
  return LTB_OK;
}

void scratch_free(ltb_scratch* s);

void plan_free(ltb_plan* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  {
    std::lock_guard<std::mutex> lk(p->pool->mu);
    for (ltb_scratch* s : p->pool->free) scratch_free(s);
    p->pool->free.clear();
    p->pool->plan_alive = false;
  }
  cudaFree(p->fhat);
  cudaFree(p->tw);
  cudaFree(p->big_tw);
  delete p;
}

__global__ void count_nonfinite_kernel(const double* x, long long n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) ++local;
  if (local) atomicAdd(bad, local);
}

ltb_status ensure_stage(ltb_scratch* s, size_t nin, size_t nout) {
  if (nin > s->stage_in_n) {
    cudaFree(s->stage_in);
    s->stage_in = nullptr;
    LTB_CUDA_TRY(cudaMalloc(&s->stage_in, sizeof(double) * nin));
    s->stage_in_n = nin;
  }
  if (nout > s->stage_out_n) {
    cudaFree(s->stage_out);
    s->stage_out = nullptr;
    LTB_CUDA_TRY(cudaMalloc(&s->stage_out, sizeof(double) * nout));
    s->stage_out_n = nout;
  }
  return LTB_OK;
}

// d = F m on device pointers, async on s->stream (fft_matvec.cpp:139-179)
ltb_status apply_dev(const ltb_plan* p, ltb_scratch* s, const double* m, double* d) {
  const cudaStream_t st = s->stream;
  cudaEvent_t* ev = timing_quad(s, 0);
  if (ev) cudaEventRecord(ev[0], st);
  // K1: pad + r2c of the n_cols input rows -> x-hat[f][c]
  RfftSrc src{m, 0, 1, 0, 0};
  LTB_LAUNCH(launch_rfft_rows(p->fft, src, p->nt, p->cols, s->xhat, p->cols, st), 1);
  if (ev) cudaEventRecord(ev[1], st);
  // K2: y-hat[f][r] = sum_c F-hat[f][c][r] x-hat[f][c]  (+ in-kernel unit
  // reduction; the launcher also zeroes the tickets with a memset node)
  LTB_LAUNCH(launch_gemv_n(p->shape, p->fhat, s->xhat, s->partials, s->dhat, s->tickets, st), 1);
  if (ev) cudaEventRecord(ev[2], st);
  // K4: c2r + truncate + 1/(2 N_t) of the rows_out output rows
  LTB_LAUNCH(launch_irfft_rows(p->fft, s->dhat, p->rows, 0, 1, p->nt, p->rows, 1.0 / p->npad, d,
                               st),
             1);
  if (ev) cudaEventRecord(ev[3], st);
  return LTB_OK;
}

// m = F* d on device pointers (fft_matvec.cpp:181-217)
ltb_status apply_adjoint_dev(const ltb_plan* p, ltb_scratch* s, const double* d, double* m) {
  const cudaStream_t st = s->stream;
  cudaEvent_t* ev = timing_quad(s, 1);
  if (ev) cudaEventRecord(ev[0], st);
  RfftSrc src{d, 0, 1, 0, 0};
  LTB_LAUNCH(launch_rfft_rows(p->fft, src, p->nt, p->rows, s->dhat, p->rows, st), 1);
  if (ev) cudaEventRecord(ev[1], st);
  LTB_LAUNCH(launch_gemv_h(p->shape, p->fhat, s->dhat, s->xhat, st), 1);
  if (ev) cudaEventRecord(ev[2], st);
  LTB_LAUNCH(launch_irfft_rows(p->fft, s->xhat, p->cols, 0, 1, p->nt, p->cols, 1.0 / p->npad, m,
                               st),
             1);
  if (ev) cudaEventRecord(ev[3], st);
  return LTB_OK;
}

using DevFn = ltb_status (*)(const ltb_plan*, ltb_scratch*, const double*, double*);

// Host-pointer applies move n_cols * N_t values one way (m in for F m, m out
// for F* d): 110 MB at Cascadia, ~2 ms over PCIe.  Cut into column chunks,
// those copies run on a second stream against the transforms and GEMVs of
// the other chunks (GEMV-N accumulates the chunks' products into y-hat in
// chunk order, so the result is deterministic).  Returns LTB_OK after the
// results are on the host.
constexpr size_t kPipeMinBytes = 16u << 20;
constexpr int kPipeGeo = 3, kPipeEven = 8, kPipeMaxChunks = 8;

ltb_status pipe_setup(ltb_scratch* s) {
  if (!s->copy_stream) LTB_CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
  for (cudaEvent_t& e : s->pipe_ev)
    if (!e) LTB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return LTB_OK;
}

// Column chunk boundaries b[0..K] of the host-pointer pipelines, in whole
// GEMV work units.  A column costs 16 Nf rows bytes of F-hat streaming and
// 8 N_t bytes of PCIe copy, so the copy runs g ~ rows / 65 times faster
// than the GEMV consumes / produces columns (HBM ~6.5 TB/s, PCIe ~50 GB/s).
// g >= 2 (Cascadia: ~9): three chunks growing by ~0.6 g from the end whose
// copy cannot overlap anything -- first for the H2D of F m, last for the D2H
// of F* d -- so each copy hides under the neighbouring chunk's GEMV, the
// short end chunk's copy is the only exposed one, and there are few GEMV
// windows (each launch has a wave tail).  g < 2 (config 2's G*: the copy is
// the critical path): kPipeEven even chunks, so the copies start early.
int pipe_bounds(const ltb_plan* p, bool short_first, long long* b) {
  // even boundaries too: the transforms pair rows (2j, 2j+1), so chunking
  // keeps the device path's pairs and its bits
  const long long cols = p->cols, u = p->shape.unit_cols * (p->shape.unit_cols % 2 ? 2 : 1);
  const double g = std::min(6.0, 0.6 * p->rows / 65.0);
  const int n = g >= 2.0 ? kPipeGeo : kPipeEven;
  const double grow = g >= 2.0 ? g : 1.0;
  long long sz[kPipeMaxChunks];
  double w = 1.0, tot = 0.0;
  for (int k = 0; k < n; ++k, w *= grow) tot += w;
  long long used = 0;
  int K = 0;
  w = 1.0;
  for (int k = 0; k < n && used < cols; ++k, w *= grow) {
    long long c = (long long)(cols * (w / tot));
    c = std::max(u, (c + u - 1) / u * u);
    if (k == n - 1 || used + c > cols) c = cols - used;
    sz[K++] = c;
    used += c;
  }
  b[0] = 0;
  for (int k = 0; k < K; ++k) b[k + 1] = b[k] + sz[short_first ? k : K - 1 - k];
  return K;
}

// F* of a device-resident d into dev_out (n_cols x N_t), GEMV-H / c2r in
// column chunks with each chunk's copy to host_out queued on the copy stream
// as soon as it is ready.  Asynchronous: the copy stream is joined back into
// the compute stream at the end (later work on it waits for the copies).
ltb_status adjoint_chunks_to_host(const ltb_plan* p, ltb_scratch* s, const double* d_dev, double* dev_out,
                                  double* host_out) {
  ltb_status st = pipe_setup(s);
  if (st != LTB_OK) return st;
  const cudaStream_t cs = s->stream, xs = s->copy_stream;
  const long long cols = p->cols, nt = p->nt;
  long long b[kPipeMaxChunks + 1];
  const int K = pipe_bounds(p, false, b);
  RfftSrc src{d_dev, 0, 1, 0, 0};
  LTB_LAUNCH(launch_rfft_rows(p->fft, src, p->nt, p->rows, s->dhat, p->rows, cs), 1);
  for (int k = 0; k < K; ++k) {
    const long long c0 = b[k], nc = b[k + 1] - b[k];
    LTB_LAUNCH(launch_gemv_h(gemv_window(p->shape, c0, nc, 0), p->fhat, s->dhat, s->xhat, cs), 1);
    LTB_LAUNCH(launch_irfft_rows(p->fft, s->xhat + c0, cols, 0, 1, p->nt, nc, 1.0 / p->npad, dev_out + c0 * nt, cs),
               1);
    LTB_CUDA_TRY(cudaEventRecord(s->pipe_ev[k], cs));
    LTB_CUDA_TRY(cudaStreamWaitEvent(xs, s->pipe_ev[k], 0));
    LTB_CUDA_TRY(cudaMemcpyAsync(host_out + c0 * nt, dev_out + c0 * nt, sizeof(double) * nc * nt,
                                 cudaMemcpyDeviceToHost, xs));
  }
  LTB_CUDA_TRY(cudaEventRecord(s->pipe_ev[16], xs));
  LTB_CUDA_TRY(cudaStreamWaitEvent(cs, s->pipe_ev[16], 0));
  return LTB_OK;
}

// d_dev = F m of a HOST m, enqueued on s->stream (nothing synchronized):
// the pipelined column chunks above 16 MB of field, else one copy + the
// device path.  The copy stream is joined back into the compute stream.
ltb_status fm_host_enqueue(const ltb_plan* p, ltb_scratch* s, const double* in, double* d_dev) {
  const cudaStream_t cs = s->stream;
  const long long cols = p->cols, nt = p->nt;
  ltb_status st = ensure_stage(s, (size_t)std::max(cols, (long long)p->rows) * nt,
                               (size_t)std::max(cols, (long long)p->rows) * nt);
  if (st != LTB_OK) return st;
  if (s->timing || (size_t)cols * nt * sizeof(double) < kPipeMinBytes) {
    LTB_CUDA_TRY(cudaMemcpyAsync(s->stage_in, in, sizeof(double) * cols * nt, cudaMemcpyHostToDevice, cs));
    return apply_dev(p, s, s->stage_in, d_dev);
  }
  if ((st = pipe_setup(s)) != LTB_OK) return st;
  const cudaStream_t xs = s->copy_stream;
  long long b[kPipeMaxChunks + 1];
  const int K = pipe_bounds(p, true, b);
  // order the copy stream after everything already queued on the compute stream
  LTB_CUDA_TRY(cudaEventRecord(s->pipe_ev[16], cs));
  LTB_CUDA_TRY(cudaStreamWaitEvent(xs, s->pipe_ev[16], 0));
  for (int k = 0; k < K; ++k) {
    const long long c0 = b[k], nc = b[k + 1] - b[k];
    LTB_CUDA_TRY(cudaMemcpyAsync(s->stage_in + c0 * nt, in + c0 * nt, sizeof(double) * nc * nt,
                                 cudaMemcpyHostToDevice, xs));
    LTB_CUDA_TRY(cudaEventRecord(s->pipe_ev[k], xs));
  }
  for (int k = 0; k < K; ++k) {
    const long long c0 = b[k], nc = b[k + 1] - b[k];
    LTB_CUDA_TRY(cudaStreamWaitEvent(cs, s->pipe_ev[k], 0));
    RfftSrc src{s->stage_in + c0 * nt, 0, 1, 0, 0};
    LTB_LAUNCH(launch_rfft_rows(p->fft, src, p->nt, nc, s->xhat + c0, cols, cs), 1);
    LTB_LAUNCH(launch_gemv_n(gemv_window(p->shape, c0, nc, k > 0), p->fhat, s->xhat, s->partials, s->dhat,
                             s->tickets, cs),
               1);
  }
  LTB_LAUNCH(launch_irfft_rows(p->fft, s->dhat, p->rows, 0, 1, p->nt, p->rows, 1.0 / p->npad, d_dev, cs), 1);
  return LTB_OK;
}

ltb_status apply_host_pipelined(const ltb_plan* p, ltb_scratch* s, const double* in, double* out,
                                bool adjoint) {
  ltb_status st = pipe_setup(s);
  if (st != LTB_OK) return st;
  const cudaStream_t cs = s->stream, xs = s->copy_stream;
  const long long nt = p->nt;
  if (!adjoint) {
    if ((st = fm_host_enqueue(p, s, in, s->stage_out)) != LTB_OK) return st;
    LTB_CUDA_TRY(cudaMemcpyAsync(out, s->stage_out, sizeof(double) * p->rows * nt, cudaMemcpyDeviceToHost, cs));
    LTB_CUDA_TRY(cudaStreamSynchronize(cs));
    LTB_CUDA_TRY(cudaStreamSynchronize(xs));
    return LTB_OK;
  }
  LTB_CUDA_TRY(cudaMemcpyAsync(s->stage_in, in, sizeof(double) * p->rows * nt, cudaMemcpyHostToDevice, cs));
  st = adjoint_chunks_to_host(p, s, s->stage_in, s->stage_out, out);
  if (st != LTB_OK) return st;
  LTB_CUDA_TRY(cudaStreamSynchronize(cs));
  LTB_CUDA_TRY(cudaStreamSynchronize(xs));
  return LTB_OK;
}

ltb_status run_apply(const ltb_plan* p, ltb_scratch* s, const double* in, double* out,
                     int ptr_kind, bool adjoint) {
  if (!p || !s) return fail(LTB_INVALID, "apply: null plan or scratch");
  if (s->plan != p) return fail(LTB_INVALID, "apply: scratch was created for another plan");
  if (!in || !out) return fail(LTB_INVALID, "apply: null input/output");
  DeviceGuard g(p->device);
  const size_t nin = (size_t)(adjoint ? p->rows : p->cols) * p->nt;
  const size_t nout = (size_t)(adjoint ? p->cols : p->rows) * p->nt;
  DevFn fn = adjoint ? apply_adjoint_dev : apply_dev;
  if (ptr_kind == LTB_PTR_DEVICE) return fn(p, s, in, out);
  if (ptr_kind != LTB_PTR_HOST) return fail(LTB_INVALID, "apply: bad ptr_kind %d", ptr_kind);
  ltb_status st = ensure_stage(s, std::max(nin, nout), std::max(nin, nout));
  if (st != LTB_OK) return st;
  if (!s->timing && (size_t)p->cols * p->nt * sizeof(double) >= kPipeMinBytes)
    return apply_host_pipelined(p, s, in, out, adjoint);
  LTB_CUDA_TRY(cudaMemcpyAsync(s->stage_in, in, sizeof(double) * nin, cudaMemcpyHostToDevice, s->stream));
  st = fn(p, s, s->stage_in, s->stage_out);
  if (st != LTB_OK) return st;
  LTB_CUDA_TRY(cudaMemcpyAsync(out, s->stage_out, sizeof(double) * nout, cudaMemcpyDeviceToHost, s->stream));
  LTB_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return LTB_OK;
}

}  // namespace

extern "C" {

ltb_status ltb_plan_create(const double* kernel, int rows, int cols, int nt, int tag, int ptr_kind,
                           const ltb_opts* opts, ltb_plan** out) {
  if (!out) return fail(LTB_INVALID, "ltb_plan_create: null out");
  *out = nullptr;
  if (!kernel) return fail(LTB_INVALID, "ltb_plan_create: null kernel");
  if (rows < 1 || cols < 1 || nt < 1)
    return fail(LTB_DIMENSION, "MatvecPlan: kernel tensor size does not match dims");
  const size_t n = (size_t)rows * cols * nt;
  // core.cpp:73-77: reject non-finite kernel entries
  if (ptr_kind == LTB_PTR_HOST) {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(kernel[i])) return fail(LTB_NUMERICAL, "MatvecPlan: non-finite kernel entry");
  }
  ltb_plan* p = new ltb_plan();
  ltb_status st = plan_init(p, rows, cols, nt, tag, opts);
  if (st != LTB_OK) {
    plan_free(p);
    return st;
  }
  DeviceGuard g(p->device);
  double* dk = nullptr;
  unsigned long long* bad = nullptr;
  auto cleanup = [&](ltb_status s_) {
    cudaFree(dk);
    cudaFree(bad);
    if (s_ != LTB_OK) plan_free(p);
    return s_;
  };
  const double* src_ptr = kernel;
  if (ptr_kind == LTB_PTR_HOST) {
    if (cudaMalloc(&dk, sizeof(double) * n) != cudaSuccess ||
        cudaMemcpy(dk, kernel, sizeof(double) * n, cudaMemcpyHostToDevice) != cudaSuccess)
      return cleanup(fail(LTB_CUDA, "MatvecPlan: kernel upload failed: %s",
                          cudaGetErrorString(cudaGetLastError())));
    src_ptr = dk;
  } else {
    if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess)
      return cleanup(fail(LTB_CUDA, "MatvecPlan: alloc failed"));
    cudaMemset(bad, 0, sizeof(unsigned long long));
    count_nonfinite_kernel<<<148 * 8, 256>>>(kernel, (long long)n, bad);
    g_launches += 1;
    unsigned long long hb = 0;
    cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
    if (hb) return cleanup(fail(LTB_NUMERICAL, "MatvecPlan: non-finite kernel entry"));
  }
  // K7: F-hat[f][c][r] = r2c(pad(k[r][c][:]))[f]; logical row g = c*rows + r
  RfftSrc src{src_ptr, 0, rows, (long long)cols, 0};
  cudaError_t e = launch_rfft_rows(p->fft, src, nt, (long long)rows * cols, p->fhat,
                                   (long long)rows * cols, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(fail(LTB_CUDA, "MatvecPlan: plan build: %s", cudaGetErrorString(e)));
  g_launches += 1;
  *out = p;
  return cleanup(LTB_OK);
}

ltb_status ltb_plan_create_generated(int rows, int cols, int nt, int tag, uint64_t seed,
                                     uint64_t stream, long long nm_total, long long c0,
                                     const ltb_opts* opts, ltb_plan** out) {
  if (!out) return fail(LTB_INVALID, "ltb_plan_create_generated: null out");
  *out = nullptr;
  if (c0 < 0 || nm_total < c0 + cols)
    return fail(LTB_DIMENSION, "generated plan: shard [%lld, %lld) outside nm_total=%lld", c0,
                c0 + cols, nm_total);
  ltb_plan* p = new ltb_plan();
  ltb_status st = plan_init(p, rows, cols, nt, tag, opts);
  if (st != LTB_OK) {
    plan_free(p);
    return st;
  }
  DeviceGuard g(p->device);
  RfftSrc src{nullptr, gen_key(seed, stream), rows, nm_total, c0};
  cudaError_t e = launch_rfft_rows(p->fft, src, nt, (long long)rows * cols, p->fhat,
                                   (long long)rows * cols, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    plan_free(p);
    return fail(LTB_CUDA, "generated plan build: %s", cudaGetErrorString(e));
  }
  g_launches += 1;
  *out = p;
  return LTB_OK;
}

ltb_status ltb_plan_destroy(ltb_plan* p) {
  plan_free(p);
  return LTB_OK;
}

ltb_status ltb_plan_dims(const ltb_plan* p, int* rows, int* cols, int* nt, int* npad, int* nf,
                         int* tag) {
  if (!p) return fail(LTB_INVALID, "ltb_plan_dims: null plan");
  if (rows) *rows = p->rows;
  if (cols) *cols = p->cols;
  if (nt) *nt = p->nt;
  if (npad) *npad = p->npad;
  if (nf) *nf = p->nf;
  if (tag) *tag = p->tag;
  return LTB_OK;
}

ltb_status ltb_plan_bytes(const ltb_plan* p, size_t* bytes) {
  if (!p || !bytes) return fail(LTB_INVALID, "ltb_plan_bytes: null argument");
  *bytes = p->bytes;
  return LTB_OK;
}

ltb_status ltb_kernel_hat_sqnorm(const ltb_plan* p, double* out) {
  if (!p || !out) return fail(LTB_INVALID, "ltb_kernel_hat_sqnorm: null argument");
  DeviceGuard g(p->device);
  double* work = nullptr;
  LTB_CUDA_TRY(cudaMalloc(&work, sizeof(double) * (1024 + 4)));
  const long long bc = (long long)p->rows * p->cols;
  double h[3];
  cudaError_t e = launch_sqnorm(p->fhat, bc * p->nf, work, work + 1024, 0);
  if (e == cudaSuccess) e = launch_sqnorm(p->fhat, bc, work, work + 1025, 0);
  if (e == cudaSuccess) e = launch_sqnorm(p->fhat + bc * (p->nf - 1), bc, work, work + 1026, 0);
  if (e == cudaSuccess) e = cudaMemcpy(h, work + 1024, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(work);
  if (e != cudaSuccess) return fail(LTB_CUDA, "kernel_hat_sqnorm: %s", cudaGetErrorString(e));
  g_launches += 6;
  // interior frequencies appear twice in the full circulant spectrum
  *out = 2 * h[0] - (h[1] + h[2]);
  return LTB_OK;
}

ltb_status ltb_plan_copy_kernel_hat(const ltb_plan* p, int f0, int nfreq, double* host_out) {
  if (!p || !host_out) return fail(LTB_INVALID, "copy_kernel_hat: null argument");
  if (f0 < 0 || nfreq < 0 || f0 + nfreq > p->nf)
    return fail(LTB_DIMENSION, "copy_kernel_hat: frequency range out of bounds");
  DeviceGuard g(p->device);
  const size_t bc = (size_t)p->rows * p->cols;
  LTB_CUDA_TRY(cudaMemcpy(host_out, p->fhat + bc * f0, sizeof(double2) * bc * nfreq,
                          cudaMemcpyDeviceToHost));
  return LTB_OK;
}

}  // extern "C"

namespace {
void scratch_free(ltb_scratch* s) {
  DeviceGuard g(s->device);
  if (s->priv) cudaStreamSynchronize(s->priv);
  cudaFree(s->xhat);
  cudaFree(s->dhat);
  cudaFree(s->partials);
  cudaFree(s->tickets);
  cudaFree(s->red);
  cudaFree(s->stage_in);
  cudaFree(s->stage_out);
  for (cudaEvent_t e : s->events) cudaEventDestroy(e);
  for (cudaEvent_t e : s->pipe_ev)
    if (e) cudaEventDestroy(e);
  if (s->released) cudaEventDestroy(s->released);
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  if (s->priv) cudaStreamDestroy(s->priv);
  delete s;
}

// bind a (new or pooled) scratch to the caller's stream, or its private one
cudaError_t scratch_bind(ltb_scratch* s, void* stream) {
  if (stream) {
    s->stream = (cudaStream_t)stream;
  } else {
    if (!s->priv) {
      cudaError_t e = cudaStreamCreateWithFlags(&s->priv, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    s->stream = s->priv;
  }
  // whatever the previous owner queued on its stream finishes first
  return s->released ? cudaStreamWaitEvent(s->stream, s->released, 0) : cudaSuccess;
}
}  // namespace

extern "C" {

ltb_status ltb_scratch_create(const ltb_plan* p, void* stream, ltb_scratch** out) {
  if (!p || !out) return fail(LTB_INVALID, "ltb_scratch_create: null argument");
  *out = nullptr;
  DeviceGuard g(p->device);
  ltb_scratch* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(p->pool->mu);
    if (!p->pool->free.empty()) {
      s = p->pool->free.back();
      p->pool->free.pop_back();
    }
  }
  if (s) {
    cudaError_t e = scratch_bind(s, stream);
    if (e != cudaSuccess) {
      scratch_free(s);
      return fail(LTB_CUDA, "ltb_scratch_create: %s", cudaGetErrorString(e));
    }
    *out = s;
    return LTB_OK;
  }
  s = new ltb_scratch();
  s->plan = p;
  s->pool = p->pool;
  s->device = p->device;
  auto bail = [&](cudaError_t e) {
    scratch_free(s);
    return fail(LTB_CUDA, "ltb_scratch_create: %s", cudaGetErrorString(e));
  };
  cudaError_t e;
  if ((e = scratch_bind(s, stream)) != cudaSuccess) return bail(e);
  const size_t nx = (size_t)p->nf * p->cols, nd = (size_t)p->nf * p->rows;
  if ((e = cudaMalloc(&s->xhat, sizeof(double2) * nx)) != cudaSuccess) return bail(e);
  if ((e = cudaMalloc(&s->dhat, sizeof(double2) * nd)) != cudaSuccess) return bail(e);
  if ((e = cudaMalloc(&s->partials, sizeof(double2) * gemv_n_partials(p->shape))) != cudaSuccess) return bail(e);
  if ((e = cudaMalloc(&s->tickets, sizeof(unsigned) * (size_t)p->nf * gemv_n_row_tiles(p->shape))) != cudaSuccess) return bail(e);
  if ((e = cudaMalloc(&s->red, sizeof(double) * (1024 + 8))) != cudaSuccess) return bail(e);
  *out = s;
  return LTB_OK;
}

// Returns the scratch to its plan's pool (workspaces and private stream
// kept; work still queued on its stream is fenced by an event the next owner
// waits on), or frees it when the pool is full.
ltb_status ltb_scratch_destroy(ltb_scratch* s) {
  if (!s) return LTB_OK;
  DeviceGuard g(s->device);
  s->timing = false;
  s->next_quad = 0;
  bool pooled = false;
  if (s->pool && (s->released || cudaEventCreateWithFlags(&s->released, cudaEventDisableTiming) == cudaSuccess) &&
      cudaEventRecord(s->released, s->stream) == cudaSuccess) {
    std::lock_guard<std::mutex> lk(s->pool->mu);
    if (s->pool->plan_alive && s->pool->free.size() < kScratchPoolMax) {
      s->pool->free.push_back(s);
      pooled = true;
    }
  }
  cudaGetLastError();
  if (!pooled) {
    // a borrowed stream may already be gone (its owner tears down first);
    // cudaFree in scratch_free synchronizes the device anyway
    scratch_free(s);
  }
  return LTB_OK;
}

ltb_status ltb_scratch_sync(ltb_scratch* s) {
  if (!s) return fail(LTB_INVALID, "ltb_scratch_sync: null scratch");
  DeviceGuard g(s->device);
  LTB_CUDA_TRY(cudaStreamSynchronize(s->stream));
  return LTB_OK;
}

void* ltb_scratch_stream(ltb_scratch* s) { return s ? (void*)s->stream : nullptr; }

ltb_status ltb_scratch_timing(ltb_scratch* s, int enable) {
  if (!s) return fail(LTB_INVALID, "ltb_scratch_timing: null scratch");
  DeviceGuard g(s->device);
  LTB_CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->timing = enable != 0;
  s->next_quad = 0;
  return LTB_OK;
}

ltb_status ltb_scratch_stage_ms(ltb_scratch* s, double* ms6, int* calls2) {
  if (!s || !ms6 || !calls2) return fail(LTB_INVALID, "ltb_scratch_stage_ms: null argument");
  DeviceGuard g(s->device);
  LTB_CUDA_TRY(cudaStreamSynchronize(s->stream));
  for (int k = 0; k < 6; ++k) ms6[k] = 0.0;
  calls2[0] = calls2[1] = 0;
  for (size_t q = 0; q < s->next_quad; ++q) {
    const int dir = s->event_dir[q];
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      LTB_CUDA_TRY(cudaEventElapsedTime(&ms, s->events[4 * q + k], s->events[4 * q + k + 1]));
      ms6[3 * dir + k] += ms;
    }
    calls2[dir] += 1;
  }
  return LTB_OK;
}

ltb_status ltb_apply(const ltb_plan* p, ltb_scratch* s, const double* in, double* out, int ptr_kind) {
  return run_apply(p, s, in, out, ptr_kind, false);
}

ltb_status ltb_apply_adjoint(const ltb_plan* p, ltb_scratch* s, const double* in, double* out,
                             int ptr_kind) {
  return run_apply(p, s, in, out, ptr_kind, true);
}

static ltb_status check_series(const ltb_plan* p, int n_rows, int n_time, int layout, bool adjoint) {
  if (!p) return fail(LTB_INVALID, "apply: null plan");
  const char* what = adjoint ? "MatvecPlan::apply_adjoint" : "MatvecPlan::apply";
  // BlockSeries::check_consistent (core.cpp:29-38)
  if (n_rows < 1 || n_time < 1) return fail(LTB_DIMENSION, "%s: series dims must be >= 1", what);
  // check_layout (fft_matvec.cpp:221-228)
  if (layout != LTB_SPACE_MAJOR_ROWS)
    return fail(LTB_LAYOUT, "%s: requires SpaceMajorRows input, got TimeMajorBlocks (no silent reindex)",
                what);
  const int want_rows = adjoint ? p->rows : p->cols;
  if (n_rows != want_rows || n_time != p->nt)
    return fail(LTB_DIMENSION, "%s: input dims (%d,%d) do not match kernel (%d,%d)", what, n_rows,
                n_time, want_rows, p->nt);
  return LTB_OK;
}

ltb_status ltb_apply_series(const ltb_plan* p, ltb_scratch* s, const double* in, int n_rows,
                            int n_time, int layout, double* out, int ptr_kind) {
  ltb_status st = check_series(p, n_rows, n_time, layout, false);
  return st != LTB_OK ? st : run_apply(p, s, in, out, ptr_kind, false);
}

ltb_status ltb_apply_adjoint_series(const ltb_plan* p, ltb_scratch* s, const double* in,
                                    int n_rows, int n_time, int layout, double* out,
                                    int ptr_kind) {
  ltb_status st = check_series(p, n_rows, n_time, layout, true);
  return st != LTB_OK ? st : run_apply(p, s, in, out, ptr_kind, true);
}

}  // extern "C"

// ---- internal hooks for ltb_engine.cu ----
namespace ltb_internal {
// m = G* y (device y) and q = F_q m with the G* c2r and the F_q r2c fused
// (launch_c2r_r2c_rows: m is written once and never read back); with m_host
// the G* columns run in chunks and each chunk of m is copied out while the
// next ones compute.  All on sg's stream (sq must share it).
ltb_status gstar_then_fq(const ltb_plan* g, ltb_scratch* sg, const ltb_plan* fq, ltb_scratch* sq,
                         const double* y_dev, double* m_dev, double* q_dev, double* m_host) {
  if (!g || !fq || !sg || !sq || sg->plan != g || sq->plan != fq)
    return fail(LTB_INVALID, "forecast: plan / scratch mismatch");
  if (g->cols != fq->cols || g->nt != fq->nt) return fail(LTB_DIMENSION, "engine: F and Fq dims are inconsistent");
  const cudaStream_t cs = sg->stream;
  const long long cols = g->cols, nt = g->nt;
  RfftSrc src{y_dev, 0, 1, 0, 0};
  LTB_LAUNCH(launch_rfft_rows(g->fft, src, g->nt, g->rows, sg->dhat, g->rows, cs), 1);
  const bool chunked = m_host && !sg->timing && (size_t)cols * nt * sizeof(double) >= kPipeMinBytes;
  int K = 1;
  long long b[kPipeMaxChunks + 1] = {0, cols};
  if (chunked) {
    ltb_status st = pipe_setup(sg);
    if (st != LTB_OK) return st;
    K = pipe_bounds(g, false, b);
  }
  for (int k = 0; k < K; ++k) {
    const long long c0 = b[k], nc = b[k + 1] - b[k];
    LTB_LAUNCH(launch_gemv_h(gemv_window(g->shape, c0, nc, 0), g->fhat, sg->dhat, sg->xhat, cs), 1);
    LTB_LAUNCH(launch_c2r_r2c_rows(g->fft, sg->xhat + c0, cols, g->nt, nc, 1.0 / g->npad, m_dev + c0 * nt,
                                   sq->xhat + c0, cols, cs),
               1);
    if (chunked) {
      LTB_CUDA_TRY(cudaEventRecord(sg->pipe_ev[k], cs));
      LTB_CUDA_TRY(cudaStreamWaitEvent(sg->copy_stream, sg->pipe_ev[k], 0));
      LTB_CUDA_TRY(cudaMemcpyAsync(m_host + c0 * nt, m_dev + c0 * nt, sizeof(double) * nc * nt,
                                   cudaMemcpyDeviceToHost, sg->copy_stream));
    }
  }
  LTB_LAUNCH(launch_gemv_n(fq->shape, fq->fhat, sq->xhat, sq->partials, sq->dhat, sq->tickets, cs), 1);
  LTB_LAUNCH(launch_irfft_rows(fq->fft, sq->dhat, fq->rows, 0, 1, fq->nt, fq->rows, 1.0 / fq->npad, q_dev, cs), 1);
  if (chunked) {
    LTB_CUDA_TRY(cudaEventRecord(sg->pipe_ev[16], sg->copy_stream));
    LTB_CUDA_TRY(cudaStreamWaitEvent(cs, sg->pipe_ev[16], 0));
  } else if (m_host) {
    LTB_CUDA_TRY(cudaMemcpyAsync(m_host, m_dev, sizeof(double) * cols * nt, cudaMemcpyDeviceToHost, cs));
  }
  return LTB_OK;
}
ltb_status adjoint_to_host(const ltb_plan* p, ltb_scratch* s, const double* d_dev, double* dev_out,
                           double* host_out) {
  if (!p || !s || s->plan != p) return fail(LTB_INVALID, "apply: scratch was created for another plan");
  if (s->timing || (size_t)p->cols * p->nt * sizeof(double) < kPipeMinBytes) {
    ltb_status st = apply_adjoint_dev(p, s, d_dev, dev_out);
    if (st != LTB_OK) return st;
    LTB_CUDA_TRY(cudaMemcpyAsync(host_out, dev_out, sizeof(double) * p->cols * p->nt, cudaMemcpyDeviceToHost,
                                 s->stream));
    return LTB_OK;
  }
  return adjoint_chunks_to_host(p, s, d_dev, dev_out, host_out);
}
ltb_status set_error(ltb_status st, const char* msg) {
  g_err = msg;
  return st;
}
ltb_status apply_device(const ltb_plan* p, ltb_scratch* s, const double* in, double* out,
                        bool adjoint) {
  if (!p || !s) return fail(LTB_INVALID, "apply: null plan or scratch");
  if (s->plan != p) return fail(LTB_INVALID, "apply: scratch was created for another plan");
  return adjoint ? apply_adjoint_dev(p, s, in, out) : apply_dev(p, s, in, out);
}
cudaStream_t scratch_stream(ltb_scratch* s) { return s->stream; }
// the device buffers a captured apply bakes in (ltb_engine.cu's graph key);
// false while the scratch records per-stage timing events
bool scratch_graph_key(const ltb_scratch* s, const void** out4) {
  out4[0] = s->xhat;
  out4[1] = s->dhat;
  out4[2] = s->partials;
  out4[3] = s->tickets;
  return !s->timing;
}
ltb_status fm_from_host(const ltb_plan* p, ltb_scratch* s, const double* in_host, double* d_dev) {
  if (!p || !s || s->plan != p) return fail(LTB_INVALID, "apply: scratch was created for another plan");
  return fm_host_enqueue(p, s, in_host, d_dev);
}
ltb_status fstar_to_host(const ltb_plan* p, ltb_scratch* s, const double* d_dev, double* m_host) {
  if (!p || !s || s->plan != p) return fail(LTB_INVALID, "apply: scratch was created for another plan");
  ltb_status st = ensure_stage(s, (size_t)std::max(p->cols, p->rows) * p->nt,
                               (size_t)std::max(p->cols, p->rows) * p->nt);
  if (st != LTB_OK) return st;
  return adjoint_to_host(p, s, d_dev, s->stage_out, m_host);
}
double* scratch_stage_in(ltb_scratch* s, size_t n) {
  return ensure_stage(s, n, s->stage_out_n) == LTB_OK ? s->stage_in : nullptr;
}
double* scratch_stage_out(ltb_scratch* s, size_t n) {
  return ensure_stage(s, s->stage_in_n, n) == LTB_OK ? s->stage_out : nullptr;
}
int scratch_device(const ltb_scratch* s) { return s->device; }
int plan_device(const ltb_plan* p) { return p->device; }
void plan_dims(const ltb_plan* p, int* rows, int* cols, int* nt) {
  *rows = p->rows;
  *cols = p->cols;
  *nt = p->nt;
}
void count_launches(uint64_t n) { g_launches += n; }
}  // namespace ltb_internal

// ---- dense_apply (fft_matvec.cpp:267-315): FFT-free time-domain product ----
namespace {
// forward: out[r][j] = sum_c sum_{l<=j} k[r][c][l] m[c][j-l]
// adjoint: out[c][j] = sum_r sum_{l<nt-j} k[r][c][l] d[r][j+l]
__global__ void dense_apply_kernel(const double* __restrict__ k, int rows, int cols, int nt,
                                   const double* __restrict__ v, int adjoint,
                                   double* __restrict__ out) {
  const long long total = (long long)(adjoint ? cols : rows) * nt;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(o / nt), j = (int)(o % nt);
    double acc = 0.0;
    if (!adjoint) {
      for (int c = 0; c < cols; ++c) {
        const double* kr = k + ((size_t)row * cols + c) * nt;
        const double* mc = v + (size_t)c * nt;
        for (int l = 0; l <= j; ++l) acc = fma(kr[l], mc[j - l], acc);
      }
    } else {
      for (int r = 0; r < rows; ++r) {
        const double* kr = k + ((size_t)r * cols + row) * nt;
        const double* dr = v + (size_t)r * nt;
        for (int l = 0; l + j < nt; ++l) acc = fma(kr[l], dr[j + l], acc);
      }
    }
    out[o] = acc;
  }
}
}  // namespace

extern "C" ltb_status ltb_dense_apply(const double* kernel, int rows, int cols, int nt,
                                      const double* v, int adjoint, unsigned long long cap,
                                      double* out, int ptr_kind) {
  if (!kernel || !v || !out) return fail(LTB_INVALID, "dense_apply: null argument");
  if (rows < 1 || cols < 1 || nt < 1)
    return fail(LTB_DIMENSION, "dense_apply: kernel tensor size does not match dims");
  const unsigned long long implied =
      (unsigned long long)rows * nt * (unsigned long long)cols * nt * 8ull;
  if (cap != 0 && implied > cap)
    return fail(LTB_CAPACITY, "dense_apply: implied dense operator needs %llu bytes, above the cap of %llu",
                implied, cap);
  const size_t nk = (size_t)rows * cols * nt;
  const size_t nin = (size_t)(adjoint ? rows : cols) * nt, nout = (size_t)(adjoint ? cols : rows) * nt;
  const double *dk = kernel, *dv = v;
  double* dout = out;
  double *tk = nullptr, *tv = nullptr, *to = nullptr;
  auto done = [&](ltb_status s_) {
    cudaFree(tk);
    cudaFree(tv);
    cudaFree(to);
    return s_;
  };
  if (ptr_kind == LTB_PTR_HOST) {
    if (cudaMalloc(&tk, nk * 8) != cudaSuccess || cudaMalloc(&tv, nin * 8) != cudaSuccess ||
        cudaMalloc(&to, nout * 8) != cudaSuccess ||
        cudaMemcpy(tk, kernel, nk * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(tv, v, nin * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return done(fail(LTB_CUDA, "dense_apply: staging failed"));
    dk = tk;
    dv = tv;
    dout = to;
  }
  const long long blocks = std::min<long long>(((long long)nout + 255) / 256, 148 * 16);
  dense_apply_kernel<<<(unsigned)blocks, 256>>>(dk, rows, cols, nt, dv, adjoint, dout);
  g_launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ptr_kind == LTB_PTR_HOST) e = cudaMemcpy(out, to, nout * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return done(fail(LTB_CUDA, "dense_apply: %s", cudaGetErrorString(e)));
  return done(LTB_OK);
}

// ---------------------------------------------------------------------------
// Device plan build from kernel slabs: the prior premultiply that turns F
// into G* (prior.cpp:108-134) and the BTPZ1 kernel-archive loader
// (io.cpp:71-100).  Kernel rows [r0, r0+R) are one contiguous slab
// [R][cols][nt] of the kernel tensor (in the archive too), so plans of any
// size are built slab by slab without holding the time-domain kernel.
// ---------------------------------------------------------------------------
namespace {

// Cholesky of A_x = delta I - gamma L, L the Neumann Laplacian
// (prior.cpp:9-39); SPD tridiagonal: diagonal ldiag, sub-diagonal lsub
ltb_status prior_factor(int n, double h_x, double gamma, double delta, std::vector<double>& ldiag,
                        std::vector<double>& lsub) {
  if (n < 1) return fail(LTB_CONFIG, "prior: n_space must be >= 1");
  if (!(h_x > 0)) return fail(LTB_CONFIG, "prior: h_x must be positive");
  if (!(delta > 0)) return fail(LTB_CONFIG, "prior: delta must be positive");
  if (gamma < 0) return fail(LTB_CONFIG, "prior: gamma must be >= 0");
  const double w = gamma / (h_x * h_x);
  ldiag.assign(n, 0.0);
  lsub.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double diag = delta;
    if (i > 0) diag += w;
    if (i + 1 < n) diag += w;
    if (i > 0) {
      lsub[i] = -w / ldiag[i - 1];
      diag -= lsub[i] * lsub[i];
    }
    if (!(diag > 0)) return fail(LTB_NUMERICAL, "prior: factorization of A_x failed");
    ldiag[i] = std::sqrt(diag);
  }
  return LTB_OK;
}

// Gamma_x = A_x^{-2} applied along the column (space) axis of every
// (row, lag) line of a slab [R][nm][nt]: thread per line, two forward /
// backward substitution pairs; consecutive threads are consecutive lags, so
// every step of the recurrence is one coalesced row of the slab.  The loads
// of 8 steps are issued together (they do not depend on the recurrence) and
// the diagonal enters as a reciprocal, so the dependent chain per step is
// one FMA and one multiply instead of a memory round trip and a division.
constexpr int kPreBatch = 8;
__global__ void prior_premultiply_kernel(double* __restrict__ slab, int R, int nm, int nt,
                                         const double* __restrict__ rdiag,
                                         const double* __restrict__ lsub) {
  const long long lines = (long long)R * nt;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < lines;
       t += (long long)gridDim.x * blockDim.x) {
    const long long rr = t / nt, k = t - rr * nt;
    double* x = slab + rr * (long long)nm * nt + k;
    for (int pass = 0; pass < 2; ++pass) {
      double prev = 0.0;
      for (int i0 = 0; i0 < nm; i0 += kPreBatch) {
        double v[kPreBatch], ls[kPreBatch], rd[kPreBatch];
#pragma unroll
        for (int q = 0; q < kPreBatch; ++q)
          if (i0 + q < nm) {
            v[q] = x[(size_t)(i0 + q) * nt];
            ls[q] = __ldg(lsub + i0 + q);
            rd[q] = __ldg(rdiag + i0 + q);
          }
#pragma unroll
        for (int q = 0; q < kPreBatch; ++q)
          if (i0 + q < nm) {
            const int i = i0 + q;
            prev = (i > 0 ? fma(-ls[q], prev, v[q]) : v[q]) * rd[q];
            x[(size_t)i * nt] = prev;
          }
      }
      double next = 0.0;
      for (int i1 = nm - 1; i1 >= 0; i1 -= kPreBatch) {
        double v[kPreBatch], ls[kPreBatch], rd[kPreBatch];
#pragma unroll
        for (int q = 0; q < kPreBatch; ++q)
          if (i1 - q >= 0) {
            const int i = i1 - q;
            v[q] = x[(size_t)i * nt];
            ls[q] = i + 1 < nm ? __ldg(lsub + i + 1) : 0.0;
            rd[q] = __ldg(rdiag + i);
          }
#pragma unroll
        for (int q = 0; q < kPreBatch; ++q)
          if (i1 - q >= 0) {
            const int i = i1 - q;
            next = (i + 1 < nm ? fma(-ls[q], next, v[q]) : v[q]) * rd[q];
            x[(size_t)i * nt] = next;
          }
      }
    }
  }
}

__global__ void count_nonfinite_slab(const double* x, long long n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) ++local;
  if (local) atomicAdd(bad, local);
}

// F-hat columns of kernel rows [r0, r0+R) from a device slab [R][cols][nt]
// slab: R kernel rows x src_cols columns (src_cols >= c0 + p->cols); the
// plan's columns are slab columns c0 ..
cudaError_t slab_to_fhat(ltb_plan* p, const double* slab, int r0, int R, long long src_cols, long long c0,
                         cudaStream_t st) {
  RfftSrc src{slab, 0, R, src_cols, c0};
  src.oP = R;           // logical row g = c R + rr ...
  src.oQ = p->rows;     // ... lands in F-hat column c rows + r0 + rr
  src.o0 = r0;
  return launch_rfft_rows(p->fft, src, p->nt, (long long)R * p->cols, p->fhat,
                          (long long)p->rows * p->cols, st);
}

struct PriorDev {
  double* ldiag = nullptr;
  double* lsub = nullptr;
  ~PriorDev() {
    cudaFree(ldiag);
    cudaFree(lsub);
  }
};

// Source of kernel slabs: host tensor, device tensor, generator, or archive.
struct SlabSource {
  int kind = 0;  // 0 host, 1 device, 2 generated, 3 file
  const double* ptr = nullptr;
  uint64_t key = 0;
  FILE* fh = nullptr;
  long long src_cols = 0;  // generated: columns of the whole kernel (0 = the plan's)
  long long c0 = 0;        // generated: first column of the plan (a column shard)
};

// Build p->fhat slab by slab, optionally premultiplying by Gamma_x first.
ltb_status build_plan_slabs(ltb_plan* p, const SlabSource& src, const PriorDev* prior) {
  const long long src_cols = src.src_cols > 0 ? src.src_cols : p->cols;
  const size_t row_elems = (size_t)src_cols * p->nt;
  // up to 64 kernel rows / 1 GB per slab: the premultiply runs one thread per
  // (row, lag) line, so larger slabs keep more of the GPU busy
  int R = (int)std::max<size_t>(1, std::min<size_t>(64, (size_t)(1u << 30) / (row_elems * 8)));
  R = std::min(R, p->rows);
  double* slab = nullptr;
  unsigned long long* bad = nullptr;
  std::vector<double> host;
  auto done = [&](ltb_status s) {
    cudaFree(slab);
    cudaFree(bad);
    return s;
  };
  if (cudaMalloc(&slab, sizeof(double) * row_elems * R) != cudaSuccess ||
      cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess)
    return done(fail(LTB_CUDA, "plan build: slab alloc failed"));
  cudaMemset(bad, 0, sizeof(unsigned long long));
  if (src.kind == 3) host.resize(row_elems * R);
  for (int r0 = 0; r0 < p->rows; r0 += R) {
    const int rr = std::min(R, p->rows - r0);
    const size_t n = row_elems * rr;
    cudaError_t e = cudaSuccess;
    if (src.kind == 0) {
      e = cudaMemcpy(slab, src.ptr + (size_t)r0 * row_elems, sizeof(double) * n, cudaMemcpyHostToDevice);
    } else if (src.kind == 1) {
      e = cudaMemcpy(slab, src.ptr + (size_t)r0 * row_elems, sizeof(double) * n, cudaMemcpyDeviceToDevice);
    } else if (src.kind == 2) {
      e = launch_gen_fill(src.key, (uint64_t)r0 * row_elems, (long long)n, slab, 0);
      g_launches += 1;
    } else {
      if (fread(host.data(), sizeof(double), n, src.fh) != n)
        return done(fail(LTB_IO, "truncated archive while reading kernel data"));
      e = cudaMemcpy(slab, host.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) return done(fail(LTB_CUDA, "plan build: %s", cudaGetErrorString(e)));
    if (src.kind != 2) {  // core.cpp:73-77: reject non-finite kernel entries
      count_nonfinite_slab<<<148 * 4, 256>>>(slab, (long long)n, bad);
      g_launches += 1;
    }
    if (prior) {
      const long long lines = (long long)rr * p->nt;
      prior_premultiply_kernel<<<(unsigned)std::max(1ll, std::min(148ll * 16, (lines + 127) / 128)), 128>>>(
          slab, rr, (int)src_cols, p->nt, prior->ldiag, prior->lsub);
      g_launches += 1;
    }
    e = slab_to_fhat(p, slab, r0, rr, src_cols, src.c0, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return done(fail(LTB_CUDA, "plan build: %s", cudaGetErrorString(e)));
    g_launches += 1;
  }
  unsigned long long hb = 0;
  cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
  if (hb) return done(fail(LTB_NUMERICAL, "MatvecPlan: non-finite kernel entry"));
  return done(LTB_OK);
}

ltb_status make_prior(int nm, double h_x, double gamma, double delta, PriorDev& d) {
  std::vector<double> ld, ls;
  ltb_status st = prior_factor(nm, h_x, gamma, delta, ld, ls);
  if (st != LTB_OK) return st;
  LTB_CUDA_TRY(cudaMalloc(&d.ldiag, sizeof(double) * nm));
  LTB_CUDA_TRY(cudaMalloc(&d.lsub, sizeof(double) * nm));
  for (double& v : ld) v = 1.0 / v;  // the kernel multiplies by the reciprocal diagonal
  LTB_CUDA_TRY(cudaMemcpy(d.ldiag, ld.data(), sizeof(double) * nm, cudaMemcpyHostToDevice));
  LTB_CUDA_TRY(cudaMemcpy(d.lsub, ls.data(), sizeof(double) * nm, cudaMemcpyHostToDevice));
  return LTB_OK;
}

// premultiply_kernel tag rule (prior.cpp:114-120)
ltb_status premultiplied_tag(int tag, int* out) {
  if (tag == LTB_TAG_F) *out = LTB_TAG_GSTAR;
  else if (tag == LTB_TAG_FQ) *out = LTB_TAG_GQSTAR;
  else return fail(LTB_CONFIG, "premultiply_kernel: kernel already premultiplied");
  return LTB_OK;
}

ltb_status plan_from_source(int rows, int cols, int nt, int tag, const SlabSource& src,
                            const double* prior3, const ltb_opts* opts, ltb_plan** out) {
  *out = nullptr;
  int ptag = tag;
  if (prior3) {
    ltb_status st = premultiplied_tag(tag, &ptag);
    if (st != LTB_OK) return st;
  }
  ltb_plan* p = new ltb_plan();
  ltb_status st = plan_init(p, rows, cols, nt, ptag, opts);
  if (st != LTB_OK) {
    plan_free(p);
    return st;
  }
  DeviceGuard g(p->device);
  PriorDev prior;
  const int prior_cols = src.src_cols > 0 ? (int)src.src_cols : cols;
  if (prior3 && (st = make_prior(prior_cols, prior3[0], prior3[1], prior3[2], prior)) != LTB_OK) {
    plan_free(p);
    return st;
  }
  st = build_plan_slabs(p, src, prior3 ? &prior : nullptr);
  if (st != LTB_OK) {
    plan_free(p);
    return st;
  }
  *out = p;
  return LTB_OK;
}

}  // namespace

namespace ltb_internal {
// Gamma_x premultiply of a whole device kernel [rows][cols][nt] in place
// (form_K's G kernel, bayes_engine.cpp:105)
ltb_status premultiply_device(double* kernel, int rows, int cols, int nt, double h_x, double gamma,
                              double delta) {
  PriorDev prior;
  ltb_status st = make_prior(cols, h_x, gamma, delta, prior);
  if (st != LTB_OK) return st;
  const long long lines = (long long)rows * nt;
  prior_premultiply_kernel<<<(unsigned)std::max(1ll, std::min(148ll * 16, (lines + 127) / 128)), 128>>>(
      kernel, rows, cols, nt, prior.ldiag, prior.lsub);
  g_launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(LTB_CUDA, "premultiply: %s", cudaGetErrorString(e));
  return LTB_OK;
}
// non-finite scan of a device array (core.cpp:73-77)
ltb_status check_finite_device(const double* x, long long n, const char* what) {
  unsigned long long* bad = nullptr;
  if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess) return fail(LTB_CUDA, "finite scan: alloc");
  cudaMemset(bad, 0, sizeof(unsigned long long));
  count_nonfinite_slab<<<148 * 4, 256>>>(x, n, bad);
  g_launches += 1;
  unsigned long long hb = 0;
  cudaError_t e = cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  if (e != cudaSuccess) return fail(LTB_CUDA, "finite scan: %s", cudaGetErrorString(e));
  if (hb) return fail(LTB_NUMERICAL, "%s: non-finite kernel entry", what);
  return LTB_OK;
}
}  // namespace ltb_internal

extern "C" {

ltb_status ltb_plan_create_premultiplied(const double* kernel, int rows, int cols, int nt, int tag,
                                         int ptr_kind, double h_x, double gamma, double delta,
                                         const ltb_opts* opts, ltb_plan** out) {
  if (!out || !kernel) return fail(LTB_INVALID, "plan_create_premultiplied: null argument");
  if (rows < 1 || cols < 1 || nt < 1)
    return fail(LTB_DIMENSION, "premultiply_kernel: kernel tensor size does not match dims");
  SlabSource src;
  src.kind = ptr_kind == LTB_PTR_DEVICE ? 1 : 0;
  src.ptr = kernel;
  const double prior[3] = {h_x, gamma, delta};
  return plan_from_source(rows, cols, nt, tag, src, prior, opts, out);
}

ltb_status ltb_plan_create_generated_premultiplied(int rows, int cols, int nt, int tag,
                                                   uint64_t seed, uint64_t stream, double h_x,
                                                   double gamma, double delta, const ltb_opts* opts,
                                                   ltb_plan** out) {
  if (!out) return fail(LTB_INVALID, "plan_create_generated_premultiplied: null out");
  SlabSource src;
  src.kind = 2;
  src.key = gen_key(seed, stream);
  const double prior[3] = {h_x, gamma, delta};
  return plan_from_source(rows, cols, nt, tag, src, prior, opts, out);
}

ltb_status ltb_plan_create_generated_premultiplied_shard(int rows, int cols, int nt, int tag, uint64_t seed,
                                                         uint64_t stream, long long nm_total, long long c0,
                                                         double h_x, double gamma, double delta,
                                                         const ltb_opts* opts, ltb_plan** out) {
  if (!out) return fail(LTB_INVALID, "plan_create_generated_premultiplied_shard: null out");
  *out = nullptr;
  if (c0 < 0 || nm_total < c0 + cols)
    return fail(LTB_DIMENSION, "generated plan: shard [%lld, %lld) outside nm_total=%lld", c0, c0 + cols, nm_total);
  SlabSource src;
  src.kind = 2;
  src.key = gen_key(seed, stream);
  src.src_cols = nm_total;
  src.c0 = c0;
  const double prior[3] = {h_x, gamma, delta};
  return plan_from_source(rows, cols, nt, tag, src, prior, opts, out);
}

// BTPZ1 (io.cpp:71-100): "BTPZ1", u64 rows, cols, N_t, tag, then the
// [row][col][lag] doubles (little endian)
ltb_status ltb_plan_load_btpz(const char* path, const double* prior3, const ltb_opts* opts,
                              ltb_plan** out) {
  if (!out || !path) return fail(LTB_INVALID, "plan_load_btpz: null argument");
  *out = nullptr;
  FILE* fh = fopen(path, "rb");
  if (!fh) return fail(LTB_IO, "cannot open kernel archive %s", path);
  char magic[5];
  uint64_t hdr[4];
  ltb_status st = LTB_OK;
  if (fread(magic, 1, 5, fh) != 5 || memcmp(magic, "BTPZ1", 5) != 0) {
    st = fail(LTB_IO, "bad magic in %s (expected BTPZ1)", path);
  } else if (fread(hdr, sizeof(uint64_t), 4, fh) != 4) {
    st = fail(LTB_IO, "truncated archive while reading header of %s", path);
  } else if (hdr[0] == 0 || hdr[1] == 0 || hdr[2] == 0 || hdr[3] > 3 ||
             hdr[0] * hdr[1] * hdr[2] > (1ull << 40) || hdr[0] > INT32_MAX || hdr[1] > INT32_MAX ||
             hdr[2] > INT32_MAX) {
    st = fail(LTB_IO, "implausible kernel header in %s", path);
  } else {
    SlabSource src;
    src.kind = 3;
    src.fh = fh;
    st = plan_from_source((int)hdr[0], (int)hdr[1], (int)hdr[2], (int)hdr[3], src, prior3, opts, out);
  }
  fclose(fh);
  return st;
}

}  // extern "C"
