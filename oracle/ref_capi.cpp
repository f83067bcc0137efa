// ref_capi.cpp -- C entry points over the reference's OWN MatvecPlan and
// dense_apply, compiled verbatim from /root/reference/proj/src/{fft_matvec,
// core}.cpp against oracle/shim (TEST INFRASTRUCTURE ONLY).  Loaded by the
// tests (golden-vector generation, oracle pinning) and by bench.py's
// cpu_baseline / --impl reference legs.  Never part of the product path.
//
// Exceptions of the reference taxonomy (core.hpp:12-35) map to the status
// codes of include/ltb.h.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ltibayes/fft_matvec.hpp"
#include "ltb_oracle.h"

using namespace ltibayes;

namespace {
thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 1;
  } catch (const LayoutError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 4;
  } catch (const StateError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

BlockToeplitzKernel make_kernel(const double* k, int rows, int cols, int nt, int tag) {
  BlockToeplitzKernel kern(rows, cols, nt, static_cast<KernelTag>(tag));
  std::memcpy(kern.data.data(), k, sizeof(double) * kern.data.size());
  return kern;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan_create(const double* kernel, int rows, int cols, int nt, int tag, void** out) {
  *out = nullptr;
  try {
    // BlockToeplitzKernel's ctor sizes data from the dims; reject negatives
    // before allocation the way check_consistent would.
    if (rows < 1 || cols < 1 || nt < 1) throw DimensionError("ref_plan_create: dims must be >= 1");
    auto* p = new MatvecPlan(make_kernel(kernel, rows, cols, nt, tag));
    *out = p;
    return 0;
  } catch (...) {
    return map_exc();
  }
}

void ref_plan_destroy(void* p) { delete static_cast<MatvecPlan*>(p); }

void ref_plan_dims(void* h, int* rows, int* cols, int* nt, int* npad, int* nf) {
  auto* p = static_cast<MatvecPlan*>(h);
  *rows = p->rows_out();
  *cols = p->n_cols();
  *nt = p->n_time();
  *npad = p->padded_len();
  *nf = p->n_freq();
}

int ref_apply_raw(void* h, const double* in, double* out) {
  try {
    auto* p = static_cast<MatvecPlan*>(h);
    MatvecPlan::Scratch s(*p);
    p->apply_raw(in, out, s);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_apply_adjoint_raw(void* h, const double* in, double* out) {
  try {
    auto* p = static_cast<MatvecPlan*>(h);
    MatvecPlan::Scratch s(*p);
    p->apply_adjoint_raw(in, out, s);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// Typed path (fft_matvec.cpp:232-265): layout 0 = TimeMajorBlocks,
// 1 = SpaceMajorRows, exactly as ltibayes::Layout.
int ref_apply(void* h, const double* in, int n_rows, int n_time, int layout, int adjoint,
              double* out) {
  try {
    auto* p = static_cast<MatvecPlan*>(h);
    if (!adjoint) {
      SpaceTimeField m(n_rows, n_time, static_cast<Layout>(layout));
      std::memcpy(m.values.data(), in, sizeof(double) * m.values.size());
      const ObsSeries d = p->apply(m);
      std::memcpy(out, d.values.data(), sizeof(double) * d.values.size());
    } else {
      ObsSeries d(n_rows, n_time, static_cast<Layout>(layout));
      std::memcpy(d.values.data(), in, sizeof(double) * d.values.size());
      const SpaceTimeField m = p->apply_adjoint(d);
      std::memcpy(out, m.values.data(), sizeof(double) * m.values.size());
    }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

double ref_kernel_hat_sqnorm(void* h) { return static_cast<MatvecPlan*>(h)->kernel_hat_sqnorm(); }

int ref_dense_apply(const double* kernel, int rows, int cols, int nt, const double* v,
                    size_t v_len, int adjoint, unsigned long long cap, double* out) {
  try {
    if (rows < 1 || cols < 1 || nt < 1) throw DimensionError("ref_dense_apply: dims must be >= 1");
    const auto k = make_kernel(kernel, rows, cols, nt, 0);
    std::vector<double> vin(v, v + v_len);
    const auto r = dense_apply(k, vin, adjoint != 0, cap);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// Host CPU baseline: the reference apply_raw / apply_adjoint_raw on a sample
// of `nm_sample` generated columns (orc_gen_kernel, same generator and seed
// as the GPU plan), split into `threads` contiguous column shards, one
// MatvecPlan + Scratch per thread (the SURVEY section 8d recipe; the
// reference itself is single-threaded, fft_matvec.cpp has no parallel_for).
// F m sums the shard outputs; F* d is exact per shard.  Reports the median
// over `reps` of the wall time of the slowest thread.
int ref_bench(int rows, int nm_total, int nm_sample, int nt, unsigned long long seed,
              int threads, int reps, double* t_build, double* t_apply, double* t_adjoint) {
  try {
    threads = std::max(1, std::min(threads, nm_sample));
    std::vector<std::unique_ptr<MatvecPlan>> plans(threads);
    std::vector<int> c0(threads + 1);
    for (int t = 0; t <= threads; ++t) c0[t] = static_cast<int>((long long)nm_sample * t / threads);
    const double tb = now();
    {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
          const int cols = c0[t + 1] - c0[t];
          BlockToeplitzKernel k(rows, cols, nt, KernelTag::F);
          orc_gen_kernel(seed, 1, rows, nm_total, c0[t], cols, nt, k.data.data());
          plans[t] = std::make_unique<MatvecPlan>(k);
        });
      }
      for (auto& th : pool) th.join();
    }
    *t_build = now() - tb;
    std::vector<double> m(static_cast<size_t>(nm_sample) * nt), d(static_cast<size_t>(rows) * nt);
    orc_gen_fill(seed, 10, 0, m.size(), m.data());
    orc_gen_fill(seed, 11, 0, d.size(), d.data());
    std::vector<std::vector<double>> outs(threads, std::vector<double>(d.size()));
    std::vector<double> madj(m.size());
    auto run = [&](bool adjoint) {
      std::vector<double> times;
      for (int rep = 0; rep < reps; ++rep) {
        std::atomic<int> ready{0};
        std::vector<std::thread> pool;
        const double t0 = now();
        for (int t = 0; t < threads; ++t) {
          pool.emplace_back([&, t] {
            MatvecPlan::Scratch s(*plans[t]);
            ready.fetch_add(1);
            if (!adjoint) {
              plans[t]->apply_raw(m.data() + static_cast<size_t>(c0[t]) * nt, outs[t].data(), s);
            } else {
              plans[t]->apply_adjoint_raw(d.data(), madj.data() + static_cast<size_t>(c0[t]) * nt, s);
            }
          });
        }
        for (auto& th : pool) th.join();
        if (!adjoint) {  // F m = sum of shard outputs
          for (int t = 1; t < threads; ++t)
            for (size_t i = 0; i < d.size(); ++i) outs[0][i] += outs[t][i];
        }
        times.push_back(now() - t0);
      }
      std::sort(times.begin(), times.end());
      return times[times.size() / 2];
    };
    *t_apply = run(false);
    *t_adjoint = run(true);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

}  // extern "C"
