// fft_matvec_b200.cpp -- drop-in replacement for the reference's
// proj/src/fft_matvec.cpp: implements ltibayes::MatvecPlan and dense_apply
// exactly as declared in the UNCHANGED reference header
// proj/include/ltibayes/fft_matvec.hpp, on top of the C ABI in include/ltb.h
// (libltb.so, sm_100a).  A maintainer swaps this file for fft_matvec.cpp in
// proj/CMakeLists.txt and links libltb.so; every caller (InferenceEngine,
// workflow, tests) keeps working and runs its matvecs on the B200.
//
// Semantics kept from the reference:
//   * ctor: kernel.check_consistent (core.cpp:67-78: DimensionError,
//     NumericalError on non-finite entries), plan immutable afterwards
//     (fft_matvec.cpp:73-111);
//   * apply_raw / apply_adjoint_raw take HOST pointers and return with the
//     result in place (:139-217); one Scratch per concurrent caller (:26-28)
//     -- here a Scratch owns a CUDA stream and device workspace;
//   * apply / apply_adjoint check the SpaceMajorRows contract and dims
//     (:221-265), throwing LayoutError / DimensionError;
//   * kernel_hat_sqnorm (:124-137); dense_apply with CapacityError (:267-315).
// CUDA failures surface as NumericalError with the driver's message (the
// reference taxonomy has no device errors).
//
// Multi-GPU: with LTB_DEVICES=0,1,... (two or more ordinals, repeats allowed)
// every plan is built sharded over those GPUs by column ranges
// (ltb_plan_create_sharded: F m sums the shards' partial outputs on the
// first device over NVLink, F* d hands d to every shard) -- same interface,
// same results to rounding, so the engine's four plans (bayes_engine.cpp:
// 110-113) and every other caller shard without a code change.
#include "ltibayes/fft_matvec.hpp"

#include <cstdlib>
#include <string>
#include <vector>

#include "ltb.h"

namespace ltibayes {

namespace {

[[noreturn]] void raise_status(ltb_status st, const char* where) {
  const std::string msg = std::string(where) + ": " + ltb_last_error();
  switch (st) {
    case LTB_DIMENSION: throw DimensionError(msg);
    case LTB_LAYOUT: throw LayoutError(msg);
    case LTB_CAPACITY: throw CapacityError(msg);
    case LTB_STATE: throw StateError(msg);
    default: throw NumericalError(msg);
  }
}

inline void check(ltb_status st, const char* where) {
  if (st != LTB_OK) raise_status(st, where);
}

// LTB_DEVICES="0,1,2,3" -> {0,1,2,3}; fewer than two entries: single device
std::vector<int> shard_devices() {
  std::vector<int> devs;
  const char* env = std::getenv("LTB_DEVICES");
  if (!env) return devs;
  std::string s(env);
  size_t pos = 0;
  while (pos < s.size()) {
    const size_t end = s.find(',', pos);
    const std::string tok = s.substr(pos, end == std::string::npos ? std::string::npos : end - pos);
    if (!tok.empty()) devs.push_back(std::stoi(tok));
    if (end == std::string::npos) break;
    pos = end + 1;
  }
  if (devs.size() < 2) devs.clear();
  return devs;
}

void check_series(const BlockSeries& v, const char* what) {
  v.check_consistent(what);
  if (v.layout != Layout::SpaceMajorRows) {
    throw LayoutError(std::string(what) + ": requires SpaceMajorRows input, got " +
                      layout_name(v.layout) + " (no silent reindex)");
  }
}

}  // namespace

struct MatvecPlan::Impl {
  ltb_plan* plan = nullptr;      // single device
  ltb_splan* splan = nullptr;    // sharded over LTB_DEVICES
  int rows = 0, cols = 0, nt = 0;
  KernelTag tag = KernelTag::F;
  ~Impl() {
    if (plan) ltb_plan_destroy(plan);
    if (splan) ltb_splan_destroy(splan);
  }
};

struct MatvecPlan::Scratch::Impl {
  ltb_scratch* s = nullptr;
  ltb_sscratch* ss = nullptr;
  ~Impl() {
    if (s) ltb_scratch_destroy(s);
    if (ss) ltb_sscratch_destroy(ss);
  }
};

MatvecPlan::Scratch::Scratch(const MatvecPlan& plan) : impl_(std::make_unique<Impl>()) {
  if (plan.impl_->splan)
    check(ltb_sscratch_create(plan.impl_->splan, nullptr, &impl_->ss), "MatvecPlan::Scratch");
  else
    check(ltb_scratch_create(plan.impl_->plan, nullptr, &impl_->s), "MatvecPlan::Scratch");
}
MatvecPlan::Scratch::~Scratch() = default;
MatvecPlan::Scratch::Scratch(Scratch&&) noexcept = default;

MatvecPlan::MatvecPlan(const BlockToeplitzKernel& kernel) : impl_(std::make_unique<Impl>()) {
  kernel.check_consistent("MatvecPlan");
  const std::vector<int> devs = shard_devices();
  if (!devs.empty() && kernel.n_cols >= static_cast<int>(devs.size()))
    check(ltb_plan_create_sharded(kernel.data.data(), kernel.rows_out, kernel.n_cols, kernel.n_time,
                                  static_cast<int>(kernel.tag), static_cast<int>(devs.size()), devs.data(),
                                  nullptr, &impl_->splan),
          "MatvecPlan");
  else
    check(ltb_plan_create(kernel.data.data(), kernel.rows_out, kernel.n_cols, kernel.n_time,
                          static_cast<int>(kernel.tag), LTB_PTR_HOST, nullptr, &impl_->plan),
          "MatvecPlan");
  impl_->rows = kernel.rows_out;
  impl_->cols = kernel.n_cols;
  impl_->nt = kernel.n_time;
  impl_->tag = kernel.tag;
}

MatvecPlan::~MatvecPlan() = default;
MatvecPlan::MatvecPlan(MatvecPlan&&) noexcept = default;
MatvecPlan& MatvecPlan::operator=(MatvecPlan&&) noexcept = default;

int MatvecPlan::rows_out() const { return impl_->rows; }
int MatvecPlan::n_cols() const { return impl_->cols; }
int MatvecPlan::n_time() const { return impl_->nt; }
int MatvecPlan::padded_len() const { return 2 * impl_->nt; }
int MatvecPlan::n_freq() const { return impl_->nt + 1; }
KernelTag MatvecPlan::tag() const { return impl_->tag; }

double MatvecPlan::kernel_hat_sqnorm() const {
  double out = 0;
  if (impl_->splan)
    check(ltb_splan_kernel_hat_sqnorm(impl_->splan, &out), "MatvecPlan::kernel_hat_sqnorm");
  else
    check(ltb_kernel_hat_sqnorm(impl_->plan, &out), "MatvecPlan::kernel_hat_sqnorm");
  return out;
}

void MatvecPlan::apply_raw(const double* in, double* out, Scratch& scratch) const {
  if (impl_->splan)
    check(ltb_apply_sharded(impl_->splan, scratch.impl_->ss, in, out, LTB_PTR_HOST), "MatvecPlan::apply_raw");
  else
    check(ltb_apply(impl_->plan, scratch.impl_->s, in, out, LTB_PTR_HOST), "MatvecPlan::apply_raw");
}

void MatvecPlan::apply_adjoint_raw(const double* in, double* out, Scratch& scratch) const {
  if (impl_->splan)
    check(ltb_apply_adjoint_sharded(impl_->splan, scratch.impl_->ss, in, out, LTB_PTR_HOST),
          "MatvecPlan::apply_adjoint_raw");
  else
    check(ltb_apply_adjoint(impl_->plan, scratch.impl_->s, in, out, LTB_PTR_HOST),
          "MatvecPlan::apply_adjoint_raw");
}

ObsSeries MatvecPlan::apply(const SpaceTimeField& m) const {
  Scratch s(*this);
  return apply(m, s);
}

ObsSeries MatvecPlan::apply(const SpaceTimeField& m, Scratch& scratch) const {
  check_series(m, "MatvecPlan::apply");
  if (m.n_rows != n_cols() || m.n_time != n_time()) {
    throw DimensionError("MatvecPlan::apply: input dims (" + std::to_string(m.n_rows) + "," +
                         std::to_string(m.n_time) + ") do not match kernel (" +
                         std::to_string(n_cols()) + "," + std::to_string(n_time()) + ")");
  }
  ObsSeries d(rows_out(), n_time(), Layout::SpaceMajorRows);
  apply_raw(m.values.data(), d.values.data(), scratch);
  return d;
}

SpaceTimeField MatvecPlan::apply_adjoint(const ObsSeries& d) const {
  Scratch s(*this);
  return apply_adjoint(d, s);
}

SpaceTimeField MatvecPlan::apply_adjoint(const ObsSeries& d, Scratch& scratch) const {
  check_series(d, "MatvecPlan::apply_adjoint");
  if (d.n_rows != rows_out() || d.n_time != n_time()) {
    throw DimensionError("MatvecPlan::apply_adjoint: input dims do not match");
  }
  SpaceTimeField m(n_cols(), n_time(), Layout::SpaceMajorRows);
  apply_adjoint_raw(d.values.data(), m.values.data(), scratch);
  return m;
}

std::vector<double> dense_apply(const BlockToeplitzKernel& kernel, const std::vector<double>& v,
                                bool adjoint, uint64_t mem_cap_bytes) {
  kernel.check_consistent("dense_apply");
  const uint64_t implied = static_cast<uint64_t>(kernel.rows_out) * kernel.n_time *
                           kernel.n_cols * kernel.n_time * 8;
  if (mem_cap_bytes != 0 && implied > mem_cap_bytes) {
    throw CapacityError("dense_apply: implied dense operator needs " + std::to_string(implied) +
                        " bytes, above the cap of " + std::to_string(mem_cap_bytes));
  }
  const size_t in_len =
      static_cast<size_t>(adjoint ? kernel.rows_out : kernel.n_cols) * kernel.n_time;
  if (v.size() != in_len) {
    throw DimensionError("dense_apply: input length " + std::to_string(v.size()) +
                         ", expected " + std::to_string(in_len));
  }
  std::vector<double> out(
      static_cast<size_t>(adjoint ? kernel.n_cols : kernel.rows_out) * kernel.n_time);
  check(ltb_dense_apply(kernel.data.data(), kernel.rows_out, kernel.n_cols, kernel.n_time,
                        v.data(), adjoint ? 1 : 0, mem_cap_bytes, out.data(), LTB_PTR_HOST),
        "dense_apply");
  return out;
}

}  // namespace ltibayes
