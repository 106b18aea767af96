// als_gpu.cpp — drop-in replacement for the reference's core/src/als.cpp: every
// function declared in cpd/als.hpp (unchanged header) over the C-ABI of
// libcpdgpu.so.  The sweeps, the pseudo-inverse and run() execute on the B200
// (the whole Gauss-Seidel sweep is one device graph); random_init and
// rebalance_columns are host helpers as in the reference.  Semantics, errors
// and traces follow als.cpp:15-212.
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "cpd/als.hpp"
#include "cpd/errors.hpp"
#include "gpu_context.hpp"

namespace cpd {
namespace {

void check_mode(int n, std::size_t count, const char* who) {
  if (n < 1 || n > static_cast<int>(count))
    throw IndexError(std::string(who) + ": mode " + std::to_string(n) + " outside 1.." + std::to_string(count));
}

void check_factors_match(const DenseTensor& y, const FactorList& factors, const char* who) {
  if (factor_shape(factors) != y.shape())
    throw ShapeError(std::string(who) + ": factor row counts do not match the tensor");
}

}  // namespace

Eigen::MatrixXd pinv_psd(const Eigen::MatrixXd& s, double rtol) {
  if (s.rows() != s.cols()) throw ShapeError("pinv_psd: matrix must be square");
  if (rtol < 0.0) throw ArgumentError("pinv_psd: rtol must be nonnegative");
  auto& ctx = gpu::context();
  Eigen::MatrixXd out(s.rows(), s.cols());
  ctx.check(cpdgpu_pinv_psd(ctx.h, s.rows(), s.data(), rtol, out.data()));
  return out;
}

Eigen::MatrixXd als_update_mode(const Eigen::MatrixXd& m, const FactorList& factors, int n, double pinv_rtol) {
  check_mode(n, factors.size(), "als_update_mode");
  if (!m.allFinite()) throw NumericError("als_update_mode: non-finite gradient input");
  const Shape s = factor_shape(factors);
  const index_t R = factor_rank(factors);
  if (m.rows() != s.dim(n) || m.cols() != R) throw ShapeError("als_update_mode: mttkrp matrix has the wrong size");
  auto& ctx = gpu::context();
  const auto fp = gpu::cptrs(factors);
  const auto d = gpu::dims64(s);
  Eigen::MatrixXd out(m.rows(), m.cols());
  ctx.check(cpdgpu_als_update_mode(ctx.h, s.order(), d.data(), R, m.data(), fp.data(), n, pinv_rtol, out.data()));
  return out;
}

void als_sweep_direct(const DenseTensor& y, FactorList& factors, const std::vector<int>& order, double pinv_rtol,
                      CostCounter* counter) {
  for (int n : order) check_mode(n, factors.size(), "als_sweep_direct");
  check_factors_match(y, factors, "als_sweep_direct");
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  auto fp = gpu::ptrs(factors);
  uint64_t mults = 0;
  ctx.check(cpdgpu_als_sweep_direct(ctx.h, t.get(), factor_rank(factors), fp.data(), order.data(),
                                    static_cast<int>(order.size()), pinv_rtol, &mults));
  if (counter) counter->charge(mults);
}

void als_sweep_fast(const DenseTensor& y, FactorList& factors, double pinv_rtol, CostCounter* counter,
                    FastStats* stats) {
  if (y.order() < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  check_factors_match(y, factors, "cp_gradient_all");
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  auto fp = gpu::ptrs(factors);
  uint64_t mults = 0;
  int64_t peak = 0;
  ctx.check(cpdgpu_als_sweep(ctx.h, t.get(), factor_rank(factors), fp.data(), pinv_rtol, nullptr, &mults));
  if (counter) counter->charge(mults);
  if (stats) {  // the sweep's gradient workspace, as the reference reports it (see cp_gradient_all)
    std::vector<int64_t> d = gpu::dims64(y.shape());
    std::vector<int> perm(d.size()), inv(d.size());
    cpdgpu_sort_modes(static_cast<int>(d.size()), d.data(), perm.data(), inv.data());
    std::vector<int64_t> sd;
    for (int p : perm) sd.push_back(d[static_cast<size_t>(p - 1)]);
    ctx.check(cpdgpu_reference_workspace(static_cast<int>(sd.size()), sd.data(), factor_rank(factors), &peak));
    stats->peak_workspace_doubles = peak;
  }
}

void mu_sweep(const DenseTensor& y, FactorList& factors, double eps, CostCounter* counter) {
  if (eps < 0.0) throw ArgumentError("mu_sweep: eps must be nonnegative");
  check_factors_match(y, factors, "mu_sweep");
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  auto fp = gpu::ptrs(factors);
  uint64_t mults = 0;
  ctx.check(cpdgpu_mu_sweep(ctx.h, t.get(), factor_rank(factors), fp.data(), eps, &mults));
  if (counter) counter->charge(mults);
}

void gd_step(const DenseTensor& y, FactorList& factors, double eta, CostCounter* counter) {
  if (!(eta >= 0.0)) throw ArgumentError("gd_step: eta must be nonnegative");
  check_factors_match(y, factors, "gd_step");
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  auto fp = gpu::ptrs(factors);
  uint64_t mults = 0;
  ctx.check(cpdgpu_gd_step(ctx.h, t.get(), factor_rank(factors), fp.data(), eta, &mults));
  if (counter) counter->charge(mults);
}

// Reporting helper (als.cpp:103-124), host-side: equal column norms across modes.
KruskalModel rebalance_columns(const KruskalModel& model) {
  FactorList f = model.factors();
  const int N = model.order();
  for (index_t r = 0; r < model.rank(); ++r) {
    double log_sum = 0.0;
    bool dead = false;
    for (int n = 0; n < N; ++n) {
      const double nr = f[static_cast<size_t>(n)].col(r).norm();
      if (nr == 0.0) dead = true;
      else log_sum += std::log(nr);
    }
    for (int n = 0; n < N; ++n) {
      auto col = f[static_cast<size_t>(n)].col(r);
      if (dead) col.setZero();
      else col *= std::exp(log_sum / N) / col.norm();
    }
  }
  return KruskalModel(std::move(f));
}

// Uniform01 (rng.hpp:16-26) stream, column-major per factor in mode order
// (als.cpp:127-139), drawn by cpdgpu_uniform01_fill (bit-identical).
KruskalModel random_init(const Shape& shape, index_t rank, std::uint64_t seed) {
  if (rank < 1) throw ArgumentError("random_init: rank must be positive");
  index_t total = 0;
  for (int n = 1; n <= shape.order(); ++n) total += shape.dim(n) * rank;
  std::vector<double> v(static_cast<size_t>(total));
  gpu::context().check(cpdgpu_uniform01_fill(seed, total, v.data()));
  FactorList f;
  index_t at = 0;
  for (int n = 1; n <= shape.order(); ++n) {
    Eigen::MatrixXd a(shape.dim(n), rank);
    std::copy(v.begin() + at, v.begin() + at + a.size(), a.data());
    at += a.size();
    f.push_back(std::move(a));
  }
  return KruskalModel(std::move(f));
}

std::vector<int> standard_order(int order) {
  std::vector<int> v(static_cast<size_t>(order));
  std::iota(v.begin(), v.end(), 1);
  return v;
}

// run (als.cpp:147-210): every Algorithm on the device, fit by the Gram identity.
SolveResult run(const DenseTensor& y, const KruskalModel& init, Algorithm algo, const SolveOptions& opts,
                CostCounter* counter) {
  if (opts.max_iters < 1) throw ArgumentError("run: max_iters must be at least 1");
  if (opts.tol < 0.0 || opts.pinv_rtol < 0.0 || opts.mu_eps < 0.0)
    throw ArgumentError("run: tolerances must be nonnegative");
  if (init.shape() != y.shape()) throw ShapeError("run: init factors do not match the tensor");
  FactorList f = init.factors();
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  auto fp = gpu::ptrs(f);
  const size_t n = static_cast<size_t>(opts.max_iters);
  RunTrace tr;
  tr.cost.resize(n);
  tr.rel_error.resize(n);
  tr.seconds.resize(n);
  tr.mults.resize(n);
  int iters = 0;
  const int code = algo == Algorithm::als_direct ? 0 : algo == Algorithm::als_fast ? 1 : algo == Algorithm::mu ? 2 : 3;
  ctx.check(cpdgpu_run_algo(ctx.h, t.get(), init.rank(), fp.data(), code, opts.order == UpdateOrder::pivot ? 1 : 0,
                            opts.max_iters, opts.tol, opts.pinv_rtol, opts.mu_eps, opts.gd_eta, tr.cost.data(),
                            tr.rel_error.data(), tr.seconds.data(), tr.mults.data(), &iters));
  tr.iters_run = iters;
  tr.cost.resize(static_cast<size_t>(iters));
  tr.rel_error.resize(static_cast<size_t>(iters));
  tr.seconds.resize(static_cast<size_t>(iters));
  tr.mults.resize(static_cast<size_t>(iters));
  const std::uint64_t base = counter ? counter->total() : 0;
  for (auto& m : tr.mults) m = counter ? base + m : 0;  // cumulative counter totals (als.cpp:185)
  if (counter && iters > 0) counter->charge(tr.mults.back() - base);
  return SolveResult{KruskalModel(std::move(f)), std::move(tr)};
}

}  // namespace cpd
