// mttkrp_gpu.cpp — drop-in replacement for the reference's core/src/mttkrp.cpp:
// every function declared in cpd/mttkrp.hpp (unchanged header) implemented over
// the C-ABI of libcpdgpu.so (include/cpdgpu.h), so the all-mode gradient and the
// direct MTTKRP run on the B200.  Build it in place of mttkrp.cpp (and
// als_gpu.cpp in place of als.cpp) and link -lcpdgpu; INTEGRATION.md.  Inputs,
// outputs, visit order, counter charges and exception types/messages follow the
// reference (mttkrp.cpp:11-320).
#include <exception>
#include <numeric>
#include <string>
#include <vector>

#include "cpd/errors.hpp"
#include "cpd/mttkrp.hpp"
#include "cpd/tensor_ops.hpp"
#include "gpu_context.hpp"

namespace cpd {
namespace {

void check_factors_match(const DenseTensor& y, const FactorList& factors, const char* who) {
  if (factor_shape(factors) != y.shape())
    throw ShapeError(std::string(who) + ": factor row counts do not match the tensor");
}

struct HookCtx {
  const ModeHook* hook;
  CostCounter* counter;
  FactorList* factors;
  std::vector<Eigen::MatrixXd>* out;
  std::vector<std::vector<double>>* bufs;
  index_t R;
  std::exception_ptr error;
};

// Between modes (mttkrp.cpp:134-145): charge, hook(orig, G), re-read the factor.
// Nothing unwinds through the C frames: the hook's exception is held and
// rethrown unchanged after the C call returns.
int hook_tramp(void* user, int mode, const double* g, int64_t rows, int64_t rank, uint64_t mults) {
  auto* h = static_cast<HookCtx*>(user);
  try {
    if (h->counter) h->counter->charge(mults);
    Eigen::MatrixXd& G = (*h->out)[static_cast<size_t>(mode - 1)];
    if (G.data() != g) std::copy(g, g + rows * rank, G.data());
    (*h->hook)(mode, G);
    const Eigen::MatrixXd& F = (*h->factors)[static_cast<size_t>(mode - 1)];
    if (F.rows() != rows || F.cols() != h->R)
      throw ShapeError("cp_gradient_all: hook left factor of mode " + std::to_string(mode) + " with the wrong size");
    std::copy(F.data(), F.data() + rows * rank, (*h->bufs)[static_cast<size_t>(mode - 1)].data());
    return 0;
  } catch (...) {
    h->error = std::current_exception();
  }
  return CPDGPU_HOOK_ABORTED;
}

}  // namespace

Eigen::MatrixXd mttkrp_direct(const DenseTensor& y, const FactorList& factors, int n, CostCounter* counter) {
  const int N = y.order();
  if (n < 1 || n > N)
    throw IndexError("mttkrp_direct: mode " + std::to_string(n) + " outside 1.." + std::to_string(N));
  check_factors_match(y, factors, "mttkrp_direct");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  const auto fp = gpu::cptrs(factors);
  Eigen::MatrixXd out(y.shape().dim(n), R);
  uint64_t mults = 0;
  ctx.check(cpdgpu_mttkrp_direct(ctx.h, t.get(), R, fp.data(), n, out.data(), &mults));
  if (counter) counter->charge(mults);
  return out;
}

int select_pivot(const Shape& shape) {
  if (shape.order() < 2) throw ArgumentError("select_pivot: need an order-2 or higher shape");
  int p = 0;
  const auto d = gpu::dims64(shape);
  if (cpdgpu_select_pivot(shape.order(), d.data(), &p) != CPDGPU_OK)
    throw ShapeError("select_pivot: no mode satisfies J_n <= K_n; sort modes first");
  return p;
}

SortResult sort_modes(const DenseTensor& y, const FactorList& factors) {
  check_factors_match(y, factors, "sort_modes");
  const int N = y.order();
  std::vector<int> perm(static_cast<size_t>(N)), inverse(static_cast<size_t>(N));
  const auto d = gpu::dims64(y.shape());
  const int st = cpdgpu_sort_modes(N, d.data(), perm.data(), inverse.data());
  if (st != CPDGPU_OK) gpu::throw_status(st, "sort_modes: bad shape");
  bool identity = true;
  for (int j = 1; j <= N; ++j) identity &= perm[static_cast<size_t>(j - 1)] == j;
  FactorList sorted;
  sorted.reserve(factors.size());
  for (int j = 1; j <= N; ++j) sorted.push_back(factors[static_cast<size_t>(perm[static_cast<size_t>(j - 1)] - 1)]);
  // the physical copy is the reference's own permute (tensor_ops.cpp:39-71): this
  // helper is not on the gradient path (the device sorts internally)
  return SortResult{identity ? y : permute(y, perm), std::move(sorted), std::move(perm), std::move(inverse)};
}

std::vector<Eigen::MatrixXd> cp_gradient_all(const DenseTensor& y, FactorList& factors, CostCounter* counter,
                                             const ModeHook& hook, FastStats* stats) {
  const int N = y.order();
  if (N < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  check_factors_match(y, factors, "cp_gradient_all");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  const gpu::DeviceTensor t(y);
  std::vector<Eigen::MatrixXd> out(static_cast<size_t>(N));
  for (int m = 0; m < N; ++m) out[static_cast<size_t>(m)].resize(y.shape().dim(m + 1), R);
  std::vector<double*> gp;
  for (auto& g : out) gp.push_back(g.data());
  int64_t peak = 0;
  if (!hook) {
    const auto fp = gpu::cptrs(factors);
    std::vector<uint64_t> mults(static_cast<size_t>(N));
    ctx.check(cpdgpu_cp_gradient_all(ctx.h, t.get(), R, fp.data(), gp.data(), mults.data(), &peak));
    if (counter)
      for (int j = 0; j < N; ++j) counter->charge(mults[static_cast<size_t>(j)]);
  } else {
    std::vector<std::vector<double>> bufs(static_cast<size_t>(N));
    std::vector<double*> fp(static_cast<size_t>(N));
    for (int m = 0; m < N; ++m) {
      const Eigen::MatrixXd& F = factors[static_cast<size_t>(m)];
      bufs[static_cast<size_t>(m)].assign(F.data(), F.data() + F.size());
      fp[static_cast<size_t>(m)] = bufs[static_cast<size_t>(m)].data();
    }
    HookCtx hc{&hook, counter, &factors, &out, &bufs, R, nullptr};
    const int st = cpdgpu_cp_gradient_all_hook(ctx.h, t.get(), R, fp.data(), gp.data(), hook_tramp, &hc, &peak);
    if (hc.error) std::rethrow_exception(hc.error);
    ctx.check(st);
  }
  // the reference algorithm's workspace high-water mark (mttkrp.cpp:127-131,243),
  // reported for compatibility; the device's own buffers are not counted here
  if (stats) stats->peak_workspace_doubles = peak;
  return out;
}

std::vector<Eigen::MatrixXd> cp_gradient_all(const DenseTensor& y, const FactorList& factors, CostCounter* counter,
                                             FastStats* stats) {
  FactorList copy = factors;
  return cp_gradient_all(y, copy, counter, ModeHook{}, stats);
}

std::vector<int> fast_update_order(const Shape& shape) {
  if (shape.order() < 2) throw ArgumentError("fast_update_order: need an order-2 or higher shape");
  std::vector<int> order(static_cast<size_t>(shape.order()));
  const auto d = gpu::dims64(shape);
  const int st = cpdgpu_fast_update_order(shape.order(), d.data(), order.data());
  if (st != CPDGPU_OK) gpu::throw_status(st, "fast_update_order: bad shape");
  return order;
}

std::uint64_t predicted_mult_count(const Shape& shape, index_t R, int n, CountVariant variant) {
  const auto d = gpu::dims64(shape);
  uint64_t out = 0;
  const int v = variant == CountVariant::direct ? 0 : variant == CountVariant::fast ? 1 : 2;
  const int st = cpdgpu_predicted_mult_count(shape.order(), d.data(), R, n, v, &out);
  if (st == CPDGPU_INDEX_ERROR)
    throw IndexError("predicted_mult_count: mode " + std::to_string(n) + " outside 1.." +
                     std::to_string(shape.order()));
  if (st != CPDGPU_OK)
    throw ArgumentError(R < 1 ? "predicted_mult_count: rank must be positive"
                              : "predicted_mult_count: dims must be ascending");
  return out;
}

std::uint64_t fast_count_realized(const Shape& shape, index_t R, int n) {
  if (n < 1 || n > shape.order())
    throw IndexError("fast_count_realized: mode " + std::to_string(n) + " outside 1.." +
                     std::to_string(shape.order()));
  if (R < 1) throw ArgumentError("fast_count_realized: rank must be positive");
  if (!shape.ascending()) throw ArgumentError("fast_count_realized: dims must be ascending");
  const auto d = gpu::dims64(shape);
  return cpdgpu_fast_count_realized(shape.order(), d.data(), R, n);
}

}  // namespace cpd
