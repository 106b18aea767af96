// cpd_gpu/cpd.hpp — drop-in C++ adapter with the reference's hot-path API
// (/root/reference/proj/core/include/cpd/{mttkrp,als,kruskal,cost_counter,
// errors,shape,dense_tensor}.hpp) implemented over the C-ABI (include/cpdgpu.h).
//
// Same names, signatures, column-major layout, visit order and exception types
// as the reference; the arithmetic runs on a B200 through libcpdgpu.so.  Link
// with -lcpdgpu.  Define CPD_GPU_WITH_EIGEN (and have Eigen on the include
// path) to use Eigen::MatrixXd as the matrix type, exactly as the reference
// does; otherwise cpd::Matrix, a minimal column-major double matrix with the
// members the adapter needs (rows, cols, data, operator()).
//
// Header-only: every function is inline; one device context per thread
// (cpd::gpu::context()), device chosen with cpd::gpu::set_device().
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../cpdgpu.h"

#ifdef CPD_GPU_WITH_EIGEN
#include <Eigen/Core>
#endif

namespace cpd {

using index_t = std::int64_t;

// ---- errors (errors.hpp:8-35) ---------------------------------------------------
struct ShapeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct IndexError : std::out_of_range {
  using std::out_of_range::out_of_range;
};
struct ArgumentError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DomainError : std::domain_error {
  using std::domain_error::domain_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Device / driver failure (no reference counterpart).
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace gpu {
[[noreturn]] inline void throw_status(int st, const std::string& msg) {
  switch (st) {
    case CPDGPU_SHAPE_ERROR: throw ShapeError(msg);
    case CPDGPU_INDEX_ERROR: throw IndexError(msg);
    case CPDGPU_ARGUMENT_ERROR: throw ArgumentError(msg);
    case CPDGPU_NUMERIC_ERROR: throw NumericError(msg);
    case CPDGPU_DOMAIN_ERROR: throw DomainError(msg);
    case CPDGPU_PARSE_ERROR: throw ParseError(msg);
    default: throw DeviceError(msg.empty() ? "cpdgpu: device failure" : msg);
  }
}
}  // namespace gpu

// ---- matrices ---------------------------------------------------------------------
#ifdef CPD_GPU_WITH_EIGEN
using Matrix = Eigen::MatrixXd;
#else
// Column-major rows x cols doubles; the subset of Eigen::MatrixXd the adapter
// and its callers use.
class Matrix {
 public:
  Matrix() = default;
  Matrix(index_t rows, index_t cols) : rows_(rows), cols_(cols), v_(static_cast<size_t>(rows * cols), 0.0) {}
  static Matrix Zero(index_t r, index_t c) { return Matrix(r, c); }
  static Matrix Ones(index_t r, index_t c) {
    Matrix m(r, c);
    for (auto& x : m.v_) x = 1.0;
    return m;
  }
  static Matrix Identity(index_t r, index_t c) {
    Matrix m(r, c);
    for (index_t i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  index_t size() const { return rows_ * cols_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(index_t i, index_t j) { return v_[static_cast<size_t>(i + rows_ * j)]; }
  double operator()(index_t i, index_t j) const { return v_[static_cast<size_t>(i + rows_ * j)]; }
  void resize(index_t r, index_t c) {
    rows_ = r;
    cols_ = c;
    v_.assign(static_cast<size_t>(r * c), 0.0);
  }
  Matrix col(index_t j) const {
    Matrix m(rows_, 1);
    for (index_t i = 0; i < rows_; ++i) m(i, 0) = (*this)(i, j);
    return m;
  }

 private:
  index_t rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};
#endif

using FactorMatrix = Matrix;
using FactorList = std::vector<FactorMatrix>;

// ---- instrumentation (cost_counter.hpp:11-27, mttkrp.hpp:44-47) --------------------
class CostCounter {
 public:
  void charge(std::uint64_t mults) noexcept { total_ += mults; }
  void charge_gemm(std::int64_t m, std::int64_t k, std::int64_t p) noexcept {
    total_ += static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(k) * static_cast<std::uint64_t>(p);
  }
  void charge_kron(std::int64_t p, std::int64_t q) noexcept {
    total_ += static_cast<std::uint64_t>(p) * static_cast<std::uint64_t>(q);
  }
  std::uint64_t total() const noexcept { return total_; }
  void reset() noexcept { total_ = 0; }

 private:
  std::uint64_t total_ = 0;
};

struct FastStats {
  std::int64_t peak_workspace_doubles = 0;
};

using ModeHook = std::function<void(int n, const Matrix& gradient)>;

// ---- device context ------------------------------------------------------------------
namespace gpu {
struct Context {
  cpdgpu_ctx* h = nullptr;
  explicit Context(int device) {
    const int st = cpdgpu_create(&h, device);
    if (st != CPDGPU_OK) throw_status(st, "cpdgpu_create failed (no B200 device?)");
  }
  ~Context() { cpdgpu_destroy(h); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  void check(int st) const {
    if (st != CPDGPU_OK) throw_status(st, cpdgpu_last_error(h));
  }
};
inline int& device_index() {
  static thread_local int d = 0;
  return d;
}
inline std::unique_ptr<Context>& context_slot() {
  static thread_local std::unique_ptr<Context> c;
  return c;
}
inline Context& context() {
  auto& c = context_slot();
  if (!c) c = std::make_unique<Context>(device_index());
  return *c;
}
inline void set_device(int device) {
  device_index() = device;
  context_slot().reset();
}
// The device workspace the library holds besides the tensors' values, in bytes (in use,
// high-water mark): this implementation's own FastStats::peak_workspace figure
// (mttkrp.hpp:37-47); FastStats itself keeps the reference algorithm's number.
struct DeviceWorkspace {
  std::int64_t current_bytes = 0, peak_bytes = 0;
};
inline DeviceWorkspace device_workspace() {
  DeviceWorkspace w;
  auto& c = context();
  c.check(cpdgpu_device_workspace(c.h, &w.current_bytes, &w.peak_bytes));
  return w;
}
}  // namespace gpu

// ---- Shape (shape.hpp:15-42) ---------------------------------------------------------
class Shape {
 public:
  explicit Shape(std::vector<index_t> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw ShapeError("shape: need at least one mode");
    prefix_.push_back(1);
    for (size_t k = 0; k < dims_.size(); ++k) {
      if (dims_[k] < 1)
        throw ShapeError("shape: mode " + std::to_string(k + 1) + " has nonpositive extent " +
                         std::to_string(dims_[k]));
      index_t next = 0;
      if (__builtin_mul_overflow(prefix_.back(), dims_[k], &next))
        throw ShapeError("shape: entry count overflows at mode " + std::to_string(k + 1));
      prefix_.push_back(next);
    }
  }
  int order() const { return static_cast<int>(dims_.size()); }
  index_t dim(int n) const {
    if (n < 1 || n > order())
      throw IndexError("shape: mode " + std::to_string(n) + " outside 1.." + std::to_string(order()));
    return dims_[static_cast<size_t>(n - 1)];
  }
  const std::vector<index_t>& dims() const { return dims_; }
  index_t num_entries() const { return prefix_.back(); }
  index_t j_prefix(int n) const {
    if (n < 0 || n > order())
      throw IndexError("shape: prefix length " + std::to_string(n) + " outside 0.." + std::to_string(order()));
    return prefix_[static_cast<size_t>(n)];
  }
  index_t k_suffix(int n) const { return num_entries() / j_prefix(n); }
  bool ascending() const {
    for (size_t k = 1; k < dims_.size(); ++k)
      if (dims_[k] < dims_[k - 1]) return false;
    return true;
  }
  bool operator==(const Shape& o) const { return dims_ == o.dims_; }
  bool operator!=(const Shape& o) const { return !(*this == o); }

 private:
  std::vector<index_t> dims_;
  std::vector<index_t> prefix_;
};

// ---- DenseTensor (dense_tensor.hpp:15-47) ---------------------------------------------
// Immutable fp64 column-major values shared by copies; the device copy is made on
// first use and shared the same way (valid for the values' lifetime).
class DenseTensor {
 public:
  DenseTensor(Shape shape, std::vector<double> values)
      : shape_(std::move(shape)), values_(std::make_shared<const std::vector<double>>(std::move(values))),
        dev_(std::make_shared<DeviceCopy>()) {
    if (static_cast<index_t>(values_->size()) != shape_.num_entries())
      throw ShapeError("tensor: " + std::to_string(values_->size()) + " values for a shape holding " +
                       std::to_string(shape_.num_entries()) + " entries");
  }
  static DenseTensor zeros(Shape shape) {
    std::vector<double> v(static_cast<size_t>(shape.num_entries()), 0.0);
    return DenseTensor(std::move(shape), std::move(v));
  }
  const Shape& shape() const { return shape_; }
  int order() const { return shape_.order(); }
  index_t size() const { return shape_.num_entries(); }
  const double* data() const { return values_->data(); }
  const std::vector<double>& values() const { return *values_; }
  double norm() const {
    double s = 0.0;
    for (double x : *values_) s += x * x;
    return std::sqrt(s);
  }
  // device handle (uploaded once)
  cpdgpu_tensor* device() const {
    if (!dev_->t) {
      auto& ctx = gpu::context();
      std::vector<int64_t> d(shape_.dims().begin(), shape_.dims().end());
      ctx.check(cpdgpu_tensor_upload(ctx.h, data(), CPDGPU_F64, order(), d.data(), &dev_->t));
    }
    return dev_->t;
  }

 private:
  struct DeviceCopy {
    cpdgpu_tensor* t = nullptr;
    ~DeviceCopy() { cpdgpu_tensor_free(t); }
  };
  Shape shape_;
  std::shared_ptr<const std::vector<double>> values_;
  std::shared_ptr<DeviceCopy> dev_;
};

// ---- helpers ----------------------------------------------------------------------------
// factor_shape / factor_rank (kron.cpp:25-45)
inline Shape factor_shape(const FactorList& factors) {
  if (factors.empty()) throw ArgumentError("factors: empty list");
  const index_t R = factors.front().cols();
  std::vector<index_t> dims;
  for (size_t k = 0; k < factors.size(); ++k) {
    if (factors[k].cols() != R)
      throw ShapeError("factors: mode " + std::to_string(k + 1) + " has rank " + std::to_string(factors[k].cols()) +
                       ", expected " + std::to_string(R));
    if (factors[k].rows() < 1) throw ShapeError("factors: mode " + std::to_string(k + 1) + " has no rows");
    dims.push_back(factors[k].rows());
  }
  return Shape(std::move(dims));
}
inline index_t factor_rank(const FactorList& factors) {
  if (factors.empty()) throw ArgumentError("factors: empty list");
  return factors.front().cols();
}

namespace detail {
inline std::vector<int64_t> dims64(const Shape& s) { return std::vector<int64_t>(s.dims().begin(), s.dims().end()); }
inline void check_status(int st) {
  if (st != CPDGPU_OK) gpu::throw_status(st, "");
}
inline void check_factors_match(const DenseTensor& y, const FactorList& f, const char* who) {
  if (factor_shape(f) != y.shape()) throw ShapeError(std::string(who) + ": factor row counts do not match the tensor");
}
}  // namespace detail

// ---- ordering (mttkrp.hpp:24,35,73) ------------------------------------------------------
inline int select_pivot(const Shape& shape) {
  int p = 0;
  auto d = detail::dims64(shape);
  const int st = cpdgpu_select_pivot(shape.order(), d.data(), &p);
  if (st != CPDGPU_OK)
    gpu::throw_status(st, shape.order() < 2 ? "select_pivot: need an order-2 or higher shape"
                                            : "select_pivot: no mode satisfies J_n <= K_n; sort modes first");
  return p;
}

inline std::vector<int> fast_update_order(const Shape& shape) {
  std::vector<int> order(static_cast<size_t>(shape.order()));
  auto d = detail::dims64(shape);
  const int st = cpdgpu_fast_update_order(shape.order(), d.data(), order.data());
  if (st != CPDGPU_OK) gpu::throw_status(st, "fast_update_order: need an order-2 or higher shape");
  return order;
}

// Stable ascending mode order (mttkrp.cpp:67-90): perm (sorted position ->
// original mode) and inverse, both 1-based.  The device path sorts internally.
struct ModeOrder {
  std::vector<int> perm, inverse;
};
inline ModeOrder sort_mode_order(const Shape& shape) {
  ModeOrder o;
  o.perm.resize(static_cast<size_t>(shape.order()));
  o.inverse.resize(o.perm.size());
  auto d = detail::dims64(shape);
  detail::check_status(cpdgpu_sort_modes(shape.order(), d.data(), o.perm.data(), o.inverse.data()));
  return o;
}

// mttkrp.cpp:292-320 (ascending dims)
inline std::uint64_t fast_count_realized(const Shape& shape, index_t R, int n) {
  if (n < 1 || n > shape.order())
    throw IndexError("fast_count_realized: mode " + std::to_string(n) + " outside 1.." +
                     std::to_string(shape.order()));
  if (R < 1) throw ArgumentError("fast_count_realized: rank must be positive");
  if (!shape.ascending()) throw ArgumentError("fast_count_realized: dims must be ascending");
  auto d = detail::dims64(shape);
  return cpdgpu_fast_count_realized(shape.order(), d.data(), R, n);
}

// sort_modes (mttkrp.hpp:28-35, mttkrp.cpp:67-90): stable ascending mode order,
// the permuted tensor (host copy; identity sorts share the tensor) and factors.
// The device gradient sorts internally; this is the reference's helper.
struct SortResult {
  DenseTensor tensor;
  FactorList factors;
  std::vector<int> perm;
  std::vector<int> inverse;
};
inline SortResult sort_modes(const DenseTensor& y, const FactorList& factors) {
  detail::check_factors_match(y, factors, "sort_modes");
  const ModeOrder o = sort_mode_order(y.shape());
  const int N = y.order();
  bool identity = true;
  for (int j = 1; j <= N; ++j) identity &= o.perm[static_cast<size_t>(j - 1)] == j;
  FactorList sf;
  for (int j = 1; j <= N; ++j) sf.push_back(factors[static_cast<size_t>(o.perm[static_cast<size_t>(j - 1)] - 1)]);
  if (identity) return SortResult{y, std::move(sf), o.perm, o.inverse};
  // out(i_1..i_N) = y(i at positions perm): mode j of the result is mode perm[j] of y
  std::vector<index_t> od;
  for (int j = 0; j < N; ++j) od.push_back(y.shape().dim(o.perm[static_cast<size_t>(j)]));
  const Shape os(od);
  std::vector<index_t> stride(static_cast<size_t>(N));
  for (int m = 0; m < N; ++m) stride[static_cast<size_t>(m)] = y.shape().j_prefix(m);
  std::vector<double> v(static_cast<size_t>(y.size()));
  std::vector<index_t> idx(static_cast<size_t>(N), 0);
  for (index_t q = 0; q < y.size(); ++q) {
    index_t src = 0;
    for (int j = 0; j < N; ++j) src += idx[static_cast<size_t>(j)] * stride[static_cast<size_t>(o.perm[static_cast<size_t>(j)] - 1)];
    v[static_cast<size_t>(q)] = y.data()[src];
    for (int j = 0; j < N && ++idx[static_cast<size_t>(j)] == od[static_cast<size_t>(j)]; ++j) idx[static_cast<size_t>(j)] = 0;
  }
  return SortResult{DenseTensor(os, std::move(v)), std::move(sf), o.perm, o.inverse};
}

// ---- the all-mode gradient (mttkrp.hpp:59-69, mttkrp.cpp:113-253) --------------------------
namespace detail {
struct HookCtx {
  const ModeHook* hook;
  CostCounter* counter;
  FactorList* factors;
  std::vector<Matrix>* out;
  std::vector<std::vector<double>>* bufs;
  index_t R;
  std::exception_ptr error;  // whatever the hook (or the size check) threw
};
// Runs the caller's hook between modes.  Nothing may unwind through the C-ABI
// frames, so any exception is captured here (status -1 stops the sweep) and
// rethrown unchanged by cp_gradient_all once the C call has returned, exactly
// as the reference's direct hook(orig, G) call would propagate it
// (mttkrp.cpp:134-145).
inline int hook_tramp(void* user, int mode, const double* g, int64_t rows, int64_t rank, uint64_t mults) {
  auto* h = static_cast<HookCtx*>(user);
  try {
    if (h->counter) h->counter->charge(mults);  // the charge lands before the hook (test_counts.cpp:16-31)
    Matrix& G = (*h->out)[static_cast<size_t>(mode - 1)];  // the C-ABI wrote G(mode) here
    if (G.data() != g) std::copy(g, g + rows * rank, G.data());
    (*h->hook)(mode, G);
    const Matrix& F = (*h->factors)[static_cast<size_t>(mode - 1)];
    if (F.rows() != rows || F.cols() != h->R)
      throw ShapeError("cp_gradient_all: hook left factor of mode " + std::to_string(mode) + " with the wrong size");
    std::copy(F.data(), F.data() + rows * rank, (*h->bufs)[static_cast<size_t>(mode - 1)].data());
    return 0;
  } catch (...) {
    h->error = std::current_exception();
  }
  return CPDGPU_HOOK_ABORTED;
}
}  // namespace detail

inline std::vector<Matrix> cp_gradient_all(const DenseTensor& y, FactorList& factors, CostCounter* counter,
                                           const ModeHook& hook, FastStats* stats) {
  const int N = y.order();
  if (N < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  detail::check_factors_match(y, factors, "cp_gradient_all");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  std::vector<Matrix> out(static_cast<size_t>(N));
  for (int m = 0; m < N; ++m) out[static_cast<size_t>(m)].resize(y.shape().dim(m + 1), R);
  std::vector<double*> gp(static_cast<size_t>(N));
  for (int m = 0; m < N; ++m) gp[static_cast<size_t>(m)] = out[static_cast<size_t>(m)].data();
  int64_t peak = 0;
  if (!hook) {
    std::vector<const double*> fp(static_cast<size_t>(N));
    for (int m = 0; m < N; ++m) fp[static_cast<size_t>(m)] = factors[static_cast<size_t>(m)].data();
    std::vector<uint64_t> mults(static_cast<size_t>(N));
    ctx.check(cpdgpu_cp_gradient_all(ctx.h, y.device(), R, fp.data(), gp.data(), mults.data(), &peak));
    if (counter)
      for (auto m : mults) counter->charge(m);
  } else {
    std::vector<std::vector<double>> bufs(static_cast<size_t>(N));
    std::vector<double*> fp(static_cast<size_t>(N));
    for (int m = 0; m < N; ++m) {
      const Matrix& F = factors[static_cast<size_t>(m)];
      bufs[static_cast<size_t>(m)].assign(F.data(), F.data() + F.rows() * F.cols());
      fp[static_cast<size_t>(m)] = bufs[static_cast<size_t>(m)].data();
    }
    detail::HookCtx hc{&hook, counter, &factors, &out, &bufs, R, nullptr};
    const int st = cpdgpu_cp_gradient_all_hook(ctx.h, y.device(), R, fp.data(), gp.data(), detail::hook_tramp, &hc,
                                               &peak);
    if (hc.error) std::rethrow_exception(hc.error);
    ctx.check(st);
  }
  if (stats) stats->peak_workspace_doubles = peak;
  return out;
}

inline std::vector<Matrix> cp_gradient_all(const DenseTensor& y, const FactorList& factors,
                                           CostCounter* counter = nullptr, FastStats* stats = nullptr) {
  FactorList copy = factors;
  return cp_gradient_all(y, copy, counter, ModeHook{}, stats);
}

// ---- multi-GPU: the all-mode gradient over last-mode slabs ---------------------
// One process (or thread) per GPU, each holding the contiguous last-mode slab
// [lo, hi) = gpu::slab_bounds(I_N, nranks, rank) of a tensor with ascending dims.
// Each rank calls cp_gradient_all_sharded with its slab and the GLOBAL factors and
// receives every global G(n): the library computes the slab's gradient at the
// global pivot and finishes it with ONE all-reduce inside libcpdgpu.so (NCCL over
// NVLink after gpu::comm_init, or the caller's host all-reduce after
// gpu::comm_init_host).  Counter charges are the unsharded call's
// (mttkrp.hpp:59-69 semantics on the whole tensor).
namespace gpu {
inline std::vector<unsigned char> comm_unique_id() {
  std::vector<unsigned char> id(CPDGPU_COMM_ID_BYTES);
  const int st = cpdgpu_comm_unique_id(id.data());
  if (st != CPDGPU_OK) throw_status(st, "cpdgpu_comm_unique_id failed (libnccl.so.2 missing?)");
  return id;
}
// NCCL communicator on this thread's context (rank 0 made `id`, every rank passes it)
inline void comm_init(const std::vector<unsigned char>& id, int nranks, int rank) {
  auto& c = context();
  c.check(cpdgpu_comm_init(c.h, id.data(), nranks, rank));
}
// host all-reduce (MPI, gloo, ...): fn(user, buf, count) sums `count` doubles in place
inline void comm_init_host(int nranks, int rank, cpdgpu_allreduce_fn fn, void* user) {
  auto& c = context();
  c.check(cpdgpu_comm_init_host(c.h, nranks, rank, fn, user));
}
inline void comm_destroy() {
  auto& c = context();
  c.check(cpdgpu_comm_destroy(c.h));
}
inline std::pair<index_t, index_t> slab_bounds(index_t extent, int nranks, int rank) {
  int64_t lo = 0, hi = 0;
  const int st = cpdgpu_slab_bounds(extent, nranks, rank, &lo, &hi);
  if (st != CPDGPU_OK) throw_status(st, "slab_bounds: bad argument");
  return {lo, hi};
}
}  // namespace gpu

inline std::vector<Matrix> cp_gradient_all_sharded(const DenseTensor& slab, const Shape& global_shape,
                                                   const FactorList& factors, CostCounter* counter = nullptr) {
  const int N = global_shape.order();
  if (N < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  if (factor_shape(factors) != global_shape)
    throw ShapeError("cp_gradient_all: factor row counts do not match the tensor");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  const auto gd = detail::dims64(global_shape);
  std::vector<const double*> fp;
  for (const auto& f : factors) fp.push_back(f.data());
  std::vector<Matrix> out(static_cast<size_t>(N));
  std::vector<double*> gp;
  for (int m = 0; m < N; ++m) {
    out[static_cast<size_t>(m)].resize(global_shape.dim(m + 1), R);
    gp.push_back(out[static_cast<size_t>(m)].data());
  }
  std::vector<uint64_t> mults(static_cast<size_t>(N));
  ctx.check(cpdgpu_cp_gradient_all_sharded(ctx.h, slab.device(), N, gd.data(), R, fp.data(), gp.data(), mults.data()));
  if (counter)
    for (auto m : mults) counter->charge(m);
  return out;
}

// Sharded als_sweep_fast (als.cpp:69-78): every rank passes its slab and the
// GLOBAL factors, which leave identical on every rank; returns the global cost.
inline double als_sweep_fast_sharded(const DenseTensor& slab, const Shape& global_shape, FactorList& factors,
                                     double pinv_rtol = 1e-12, CostCounter* counter = nullptr) {
  const int N = global_shape.order();
  if (N < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  if (factor_shape(factors) != global_shape)
    throw ShapeError("cp_gradient_all: factor row counts do not match the tensor");
  auto& ctx = gpu::context();
  const auto gd = detail::dims64(global_shape);
  std::vector<double*> fp;
  for (auto& f : factors) fp.push_back(f.data());
  double cost = 0.0;
  uint64_t mults = 0;
  ctx.check(cpdgpu_als_sweep_sharded(ctx.h, slab.device(), N, gd.data(), factor_rank(factors), fp.data(), pinv_rtol,
                                     &cost, &mults));
  if (counter) counter->charge(mults);
  return cost;
}

// predicted_mult_count (mttkrp.hpp:76-86): the analytic count of one mode
enum class CountVariant { direct, fast, fast_derived };
inline std::uint64_t predicted_mult_count(const Shape& shape, index_t R, int n, CountVariant variant) {
  const auto d = detail::dims64(shape);
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

// ---- direct MTTKRP (mttkrp.hpp:19-20): one pass over Y per mode ----------------------------
inline Matrix mttkrp_direct(const DenseTensor& y, const FactorList& factors, int n, CostCounter* counter = nullptr) {
  const int N = y.order();
  if (n < 1 || n > N) throw IndexError("mttkrp_direct: mode " + std::to_string(n) + " outside 1.." + std::to_string(N));
  detail::check_factors_match(y, factors, "mttkrp_direct");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  std::vector<const double*> fp(factors.size());
  for (size_t k = 0; k < factors.size(); ++k) fp[k] = factors[k].data();
  Matrix out(y.shape().dim(n), R);
  uint64_t mults = 0;
  ctx.check(cpdgpu_mttkrp_direct(ctx.h, y.device(), R, fp.data(), n, out.data(), &mults));
  if (counter) counter->charge(mults);
  return out;
}

// ---- ALS (als.hpp:21-93, kruskal.hpp:14-29) -----------------------------------------------
class KruskalModel {
 public:
  KruskalModel() = default;
  explicit KruskalModel(FactorList factors) : factors_(std::move(factors)) { factor_shape(factors_); }
  int order() const { return static_cast<int>(factors_.size()); }
  index_t rank() const { return factor_rank(factors_); }
  Shape shape() const { return factor_shape(factors_); }
  const FactorList& factors() const { return factors_; }
  FactorList& factors() { return factors_; }
  const FactorMatrix& factor(int n) const {
    if (n < 1 || n > order())
      throw IndexError("model: mode " + std::to_string(n) + " outside 1.." + std::to_string(order()));
    return factors_[static_cast<size_t>(n - 1)];
  }

 private:
  FactorList factors_;
};

enum class Algorithm { als_direct, als_fast, mu, gd };
enum class UpdateOrder { standard, pivot };

struct SolveOptions {
  int max_iters = 20;
  double tol = 0.0;
  double pinv_rtol = 1e-12;
  double mu_eps = 1e-12;
  double gd_eta = 1e-3;
  UpdateOrder order = UpdateOrder::standard;
  std::uint64_t seed = 0;
};

struct RunTrace {
  std::vector<double> cost;
  std::vector<double> rel_error;
  std::vector<double> seconds;  // device-timed sweeps (CUDA events)
  std::vector<std::uint64_t> mults;
  int iters_run = 0;
};

struct SolveResult {
  KruskalModel model;
  RunTrace trace;
};

inline Matrix pinv_psd(const Matrix& s, double rtol = 1e-12) {
  if (s.rows() != s.cols()) throw ShapeError("pinv_psd: matrix must be square");
  if (rtol < 0.0) throw ArgumentError("pinv_psd: rtol must be nonnegative");
  auto& ctx = gpu::context();
  Matrix out(s.rows(), s.cols());
  ctx.check(cpdgpu_pinv_psd(ctx.h, s.rows(), s.data(), rtol, out.data()));
  return out;
}

inline Matrix als_update_mode(const Matrix& m, const FactorList& factors, int n, double pinv_rtol = 1e-12) {
  const int N = static_cast<int>(factors.size());
  if (n < 1 || n > N) throw IndexError("als_update_mode: mode " + std::to_string(n) + " outside 1.." + std::to_string(N));
  const Shape s = factor_shape(factors);
  const index_t R = factor_rank(factors);
  if (m.rows() != s.dim(n) || m.cols() != R) throw ShapeError("als_update_mode: mttkrp matrix has the wrong size");
  auto& ctx = gpu::context();
  std::vector<const double*> fp(static_cast<size_t>(N));
  for (int k = 0; k < N; ++k) fp[static_cast<size_t>(k)] = factors[static_cast<size_t>(k)].data();
  auto d = detail::dims64(s);
  Matrix out(m.rows(), m.cols());
  ctx.check(cpdgpu_als_update_mode(ctx.h, N, d.data(), R, m.data(), fp.data(), n, pinv_rtol, out.data()));
  return out;
}

inline void als_sweep_fast(const DenseTensor& y, FactorList& factors, double pinv_rtol = 1e-12,
                           CostCounter* counter = nullptr, FastStats* stats = nullptr) {
  if (y.order() < 2) throw ArgumentError("cp_gradient_all: need an order-2 or higher tensor");
  detail::check_factors_match(y, factors, "cp_gradient_all");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  std::vector<double*> fp(factors.size());
  for (size_t k = 0; k < factors.size(); ++k) fp[k] = factors[k].data();
  uint64_t mults = 0;
  ctx.check(cpdgpu_als_sweep(ctx.h, y.device(), R, fp.data(), pinv_rtol, nullptr, &mults));
  if (counter) counter->charge(mults);
  (void)stats;
}

// als_sweep_direct (als.hpp:58-60): direct MTTKRP + update per mode of `order`.
inline void als_sweep_direct(const DenseTensor& y, FactorList& factors, const std::vector<int>& order,
                             double pinv_rtol = 1e-12, CostCounter* counter = nullptr) {
  detail::check_factors_match(y, factors, "als_sweep_direct");
  const index_t R = factor_rank(factors);
  auto& ctx = gpu::context();
  std::vector<double*> fp(factors.size());
  for (size_t k = 0; k < factors.size(); ++k) fp[k] = factors[k].data();
  uint64_t mults = 0;
  ctx.check(cpdgpu_als_sweep_direct(ctx.h, y.device(), R, fp.data(), order.data(), static_cast<int>(order.size()),
                                    pinv_rtol, &mults));
  if (counter) counter->charge(mults);
}

// mu_sweep (als.hpp:68-71): multiplicative updates; negative entries -> DomainError.
inline void mu_sweep(const DenseTensor& y, FactorList& factors, double eps = 1e-12, CostCounter* counter = nullptr) {
  detail::check_factors_match(y, factors, "mu_sweep");
  auto& ctx = gpu::context();
  std::vector<double*> fp(factors.size());
  for (size_t k = 0; k < factors.size(); ++k) fp[k] = factors[k].data();
  uint64_t mults = 0;
  ctx.check(cpdgpu_mu_sweep(ctx.h, y.device(), factor_rank(factors), fp.data(), eps, &mults));
  if (counter) counter->charge(mults);
}

// gd_step (als.hpp:73-76): simultaneous gradient step.
inline void gd_step(const DenseTensor& y, FactorList& factors, double eta, CostCounter* counter = nullptr) {
  detail::check_factors_match(y, factors, "gd_step");
  auto& ctx = gpu::context();
  std::vector<double*> fp(factors.size());
  for (size_t k = 0; k < factors.size(); ++k) fp[k] = factors[k].data();
  uint64_t mults = 0;
  ctx.check(cpdgpu_gd_step(ctx.h, y.device(), factor_rank(factors), fp.data(), eta, &mults));
  if (counter) counter->charge(mults);
}

// random_init (als.hpp:84-85, als.cpp:127-139): Uniform01 (rng.hpp:16-26, the
// std::mt19937_64 stream, bit-identical) column-major per factor in mode order.
inline KruskalModel random_init(const Shape& shape, index_t rank, std::uint64_t seed) {
  if (rank < 1) throw ArgumentError("random_init: rank must be positive");
  index_t total = 0;
  for (int n = 1; n <= shape.order(); ++n) total += shape.dim(n) * rank;
  std::vector<double> v(static_cast<size_t>(total));
  detail::check_status(cpdgpu_uniform01_fill(seed, total, v.data()));
  FactorList f;
  index_t at = 0;
  for (int n = 1; n <= shape.order(); ++n) {
    Matrix a(shape.dim(n), rank);
    std::copy(v.begin() + at, v.begin() + at + shape.dim(n) * rank, a.data());
    at += shape.dim(n) * rank;
    f.push_back(std::move(a));
  }
  return KruskalModel(std::move(f));
}

// standard_order (als.hpp:87): 1..N
inline std::vector<int> standard_order(int order) {
  std::vector<int> v(static_cast<size_t>(order));
  std::iota(v.begin(), v.end(), 1);
  return v;
}

// run(y, init, algo, opts) (als.cpp:147-210) for every Algorithm on the device.
inline SolveResult run(const DenseTensor& y, const KruskalModel& init, Algorithm algo, const SolveOptions& opts = {},
                       CostCounter* counter = nullptr) {
  if (opts.max_iters < 1) throw ArgumentError("run: max_iters must be at least 1");
  if (opts.tol < 0.0 || opts.pinv_rtol < 0.0 || opts.mu_eps < 0.0)
    throw ArgumentError("run: tolerances must be nonnegative");
  if (init.shape() != y.shape()) throw ShapeError("run: init factors do not match the tensor");
  FactorList f = init.factors();
  const index_t R = init.rank();
  auto& ctx = gpu::context();
  std::vector<double*> fp(f.size());
  for (size_t k = 0; k < f.size(); ++k) fp[k] = f[k].data();
  const size_t n = static_cast<size_t>(opts.max_iters);
  RunTrace tr;
  tr.cost.resize(n);
  tr.rel_error.resize(n);
  tr.seconds.resize(n);
  tr.mults.resize(n);
  int iters = 0;
  const int code = algo == Algorithm::als_direct ? 0 : algo == Algorithm::als_fast ? 1 : algo == Algorithm::mu ? 2 : 3;
  ctx.check(cpdgpu_run_algo(ctx.h, y.device(), R, fp.data(), code, opts.order == UpdateOrder::pivot ? 1 : 0,
                            opts.max_iters, opts.tol, opts.pinv_rtol, opts.mu_eps, opts.gd_eta, tr.cost.data(),
                            tr.rel_error.data(), tr.seconds.data(), tr.mults.data(), &iters));
  tr.iters_run = iters;
  tr.cost.resize(static_cast<size_t>(iters));
  tr.rel_error.resize(static_cast<size_t>(iters));
  tr.seconds.resize(static_cast<size_t>(iters));
  tr.mults.resize(static_cast<size_t>(iters));
  const std::uint64_t base = counter ? counter->total() : 0;
  for (auto& m : tr.mults) m = counter ? base + m : 0;
  if (counter && iters > 0) counter->charge(tr.mults.back() - base);
  return SolveResult{KruskalModel(std::move(f)), std::move(tr)};
}

}  // namespace cpd
