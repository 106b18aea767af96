// gpu_context.hpp — shared plumbing of the drop-in replacement for the
// reference's core/src/mttkrp.cpp and core/src/als.cpp (mttkrp_gpu.cpp,
// als_gpu.cpp): one libcpdgpu context per host thread, status -> the
// reference's exception types (errors.hpp:8-35), and a device copy of a
// cpd::DenseTensor for the duration of one call.
#pragma once
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "cpd/dense_tensor.hpp"
#include "cpd/errors.hpp"
#include "cpd/kron.hpp"
#include "cpdgpu.h"

namespace cpd::gpu {

// Device / driver failure: no reference counterpart; surfaces as runtime_error.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

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

struct Context {
  cpdgpu_ctx* h = nullptr;
  explicit Context(int device) {
    // Load every kernel when the context is made, not on its first launch (CUDA's lazy
    // module loading): a caller that times individual calls, like the reference's
    // run_benchmark (bench.cpp:60-90, acceptance criterion 6), would otherwise charge
    // the one-time loads to whichever engine launches a kernel first.  No effect when
    // the variable is already set or CUDA is already initialised in the process.
    setenv("CUDA_MODULE_LOADING", "EAGER", 0);
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

// CPD_GPU_DEVICE selects the device (default 0); one context per host thread.
inline Context& context() {
  static thread_local std::unique_ptr<Context> c;
  if (!c) {
    const char* e = std::getenv("CPD_GPU_DEVICE");
    c = std::make_unique<Context>(e ? std::atoi(e) : 0);
  }
  return *c;
}

// The tensor's values on the device for one call (the reference's DenseTensor
// has no slot to cache a device copy in).
class DeviceTensor {
 public:
  explicit DeviceTensor(const DenseTensor& y) {
    auto& ctx = context();
    std::vector<int64_t> d(y.shape().dims().begin(), y.shape().dims().end());
    ctx.check(cpdgpu_tensor_upload(ctx.h, y.data(), CPDGPU_F64, y.order(), d.data(), &t_));
  }
  ~DeviceTensor() { cpdgpu_tensor_free(t_); }
  DeviceTensor(const DeviceTensor&) = delete;
  DeviceTensor& operator=(const DeviceTensor&) = delete;
  cpdgpu_tensor* get() const { return t_; }

 private:
  cpdgpu_tensor* t_ = nullptr;
};

inline std::vector<int64_t> dims64(const Shape& s) { return std::vector<int64_t>(s.dims().begin(), s.dims().end()); }
inline std::vector<const double*> cptrs(const FactorList& f) {
  std::vector<const double*> p;
  for (const auto& a : f) p.push_back(a.data());
  return p;
}
inline std::vector<double*> ptrs(FactorList& f) {
  std::vector<double*> p;
  for (auto& a : f) p.push_back(a.data());
  return p;
}

}  // namespace cpd::gpu
