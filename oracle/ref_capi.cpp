// ref_capi.cpp — TEST INFRASTRUCTURE ONLY (oracle/_ref/libcpdref.so).
//
// A C entry layer over the reference implementation itself, compiled from its
// own sources under /root/reference/proj/core (oracle/Makefile, target `ref`,
// reference flags -O3 -DNDEBUG, Eigen replaced by oracle/shim).  Used by the
// tests to pin the C oracle port and the GPU path to the reference's own
// results, and by bench.py's CPU-baseline / --impl reference legs (kind
// "reference").  Nothing in the product links it.
//
// Every call returns 0 or the cpdgpu-style status of the exception the reference
// threw (1 ShapeError, 2 IndexError, 3 ArgumentError, 4 NumericError, 5
// DomainError, 8 ParseError, 6 anything else); ref_last_error() has its text.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cpd/als.hpp"
#include "cpd/cost_counter.hpp"
#include "cpd/dense_tensor.hpp"
#include "cpd/errors.hpp"
#include "cpd/kruskal.hpp"
#include "cpd/mttkrp.hpp"
#include "cpd/shape.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const cpd::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const cpd::IndexError& e) {
    g_err = e.what();
    return 2;
  } catch (const cpd::ArgumentError& e) {
    g_err = e.what();
    return 3;
  } catch (const cpd::NumericError& e) {
    g_err = e.what();
    return 4;
  } catch (const cpd::DomainError& e) {
    g_err = e.what();
    return 5;
  } catch (const cpd::ParseError& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 6;
  }
}

cpd::FactorList factor_list(int N, const int64_t* dims, int64_t R, const double* const* f) {
  cpd::FactorList out;
  for (int m = 0; m < N; ++m) {
    Eigen::MatrixXd a(dims[m], R);
    std::memcpy(a.data(), f[m], static_cast<size_t>(dims[m] * R) * sizeof(double));
    out.push_back(std::move(a));
  }
  return out;
}

// A tensor split into `parts` slabs of its first (axis 0) or last (axis 1) mode,
// one reference call per slab on its own thread (the reference code is
// single-threaded): the slab gradients of the other modes sum exactly, the rows
// of the split mode's gradient stay with their slab.
struct RefTensor {
  std::vector<int64_t> dims;
  int axis = 1;
  std::vector<cpd::DenseTensor> slabs;
  std::vector<int64_t> lo;  // first index of each slab along the split mode
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_tensor_new(int N, const int64_t* dims, const double* values, int parts, int axis) {
  auto* t = new RefTensor();
  const int st = guarded([&] {
    t->dims.assign(dims, dims + N);
    t->axis = axis ? 1 : 0;
    const int m = t->axis ? N - 1 : 0;
    const int64_t I = dims[m];
    int64_t front = 1;  // entries per index of the split mode (last) / its stride (first)
    for (int k = 0; k + 1 < N; ++k) front *= dims[k];
    const int64_t total = front * dims[N - 1];
    if (parts < 1) parts = 1;
    if (parts > I) parts = static_cast<int>(I);
    for (int k = 0; k < parts; ++k) {
      const int64_t a = I * k / parts, b = I * (k + 1) / parts;
      std::vector<int64_t> d(dims, dims + N);
      d[static_cast<size_t>(m)] = b - a;
      std::vector<double> v;
      if (t->axis) {
        v.assign(values + a * front, values + b * front);
      } else {  // rows [a, b) of mode 1 from every mode-1 fibre
        v.resize(static_cast<size_t>((b - a) * (total / I)));
        for (int64_t f = 0, at = 0; f < total / I; ++f, at += b - a)
          std::copy(values + f * I + a, values + f * I + b, v.begin() + at);
      }
      t->slabs.emplace_back(cpd::Shape(d), std::move(v));
      t->lo.push_back(a);
    }
  });
  if (st != 0) {
    delete t;
    return nullptr;
  }
  return t;
}

void ref_tensor_free(void* h) { delete static_cast<RefTensor*>(h); }

// cp_gradient_all (mttkrp.hpp:59-69) of the whole tensor: one reference call per
// slab (parallel threads), combined as above; mults = the counters' total.
int ref_cp_gradient_all(void* h, int64_t R, const double* const* factors, double* const* grads, uint64_t* mults) {
  return guarded([&] {
    auto* t = static_cast<RefTensor*>(h);
    const int N = static_cast<int>(t->dims.size());
    const size_t P = t->slabs.size();
    std::vector<std::vector<Eigen::MatrixXd>> out(P);
    std::vector<uint64_t> cnt(P, 0);
    std::vector<int> status(P, 0);
    std::vector<std::string> errs(P);
    const int m = t->axis ? N - 1 : 0;  // the split mode
    auto work = [&](size_t k) {
      status[k] = guarded([&] {
        std::vector<int64_t> d = t->dims;
        const int64_t rows = t->slabs[k].shape().dim(m + 1), I = t->dims[static_cast<size_t>(m)];
        d[static_cast<size_t>(m)] = rows;
        std::vector<const double*> fk(factors, factors + N);
        std::vector<double> part(static_cast<size_t>(rows * R));
        for (int64_t r = 0; r < R; ++r)
          std::memcpy(part.data() + r * rows, factors[m] + r * I + t->lo[k], static_cast<size_t>(rows) * sizeof(double));
        fk[static_cast<size_t>(m)] = part.data();
        cpd::FactorList fl = factor_list(N, d.data(), R, fk.data());
        cpd::CostCounter c;
        out[k] = cpd::cp_gradient_all(t->slabs[k], fl, &c);
        cnt[k] = c.total();
      });
      if (status[k]) errs[k] = g_err;
    };
    if (P == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (size_t k = 0; k < P; ++k) th.emplace_back(work, k);
      for (auto& x : th) x.join();
    }
    for (size_t k = 0; k < P; ++k)
      if (status[k]) {
        g_err = errs[k];
        throw std::runtime_error(errs[k]);
      }
    for (int n = 0; n < N; ++n)
      std::memset(grads[n], 0, static_cast<size_t>(t->dims[static_cast<size_t>(n)] * R) * sizeof(double));
    uint64_t total = 0;
    for (size_t k = 0; k < P; ++k) {
      for (int n = 0; n < N; ++n) {
        const Eigen::MatrixXd& G = out[k][static_cast<size_t>(n)];
        if (n != m) {
          for (int64_t e = 0; e < G.size(); ++e) grads[n][e] += G.data()[e];
        } else {
          const int64_t I = t->dims[static_cast<size_t>(m)];
          for (int64_t r = 0; r < R; ++r)
            for (int64_t i = 0; i < G.rows(); ++i) grads[n][r * I + t->lo[k] + i] = G(i, r);
        }
      }
      total += cnt[k];
    }
    if (mults) *mults = total;
  });
}

// Seconds per cp_gradient_all call over `reps` calls (the timed window holds the
// reference calls only, as run() times its sweeps: als.cpp:176-192).
int ref_time_cp_gradient_all(void* h, int64_t R, const double* const* factors, double* const* grads, int reps,
                             double* seconds) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) {
    const int st = ref_cp_gradient_all(h, R, factors, grads, nullptr);
    if (st) return st;
  }
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
  return 0;
}

// als_sweep_fast (als.hpp:62-66) on the whole tensor (one slab), factors in place.
int ref_als_sweep_fast(void* h, int64_t R, double* const* factors, double rtol, uint64_t* mults, double* seconds) {
  return guarded([&] {
    auto* t = static_cast<RefTensor*>(h);
    if (t->slabs.size() != 1) throw cpd::ArgumentError("ref_als_sweep_fast: needs a one-slab tensor");
    const int N = static_cast<int>(t->dims.size());
    cpd::FactorList fl = factor_list(N, t->dims.data(), R, factors);
    cpd::CostCounter c;
    const auto t0 = std::chrono::steady_clock::now();
    cpd::als_sweep_fast(t->slabs[0], fl, rtol, &c);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int m = 0; m < N; ++m)
      std::memcpy(factors[m], fl[static_cast<size_t>(m)].data(),
                  static_cast<size_t>(t->dims[static_cast<size_t>(m)] * R) * sizeof(double));
    if (mults) *mults = c.total();
  });
}

// run() (als.hpp:88-93) with `algo` (Algorithm order) and the reference trace.
int ref_run(void* h, int64_t R, double* const* factors, int algo, int pivot_order, int max_iters, double tol,
            double* cost, double* rel, int* iters) {
  return guarded([&] {
    auto* t = static_cast<RefTensor*>(h);
    if (t->slabs.size() != 1) throw cpd::ArgumentError("ref_run: needs a one-slab tensor");
    const int N = static_cast<int>(t->dims.size());
    cpd::KruskalModel init(factor_list(N, t->dims.data(), R, factors));
    cpd::SolveOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.order = pivot_order ? cpd::UpdateOrder::pivot : cpd::UpdateOrder::standard;
    const cpd::SolveResult res = cpd::run(t->slabs[0], init, static_cast<cpd::Algorithm>(algo), o);
    *iters = res.trace.iters_run;
    for (int i = 0; i < res.trace.iters_run; ++i) {
      cost[i] = res.trace.cost[static_cast<size_t>(i)];
      rel[i] = res.trace.rel_error[static_cast<size_t>(i)];
    }
    for (int m = 0; m < N; ++m)
      std::memcpy(factors[m], res.model.factor(m + 1).data(),
                  static_cast<size_t>(t->dims[static_cast<size_t>(m)] * R) * sizeof(double));
  });
}

int ref_mttkrp_direct(void* h, int64_t R, const double* const* factors, int n, double* out) {
  return guarded([&] {
    auto* t = static_cast<RefTensor*>(h);
    if (t->slabs.size() != 1) throw cpd::ArgumentError("ref_mttkrp_direct: needs a one-slab tensor");
    const int N = static_cast<int>(t->dims.size());
    const Eigen::MatrixXd m = cpd::mttkrp_direct(t->slabs[0], factor_list(N, t->dims.data(), R, factors), n);
    std::memcpy(out, m.data(), static_cast<size_t>(m.size()) * sizeof(double));
  });
}

int ref_select_pivot(int N, const int64_t* dims, int* out) {
  return guarded([&] { *out = cpd::select_pivot(cpd::Shape(std::vector<int64_t>(dims, dims + N))); });
}

int ref_counts(int N, const int64_t* dims, int64_t R, int n, uint64_t* direct, uint64_t* fast, uint64_t* derived,
               uint64_t* realized) {
  return guarded([&] {
    const cpd::Shape s(std::vector<int64_t>(dims, dims + N));
    *direct = cpd::predicted_mult_count(s, R, n, cpd::CountVariant::direct);
    *fast = cpd::predicted_mult_count(s, R, n, cpd::CountVariant::fast);
    *derived = cpd::predicted_mult_count(s, R, n, cpd::CountVariant::fast_derived);
    *realized = cpd::fast_count_realized(s, R, n);
  });
}

int ref_pinv_psd(int64_t n, const double* s, double rtol, double* out) {
  return guarded([&] {
    Eigen::MatrixXd m(n, n);
    std::memcpy(m.data(), s, static_cast<size_t>(n * n) * sizeof(double));
    const Eigen::MatrixXd p = cpd::pinv_psd(m, rtol);
    std::memcpy(out, p.data(), static_cast<size_t>(n * n) * sizeof(double));
  });
}

}  // extern "C"
