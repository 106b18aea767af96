// C++ drop-in adapter tests (include/cpd_gpu/cpd.hpp over libcpdgpu.so), written
// the way the reference's own C++ tests are: known answers, fast == brute,
// permutation equivariance, the Gauss-Seidel hook contract, counts, ALS
// behaviour (/root/reference/proj/core/tests/test_mttkrp.cpp, test_counts.cpp,
// test_als.cpp).  The brute-force MTTKRP below is test infrastructure, not the
// product.  Needs a B200; driven by tests/test_cpp_adapter.py (marked gpu).
#include <cpd_gpu/cpd.hpp>

#include <cstdio>
#include <cstdlib>
#include <string>

namespace {

int g_failed = 0;
int g_checks = 0;

#define CHECK_LT(a, b)                                                                  \
  do {                                                                                  \
    ++g_checks;                                                                         \
    const double va_ = (a), vb_ = (b);                                                  \
    if (!(va_ < vb_)) {                                                                 \
      ++g_failed;                                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s = %.3e !< %.3e\n", __FILE__, __LINE__, #a, va_, vb_); \
    }                                                                                   \
  } while (0)

#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_failed;                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                   \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

std::uint64_t mix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
double unif(std::uint64_t seed, std::uint64_t i) {
  return static_cast<double>(mix(mix(seed) + i) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

cpd::DenseTensor random_tensor(const std::vector<cpd::index_t>& dims, std::uint64_t seed) {
  cpd::Shape s(dims);
  std::vector<double> v(static_cast<size_t>(s.num_entries()));
  for (size_t i = 0; i < v.size(); ++i) v[i] = unif(seed, i);
  return cpd::DenseTensor(s, std::move(v));
}
cpd::FactorList random_factors(const std::vector<cpd::index_t>& dims, cpd::index_t R, std::uint64_t seed) {
  cpd::FactorList f;
  for (size_t k = 0; k < dims.size(); ++k) {
    cpd::Matrix a(dims[k], R);
    for (cpd::index_t i = 0; i < dims[k] * R; ++i) a.data()[i] = unif(seed * 31 + k, static_cast<std::uint64_t>(i));
    f.push_back(a);
  }
  return f;
}

// Brute force G(n)[i, r] = sum over all entries with i_n = i of y * prod_{m != n} A_m[i_m, r].
cpd::Matrix brute(const cpd::DenseTensor& y, const cpd::FactorList& f, int n) {
  const auto& d = y.shape().dims();
  const cpd::index_t R = f[0].cols();
  cpd::Matrix g(d[static_cast<size_t>(n - 1)], R);
  std::vector<cpd::index_t> idx(d.size(), 0);
  for (cpd::index_t e = 0; e < y.size(); ++e) {
    cpd::index_t rem = e;
    for (size_t k = 0; k < d.size(); ++k) {
      idx[k] = rem % d[k];
      rem /= d[k];
    }
    for (cpd::index_t r = 0; r < R; ++r) {
      double p = y.data()[e];
      for (size_t k = 0; k < d.size(); ++k)
        if (static_cast<int>(k) != n - 1) p *= f[k](idx[k], r);
      g(idx[static_cast<size_t>(n - 1)], r) += p;
    }
  }
  return g;
}

double max_rel_diff(const cpd::Matrix& a, const cpd::Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return 1e300;
  double num = 0.0, den = 0.0;
  for (cpd::index_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a.data()[i] - b.data()[i]));
    den = std::max(den, std::abs(b.data()[i]));
  }
  return den > 0 ? num / den : num;
}

void test_ladder_kat() {  // test_mttkrp.cpp:13-35
  std::vector<double> v(8);
  for (int i = 0; i < 8; ++i) v[static_cast<size_t>(i)] = i + 1;
  cpd::DenseTensor y(cpd::Shape({2, 2, 2}), v);
  cpd::FactorList f(3, cpd::Matrix::Ones(2, 2));
  auto g = cpd::cp_gradient_all(y, f);
  const double want[3][2] = {{16, 20}, {14, 22}, {10, 26}};
  for (int n = 0; n < 3; ++n)
    for (int r = 0; r < 2; ++r)
      for (int i = 0; i < 2; ++i) CHECK(g[static_cast<size_t>(n)](i, r) == want[n][i]);
}

void test_unit_basis() {  // test_mttkrp.cpp:37-51
  std::vector<double> v(8);
  for (int i = 0; i < 8; ++i) v[static_cast<size_t>(i)] = i + 1;
  cpd::DenseTensor y(cpd::Shape({2, 2, 2}), v);
  cpd::Matrix e1(2, 1);
  e1(0, 0) = 1.0;
  auto g = cpd::cp_gradient_all(y, cpd::FactorList(3, e1));
  CHECK(g[0](0, 0) == 1.0 && g[0](1, 0) == 2.0);
  CHECK(g[2](0, 0) == 1.0 && g[2](1, 0) == 5.0);
}

void test_ordering_kats() {  // test_mttkrp.cpp:62-100, 151-157
  CHECK(cpd::select_pivot(cpd::Shape({10, 10, 10})) == 1);
  CHECK(cpd::select_pivot(cpd::Shape({10, 10, 10, 10})) == 2);
  CHECK(cpd::select_pivot(cpd::Shape({2, 3, 4, 5})) == 2);
  CHECK(cpd::select_pivot(cpd::Shape({3, 5})) == 1);
  CHECK(cpd::select_pivot(cpd::Shape({2, 2, 3, 3, 4})) == 3);
  CHECK(throws<cpd::ArgumentError>([] { cpd::select_pivot(cpd::Shape({7})); }));
  auto o = cpd::sort_mode_order(cpd::Shape({5, 3, 4}));
  CHECK((o.perm == std::vector<int>{2, 3, 1}) && (o.inverse == std::vector<int>{3, 1, 2}));
  CHECK((cpd::sort_mode_order(cpd::Shape({4, 4, 4})).perm == std::vector<int>{1, 2, 3}));
  CHECK((cpd::fast_update_order(cpd::Shape({2, 3, 4, 5})) == std::vector<int>{2, 1, 3, 4}));
  CHECK((cpd::fast_update_order(cpd::Shape({10, 10, 10})) == std::vector<int>{1, 2, 3}));
  CHECK((cpd::fast_update_order(cpd::Shape({5, 3, 4})) == std::vector<int>{2, 3, 1}));
}

void test_fast_equals_brute() {  // test_mttkrp.cpp:102-119
  const std::vector<std::vector<cpd::index_t>> shapes = {{2, 3, 4}, {4, 3, 2}, {3, 1, 4}, {2, 2},
                                                          {2, 3, 2, 4}, {1, 5, 2}, {6, 6}, {7, 5, 9, 4}};
  for (const auto& d : shapes)
    for (cpd::index_t R : {1, 3, 17}) {
      auto y = random_tensor(d, 100 + static_cast<std::uint64_t>(R));
      auto f = random_factors(d, R, 200 + static_cast<std::uint64_t>(R));
      auto g = cpd::cp_gradient_all(y, f);
      for (int n = 1; n <= static_cast<int>(d.size()); ++n)
        CHECK_LT(max_rel_diff(g[static_cast<size_t>(n - 1)], brute(y, f, n)), 1e-12);
    }
}

void test_permutation_equivariance() {  // test_mttkrp.cpp:121-136
  const std::vector<cpd::index_t> d = {3, 4, 2, 3};
  auto y = random_tensor(d, 301);
  auto f = random_factors(d, 2, 302);
  auto base = cpd::cp_gradient_all(y, f);
  const int perm[4] = {3, 1, 4, 2};
  std::vector<cpd::index_t> pd;
  for (int p : perm) pd.push_back(d[static_cast<size_t>(p - 1)]);
  cpd::Shape ps(pd);
  std::vector<double> pv(static_cast<size_t>(y.size()));
  for (cpd::index_t e = 0; e < y.size(); ++e) {  // permuted entry e -> source index
    cpd::index_t rem = e, src = 0;
    std::vector<cpd::index_t> idx(4);
    for (int k = 0; k < 4; ++k) {
      idx[static_cast<size_t>(perm[k] - 1)] = rem % pd[static_cast<size_t>(k)];
      rem /= pd[static_cast<size_t>(k)];
    }
    for (int k = 3; k >= 0; --k) src = src * d[static_cast<size_t>(k)] + idx[static_cast<size_t>(k)];
    pv[static_cast<size_t>(e)] = y.data()[src];
  }
  cpd::FactorList pf;
  for (int p : perm) pf.push_back(f[static_cast<size_t>(p - 1)]);
  auto moved = cpd::cp_gradient_all(cpd::DenseTensor(ps, pv), pf);
  for (int k = 0; k < 4; ++k) CHECK_LT(max_rel_diff(moved[static_cast<size_t>(k)], base[static_cast<size_t>(perm[k] - 1)]), 1e-12);
}

void test_hook_gauss_seidel() {  // test_mttkrp.cpp:159-186
  const std::vector<cpd::index_t> d = {3, 4, 2, 3};
  auto y = random_tensor(d, 501);
  auto f0 = random_factors(d, 2, 502);
  cpd::FactorList ref = f0;
  std::vector<cpd::Matrix> ref_grad(4);
  for (int n : cpd::fast_update_order(y.shape())) {
    ref_grad[static_cast<size_t>(n - 1)] = brute(y, ref, n);
    ref[static_cast<size_t>(n - 1)] = random_factors(d, 2, 600 + static_cast<std::uint64_t>(n))[static_cast<size_t>(n - 1)];
  }
  cpd::FactorList f = f0;
  std::vector<cpd::Matrix> got(4);
  std::vector<int> visited;
  cpd::cp_gradient_all(y, f, nullptr, [&](int n, const cpd::Matrix& g) {
    visited.push_back(n);
    got[static_cast<size_t>(n - 1)] = g;
    f[static_cast<size_t>(n - 1)] = random_factors(d, 2, 600 + static_cast<std::uint64_t>(n))[static_cast<size_t>(n - 1)];
  }, nullptr);
  CHECK(visited == cpd::fast_update_order(y.shape()));
  for (int n = 0; n < 4; ++n) {
    CHECK_LT(max_rel_diff(got[static_cast<size_t>(n)], ref_grad[static_cast<size_t>(n)]), 1e-12);
    CHECK(max_rel_diff(f[static_cast<size_t>(n)], ref[static_cast<size_t>(n)]) == 0.0);
  }
  // a hook that leaves a factor of the wrong size is a ShapeError
  cpd::FactorList bad = f0;
  CHECK(throws<cpd::ShapeError>([&] {
    cpd::cp_gradient_all(y, bad, nullptr, [&](int n, const cpd::Matrix&) { bad[static_cast<size_t>(n - 1)] = cpd::Matrix(1, 1); }, nullptr);
  }));
  // whatever the hook throws reaches the caller unchanged, as the reference's direct
  // hook(orig, G) call propagates it (mttkrp.cpp:134-145): reference types, user types,
  // non-std exceptions; the context stays usable afterwards
  struct UserError {
    int code;
  };
  cpd::FactorList h = f0;
  CHECK(throws<cpd::DomainError>([&] {
    cpd::cp_gradient_all(y, h, nullptr, [](int, const cpd::Matrix&) { throw cpd::DomainError("hook domain"); }, nullptr);
  }));
  CHECK(throws<cpd::ParseError>([&] {
    cpd::cp_gradient_all(y, h, nullptr, [](int, const cpd::Matrix&) { throw cpd::ParseError("hook parse"); }, nullptr);
  }));
  int caught = 0;
  try {
    cpd::cp_gradient_all(y, h, nullptr, [](int n, const cpd::Matrix&) { throw UserError{n}; }, nullptr);
  } catch (const UserError& e) {
    caught = e.code;
  }
  CHECK(caught == cpd::fast_update_order(y.shape()).front());
  CHECK_LT(max_rel_diff(cpd::cp_gradient_all(y, f0)[0], brute(y, f0, 1)), 1e-12);
}

void test_counts_and_workspace() {  // test_counts.cpp:16-31, test_mttkrp.cpp:188-198
  const std::vector<cpd::index_t> d = {4, 5, 6, 7};
  auto y = random_tensor(d, 601);
  auto f = random_factors(d, 3, 602);
  cpd::CostCounter c;
  cpd::FastStats st;
  cpd::cp_gradient_all(y, f, &c, &st);
  std::uint64_t want = 0;
  for (int n = 1; n <= 4; ++n) want += cpd::fast_count_realized(y.shape(), 3, n);
  CHECK(c.total() == want);
  const cpd::index_t J = 4 * 5, big = std::max<cpd::index_t>(J, 6 * 7);
  CHECK(st.peak_workspace_doubles > 0 && st.peak_workspace_doubles <= 2 * 3 * big + big);
  // the device's own workspace (bytes in use / high-water mark) is reported beside it
  const auto ws = cpd::gpu::device_workspace();
  CHECK(ws.peak_bytes >= ws.current_bytes && ws.peak_bytes >= 8 * st.peak_workspace_doubles);
  // per-mode charges land before the hook
  cpd::CostCounter c2;
  std::vector<std::uint64_t> seen;
  cpd::FactorList f2 = f;
  cpd::cp_gradient_all(y, f2, &c2, [&](int, const cpd::Matrix&) { seen.push_back(c2.total()); }, nullptr);
  CHECK(seen.size() == 4 && seen.back() == want);
  std::uint64_t acc = 0;
  auto order = cpd::fast_update_order(y.shape());
  for (size_t k = 0; k < order.size(); ++k) {
    acc += cpd::fast_count_realized(y.shape(), 3, order[k]);
    CHECK(seen[k] == acc);
  }
  CHECK(throws<cpd::IndexError>([&] { cpd::fast_count_realized(y.shape(), 3, 0); }));
}

void test_direct() {  // mttkrp_direct (test_mttkrp.cpp-style: equals brute force for every mode)
  const std::vector<cpd::index_t> d = {5, 4, 6, 3};
  auto y = random_tensor(d, 77);
  auto f = random_factors(d, 4, 78);
  for (int n = 1; n <= 4; ++n) CHECK_LT(max_rel_diff(cpd::mttkrp_direct(y, f, n), brute(y, f, n)), 1e-12);
  CHECK(throws<cpd::IndexError>([&] { cpd::mttkrp_direct(y, f, 5); }));
  cpd::FactorList a = f, b = f;
  cpd::als_sweep_direct(y, a, {1, 2, 3, 4});
  for (int n = 1; n <= 4; ++n) b[static_cast<size_t>(n - 1)] = cpd::als_update_mode(brute(y, b, n), b, n);
  for (int k = 0; k < 4; ++k) CHECK_LT(max_rel_diff(a[static_cast<size_t>(k)], b[static_cast<size_t>(k)]), 1e-10);
}

void test_errors() {  // errors.hpp mapping
  auto y = random_tensor({3, 4, 5}, 7);
  auto f = random_factors({3, 4, 6}, 2, 8);
  CHECK(throws<cpd::ShapeError>([&] { cpd::cp_gradient_all(y, f); }));
  CHECK(throws<cpd::ShapeError>([] { cpd::Shape({3, 0}); }));
  CHECK(throws<cpd::ShapeError>([] { cpd::pinv_psd(cpd::Matrix(2, 3)); }));
  CHECK(throws<cpd::ArgumentError>([] { cpd::pinv_psd(cpd::Matrix::Identity(2, 2), -1.0); }));
}

void test_pinv_and_als() {  // test_als.cpp
  cpd::Matrix s(2, 2);
  s(0, 0) = 4.0;
  s(1, 1) = 0.25;
  auto p = cpd::pinv_psd(s);
  CHECK(std::abs(p(0, 0) - 0.25) < 1e-15 && std::abs(p(1, 1) - 4.0) < 1e-14 && p(0, 1) == 0.0);
  cpd::Matrix z(2, 2);
  auto pz = cpd::pinv_psd(z);
  CHECK(pz(0, 0) == 0.0 && pz(1, 1) == 0.0);

  // exact rank-2 tensor is recovered by the fast engine
  const std::vector<cpd::index_t> d = {6, 7, 8, 5};
  auto truth = random_factors(d, 2, 901);
  cpd::Shape sh(d);
  std::vector<double> v(static_cast<size_t>(sh.num_entries()), 0.0);
  for (cpd::index_t e = 0; e < sh.num_entries(); ++e) {
    cpd::index_t rem = e;
    std::vector<cpd::index_t> idx(4);
    for (int k = 0; k < 4; ++k) {
      idx[static_cast<size_t>(k)] = rem % d[static_cast<size_t>(k)];
      rem /= d[static_cast<size_t>(k)];
    }
    for (int r = 0; r < 2; ++r) {
      double prod = 1.0;
      for (int k = 0; k < 4; ++k) prod *= truth[static_cast<size_t>(k)](idx[static_cast<size_t>(k)], r);
      v[static_cast<size_t>(e)] += prod;
    }
  }
  cpd::DenseTensor y(sh, v);
  cpd::SolveOptions opt;
  opt.max_iters = 200;
  opt.tol = 0.0;
  cpd::CostCounter c;
  auto res = cpd::run(y, cpd::KruskalModel(random_factors(d, 2, 902)), cpd::Algorithm::als_fast, opt, &c);
  CHECK(res.trace.iters_run == 200);
  CHECK(res.trace.rel_error.back() < 1e-8);
  // monotone up to the rounding of the Gram-identity fit (|Y|^2 - 2<Y,Yhat> + |Yhat|^2)
  const double y2 = y.norm() * y.norm();
  for (size_t i = 1; i < res.trace.cost.size(); ++i) CHECK(res.trace.cost[i] <= res.trace.cost[i - 1] + 1e-12 * y2);
  CHECK(c.total() == res.trace.mults.back() && c.total() > 0);
  // every Algorithm runs and fills the trace (test_als.cpp:198-221)
  for (auto algo : {cpd::Algorithm::als_direct, cpd::Algorithm::als_fast, cpd::Algorithm::mu, cpd::Algorithm::gd}) {
    cpd::SolveOptions o;
    o.max_iters = 4;
    o.gd_eta = 1e-4;
    cpd::FactorList pos = random_factors(d, 2, 905);
    for (auto& a : pos)
      for (cpd::index_t i = 0; i < a.size(); ++i) a.data()[i] = std::abs(a.data()[i]);
    std::vector<double> vy(y.values());
    for (auto& v : vy) v = std::abs(v);
    cpd::DenseTensor ypos(y.shape(), vy);
    auto r = cpd::run(ypos, cpd::KruskalModel(pos), algo, o);
    CHECK(r.trace.iters_run == 4 && r.trace.rel_error.size() == 4);
    for (size_t i = 0; i < 4; ++i)
      CHECK(std::abs(r.trace.rel_error[i] - std::sqrt(r.trace.cost[i]) / ypos.norm()) <= 1e-12 * r.trace.rel_error[i]);
  }

  // one sweep: als_sweep_fast == gradient + als_update_mode in Gauss-Seidel order
  cpd::FactorList a = random_factors(d, 3, 903), b = a;
  cpd::als_sweep_fast(y, a);
  cpd::cp_gradient_all(y, b, nullptr, [&](int n, const cpd::Matrix& g) {
    b[static_cast<size_t>(n - 1)] = cpd::als_update_mode(g, b, n);
  }, nullptr);
  for (int k = 0; k < 4; ++k) CHECK_LT(max_rel_diff(a[static_cast<size_t>(k)], b[static_cast<size_t>(k)]), 1e-10);
}

// sort_modes / random_init / standard_order / predicted_mult_count (mttkrp.hpp:28-35,76-86;
// als.hpp:84-87) and the sharded gradient on one rank (host communicator)
int host_sum(void*, double*, int64_t) { return 0; }  // world size 1: the sum is the local buffer

void test_helpers_and_sharded() {
  const std::vector<cpd::index_t> d{4, 2, 5, 3};
  cpd::DenseTensor y = random_tensor(d, 77);
  cpd::FactorList f = random_factors(d, 3, 78);
  cpd::SortResult s = cpd::sort_modes(y, f);
  CHECK((s.perm == std::vector<int>{2, 4, 1, 3}));
  CHECK((s.inverse == std::vector<int>{3, 1, 4, 2}));
  CHECK((s.tensor.shape().dims() == std::vector<cpd::index_t>{2, 3, 4, 5}));
  // entry (i2, i4, i1, i3) of the sorted tensor is y(i1, i2, i3, i4)
  CHECK(s.tensor.data()[1 + 2 * (2 + 3 * (3 + 4 * 4))] == y.data()[3 + 4 * (1 + 2 * (4 + 5 * 2))]);
  auto gs = cpd::cp_gradient_all(s.tensor, s.factors);
  auto g = cpd::cp_gradient_all(y, f);
  for (int j = 1; j <= 4; ++j)
    CHECK_LT(max_rel_diff(gs[static_cast<size_t>(j - 1)], g[static_cast<size_t>(s.perm[static_cast<size_t>(j - 1)] - 1)]), 1e-13);

  const cpd::KruskalModel m = cpd::random_init(cpd::Shape({2, 3}), 2, 5);
  CHECK(m.order() == 2 && m.rank() == 2 && m.factor(2).rows() == 3);
  for (int n = 1; n <= 2; ++n)
    for (cpd::index_t i = 0; i < m.factor(n).size(); ++i)
      CHECK(m.factor(n).data()[i] >= 0.0 && m.factor(n).data()[i] < 1.0);
  CHECK(throws<cpd::ArgumentError>([] { cpd::random_init(cpd::Shape({2, 3}), 0, 5); }));
  CHECK((cpd::standard_order(3) == std::vector<int>{1, 2, 3}));

  const cpd::Shape asc({2, 3, 4, 5});
  for (int n = 1; n <= 4; ++n) {
    CHECK(cpd::predicted_mult_count(asc, 3, n, cpd::CountVariant::fast) <=
          cpd::predicted_mult_count(asc, 3, n, cpd::CountVariant::direct));
    CHECK(cpd::predicted_mult_count(asc, 3, n, cpd::CountVariant::fast_derived) <=
          cpd::predicted_mult_count(asc, 3, n, cpd::CountVariant::fast));
  }
  CHECK(throws<cpd::IndexError>([&] { cpd::predicted_mult_count(asc, 3, 5, cpd::CountVariant::fast); }));
  CHECK(throws<cpd::ArgumentError>([] { cpd::predicted_mult_count(cpd::Shape({3, 2}), 3, 1, cpd::CountVariant::fast); }));

  // sharded gradient, world size 1: equals the plain one
  const std::vector<cpd::index_t> ad{3, 4, 5, 6};
  cpd::DenseTensor ya = random_tensor(ad, 91);
  cpd::FactorList fa = random_factors(ad, 4, 92);
  cpd::gpu::comm_init_host(1, 0, host_sum, nullptr);
  const auto b = cpd::gpu::slab_bounds(6, 1, 0);
  CHECK(b.first == 0 && b.second == 6);
  cpd::CostCounter cs, cp;
  auto gsh = cpd::cp_gradient_all_sharded(ya, ya.shape(), fa, &cs);
  auto gpl = cpd::cp_gradient_all(ya, fa, &cp);
  for (int k = 0; k < 4; ++k) CHECK_LT(max_rel_diff(gsh[static_cast<size_t>(k)], gpl[static_cast<size_t>(k)]), 1e-13);
  CHECK(cs.total() == cp.total());
  // sharded ALS sweep, world size 1: equals the plain sweep
  cpd::FactorList fs = fa, fp = fa;
  cpd::CostCounter ss, sp;
  const double cost = cpd::als_sweep_fast_sharded(ya, ya.shape(), fs, 1e-12, &ss);
  cpd::als_sweep_fast(ya, fp, 1e-12, &sp);
  for (int k = 0; k < 4; ++k) CHECK_LT(max_rel_diff(fs[static_cast<size_t>(k)], fp[static_cast<size_t>(k)]), 1e-11);
  CHECK(ss.total() == sp.total());
  CHECK(cost >= 0.0);
  cpd::gpu::comm_destroy();
  CHECK(throws<cpd::ArgumentError>([&] { cpd::cp_gradient_all_sharded(ya, ya.shape(), fa); }));  // no communicator
}

}  // namespace

int main() {
  try {
    test_ladder_kat();
    test_unit_basis();
    test_ordering_kats();
    test_fast_equals_brute();
    test_permutation_equivariance();
    test_hook_gauss_seidel();
    test_counts_and_workspace();
    test_errors();
    test_direct();
    test_pinv_and_als();
    test_helpers_and_sharded();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed ? 1 : 0;
}
