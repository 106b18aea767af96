"""The other consumers of the gradient on the device:
multiplicative updates (mu_sweep, als.cpp:80-91), gradient descent (gd_step,
als.cpp:93-101), the direct ALS engine, and run() for every Algorithm
(als.cpp:147-210) — against the oracle's restatements and the reference's own
test expectations (test_als.cpp:114-245)."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_mu_sweep_matches_oracle(gpu_ctx, oracle):
    dims = [4, 3, 5]
    yv = oracle.random_tensor(dims, 61)  # uniform(0,1): nonnegative
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    f = oracle.random_factors(dims, 3, 62)
    g = [a.copy() for a in f]
    for _ in range(5):
        f, _ = oracle.mu_sweep(yv, dims, f)
        cpd.mu_sweep(y, g)
        assert all((a >= 0).all() for a in g)
    for a, b in zip(g, f):
        assert rel(a, b) <= 1e-10


def test_mu_sweep_errors(gpu_ctx, oracle):
    dims = [3, 4, 3]
    t = oracle.random_factors(dims, 2, 63)
    yt = oracle.full(dims, t)
    bad = yt.copy()
    bad[0] = -bad[0]
    with pytest.raises(cpd.DomainError):
        cpd.mu_sweep(cpd.DenseTensor.from_values(bad, dims, ctx=gpu_ctx), [a.copy() for a in t])
    fneg = [a.copy() for a in t]
    fneg[1][0, 0] = -1.0
    y = cpd.DenseTensor.from_values(yt, dims, ctx=gpu_ctx)
    with pytest.raises(cpd.DomainError):
        cpd.mu_sweep(y, fneg)
    with pytest.raises(cpd.ArgumentError):
        cpd.mu_sweep(y, [a.copy() for a in t], eps=-1e-3)
    t2 = [a.copy() for a in t]  # exact nonnegative fit is (nearly) a fixed point
    cpd.mu_sweep(y, t2)
    for a, b in zip(t2, t):
        assert rel(a, b) < 1e-9


def test_gd_step_matches_oracle(gpu_ctx, oracle):
    dims = [3, 4, 4]
    yv = oracle.random_tensor(dims, 71)
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    f = oracle.random_factors(dims, 2, 72)
    frozen = [a.copy() for a in f]
    cpd.gd_step(y, frozen, 0.0)
    for a, b in zip(frozen, f):
        assert np.abs(a - b).max() == 0.0
    with pytest.raises(cpd.ArgumentError):
        cpd.gd_step(y, [a.copy() for a in f], -1e-6)
    g = [a.copy() for a in f]
    cpd.gd_step(y, g, 1e-4)
    want, _ = oracle.gd_step(yv, dims, f, 1e-4)
    for a, b in zip(g, want):
        assert rel(a, b) <= 1e-12
    assert oracle.cost(yv, dims, g) < oracle.cost(yv, dims, f)


@pytest.mark.parametrize("algo", ["als_direct", "als_fast", "mu", "gd"])
@pytest.mark.parametrize("dims", [[4, 3, 5], [12, 10, 14, 9]])
def test_run_every_algorithm_matches_oracle(gpu_ctx, oracle, algo, dims):
    yv = oracle.random_tensor(dims, 91)
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    init = oracle.random_factors(dims, 2, 92)
    opts = cpd.SolveOptions(max_iters=6, gd_eta=1e-4)
    c = cpd.CostCounter()
    res = cpd.run(y, init, opts, counter=c, algo=algo)
    _, tr = oracle.run(yv, dims, init, algo, max_iters=6, gd_eta=1e-4)
    assert res.trace.iters_run == 6
    assert np.allclose(res.trace.rel_error, tr["rel_error"], rtol=1e-9, atol=1e-12), (res.trace.rel_error, tr)
    assert res.trace.mults == tr["mults"]
    assert all(s > 0 for s in res.trace.seconds)


def test_run_fast_equals_direct_pivot_on_unsorted(gpu_ctx, oracle):
    dims = [5, 3, 4]  # test_als.cpp:223-238
    yv = oracle.random_tensor(dims, 101)
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    init = oracle.random_factors(dims, 2, 102)
    fast = cpd.run(y, init, cpd.SolveOptions(max_iters=6))
    direct = cpd.run(y, init, cpd.SolveOptions(max_iters=6, order="pivot"), algo="als_direct")
    for a, b in zip(fast.factors, direct.factors):
        assert rel(a, b) < 1e-10
    assert np.allclose(fast.trace.cost, direct.trace.cost, rtol=1e-10)
