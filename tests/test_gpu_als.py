"""GPU parity of the fast CP_ALS path (pinv_psd, als_update_mode, als_sweep_fast,
run) through the C-ABI.  Mirrors proj/tests/test_als.cpp and acceptance
criterion 5 (acceptance_main.cpp:301-363), plus BASELINE config 4's shape
(rank-16 model + 20 dB noise, per-sweep fit against the oracle)."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def max_rel_diff(a, b):
    scale = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), 1e-30)
    return float(np.abs(np.asarray(a) - np.asarray(b)).max(initial=0.0) / scale)


def tensor(ctx, values, dims):
    return cpd.DenseTensor.from_values(values, dims, ctx=ctx)


def test_pinv_psd(gpu_ctx, oracle):
    # test_als.cpp:21-43
    eye = np.eye(4)
    assert max_rel_diff(cpd.pinv_psd(eye, ctx=gpu_ctx), eye) < 1e-14
    d = np.zeros((2, 2))
    d[0, 0] = 2.0
    dp = cpd.pinv_psd(d, ctx=gpu_ctx)
    assert abs(dp[0, 0] - 0.5) <= 0.5 * 1e-14
    assert dp[1, 1] == 0.0
    assert np.abs(cpd.pinv_psd(np.zeros((3, 3)), ctx=gpu_ctx)).max() == 0.0
    x = np.random.default_rng(5).uniform(-1, 1, (3, 5))
    s = x.T @ x  # rank 3
    sp = cpd.pinv_psd(s, ctx=gpu_ctx)
    assert max_rel_diff(s @ sp @ s, s) < 1e-10
    assert max_rel_diff(sp @ s @ sp, sp) < 1e-10
    assert max_rel_diff(sp, sp.T) < 1e-12
    assert max_rel_diff(sp, oracle.pinv_psd(s)) < 1e-10
    with pytest.raises(cpd.ShapeError):
        cpd.pinv_psd(np.zeros((2, 3)), ctx=gpu_ctx)
    with pytest.raises(cpd.ArgumentError):
        cpd.pinv_psd(eye, -1.0, ctx=gpu_ctx)


@pytest.mark.parametrize("R", [1, 2, 5, 16, 33, 64])
def test_pinv_matches_oracle(gpu_ctx, oracle, R):
    a = np.random.default_rng(R).standard_normal((R + 3, R))
    s = a.T @ a
    assert max_rel_diff(cpd.pinv_psd(s, ctx=gpu_ctx), oracle.pinv_psd(s)) < 1e-9


def test_update_stationary_and_errors(gpu_ctx, oracle):
    # test_als.cpp:45-61
    dims = [3, 4, 2]
    f = oracle.random_factors(dims, 2, 11)
    yv = oracle.full(dims, f)
    g = cpd.cp_gradient_all(tensor(gpu_ctx, yv, dims), f)
    for n in range(1, 4):
        upd = cpd.als_update_mode(g[n - 1], f, n, ctx=gpu_ctx)
        assert max_rel_diff(upd, f[n - 1]) < 1e-10
        assert max_rel_diff(upd, oracle.als_update_mode(g[n - 1], f, n)) < 1e-12
    z = cpd.cp_gradient_all(tensor(gpu_ctx, np.zeros(24), dims), f)
    assert np.abs(cpd.als_update_mode(z[0], f, 1, ctx=gpu_ctx)).max() == 0.0
    with pytest.raises(cpd.NumericError):
        cpd.als_update_mode(np.full((3, 2), np.nan), f, 1, ctx=gpu_ctx)
    with pytest.raises(cpd.IndexError):
        cpd.als_update_mode(g[0], f, 0, ctx=gpu_ctx)


@pytest.mark.parametrize("dims", [[3, 4, 5], [5, 3, 4], [2, 6, 3, 2]], ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("seed", [31, 32, 33])
def test_sweeps_match_oracle(gpu_ctx, oracle, dims, seed):
    # test_als.cpp:72-87: five sweeps, device vs the CPU restatement
    yv = oracle.random_tensor(dims, seed)
    a = oracle.random_factors(dims, 3, seed + 100)
    b = [x.copy() for x in a]
    y = tensor(gpu_ctx, yv, dims)
    for _ in range(5):
        oracle.als_sweep_fast(yv, dims, a)
        cpd.als_sweep_fast(y, b)
    for n in range(len(dims)):
        assert max_rel_diff(a[n], b[n]) < 1e-9


def test_cost_never_increases(gpu_ctx, oracle):
    # test_als.cpp:89-104
    dims = [4, 5, 3]
    yv = oracle.random_tensor(dims, 41)
    f = oracle.random_factors(dims, 3, 42)
    y = tensor(gpu_ctx, yv, dims)
    prev = oracle.cost(yv, dims, f)
    for _ in range(20):
        cpd.als_sweep_fast(y, f)
        d = oracle.cost(yv, dims, f)
        assert d <= prev * (1.0 + 1e-10) + 1e-12
        prev = d


def test_exact_fit_fixed_point(gpu_ctx, oracle):
    # test_als.cpp:106-112
    dims = [3, 3, 4]
    f = oracle.random_factors(dims, 2, 51)
    g = [x.copy() for x in f]
    cpd.als_sweep_fast(tensor(gpu_ctx, oracle.full(dims, f), dims), g)
    for n in range(3):
        assert max_rel_diff(f[n], g[n]) < 1e-9


def test_run_fills_trace(gpu_ctx, oracle):
    # test_als.cpp:198-222 (als_fast)
    dims = [4, 3, 5]
    yv = oracle.random_tensor(dims, 91)
    init = oracle.random_factors(dims, 2, 92)
    c = cpd.CostCounter()
    res = cpd.run(tensor(gpu_ctx, yv, dims), init, cpd.SolveOptions(max_iters=4), c)
    tr = res.trace
    assert tr.iters_run == 4 and len(tr.cost) == 4 and len(tr.rel_error) == 4
    assert len(tr.seconds) == 4 and len(tr.mults) == 4
    assert all(tr.mults[i] >= tr.mults[i - 1] for i in range(1, 4))
    yn = float(np.linalg.norm(yv))
    for i in range(4):
        assert abs(tr.rel_error[i] - np.sqrt(tr.cost[i]) / yn) <= 1e-12 * tr.rel_error[i]
    _, ot = oracle.run_als_fast(yv, dims, init, max_iters=4)
    for i in range(4):
        assert abs(tr.cost[i] - ot["cost"][i]) <= 1e-9 * max(ot["cost"][i], 1e-12) + 1e-12 * yn * yn


def test_run_unsorted_matches_oracle(gpu_ctx, oracle):
    # test_als.cpp:224-238
    dims = [5, 3, 4]
    yv = oracle.random_tensor(dims, 101)
    init = oracle.random_factors(dims, 2, 102)
    res = cpd.run(tensor(gpu_ctx, yv, dims), init, cpd.SolveOptions(max_iters=6))
    of, ot = oracle.run_als_fast(yv, dims, init, max_iters=6)
    for n in range(3):
        assert max_rel_diff(res.factors[n], of[n]) < 1e-9
    for i in range(6):
        assert abs(res.trace.cost[i] - ot["cost"][i]) <= 1e-9 * ot["cost"][i] + 1e-13


def test_run_early_stop_and_validation(gpu_ctx, oracle):
    # test_als.cpp:240-262
    truth = oracle.random_factors([4, 4, 4], 1, 111)
    y = tensor(gpu_ctx, oracle.full([4, 4, 4], truth), [4, 4, 4])
    res = cpd.run(y, oracle.random_factors([4, 4, 4], 1, 112), cpd.SolveOptions(max_iters=50, tol=1e-6))
    assert 2 <= res.trace.iters_run < 50
    y2 = tensor(gpu_ctx, oracle.random_tensor([3, 4], 121), [3, 4])
    with pytest.raises(cpd.ShapeError):
        cpd.run(y2, oracle.random_factors([4, 3], 2, 122))
    with pytest.raises(cpd.ArgumentError):
        cpd.run(y2, oracle.random_factors([3, 4], 2, 123), cpd.SolveOptions(max_iters=0))
    with pytest.raises(cpd.ArgumentError):
        cpd.run(y2, oracle.random_factors([3, 4], 2, 123), cpd.SolveOptions(max_iters=1, tol=-1.0))


def test_recovery_6cubed(gpu_ctx, oracle):
    # test_als.cpp:264-279
    truth = oracle.random_factors([6, 6, 6], 2, 131)
    y = tensor(gpu_ctx, oracle.full([6, 6, 6], truth), [6, 6, 6])
    ok = False
    for seed in (201, 202, 203):
        init = oracle.random_factors([6, 6, 6], 2, seed)
        res = cpd.run(y, init, cpd.SolveOptions(max_iters=150))
        if res.trace.rel_error[-1] < 1e-4:
            ok = True
            break
    assert ok


def test_acceptance_criterion_5_recovery(gpu_ctx, oracle):
    # acceptance_main.cpp:338-353: 20^3 rank-3 recovered to <= 1e-4 within 500 sweeps
    truth = oracle.random_factors([20, 20, 20], 3, 424242)
    y = tensor(gpu_ctx, oracle.full([20, 20, 20], truth), [20, 20, 20])
    best = 1.0
    for seed in (1, 2, 3):
        res = cpd.run(y, oracle.random_factors([20, 20, 20], 3, seed), cpd.SolveOptions(max_iters=500))
        best = min(best, min(res.trace.rel_error))
        if best <= 1e-4:
            break
    assert best <= 1e-4


def _c4_like(ctx, oracle, I, R, N=5, seed=4):
    """BASELINE config 4 construction: rank-R N(0,1) model + Gaussian noise at 20 dB."""
    dims = [I] * N
    truth = [oracle.fill_normal(seed * 100 + k, I * R).reshape(I, R, order="F") for k in range(N)]
    y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=seed, ctx=ctx)
    e2 = y.norm2()
    # Y = sigma E + full(model) with sigma = |full| / (10 |E|) (SNR 20 dB)
    t = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=seed, ctx=ctx)
    t.axpby_kruskal(0.0, 1.0, truth)
    full2 = t.norm2()
    t.free()
    sigma = np.sqrt(full2) / (10.0 * np.sqrt(e2))
    y.axpby_kruskal(sigma, 1.0, truth)
    init = [oracle.fill_normal(seed * 1000 + 7 + k, I * R).reshape(I, R, order="F") for k in range(N)]
    return y, dims, init


def test_c4_like_fit_trace_vs_oracle(gpu_ctx, oracle):
    """Config-4 construction at 24^5 (7.96M entries), R=16, 50 sweeps:
    every sweep's relative fit against the oracle's (<= 1e-9 relative)."""
    y, dims, init = _c4_like(gpu_ctx, oracle, 24, 16)
    yv = y.values()
    res = cpd.run(y, init, cpd.SolveOptions(max_iters=50))
    _, ot = oracle.run_als_fast(yv, dims, init, max_iters=50)
    for i in range(50):
        assert abs(res.trace.rel_error[i] - ot["rel_error"][i]) <= 1e-9 * ot["rel_error"][i], i


@pytest.mark.slow
def test_c4_full_fit_trace_vs_oracle(gpu_ctx, oracle):
    """BASELINE config 4 at full size (60^5, 6.2 GB), 50 sweeps vs the oracle."""
    y, dims, init = _c4_like(gpu_ctx, oracle, 60, 16)
    yv = y.values()
    res = cpd.run(y, init, cpd.SolveOptions(max_iters=50))
    _, ot = oracle.run_als_fast(yv, dims, init, max_iters=50)
    for i in range(50):
        assert abs(res.trace.rel_error[i] - ot["rel_error"][i]) <= 1e-9 * ot["rel_error"][i], i
