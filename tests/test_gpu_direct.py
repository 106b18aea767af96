"""Direct mode-n MTTKRP (mttkrp_direct, mttkrp.hpp:19-20) and the direct ALS sweep
(als_sweep_direct, als.hpp:58-60) on the device: one pass over Y per mode (the
paper's Algorithm 1 cost model).  Checked against the
oracle's brute-force MTTKRP for every mode (fp64 <= 1e-12, fp32 <= 1e-5), the
reference's multiplication charge, and a host-orchestrated oracle sweep."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dims,R", [([4, 5, 6, 7], 3), ([7, 5, 6], 9), ([30, 40], 5), ([6, 7, 8, 5, 4], 20),
                                    ([60, 60, 60], 40), ([2, 1, 3], 2)])
def test_direct_equals_brute(gpu_ctx, oracle, dims, R):
    yv = oracle.random_tensor(dims, 71)
    f = oracle.random_factors(dims, R, 72)
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    for n in range(1, len(dims) + 1):
        got = cpd.mttkrp_direct(y, f, n)
        assert rel(got, oracle.brute_mttkrp(yv, dims, f, n)) <= 1e-12, n


def test_direct_fp32(gpu_ctx, oracle):
    dims, R = [40, 40, 40, 40], 64
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=5, ctx=gpu_ctx, dtype=cpd.F32)
    yv = y.values().astype(np.float64)
    f = [oracle.fill_normal(80 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
    want, _, _ = oracle.cp_gradient_all(yv, dims, f)
    for n in range(1, 5):
        assert rel(cpd.mttkrp_direct(y, f, n), want[n - 1]) <= 1e-5, n


def test_direct_charges_match_reference(gpu_ctx, oracle):
    dims, R = [3, 4, 5, 6], 7
    y = cpd.DenseTensor.from_values(oracle.random_tensor(dims, 1), dims, ctx=gpu_ctx)
    f = oracle.random_factors(dims, R, 2)
    for n in range(1, 5):
        c = cpd.CostCounter()
        cpd.mttkrp_direct(y, f, n, counter=c)
        assert c.total() == oracle.predicted_mult_count(dims, R, n, "direct"), n


def test_direct_errors(gpu_ctx, oracle):
    dims = [3, 4, 5]
    y = cpd.DenseTensor.from_values(oracle.random_tensor(dims, 1), dims, ctx=gpu_ctx)
    f = oracle.random_factors(dims, 2, 2)
    with pytest.raises(cpd.IndexError):
        cpd.mttkrp_direct(y, f, 0)
    with pytest.raises(cpd.IndexError):
        cpd.mttkrp_direct(y, f, 4)
    with pytest.raises(cpd.ShapeError):
        cpd.mttkrp_direct(y, oracle.random_factors([3, 4, 6], 2, 2), 1)


def test_als_sweep_direct_matches_oracle(gpu_ctx, oracle):
    dims, R = [5, 6, 7, 4], 3
    yv = oracle.random_tensor(dims, 91)
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    f0 = oracle.random_factors(dims, R, 92)
    order = [1, 2, 3, 4]
    ref = [a.copy(order="F") for a in f0]
    for n in order:  # als.cpp:58-67
        ref[n - 1] = oracle.als_update_mode(oracle.brute_mttkrp(yv, dims, ref, n), ref, n)
    got = [a.copy(order="F") for a in f0]
    c = cpd.CostCounter()
    cpd.als_sweep_direct(y, got, order, counter=c)
    for k in range(4):
        assert rel(got[k], ref[k]) <= 1e-10, k
    assert c.total() == sum(oracle.predicted_mult_count(dims, R, n, "direct") for n in order)
