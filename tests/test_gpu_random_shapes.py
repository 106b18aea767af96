"""Randomized parity sweep on the device: seeded random orders (2..6), extents
(1..23, unsorted, repeated), ranks (1..70) — fp64 against the oracle at 1e-10,
fp32 at 1e-5, the direct MTTKRP of a random mode, and one fast ALS sweep.
Every case is reproducible from its index (numpy Generator(seed=case))."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def _shape(rng):
    N = int(rng.integers(2, 7))
    cap = {2: 23, 3: 23, 4: 14, 5: 9, 6: 6}[N]
    dims = [int(rng.integers(1, cap + 1)) for _ in range(N)]
    R = int(rng.choice([1, 2, 3, 7, 8, 9, 16, 20, 31, 33, 64, 70]))
    return dims, R


def _rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


@pytest.mark.parametrize("case", range(24))
def test_random_shape_fp64(gpu_ctx, oracle, case):
    rng = np.random.default_rng(1000 + case)
    dims, R = _shape(rng)
    yv = rng.standard_normal(int(np.prod(dims)))
    f = [rng.standard_normal((d, R)) for d in dims]
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
    got = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(yv, dims, f)
    assert max(_rel(a, b) for a, b in zip(got, want)) <= 1e-10, (dims, R)
    n = int(rng.integers(1, len(dims) + 1))
    assert _rel(cpd.mttkrp_direct(y, f, n), want[n - 1]) <= 1e-10, (dims, R, n)
    if R <= 64 and min(dims) > 1:
        g = [a.copy(order="F") for a in f]
        cpd.als_sweep_fast(y, g)
        h = oracle.als_sweep_fast(yv, dims, [a.copy(order="F") for a in f])
        assert max(_rel(a, b) for a, b in zip(g, h)) <= 1e-8, (dims, R)


@pytest.mark.parametrize("case", range(12))
def test_random_shape_fp32(gpu_ctx, oracle, case):
    rng = np.random.default_rng(5000 + case)
    dims, R = _shape(rng)
    yv = rng.uniform(-1, 1, int(np.prod(dims))).astype(np.float32)
    f = [rng.standard_normal((d, R)) for d in dims]
    y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx, dtype=cpd.F32)
    got = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(yv.astype(np.float64), dims, f)
    assert max(_rel(a, b) for a, b in zip(got, want)) <= 1e-5, (dims, R)
