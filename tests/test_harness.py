"""Host-side parts of the benchmark harness and problem generation (no GPU):
the reference's analytic counts, working-set estimate, grid, speed ratio, and
the Uniform01 stream (bench.cpp, mttkrp.cpp:255-290, rng.hpp:9-26)."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd
from paper_1204_1586_b200 import harness as H


@pytest.mark.parametrize("dims", [[10, 10, 10], [2, 3, 4, 5], [14] * 7, [60] * 5, [3, 3, 4, 4, 5], [4, 5]])
def test_predicted_counts_match_oracle(oracle, dims):
    for R in (1, 7):
        for n in range(1, len(dims) + 1):
            for v in ("direct", "fast", "fast_derived"):
                assert H.predicted_mult_count(dims, R, n, v) == oracle.predicted_mult_count(dims, R, n, v)


def test_speed_ratio_and_grid():
    assert H.speed_ratio(3.0, 1.5) == 2.0
    with pytest.raises(cpd.ArgumentError):
        H.speed_ratio(0.0, 1.0)
    with pytest.raises(cpd.ArgumentError):
        H.speed_ratio(1.0, -1.0)
    grid = H.default_grid()
    assert len(grid) == 5 * (2 + 3)  # R in {1, 10} for I = 10, {1, 10, 20} for I = 20
    assert ([10, 10, 10], 1) in grid and ([20] * 7, 20) in grid


def test_estimate_cell_bytes():
    # bench.cpp:145-160 for 10^3, R = 10: p* = 1, fast ws = 10 (10 + 100), direct ws = 10 * 100
    assert H.estimate_cell_bytes([10, 10, 10], 10) == 8 * (2 * 1000 + max(10 * 110, 1000) + 4 * 300)


def test_uniform01_is_the_reference_stream(oracle):
    assert np.array_equal(cpd.uniform01(1234, 4096), oracle.uniform01(1234, 4096))
    f = cpd.random_init([3, 4], 2, 9)  # test_als.cpp:190-201
    g = cpd.random_init([3, 4], 2, 9)
    assert all(np.array_equal(a, b) for a, b in zip(f, g))
    assert all(((a > 0) & (a < 1)).all() for a in f)
    assert not np.array_equal(cpd.random_init([3, 4], 2, 10)[0], f[0])
    with pytest.raises(cpd.ArgumentError):
        cpd.random_init([3, 4], 0, 1)


def test_csv_header_is_the_reference_column_set():
    import io
    rec = H.BenchRecord(dims=[10, 10, 10], rank=10, iters=2, reps=1, t_baseline=2e-3, t_fast=1e-3, rho=2.0,
                        mults_baseline=300, mults_fast=150, count_ratio=2.0)
    buf = io.StringIO()
    H.write_csv(buf, [rec])
    lines = buf.getvalue().splitlines()
    assert lines[0] == "N,dims,R,iters,reps,t_direct,t_fast,rho,mults_direct,mults_fast,count_ratio"
    assert lines[1] == "3,10x10x10,10,2,1,0.002,0.001,2,300,150,2"
