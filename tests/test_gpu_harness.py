"""The reference's benchmark harness and gradcheck flow on the device
(bench.cpp:59-196, cpd_main.cpp:63-120), and the device cost (kruskal.cpp:58-77)."""
import io

import numpy as np
import pytest

import paper_1204_1586_b200 as cpd
from paper_1204_1586_b200 import harness as H

pytestmark = pytest.mark.gpu


def test_device_cost_matches_oracle(gpu_ctx, oracle):
    for dims, R in [([4, 5, 6], 3), ([12, 10, 14, 9], 5)]:
        yv = oracle.random_tensor(dims, 3)
        f = oracle.random_factors(dims, R, 4)
        y = cpd.DenseTensor.from_values(yv, dims, ctx=gpu_ctx)
        want = oracle.cost(yv, dims, f)
        assert abs(cpd.cost(y, f) - want) <= 1e-10 * want
        assert abs(cpd.relative_error(y, f) - np.sqrt(want) / np.linalg.norm(yv)) <= 1e-10


def test_generate_problem_matches_reference_stream(gpu_ctx, oracle):
    y, init = cpd.generate_problem([4, 3, 5], 2, 42, ctx=gpu_ctx)
    assert np.array_equal(y.values(), oracle.uniform01(42, 60))
    assert np.array_equal(np.concatenate([a.reshape(-1, order="F") for a in init]), oracle.uniform01(43, 24))


def test_run_benchmark_cell(gpu_ctx):
    cfg = H.BenchConfig(dims=[10, 10, 10], rank=4, iters=3, reps=2)
    log = io.StringIO()
    recs = H.run_benchmark(cfg, log=log)
    assert len(recs) == 1 and log.getvalue() == ""
    r = recs[0]
    assert r.t_baseline > 0 and r.t_fast > 0 and abs(r.rho - r.t_baseline / r.t_fast) < 1e-12
    pd, pf = H.predicted_sweep_counts([10, 10, 10], 4)
    assert r.mults_baseline == pd and r.count_ratio == pd / pf
    assert r.mults_fast == sum(cpd.fast_count_realized([10, 10, 10], 4, n) for n in (1, 2, 3))
    buf = io.StringIO()
    H.write_csv(buf, recs)
    assert buf.getvalue().splitlines()[1].startswith("3,10x10x10,4,3,2,")
    skip = H.run_benchmark(H.BenchConfig(dims=[10, 10, 10], rank=4, iters=1, reps=1, mem_budget=10), log=log)
    assert skip == [] and "skip 10x10x10" in log.getvalue()


@pytest.mark.parametrize("dims,rank", [([4, 5, 6], 3), ([3, 4, 2, 3], 2)])
def test_gradcheck_passes(gpu_ctx, dims, rank):
    out = io.StringIO()
    assert H.gradcheck(dims, rank, trials=2, out=out) == 0, out.getvalue()
    assert "all 2 trials passed" in out.getvalue()
