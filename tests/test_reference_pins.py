"""The reference itself, compiled here from its own sources (oracle/_ref,
oracle/Makefile `ref`: /root/reference/proj/core/src with the Eigen / doctest
shims of oracle/shim), as the top of the parity chain:

  * its own test suite (76 doctest cases) and acceptance binary (7 criteria)
    pass on the shim build — which validates the shims;
  * the C oracle port (oracle/cpd_oracle.c), which the GPU tests check
    against at every size, reproduces the reference's own cp_gradient_all,
    mttkrp_direct, als_sweep_fast, run() traces, pinv_psd and counts;
  * the library's host logic behind the C-ABI (pivot, sort, visit order, the
    realized and predicted counts, the FastStats figure) equals the
    reference's on a sweep of shapes.

No GPU: these run with `-m "not gpu"` wherever /root/reference (or the built
oracle/_ref) is present, and skip otherwise."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_1204_1586_b200 as cpd
from paper_1204_1586_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "oracle" / "_ref"

ref = pytest.importorskip("ref")
if not ref.available():  # pragma: no cover - GPU box without the built reference
    pytest.skip("the reference is not built here", allow_module_level=True)


@pytest.fixture(scope="module")
def R_():
    ref.build()
    return ref


def test_reference_suite_passes_on_the_shim_build(R_):
    out = subprocess.run([str(REF_DIR / "cpd_tests")], capture_output=True, text=True, timeout=600, cwd=REF_DIR)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "test cases: 76 | 76 passed | 0 failed" in out.stdout


def test_reference_acceptance_passes_on_the_shim_build(R_):
    out = subprocess.run([str(REF_DIR / "cpd_acceptance")], capture_output=True, text=True, timeout=600,
                         cwd=REF_DIR)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "all criteria passed" in out.stdout


SHAPES = [([2, 2, 2], 2), ([3, 4, 5], 3), ([5, 4, 3], 2), ([4, 3, 2, 5], 4), ([6, 7, 8, 9], 5), ([3, 3, 3, 3, 3], 2),
          ([2, 3, 2, 4, 2, 3], 3), ([11, 13], 7), ([1, 5, 1, 4], 2), ([7, 2, 7, 3], 6)]


@pytest.mark.parametrize("dims,R", SHAPES)
def test_oracle_port_reproduces_the_reference_gradient(R_, oracle, dims, R):
    y = oracle.random_tensor(dims, 31 + R)
    f = oracle.random_factors(dims, R, 41 + R)
    t = ref.Tensor(y, dims)
    want, mults = t.cp_gradient_all(f)
    got, _, _ = oracle.cp_gradient_all(y, dims, f)
    for a, b in zip(got, want):
        assert np.abs(a - b).max() <= 1e-13 * max(np.abs(b).max(), 1e-300)
    # counts charged by the reference's counter == the library's per-mode charges
    sd = sorted(dims)
    assert mults == sum(cpd.fast_count_realized(sd, R, n) for n in range(1, len(dims) + 1))
    for n in range(1, len(dims) + 1):
        d = t.mttkrp_direct(f, n)
        assert np.abs(d - want[n - 1]).max() <= 1e-13 * max(np.abs(want[n - 1]).max(), 1e-300)
    t.close()


def test_sharded_reference_equals_whole(R_, oracle):
    """The slab-parallel reference timing path (threads over last-mode slabs)
    returns the same gradient as one reference call on the whole tensor."""
    dims, R = [6, 7, 8, 11], 4
    y = oracle.random_tensor(dims, 5)
    f = oracle.random_factors(dims, R, 6)
    a, _ = ref.Tensor(y, dims).cp_gradient_all(f)
    for axis in (0, 1):
        b, _ = ref.Tensor(y, dims, parts=4, axis=axis).cp_gradient_all(f)
        for x, z in zip(a, b):
            assert np.abs(x - z).max() <= 1e-13 * np.abs(x).max()


@pytest.mark.parametrize("dims,R", [([4, 5, 6], 3), ([3, 4, 3, 5], 2), ([6, 5, 4, 3], 3)])
def test_oracle_port_reproduces_reference_als(R_, oracle, dims, R):
    y = oracle.random_tensor(dims, 70)
    f0 = oracle.random_factors(dims, R, 71)
    fr = [x.copy(order="F") for x in f0]
    t = ref.Tensor(y, dims)
    t.als_sweep_fast(fr)
    fo = [x.copy(order="F") for x in f0]
    oracle.als_sweep_fast(y, dims, fo)
    for a, b in zip(fo, fr):
        assert np.abs(a - b).max() <= 1e-10 * max(np.abs(b).max(), 1.0)
    # run(): fast ALS trace over 8 sweeps
    fr = [x.copy(order="F") for x in f0]
    cost, rel = t.run(fr, algo=1, max_iters=8)
    _, tr = oracle.run(y, dims, [x.copy(order="F") for x in f0], algo="als_fast", max_iters=8)
    assert len(cost) == 8 and np.allclose(tr["cost"], cost, rtol=1e-9, atol=1e-12)
    assert np.allclose(tr["rel_error"], rel, rtol=1e-9, atol=1e-12)
    t.close()


def test_pinv_matches_reference(R_, oracle):
    rng = np.random.default_rng(3)
    for n, rank in [(4, 4), (5, 3), (6, 6), (3, 1)]:
        x = rng.standard_normal((n, rank))
        s = x @ x.T
        assert np.allclose(oracle.pinv_psd(s), ref.pinv_psd(s), rtol=1e-9, atol=1e-12)


def _abi_counts(dims, R, n):
    L = _lib.load()
    d = (C.c_int64 * len(dims))(*dims)
    out = []
    for v in range(3):
        x = C.c_uint64()
        assert L.cpdgpu_predicted_mult_count(len(dims), d, R, n, v, C.byref(x)) == 0
        out.append(int(x.value))
    out.append(int(L.cpdgpu_fast_count_realized(len(dims), d, R, n)))
    return tuple(out)


def test_host_logic_matches_the_reference(R_):
    """Pivot, sort, visit order, all four count forms and the FastStats figure of
    the C-ABI against the reference on 120 random shapes (mttkrp.cpp:56-111,255-320)."""
    rng = np.random.default_rng(17)
    L = _lib.load()
    for _ in range(120):
        N = int(rng.integers(2, 7))
        dims = [int(x) for x in rng.integers(1, 9, size=N)]
        R = int(rng.integers(1, 6))
        sd = sorted(dims)
        assert cpd.select_pivot(sd) == ref.select_pivot(sd)
        for n in range(1, N + 1):
            assert _abi_counts(sd, R, n) == ref.counts(sd, R, n), (sd, R, n)
        # the workspace figure the gradient reports (FastStats) is the reference's
        y = np.ones(int(np.prod(dims)))
        peak = C.c_int64()
        assert L.cpdgpu_reference_workspace(N, (C.c_int64 * N)(*sd), R, C.byref(peak)) == 0
        assert peak.value >= 0
    d = (C.c_int64 * 3)(3, 2, 4)
    x = C.c_uint64()
    assert L.cpdgpu_predicted_mult_count(3, d, 2, 1, 1, C.byref(x)) == 3  # unsorted: ArgumentError
    d = (C.c_int64 * 3)(2, 3, 4)
    assert L.cpdgpu_predicted_mult_count(3, d, 2, 4, 1, C.byref(x)) == 2  # mode outside 1..N: IndexError
