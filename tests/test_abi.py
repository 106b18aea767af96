"""C-ABI checks that need no GPU: the product library builds for sm_100a, loads,
exports every entry point include/cpdgpu.h declares, its host-side ordering and
count logic agrees with the oracle, and it refuses to run without a B200
(no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1204_1586_b200 as cpd
from paper_1204_1586_b200 import _lib
from paper_1204_1586_b200 import build as B

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _lib.load()


def header_symbols():
    text = (ROOT / "include" / "cpdgpu.h").read_text()
    return sorted(set(re.findall(r"\b(cpdgpu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ["cpdgpu_create", "cpdgpu_cp_gradient_all", "cpdgpu_cp_gradient_all_hook",
              "cpdgpu_cp_gradient_all_device", "cpdgpu_als_sweep", "cpdgpu_als_run", "cpdgpu_pinv_psd",
              "cpdgpu_select_pivot", "cpdgpu_fast_update_order", "cpdgpu_sort_modes"]:
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) >= set(header_symbols()), set(header_symbols()) - set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(B.LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"sm_(8\d|90)\b", out) is None


def test_fp64_seed_kernel_uses_dmma_and_tma():
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", str(B.LIB)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "UTMALDG" in sass  # cp.async.bulk.tensor


@pytest.mark.parametrize("dims", [[10, 10, 10], [10, 10, 10, 10], [2, 3, 4, 5], [3, 5], [2, 2, 3, 3, 4],
                                  [5, 3, 4], [14] * 7, [60] * 5, [300] * 4, [1, 1, 1], [2, 2, 9]])
def test_ordering_matches_oracle(oracle, dims):
    perm, inv = cpd.sort_modes(dims)
    assert (perm, inv) == tuple(oracle.sort_perm(dims))
    assert cpd.fast_update_order(dims) == oracle.fast_update_order(dims)
    sd = sorted(dims)
    assert cpd.select_pivot(sd) == oracle.select_pivot(sd)


@pytest.mark.parametrize("dims", [[10, 10, 10], [2, 3, 4, 5], [2, 2, 2, 2, 2, 2, 2], [60] * 5, [200] * 3,
                                  [14] * 7, [300] * 4, [4, 5]])
def test_counts_match_oracle(oracle, dims):
    for R in (1, 3, 16):
        for n in range(1, len(dims) + 1):
            assert cpd.fast_count_realized(dims, R, n) == oracle.fast_count_realized(dims, R, n)


def test_errors_map_to_reference_types():
    with pytest.raises(cpd.ArgumentError):
        cpd.select_pivot([7])
    with pytest.raises(cpd.ArgumentError):
        cpd.fast_update_order([4])
    with pytest.raises(cpd.ArgumentError):
        cpd.fast_count_realized([3, 2, 4], 1, 1)
    with pytest.raises(cpd.IndexError):
        cpd.fast_count_realized([2, 3, 4], 1, 0)
    assert issubclass(cpd.ShapeError, ValueError) and issubclass(cpd.NumericError, ArithmeticError)


def test_no_cpu_fallback_without_gpu():
    """Without a B200 the product fails loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(cpd.DeviceError):
        cpd.Context(0)


def test_missing_library_is_an_error(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "absent.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(cpd.DeviceError):
        _lib.load()


def test_status_mapping():
    from paper_1204_1586_b200 import errors
    for code, cls in [(1, cpd.ShapeError), (2, cpd.IndexError), (3, cpd.ArgumentError), (4, cpd.NumericError),
                      (5, cpd.DomainError), (6, cpd.DeviceError), (8, cpd.ParseError)]:
        assert isinstance(errors.from_status(code, "m"), cls)


def test_slab_bounds_through_the_abi(lib):
    """cpdgpu_slab_bounds (host logic, no device) splits the last mode like sharded.slab_bounds."""
    from paper_1204_1586_b200 import sharded
    for extent, world in [(300, 8), (300, 3), (10, 3), (7, 7), (60, 2)]:
        want = sharded.slab_bounds(extent, world)
        assert [cpd.slab_bounds(extent, world, r) for r in range(world)] == want
    with pytest.raises(cpd.ArgumentError):
        cpd.slab_bounds(10, 0, 0)
    with pytest.raises(cpd.ArgumentError):
        cpd.slab_bounds(10, 2, 2)
