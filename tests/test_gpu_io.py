"""TDNB tensor files streamed to the device (io.hpp:10-12,
io.cpp:162-216): bit-exact round trips, last-mode slab loads for sharded ranks,
and the reference parser's errors with byte offsets (test_io.cpp:46-118)."""
import struct

import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def tdnb_bytes(dims, values):
    """The binary writer of io.cpp:192-203, restated (test infrastructure)."""
    return b"TDNB" + struct.pack("<I", len(dims)) + struct.pack(f"<{len(dims)}I", *dims) + \
        np.asarray(values, dtype="<f8").tobytes()


def test_round_trip_bitwise(gpu_ctx, oracle, tmp_path):
    dims = [3, 4, 2, 2]
    v = oracle.random_tensor(dims, 999)
    f = tmp_path / "r.tdnb"
    f.write_bytes(tdnb_bytes(dims, v))
    t = cpd.DenseTensor.load_tdnb(f, ctx=gpu_ctx)
    assert list(t.dims) == dims
    assert t.values().tobytes() == v.astype("<f8").tobytes()
    g = tmp_path / "back.tdnb"
    t.save_tdnb(g)
    assert g.read_bytes() == f.read_bytes()
    special = np.array([0.0, -0.0, 5e-324, 1.7e308, -3.25])  # test_io.cpp:54-58
    (tmp_path / "s.tdnb").write_bytes(tdnb_bytes([5], special))
    s = cpd.DenseTensor.load_tdnb(tmp_path / "s.tdnb", ctx=gpu_ctx)
    assert s.values().tobytes() == special.tobytes()


def test_fp32_tensor_saves_widened(gpu_ctx, oracle, tmp_path):
    dims = [6, 5, 4]
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=3, ctx=gpu_ctx, dtype=cpd.F32)
    y.save_tdnb(tmp_path / "w.tdnb")
    assert (tmp_path / "w.tdnb").read_bytes() == tdnb_bytes(dims, y.values().astype(np.float64))


def test_slab_load_and_gradient(gpu_ctx, oracle, tmp_path):
    dims, R = [7, 8, 9, 10], 4
    v = oracle.random_tensor(dims, 5)
    f = tmp_path / "y.tdnb"
    f.write_bytes(tdnb_bytes(dims, v))
    full = v.reshape(dims, order="F")
    for lo, hi in [(0, 3), (3, 10), (9, 10)]:
        t = cpd.DenseTensor.load_tdnb(f, slab=(lo, hi), ctx=gpu_ctx)
        assert list(t.dims) == dims[:-1] + [hi - lo]
        assert np.array_equal(t.values(), full[..., lo:hi].reshape(-1, order="F"))
    fac = oracle.random_factors(dims, R, 6)
    got = cpd.cp_gradient_all(cpd.DenseTensor.load_tdnb(f, ctx=gpu_ctx), fac)
    want, _, _ = oracle.cp_gradient_all(v, dims, fac)
    for a, b in zip(got, want):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    with pytest.raises(cpd.IndexError):
        cpd.DenseTensor.load_tdnb(f, slab=(4, 11), ctx=gpu_ctx)


@pytest.mark.parametrize("mutate,word", [
    (lambda b: b[:-3], "truncated"),          # mid-value cut
    (lambda b: b[:10], "truncated"),          # mid-dimension cut
    (lambda b: b + b"x", "trailing"),
    (lambda b: b"NOPE" + b[4:], "magic"),
    (lambda b: b[:4] + struct.pack("<I", 0) + b[8:], "implausible"),
    (lambda b: b[:8] + struct.pack("<I", 0) + b[12:], "nonpositive"),
])
def test_parser_errors_carry_byte_offsets(gpu_ctx, tmp_path, mutate, word):
    good = tdnb_bytes([2, 2, 2], np.arange(1.0, 9.0))  # t8 of test_io.cpp
    assert len(good) == 4 + 4 + 3 * 4 + 8 * 8
    f = tmp_path / "bad.tdnb"
    f.write_bytes(mutate(good))
    with pytest.raises(cpd.ParseError) as e:
        cpd.DenseTensor.load_tdnb(f, ctx=gpu_ctx)
    assert word in str(e.value) and "byte" in str(e.value) and str(f) in str(e.value)


def test_missing_file(gpu_ctx, tmp_path):
    with pytest.raises(cpd.ParseError):
        cpd.DenseTensor.load_tdnb(tmp_path / "does_not_exist.tdnb", ctx=gpu_ctx)


@pytest.mark.parametrize("staged", ["1", "0"])
def test_pageable_upload_roundtrip(gpu_ctx, monkeypatch, staged):
    """Uploads from pageable host memory (numpy arrays; the reference's DenseTensor is a
    std::vector) of more than 32 MB go through the library's pinned staging buffers,
    filled by several host threads: upload and update return the exact bytes, ragged last
    chunk included; CPDGPU_STAGED_UPLOAD=0 takes the plain copy."""
    monkeypatch.setenv("CPDGPU_STAGED_UPLOAD", staged)
    rng = np.random.default_rng(5)
    dims = [301, 299, 101]  # 72.7 MB of fp64: 8 MB chunks with a ragged tail
    y = rng.standard_normal(int(np.prod(dims)))
    t = cpd.DenseTensor.from_values(y, dims, ctx=gpu_ctx)
    assert np.array_equal(t.values().reshape(-1), y)
    y2 = rng.standard_normal(y.size)
    t.update(y2.ctypes.data)
    assert np.array_equal(t.values().reshape(-1), y2)
    y32 = rng.standard_normal(y.size).astype(np.float32)
    t32 = cpd.DenseTensor.from_values(y32, dims, ctx=gpu_ctx, dtype=cpd.F32)
    assert np.array_equal(t32.values().reshape(-1), y32)
    t.free()
    t32.free()
