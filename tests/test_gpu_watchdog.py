"""Pipeline watchdog of the seed kernels: a barrier wait that never completes is
reported, not trapped.  CPDGPU_FORCE_STALL=1 (test hook, read per launch) makes
the producer announce its first Y tile without requesting it; every wait of the
CTA then times out, the kernel unwinds and exits, the fault word (mapped host
memory) turns the call into CPDGPU_CUDA_ERROR (DeviceError), and the SAME context
computes the next gradient correctly (a __trap would have poisoned it; errors
surface as the reference's exceptions do, errors.hpp:8-35)."""
import ctypes as C

import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu


def _grad_ok(y, f, oracle, tol):
    g = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(y.values().astype(np.float64), y.dims, f)
    for a, b in zip(g, want):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= tol


@pytest.mark.parametrize("path", ["i8", "f32"])
def test_forced_stall_is_an_error_not_a_trap(gpu_ctx, oracle, monkeypatch, path):
    ctx = cpd.Context(0)  # a context of its own: graphs off so the stall flag is read per launch
    try:
        C_ = ctx._L
        assert C_.cpdgpu_set_graphs(ctx.h, 0) == 0
        R = 5 if path == "i8" else 64
        if path == "i8":
            monkeypatch.setenv("CPDGPU_I8", "1")
            dims = [16, 12, 10, 8]
            y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=5, ctx=ctx)
            want_path, tol = 1, 1e-10
        else:
            dims = [24, 24, 24, 24]
            y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=5, ctx=ctx, dtype=cpd.F32)
            want_path, tol = 4, 1e-5
        f = [oracle.fill_normal(60 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        _grad_ok(y, f, oracle, tol)
        assert ctx.last_seed_path() == want_path
        monkeypatch.setenv("CPDGPU_FORCE_STALL", "1")
        with pytest.raises(cpd.DeviceError, match="watchdog"):
            cpd.cp_gradient_all(y, f)
        monkeypatch.delenv("CPDGPU_FORCE_STALL")
        _grad_ok(y, f, oracle, tol)  # same context, still healthy
        assert ctx.last_seed_path() == want_path
    finally:
        ctx.close()
