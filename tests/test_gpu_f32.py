"""fp32 tensors on the tensor-core path (seed_f32.cu: tcgen05 kind::f16 with
hi/lo operand splitting, fp64 drains).  Parity bar from the north star: relative
Frobenius error <= 1e-5 per mode against the fp64 oracle run on the same fp32
values (upcast), BASELINE config 5 construction (U(-1,1) fp32 tensor, N(0,1)
factors) at sizes the oracle finishes in seconds, plus the edge shapes the
fp32 path handles specially (rows padded to a multiple of 8, R > 64 chunks,
unsorted modes, partial tiles)."""
import numpy as np
import pytest

import paper_1204_1586_b200 as cpd

pytestmark = pytest.mark.gpu

TOL = 1e-5  # fp32 bar (BASELINE.json north star)


def rel_errs(got, want):
    return [float(np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-300)) for g, w in zip(got, want)]


def _case(ctx, oracle, dims, R, seed=11):
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=seed, ctx=ctx, dtype=cpd.F32)
    yv = y.values().astype(np.float64)
    f = [oracle.fill_normal(seed * 10 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
    return y, yv, f


@pytest.mark.parametrize("dims,R", [
    ([16, 16, 16, 16], 5),
    ([40, 40, 40, 40], 64),      # config-5 shape family, full 64-column pass
    ([24, 30, 40], 33),
    ([7, 9, 11, 13], 8),         # J_p = 63: rows padded to 64
    ([300, 300, 20], 16),        # long K, several fp32 accumulation chunks
    ([130, 257], 3),             # N = 2, partial row block and k-tile
    ([12, 10, 14, 9, 8], 70),    # R > 64: two rank chunks, unsorted modes
])
def test_f32_gradient_matches_oracle(gpu_ctx, oracle, dims, R):
    y, yv, f = _case(gpu_ctx, oracle, dims, R)
    got = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(yv, dims, f)
    errs = rel_errs(got, want)
    assert max(errs) <= TOL, errs


def test_f32_scaling_extremes(gpu_ctx, oracle):
    """Y and factor magnitudes far outside fp16 range: power-of-two scaling keeps accuracy."""
    dims, R = [20, 24, 28], 6
    vals = (np.random.default_rng(3).uniform(-1, 1, int(np.prod(dims))) * 3e7).astype(np.float32)
    y = cpd.DenseTensor.from_values(vals, dims, ctx=gpu_ctx, dtype=cpd.F32)
    f = [np.random.default_rng(10 + k).normal(size=(d, R)) * s for k, (d, s) in
         enumerate(zip(dims, [1e-6, 1e5, 3.0]))]
    got = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(vals.astype(np.float64), dims, f)
    assert max(rel_errs(got, want)) <= TOL


def test_f32_update_refreshes_scale(gpu_ctx, oracle):
    dims, R = [16, 24, 32], 4
    y, yv, f = _case(gpu_ctx, oracle, dims, R)
    cpd.cp_gradient_all(y, f)
    big = (yv * 1000.0).astype(np.float32)
    y.update(big.ctypes.data)
    got = cpd.cp_gradient_all(y, f)
    want, _, _ = oracle.cp_gradient_all(big.astype(np.float64), dims, f)
    assert max(rel_errs(got, want)) <= TOL


def test_f32_deterministic(gpu_ctx, oracle):
    """Deterministic mode: bitwise-identical repeats; the default (left partials
    added in L2 by red.add) repeats within the path's error and both modes agree
    with the oracle."""
    y, yv, f = _case(gpu_ctx, oracle, [32, 32, 32, 32], 64)
    want, _, _ = oracle.cp_gradient_all(yv, [32, 32, 32, 32], f)
    fast = cpd.cp_gradient_all(y, f)
    assert max(rel_errs(fast, want)) <= TOL
    assert max(rel_errs(cpd.cp_gradient_all(y, f), fast)) <= 1e-6
    gpu_ctx.set_deterministic(True)
    try:
        a = cpd.cp_gradient_all(y, f)
        b = cpd.cp_gradient_all(y, f)
        for x, z in zip(a, b):
            assert np.array_equal(x, z)
        assert max(rel_errs(a, want)) <= TOL
    finally:
        gpu_ctx.set_deterministic(False)
    assert max(rel_errs(cpd.cp_gradient_all(y, f), want)) <= TOL  # back to the default (graphs re-recorded)


def test_f32_hook_gauss_seidel(gpu_ctx, oracle):
    dims, R = [12, 16, 10, 14], 7
    y, yv, f0 = _case(gpu_ctx, oracle, dims, R)
    f = [a.copy(order="F") for a in f0]
    ref = [a.copy(order="F") for a in f0]
    got = [None] * 4

    def hook(n, g):
        got[n - 1] = g
        f[n - 1] = oracle.fill_normal(900 + n, dims[n - 1] * R).reshape(dims[n - 1], R, order="F")

    cpd.cp_gradient_all(y, f, hook=hook)
    for n in oracle.fast_update_order(dims):
        want = oracle.brute_mttkrp(yv, dims, ref, n)
        assert rel_errs([got[n - 1]], [want])[0] <= TOL
        ref[n - 1] = oracle.fill_normal(900 + n, dims[n - 1] * R).reshape(dims[n - 1], R, order="F")


def test_f32_als_fit_trace(gpu_ctx, oracle):
    dims, R = [20, 22, 24, 18], 5
    y, yv, f = _case(gpu_ctx, oracle, dims, R)
    res = cpd.run(y, f, cpd.SolveOptions(max_iters=8))
    _, ot = oracle.run_als_fast(yv, dims, f, max_iters=8)
    for i in range(8):
        assert abs(res.trace.rel_error[i] - ot["rel_error"][i]) <= 1e-5 * ot["rel_error"][i]


@pytest.mark.slow
def test_f32_full_c5_matches_streaming_oracle(gpu_ctx, oracle):
    """BASELINE config 5 at full size (300^4 fp32 U(-1,1), N(0,1) factors, R=64)
    against the CPU oracle: the reference algorithm (mttkrp.cpp:149-241) in fp64 on
    the upcast fp32 values, with both seeds streamed over the generated tensor
    (oracle ora_cp_gradient_all_upm1_f32: same generator, never materialised)."""
    dims, R = [300] * 4, 64
    f = [oracle.fill_normal(500 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
    y32 = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=7, ctx=gpu_ctx, dtype=cpd.F32)
    g32 = cpd.cp_gradient_all(y32, f)
    y32.free()
    want = oracle.cp_gradient_all_upm1_f32(dims, 7, f)
    errs = rel_errs(g32, want)
    print("c5 full-size rel. Frobenius per mode vs the streaming oracle:", errs)
    assert max(errs) <= TOL, errs


def test_f32_streaming_oracle_slab(gpu_ctx, oracle):
    """A last-mode slab of a config-5-like tensor at the global pivot (the sharded
    layout, raw frame): device gradient of the generated slab vs the streaming
    oracle on the same slab (same global indices)."""
    import torch
    dims, R, lo, hi = [40, 40, 40, 40], 64, 13, 27
    slab = dims[:3] + [hi - lo]
    off = lo * 40 ** 3
    f = [oracle.fill_normal(90 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(slab)]
    y = cpd.DenseTensor.generate(slab, cpd.DIST_UNIFORM_PM1, seed=5, ctx=gpu_ctx, dtype=cpd.F32, offset=off)
    fd = torch.from_numpy(np.concatenate([x.reshape(-1, order="F") for x in f])).cuda()
    gd = torch.zeros_like(fd)
    cpd.cp_gradient_all_device(y, R, fd.data_ptr(), gd.data_ptr(), 2)
    torch.cuda.synchronize()
    flat, got, at = gd.cpu().numpy(), [], 0
    for d in slab:
        got.append(flat[at:at + d * R].reshape(d, R, order="F"))
        at += d * R
    y.free()
    want = oracle.cp_gradient_all_upm1_f32(slab, 5, f, offset=off, pivot=2)
    assert max(rel_errs(got, want)) <= TOL


def test_f32_default_path_is_operand_image(gpu_ctx, oracle):
    """Hook-free fp32 gradients with R <= 64 run the one-pass seed over the tensor's
    cached fp16 operand image (seed path 4), rebuilt when the values change."""
    dims, R = [24, 20, 16, 12], 9
    y, yv, f = _case(gpu_ctx, oracle, dims, R, seed=21)
    got = cpd.cp_gradient_all(y, f)
    assert gpu_ctx.last_seed_path() == 4
    want, _, _ = oracle.cp_gradient_all(yv, dims, f)
    assert max(rel_errs(got, want)) <= TOL
    vals2 = np.random.default_rng(8).uniform(-1, 1, yv.size).astype(np.float32)
    y.update(vals2.ctypes.data)  # new version: the operand image is rebuilt
    got2 = cpd.cp_gradient_all(y, f)
    assert gpu_ctx.last_seed_path() == 4
    want2, _, _ = oracle.cp_gradient_all(vals2.astype(np.float64), dims, f)
    assert max(rel_errs(got2, want2)) <= TOL


_PATH_CHECK = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle')
import oracle as O, paper_1204_1586_b200 as cpd
ctx = cpd.Context(0)
out = []
for dims, R in [([40, 40, 40, 40], 64), ([7, 9, 11, 13], 8), ([130, 257], 3), ([300, 300, 20], 16)]:
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=11, ctx=ctx, dtype=cpd.F32)
    yv = y.values().astype(np.float64)
    f = [O.fill_normal(110 + k, d * R).reshape(d, R, order='F') for k, d in enumerate(dims)]
    g = cpd.cp_gradient_all(y, f)
    w, _, _ = O.cp_gradient_all(yv, dims, f)
    err = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(g, w))
    out.append([ctx.last_seed_path(), err])
print(json.dumps(out))
"""


@pytest.mark.parametrize("env,path", [({"CPDGPU_F32_IMAGE": "0"}, 3), ({"CPDGPU_F32_FUSED": "0"}, 2),
                                      ({"CPDGPU_F32_BAND": "2"}, 4), ({"CPDGPU_F32_IMG_CHUNK": "0"}, 4),
                                      ({"CPDGPU_F32_BAND": "2", "CPDGPU_F32_IMG_CHUNK": "0"}, 4),
                                      ({"CPDGPU_F32_LEFT_M64": "0"}, 4)])
def test_f32_alternate_seed_paths(env, path):
    """The fused pass with the split inside the kernel (3, used when the operand
    image does not fit in memory), the two-pass seed (2), and the operand-image pass (4)
    with bands of two row tiles (stacked right product, left-only drain warps) and / or
    the whole-column image layout, and with the lo * lo left product kept (M = 128), against
    the oracle (the defaults: bands of three over the 64-row-chunked image, M = 64 for the
    Y_lo left product)."""
    import json, os, subprocess, sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    res = subprocess.run([sys.executable, "-c", _PATH_CHECK.format(root=root)], env={**os.environ, **env},
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    for got_path, err in json.loads(res.stdout.strip().splitlines()[-1]):
        assert got_path == path and err <= TOL, (got_path, err)


def _rand_shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        N = int(rng.integers(3, 6))
        dims = sorted(int(x) for x in rng.integers(3, 60, size=N))
        if np.prod(dims) > 4_000_000 or np.prod(dims) < 2000:
            continue
        out.append((dims, int(rng.choice([7, 16, 33, 64]))))
    return out


@pytest.mark.parametrize("dims,R", _rand_shapes(2026, 10))
def test_f32_fused_random_shapes(gpu_ctx, oracle, dims, R):
    """Random ascending fp32 shapes through the default path (the fused pass over
    the operand image: ragged bands, ragged column tiles, the first level fused
    with the partial reductions) against the fp64 oracle on the same values."""
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=sum(dims), ctx=gpu_ctx, dtype=cpd.F32)
    f = [oracle.fill_normal(700 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
    g = cpd.cp_gradient_all(y, f)
    want = oracle.cp_gradient_all(y.values().astype(np.float64), dims, f)[0]
    errs = rel_errs(g, want)
    assert max(errs) <= TOL, (dims, R, errs)
    y.free()
