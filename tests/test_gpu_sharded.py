"""The slab-sharded gradient's device side on one GPU: every rank's slab runs
cp_gradient_all_device with the global pivot (the call bench.py makes per rank
under NCCL), and combining the slabs the way sharded.exchange does (sum of the
partial G(1..N-1), concatenation of the G(N) rows) reproduces the unsharded
gradient.  The NCCL collective itself is covered by the gloo tests
(test_sharded_gloo.py); this pins the per-slab compute, fp64 and fp32."""
import numpy as np
import pytest
import torch

import paper_1204_1586_b200 as cpd
from paper_1204_1586_b200 import sharded

pytestmark = pytest.mark.gpu


def _slab_gradients(ctx, gdims, R, world, dist, dtype, factors):
    outs = []
    for rank in range(world):
        plan = sharded.make_plan(gdims, R, rank, world)
        a, b = plan.bounds
        y = cpd.DenseTensor.generate(plan.local_dims, dist, seed=3, ctx=ctx, dtype=dtype,
                                     offset=a * int(np.prod(gdims[:-1])))
        f = torch.from_numpy(sharded.pack_local_factors(plan, factors, np)).cuda()
        g = torch.zeros_like(f)
        cpd.cp_gradient_all_device(y, R, f.data_ptr(), g.data_ptr(), plan.pivot)
        torch.cuda.synchronize()
        outs.append((plan, g.cpu().numpy()))
        y.free()
    plan0 = outs[0][0]
    P = plan0.partial_len
    partial = torch.from_numpy(sum(o[:P] for _, o in outs))
    rows = [torch.from_numpy(o[P:].reshape(R, -1)) for _, o in outs]  # (R, rows) views
    return sharded.unpack(plan0, partial, torch.cat(rows, dim=1))


@pytest.mark.parametrize("gdims,R,world,f32", [
    ([12, 14, 15, 22], 6, 2, False),
    ([12, 14, 15, 22], 6, 3, False),
    ([20, 30, 40], 9, 4, False),
    ([40, 40, 40, 40], 64, 2, True),
    ([48, 48, 48, 64], 64, 8, True),
])
def test_slabs_reproduce_unsharded(gpu_ctx, oracle, gdims, R, world, f32):
    dtype = cpd.F32 if f32 else cpd.F64
    dist = cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL
    factors = [oracle.fill_normal(40 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(gdims)]
    got = _slab_gradients(gpu_ctx, gdims, R, world, dist, dtype, factors)
    yfull = cpd.DenseTensor.generate(gdims, dist, seed=3, ctx=gpu_ctx, dtype=dtype)
    want, _, _ = oracle.cp_gradient_all(yfull.values().astype(np.float64), gdims, factors)
    tol = 1e-5 if f32 else 1e-10
    for k in range(len(gdims)):
        err = np.linalg.norm(got[k] - want[k]) / np.linalg.norm(want[k])
        assert err <= tol, (k, err)


@pytest.mark.parametrize("gdims,R,world", [([32, 34, 36, 40], 12, 2), ([20, 30, 64], 20, 4)])
def test_int8_slabs_reproduce_unsharded(gpu_ctx, oracle, monkeypatch, gdims, R, world):
    # the same per-slab calls on the int8 seed path (global pivot, raw frame)
    monkeypatch.setenv("CPDGPU_I8", "1")
    factors = [oracle.fill_normal(70 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(gdims)]
    got = _slab_gradients(gpu_ctx, gdims, R, world, cpd.DIST_NORMAL, cpd.F64, factors)
    assert gpu_ctx.last_seed_path() == 1
    yfull = cpd.DenseTensor.generate(gdims, cpd.DIST_NORMAL, seed=3, ctx=gpu_ctx)
    want, _, _ = oracle.cp_gradient_all(yfull.values(), gdims, factors)
    for k in range(len(gdims)):
        err = np.linalg.norm(got[k] - want[k]) / np.linalg.norm(want[k])
        assert err <= 1e-10, (k, err)
