"""Multi-process (gloo, CPU) test of the slab-sharded all-mode gradient host
logic (paper_1204_1586_b200/sharded.py): last-mode slabs, one all_reduce of the
packed partial G(1..N-1), one all_gather of the G(N) rows.  The per-slab compute
is the CPU oracle standing in for the device (test infrastructure only); on the
B200 box the same exchange runs over NCCL after cpdgpu_cp_gradient_all_device."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1204_1586_b200 import sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, R, out_q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = sharded.make_plan(dims, R, rank, world)
        n = int(np.prod(dims))
        y = O.fill_normal(5, n)
        f = [O.fill_normal(6 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        a, b = plan.bounds
        slab = int(np.prod(dims[:-1]))
        local = plan.local_dims
        fl = [f[k] if k < len(dims) - 1 else f[-1][a:b] for k in range(len(dims))]
        g, _, _ = O.cp_gradient_all(y[a * slab:b * slab], local, fl)
        packed = torch.from_numpy(np.concatenate([x.reshape(-1, order="F") for x in g]))
        assert packed.numel() == plan.local_factor_offsets()[-1]
        partial, gN = sharded.exchange(plan, packed, dist)
        got = sharded.unpack(plan, partial, gN)
        if rank == 0:
            want, _, _ = O.cp_gradient_all(y, dims, f)
            errs = [float(np.linalg.norm(got[k] - want[k]) / np.linalg.norm(want[k])) for k in range(len(dims))]
            out_q.put(errs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,R,world", [([4, 5, 6, 7], 3, 2), ([3, 4, 5, 9], 2, 2), ([6, 6, 13], 4, 2)])
def test_sharded_matches_unsharded(dims, R, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    errs = q.get(timeout=10)
    assert max(errs) <= 1e-12, errs


def test_slab_bounds_balanced():
    assert [b - a for a, b in sharded.slab_bounds(300, 8)] == [38, 38, 38, 38, 37, 37, 37, 37]
    assert sharded.slab_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    p = sharded.make_plan([300] * 4, 64, 7, 8)
    assert p.pivot == 2 and p.bounds == (263, 300) and p.max_rows == 38 and p.partial_len == 900 * 64
    with pytest.raises(ValueError):
        sharded.make_plan([5, 3, 4], 2, 0, 2)  # not ascending
    with pytest.raises(ValueError):
        sharded.make_plan([4, 3], 2, 0, 8)  # fewer slices than ranks
