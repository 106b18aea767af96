"""The sharded all-mode gradient behind the C-ABI (cpdgpu_comm_init_host /
cpdgpu_cp_gradient_all_sharded[_device]): two processes (world size 2, gloo as
the library's host all-reduce) each hold one last-mode slab of a tensor on the
one GPU of the box, and both receive the GLOBAL gradients, compared with the
CPU oracle's unsharded gradient (mttkrp.cpp:113-253).  The ranks never wait on
each other inside a kernel (the exchange is a host collective), so sharing one
device is safe; on an 8-GPU box the same entry points run NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, R, f32, out_q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import torch
    import torch.distributed as dist
    import oracle as O
    import paper_1204_1586_b200 as cpd
    from paper_1204_1586_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = cpd.Context(0)
        comm = sharded.library_comm(ctx, dist)
        lo, hi = comm.bounds(dims[-1])
        ldims = list(dims[:-1]) + [hi - lo]
        front = int(np.prod(dims[:-1]))
        y = cpd.DenseTensor.generate(ldims, cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL, seed=11,
                                     ctx=ctx, offset=lo * front, dtype=cpd.F32 if f32 else cpd.F64)
        f = [O.fill_normal(30 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        counter = cpd.CostCounter()
        got = cpd.cp_gradient_all_sharded(y, dims, f, counter)
        # device form: packed slab factors in, packed global result out
        packed = np.concatenate([x.reshape(-1, order="F") for x in f[:-1]] +
                                [f[-1][lo:hi].reshape(-1, order="F")])
        fd = torch.from_numpy(packed).cuda()
        out = torch.zeros(sum(dims) * R, dtype=torch.float64, device="cuda")
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        cpd.cp_gradient_all_sharded_device(y, dims, R, fd.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        dev, at = [], 0
        for d in dims:
            dev.append(o[at:at + d * R].reshape(d, R, order="F"))
            at += d * R
        comm.close()
        # oracle: the whole tensor (the same counter-based values) on the CPU
        full = cpd.DenseTensor.generate(list(dims), cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL, seed=11,
                                        ctx=ctx, dtype=cpd.F32 if f32 else cpd.F64)
        want, _, _ = O.cp_gradient_all(full.values().astype(np.float64), list(dims), f)
        errs = [float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(got, want)]
        errs += [float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(dev, want)]
        want_mults = sum(cpd.fast_count_realized(dims, R, n) for n in range(1, len(dims) + 1))
        out_q.put((rank, errs, counter.total() == want_mults))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,R,f32", [([6, 7, 8, 9], 5, False), ([12, 14, 16, 20], 20, False),
                                        ([5, 6, 7], 3, False), ([16, 16, 16, 17], 64, True)])
def test_sharded_abi_matches_oracle(dims, R, f32):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, R, f32, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    tol = 1e-5 if f32 else 1e-12
    for rank, errs, counted in res:
        assert max(errs) <= tol, (rank, errs)
        assert counted


def test_sharded_needs_a_communicator(gpu_ctx):
    import paper_1204_1586_b200 as cpd
    y = cpd.DenseTensor.generate([4, 5, 3], cpd.DIST_NORMAL, seed=1, ctx=gpu_ctx)
    f = [np.ones((d, 2)) for d in [4, 5, 6]]
    with pytest.raises(cpd.ArgumentError):
        cpd.cp_gradient_all_sharded(y, [4, 5, 6], f)


def test_sharded_single_rank_is_the_plain_gradient(gpu_ctx, oracle):
    """World size 1 through the host communicator: the slab is the whole tensor."""
    import paper_1204_1586_b200 as cpd
    dims, R = [5, 6, 7, 8], 4
    comm = cpd.Communicator(gpu_ctx, 1, 0, host_allreduce=lambda buf: None)
    try:
        y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=2, ctx=gpu_ctx)
        f = [oracle.fill_normal(50 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        got = cpd.cp_gradient_all_sharded(y, dims, f)
        want, _, _ = oracle.cp_gradient_all(y.values(), dims, f)
        for g, w in zip(got, want):
            assert np.linalg.norm(g - w) / np.linalg.norm(w) <= 1e-12
        with pytest.raises(cpd.ShapeError):  # slab extent disagrees with the global dims
            cpd.cp_gradient_all_sharded(y, [5, 6, 7, 9], [np.ones((d, R)) for d in [5, 6, 7, 9]])
    finally:
        comm.close()


def _als_worker(rank, world, port, dims, R, iters, f32, out_q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import torch.distributed as dist
    import oracle as O
    import paper_1204_1586_b200 as cpd
    from paper_1204_1586_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = cpd.Context(0)
        comm = sharded.library_comm(ctx, dist)
        lo, hi = comm.bounds(dims[-1])
        front = int(np.prod(dims[:-1]))
        dist_kind = cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL
        dt = cpd.F32 if f32 else cpd.F64
        y = cpd.DenseTensor.generate(list(dims[:-1]) + [hi - lo], dist_kind, seed=13, ctx=ctx, offset=lo * front,
                                     dtype=dt)
        init = cpd.random_init(dims, R, 5)
        fr = [f.copy(order="F") for f in init]
        trace = cpd.als_run_sharded(y, dims, fr, max_iters=iters)
        fs = [f.copy(order="F") for f in init]
        counter = cpd.CostCounter()
        c1 = cpd.als_sweep_sharded(y, dims, fs, counter=counter)
        comm.close()
        full = cpd.DenseTensor.generate(list(dims), dist_kind, seed=13, ctx=ctx, dtype=dt)
        yv = full.values().astype(np.float64)
        of, ot = O.run_als_fast(yv, dims, init, max_iters=iters)
        o1 = O.als_sweep_fast(yv, dims, [f.copy(order="F") for f in init])
        ferr = max(float(np.max(np.abs(a - b)) / np.max(np.abs(b))) for a, b in zip(fr, of))
        cerr = max(abs(a - b) / b for a, b in zip(trace.cost, ot["cost"]))
        serr = max(float(np.max(np.abs(a - b)) / np.max(np.abs(b))) for a, b in zip(fs, o1))
        c1err = abs(c1 - O.cost(yv, dims, o1)) / c1
        want_mults = sum(cpd.fast_count_realized(dims, R, n) for n in range(1, len(dims) + 1))
        digest = float(sum(np.sum(f * (k + 1)) for k, f in enumerate(fr)))
        out_q.put((rank, trace.iters_run, ferr, cerr, serr, c1err, counter.total() == want_mults, digest))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,R,f32", [([6, 7, 8, 9], 5, False), ([12, 14, 16, 20], 12, False),
                                        ([5, 6, 7], 3, False), ([16, 16, 16, 17], 8, True)])
def test_sharded_als_matches_oracle(dims, R, f32):
    """Sharded fast ALS (cpdgpu_als_run_sharded / cpdgpu_als_sweep_sharded) over two
    last-mode slabs against the oracle's unsharded run on the whole tensor
    (als.cpp:69-78, 147-210): same Gauss-Seidel order, so the factors and the
    cost trace agree to summation order; both ranks hold identical factors."""
    world, iters = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_als_worker, args=(r, world, port, dims, R, iters, f32, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    tol = 1e-4 if f32 else 1e-9  # ALS amplifies the gradient's rounding by the Gram conditioning
    for rank, done, ferr, cerr, serr, c1err, counted, _ in res:
        assert done == iters
        assert ferr <= tol and serr <= tol, (rank, ferr, serr)
        assert cerr <= tol and c1err <= tol, (rank, cerr, c1err)
        assert counted
    assert res[0][-1] == res[1][-1]  # every rank leaves with the same factors


def test_sharded_nccl_world_size_one(gpu_ctx, oracle):
    """The library's NCCL communicator itself (libnccl dlopen'ed, ncclGetUniqueId,
    ncclCommInitRank, the in-place ncclAllReduce on the context stream, destroy) on
    the one GPU of the box as a world of one rank: the sharded gradient, device
    form and ALS sweep through it equal the oracle's unsharded results.  (With more
    GPUs the same calls run one rank per GPU; the slab split itself is covered by
    the two-process test above over the host all-reduce.)"""
    import torch
    import paper_1204_1586_b200 as cpd
    dims, R = [9, 10, 11, 12], 7
    comm = cpd.Communicator(gpu_ctx, 1, 0, unique_id=cpd.comm_unique_id())
    try:
        assert comm.bounds(dims[-1]) == (0, dims[-1])
        y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=21, ctx=gpu_ctx)
        f = [oracle.fill_normal(70 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        want, _, _ = oracle.cp_gradient_all(y.values(), dims, f)
        got = cpd.cp_gradient_all_sharded(y, dims, f)
        for g, w in zip(got, want):
            assert np.linalg.norm(g - w) / np.linalg.norm(w) <= 1e-12
        packed = np.concatenate([x.reshape(-1, order="F") for x in f])
        fd = torch.from_numpy(packed).cuda()
        out = torch.zeros(sum(dims) * R, dtype=torch.float64, device="cuda")
        gpu_ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        cpd.cp_gradient_all_sharded_device(y, dims, R, fd.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        gpu_ctx.set_stream(0)
        o, at = out.cpu().numpy(), 0
        for d, w in zip(dims, want):
            g = o[at:at + d * R].reshape(d, R, order="F")
            at += d * R
            assert np.linalg.norm(g - w) / np.linalg.norm(w) <= 1e-12
        f2 = [x.copy() for x in f]
        cost = cpd.als_sweep_sharded(y, dims, f2)
        f3 = [x.copy() for x in f]
        oracle.als_sweep_fast(y.values(), dims, f3)
        for a, b in zip(f2, f3):
            assert np.abs(a - b).max() <= 1e-9 * np.abs(b).max()
        assert np.isfinite(cost)
    finally:
        comm.close()
