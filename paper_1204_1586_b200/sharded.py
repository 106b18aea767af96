"""Slab sharding of the all-mode gradient across GPUs.

Y is split along its last mode into contiguous slabs, one per rank (column-major,
so a slab is a contiguous byte range).  With the global pivot p* forced on every
slab, the right seed and every G(1..N-1) are linear sums over slabs, while the
rows of G(N) are owned by the slab that holds them:

    local step   : cpdgpu_cp_gradient_all_device(slab, pivot = p*)   (no collective)
    exchange     : one all_reduce(SUM) of [partial G(1..N-1) | G(N) rows at the
                   slab's offset, zeros elsewhere]                    (one NCCL call)

The collective is torch.distributed (NCCL over NVLink on the B200 box, gloo in the
CPU tests); the per-slab compute is injected so the host logic can be tested with
the CPU oracle standing in for the device on a machine without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np


def slab_bounds(extent: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced split of the last mode: sizes differ by at most one
    (300 over 8 ranks -> 38,38,38,38,37,37,37,37)."""
    base, extra = divmod(int(extent), int(world))
    out, at = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((at, at + n))
        at += n
    return out


@dataclass
class SlabPlan:
    dims: tuple            # global dims (ascending; the shard frame is the sorted frame)
    R: int
    rank: int
    world: int
    pivot: int

    @property
    def bounds(self) -> tuple[int, int]:
        return slab_bounds(self.dims[-1], self.world)[self.rank]

    @property
    def local_dims(self) -> list[int]:
        a, b = self.bounds
        return list(self.dims[:-1]) + [b - a]

    @property
    def max_rows(self) -> int:
        return max(b - a for a, b in slab_bounds(self.dims[-1], self.world))

    @property
    def partial_len(self) -> int:  # packed G(1..N-1)
        return sum(int(d) for d in self.dims[:-1]) * self.R

    def local_factor_offsets(self) -> list[int]:
        offs, at = [], 0
        for d in self.local_dims:
            offs.append(at)
            at += int(d) * self.R
        return offs + [at]


def make_plan(dims: Sequence[int], R: int, rank: int, world: int) -> SlabPlan:
    dims = tuple(int(d) for d in dims)
    if list(dims) != sorted(dims):
        raise ValueError("sharded gradient: global dims must be ascending (sort modes first)")
    if len(dims) < 2:
        raise ValueError("sharded gradient: need an order-2 or higher tensor")
    if dims[-1] < world:
        raise ValueError(f"sharded gradient: last mode {dims[-1]} has fewer slices than ranks {world}")
    J = np.cumprod([1] + list(dims))
    p = max(n for n in range(1, len(dims) + 1) if J[n] <= J[-1] // J[n])
    if p >= len(dims):
        raise ValueError("sharded gradient: pivot equals the last mode; nothing to shard")
    return SlabPlan(dims, int(R), int(rank), int(world), p)


def pack_local_factors(plan: SlabPlan, factors: Sequence, xp):
    """Local packed factor buffer: modes 1..N-1 whole, mode N rows of this slab.
    `xp` is numpy or torch; factors are column-major I_n x R arrays."""
    a, b = plan.bounds
    parts = []
    for k, f in enumerate(factors):
        blk = f[a:b] if k == len(factors) - 1 else f
        parts.append(blk.T.reshape(-1) if xp is not np else np.asarray(blk).reshape(-1, order="F"))
    return xp.concatenate(parts) if xp is np else xp.cat(parts)


def exchange(plan: SlabPlan, local_out, dist, group=None):
    """One all_reduce(SUM) carrying both results: the partial G(1..N-1) and the
    G(N) rows, each rank's rows placed at its slab offset of a zero I_N x R block
    (a single latency-bound collective instead of an all_reduce plus an
    all_gather).  local_out: 1-D torch tensor (packed local gradients, caller mode
    order).  Returns (packed summed G(1..N-1), G(N) as an I_N x R column-major
    tensor viewed (R, I_N))."""
    import torch
    P = plan.partial_len
    a, b = plan.bounds
    IN = int(plan.dims[-1])
    buf = torch.zeros(P + plan.R * IN, dtype=local_out.dtype, device=local_out.device)
    buf[:P] = local_out[:P]
    buf[P:].view(plan.R, IN)[:, a:b] = local_out[P:].view(plan.R, b - a)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf[:P], buf[P:].view(plan.R, IN)


def unpack(plan: SlabPlan, partial, gN_rt) -> list[np.ndarray]:
    """Host copies of every G(n), I_n x R, caller mode order."""
    out, at = [], 0
    part = partial.detach().cpu().numpy()
    for d in plan.dims[:-1]:
        n = int(d) * plan.R
        out.append(part[at:at + n].reshape(int(d), plan.R, order="F"))
        at += n
    out.append(np.ascontiguousarray(gN_rt.detach().cpu().numpy().T))
    return out


def sharded_gradient(plan: SlabPlan, local_compute: Callable, dist, group=None):
    """One sharded all-mode gradient: local_compute() -> packed local gradients
    (1-D torch tensor); then the exchange."""
    local_out = local_compute()
    return exchange(plan, local_out, dist, group)


def library_comm(ctx, dist, group=None):
    """The library-side communicator (cpdgpu_comm_*) of this rank, built from an
    initialised torch.distributed group: NCCL backends get an NCCL communicator
    inside libcpdgpu.so (rank 0's unique id broadcast over the group), anything
    else (gloo) a host all-reduce through the group."""
    import torch
    from . import api
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        obj = [api.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return api.Communicator(ctx, world, rank, unique_id=obj[0])

    def host_allreduce(buf):
        t = torch.from_numpy(buf)  # shares the library's pinned host buffer
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return api.Communicator(ctx, world, rank, host_allreduce=host_allreduce)
