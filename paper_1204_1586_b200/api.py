"""Host-side mirror of the reference's hot-path API (proj/core/include/cpd/
{mttkrp,als,kruskal,cost_counter}.hpp) over the C-ABI.

Same names, argument meaning, column-major layout and error behaviour as the
reference; arrays are numpy.  Every numeric call runs on the B200 through
libcpdgpu.so — nothing here computes the gradient on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib, errors

F64, F32 = 0, 1
DIST_NORMAL, DIST_UNIFORM_PM1 = 0, 1


# ---- instrumentation (cost_counter.hpp:11-27, mttkrp.hpp:44-47) -------------

class CostCounter:
    """Running tally of scalar multiplications (cost_counter.hpp:11-27)."""

    def __init__(self) -> None:
        self._total = 0

    def charge(self, mults: int) -> None:
        self._total += int(mults)

    def charge_gemm(self, m: int, k: int, p: int) -> None:
        self._total += int(m) * int(k) * int(p)

    def charge_kron(self, p: int, q: int) -> None:
        self._total += int(p) * int(q)

    def total(self) -> int:
        return self._total

    def reset(self) -> None:
        self._total = 0


@dataclass
class FastStats:
    """mttkrp.hpp:44-47: high-water mark of workspace doubles (outputs excluded)."""
    peak_workspace_doubles: int = 0


# ---- context and tensors (dense_tensor.hpp:15-47) ----------------------------

class Context:
    """One B200 device plus a CUDA stream (cpdgpu_ctx)."""

    def __init__(self, device: int = 0) -> None:
        self._L = _lib.load()
        h = C.c_void_p()
        _lib.check(self._L.cpdgpu_create(C.byref(h), int(device)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self._L.cpdgpu_destroy(self.h)
            self.h = None

    def __del__(self) -> None:  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        """Order all work on an external cudaStream_t (e.g. torch's current stream)."""
        _lib.check(self._L.cpdgpu_set_stream(self.h, C.c_void_p(stream_ptr)), self.h)

    def synchronize(self) -> None:
        _lib.check(self._L.cpdgpu_synchronize(self.h), self.h)

    def launch_count(self) -> int:
        return int(self._L.cpdgpu_launch_count(self.h))

    def device_workspace(self) -> tuple[int, int]:
        """(bytes now, high-water bytes) of device workspace the library holds besides the
        tensors' own values: this implementation's FastStats::peak_workspace figure
        (mttkrp.hpp:37-47); the gradient calls report the reference algorithm's."""
        cur, peak = C.c_int64(), C.c_int64()
        _lib.check(self._L.cpdgpu_device_workspace(self.h, C.byref(cur), C.byref(peak)), self.h)
        return int(cur.value), int(peak.value)

    def set_timing(self, enabled: bool) -> None:
        _lib.check(self._L.cpdgpu_set_timing(self.h, int(bool(enabled))), self.h)

    def set_graphs(self, enabled: bool) -> None:
        _lib.check(self._L.cpdgpu_set_graphs(self.h, int(bool(enabled))), self.h)

    def set_deterministic(self, enabled: bool) -> None:
        """Bitwise-reproducible results run to run (cpdgpu_set_deterministic): the
        fused fp32 and int8 fp64 seeds then sum their left partials in a fixed
        order instead of by red.add in L2."""
        _lib.check(self._L.cpdgpu_set_deterministic(self.h, int(bool(enabled))), self.h)

    def last_seed_path(self) -> int:
        """0: fp64 DMMA seed pass, 1: fused int8 tensor-core pass, 2: fp32 pass."""
        return int(self._L.cpdgpu_last_seed_path(self.h))

    def last_seed_ms(self) -> float:
        v = C.c_double()
        _lib.check(self._L.cpdgpu_last_seed_ms(self.h, C.byref(v)), self.h)
        return float(v.value)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _dims_arg(dims: Sequence[int]):
    arr = (C.c_int64 * len(dims))(*[int(d) for d in dims])
    return arr


class DenseTensor:
    """Immutable dense column-major tensor resident on the device.

    Mirrors cpd::DenseTensor (dense_tensor.hpp:15-47): entry (i_1..i_N) lives at
    the vectorization-order position; values never change after creation.
    """

    def __init__(self, ctx: Context, handle: C.c_void_p, dims: Sequence[int], dtype: int) -> None:
        self.ctx, self.h, self.dims, self.dtype = ctx, handle, tuple(int(d) for d in dims), dtype

    # constructors -----------------------------------------------------------
    @classmethod
    def from_values(cls, values, dims: Sequence[int], ctx: Optional[Context] = None,
                    dtype: int = F64) -> "DenseTensor":
        """values: flat vector in vectorization order (first index fastest), or an
        N-d numpy array (interpreted by its logical indices, any memory order)."""
        ctx = ctx or default_context()
        np_dtype = np.float64 if dtype == F64 else np.float32
        a = np.asarray(values)
        if a.ndim > 1:
            if tuple(a.shape) != tuple(dims):
                raise errors.ShapeError(f"tensor: array shape {a.shape} != dims {tuple(dims)}")
            flat = np.asarray(a, dtype=np_dtype).reshape(-1, order="F")
        else:
            flat = np.ascontiguousarray(a, dtype=np_dtype)
        n = int(np.prod([int(d) for d in dims])) if len(dims) else 0
        if flat.size != n:
            raise errors.ShapeError(f"tensor: {flat.size} values for a shape holding {n} entries")
        h = C.c_void_p()
        d = _dims_arg(dims)
        _lib.check(ctx._L.cpdgpu_tensor_upload(ctx.h, flat.ctypes.data_as(C.c_void_p), dtype,
                                               len(dims), d, C.byref(h)), ctx.h)
        return cls(ctx, h, dims, dtype)

    @classmethod
    def generate(cls, dims: Sequence[int], dist: int = DIST_NORMAL, seed: int = 0,
                 ctx: Optional[Context] = None, dtype: int = F64, offset: int = 0) -> "DenseTensor":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _lib.check(ctx._L.cpdgpu_tensor_generate(ctx.h, dtype, len(dims), _dims_arg(dims), dist,
                                                 C.c_uint64(seed), int(offset), C.byref(h)), ctx.h)
        return cls(ctx, h, dims, dtype)

    @classmethod
    def load_tdnb(cls, path: str, slab: Optional[tuple] = None, ctx: Optional[Context] = None) -> "DenseTensor":
        """Binary tensor file (io.cpp:162-181) streamed through pinned buffers to the
        device; slab=(lo, hi) loads only last-mode slices [lo, hi) (a rank's shard)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        lo, hi = (int(slab[0]), int(slab[1])) if slab else (0, 0)
        _lib.check(ctx._L.cpdgpu_tensor_load_tdnb(ctx.h, str(path).encode(), lo, hi, C.byref(h)), ctx.h)
        with open(path, "rb") as f:
            head = f.read(8)
            n = int.from_bytes(head[4:8], "little")
            dims = [int.from_bytes(f.read(4), "little") for _ in range(n)]
        if slab:
            dims[-1] = hi - lo
        return cls(ctx, h, dims, F64)

    def save_tdnb(self, path: str) -> None:
        """Write the binary tensor file (io.cpp:192-203), f64 little-endian."""
        _lib.check(self.ctx._L.cpdgpu_tensor_save_tdnb(self.ctx.h, self.h, str(path).encode()), self.ctx.h)

    @classmethod
    def wrap_device(cls, ptr: int, dims: Sequence[int], ctx: Optional[Context] = None,
                    dtype: int = F64) -> "DenseTensor":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _lib.check(ctx._L.cpdgpu_tensor_wrap_device(ctx.h, C.c_void_p(ptr), dtype, len(dims),
                                                    _dims_arg(dims), C.byref(h)), ctx.h)
        return cls(ctx, h, dims, dtype)

    # queries ------------------------------------------------------------------
    def order(self) -> int:
        return len(self.dims)

    def size(self) -> int:
        return int(np.prod(self.dims))

    def values(self) -> np.ndarray:
        out = np.empty(self.size(), dtype=np.float64 if self.dtype == F64 else np.float32)
        _lib.check(self.ctx._L.cpdgpu_tensor_download(self.ctx.h, self.h,
                                                      out.ctypes.data_as(C.c_void_p)), self.ctx.h)
        return out

    def update(self, host_ptr: int) -> None:
        """H2D refresh of the values from host memory at host_ptr (same dims/dtype)."""
        _lib.check(self.ctx._L.cpdgpu_tensor_update(self.ctx.h, self.h, C.c_void_p(host_ptr)), self.ctx.h)

    def norm2(self) -> float:
        v = C.c_double()
        _lib.check(self.ctx._L.cpdgpu_tensor_norm2(self.ctx.h, self.h, C.byref(v)), self.ctx.h)
        return float(v.value)

    def norm(self) -> float:
        return float(np.sqrt(self.norm2()))

    def device_ptr(self) -> int:
        p = C.c_void_p()
        _lib.check(self.ctx._L.cpdgpu_tensor_device_ptr(self.h, C.byref(p)))
        return int(p.value or 0)

    def axpby_kruskal(self, alpha: float, beta: float, factors: Sequence[np.ndarray]) -> None:
        """Y <- alpha Y + beta full(model) on the device (setup helper)."""
        bufs = _factor_bufs(factors, self.dims)
        _lib.check(self.ctx._L.cpdgpu_tensor_axpby_kruskal(self.ctx.h, self.h, alpha, beta,
                                                           _ptr_array(bufs), bufs[0].shape[1]),
                   self.ctx.h)

    def free(self) -> None:
        if self.h:
            self.ctx._L.cpdgpu_tensor_free(self.h)
            self.h = None

    def __del__(self) -> None:  # pragma: no cover
        try:
            if self.h and self.ctx.h:
                self.free()
        except Exception:
            pass


# ---- helpers ---------------------------------------------------------------------

def _factor_bufs(factors: Sequence[np.ndarray], dims: Sequence[int]) -> list:
    """Column-major float64 copies; validates factor_shape (kron.cpp:25-45)."""
    if len(factors) == 0:
        raise errors.ArgumentError("factors: empty list")
    bufs = [np.asfortranarray(np.asarray(f, dtype=np.float64)) for f in factors]
    for k, b in enumerate(bufs):
        if b.ndim == 1:
            bufs[k] = b = np.asfortranarray(b.reshape(-1, 1))
        if b.ndim != 2:
            raise errors.ShapeError(f"factors: mode {k + 1} is not a matrix")
    R = bufs[0].shape[1]
    for k, b in enumerate(bufs):
        if b.shape[1] != R:
            raise errors.ShapeError(f"factors: mode {k + 1} has rank {b.shape[1]}, expected {R}")
        if b.shape[0] < 1:
            raise errors.ShapeError(f"factors: mode {k + 1} has no rows")
    if len(bufs) != len(dims) or any(b.shape[0] != d for b, d in zip(bufs, dims)):
        raise errors.ShapeError("cp_gradient_all: factor row counts do not match the tensor")
    return bufs


def _ptr_array(bufs: Sequence[np.ndarray]):
    arr = (_lib.c_dbl_p * len(bufs))()
    for i, b in enumerate(bufs):
        arr[i] = b.ctypes.data_as(_lib.c_dbl_p)
    return arr


# ---- ordering helpers (mttkrp.hpp:24,35,73) ------------------------------------

def select_pivot(dims: Sequence[int]) -> int:
    L = _lib.load()
    p = C.c_int()
    _lib.check(L.cpdgpu_select_pivot(len(dims), _dims_arg(dims), C.byref(p)))
    return p.value


def sort_modes(dims: Sequence[int]) -> tuple[list[int], list[int]]:
    """(perm, inverse), 1-based, as SortResult::perm / ::inverse (mttkrp.hpp:28-33)."""
    L = _lib.load()
    n = len(dims)
    perm, inv = (C.c_int * max(n, 1))(), (C.c_int * max(n, 1))()
    _lib.check(L.cpdgpu_sort_modes(n, _dims_arg(dims), perm, inv))
    return list(perm)[:n], list(inv)[:n]


def fast_update_order(dims: Sequence[int]) -> list[int]:
    L = _lib.load()
    n = len(dims)
    out = (C.c_int * max(n, 1))()
    _lib.check(L.cpdgpu_fast_update_order(n, _dims_arg(dims), out))
    return list(out)[:n]


def fast_count_realized(dims: Sequence[int], R: int, n: int) -> int:
    L = _lib.load()
    if list(dims) != sorted(dims):
        raise errors.ArgumentError("fast_count_realized: dims must be ascending")
    if R < 1:
        raise errors.ArgumentError("fast_count_realized: rank must be positive")
    if n < 1 or n > len(dims):
        raise errors.IndexError(f"fast_count_realized: mode {n} outside 1..{len(dims)}")
    return int(L.cpdgpu_fast_count_realized(len(dims), _dims_arg(dims), R, n))


# ---- the all-mode gradient (mttkrp.hpp:59-69) ----------------------------------

ModeHook = Callable[[int, np.ndarray], None]


def cp_gradient_all(y: DenseTensor, factors: list, counter: Optional[CostCounter] = None,
                    hook: Optional[ModeHook] = None,
                    stats: Optional[FastStats] = None) -> list[np.ndarray]:
    """All-mode CP gradients G^(n) = Y_(n) (KR_{k != n} A^(k)) (mttkrp.cpp:113-253).

    With a hook, ``hook(n, G)`` runs right after mode n's gradient is ready (in
    fast_update_order) and may replace ``factors[n-1]``; the sweep re-reads it
    (mttkrp.cpp:134-145).  The counter is charged per mode before the hook.
    """
    if y.order() < 2:
        raise errors.ArgumentError("cp_gradient_all: need an order-2 or higher tensor")
    bufs = _factor_bufs(factors, y.dims)
    R = bufs[0].shape[1]
    grads = [np.empty((d, R), dtype=np.float64, order="F") for d in y.dims]
    fptr, gptr = _ptr_array(bufs), _ptr_array(grads)
    peak = C.c_int64()
    ctx = y.ctx
    if hook is None:
        mults = (C.c_uint64 * len(y.dims))()
        _lib.check(ctx._L.cpdgpu_cp_gradient_all(ctx.h, y.h, R, fptr, gptr, mults, C.byref(peak)), ctx.h)
        if counter is not None:
            counter.charge(sum(int(m) for m in mults))
    else:
        err: list = []

        def _cb(user, mode, g, rows, rank, m):  # runs on the caller's thread
            try:
                if counter is not None:
                    counter.charge(int(m))
                hook(mode, grads[mode - 1].copy(order="F"))
                F = np.asarray(factors[mode - 1], dtype=np.float64)
                if F.ndim == 1:
                    F = F.reshape(-1, 1)
                if F.shape != (y.dims[mode - 1], R):
                    raise errors.ShapeError(
                        f"cp_gradient_all: hook left factor of mode {mode} with the wrong size")
                bufs[mode - 1][...] = F
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised below
                err.append(e)
                return 9  # CPDGPU_HOOK_ABORTED: the hook's own exception is re-raised below

        cb = _lib.HOOK(_cb)
        st = ctx._L.cpdgpu_cp_gradient_all_hook(ctx.h, y.h, R, fptr, gptr, cb, None, C.byref(peak))
        if err:
            raise err[0]
        _lib.check(st, ctx.h)
    if stats is not None:
        stats.peak_workspace_doubles = int(peak.value)
    return grads


def cp_gradient_all_device(y: DenseTensor, R: int, factors_dev_ptr: int, grads_dev_ptr: int,
                           pivot: int = 0) -> None:
    """Device-buffer form (packed factors/gradients in caller mode order), ordered on
    the context stream; used by the sharded multi-GPU driver."""
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_cp_gradient_all_device(ctx.h, y.h, int(R), C.c_void_p(factors_dev_ptr),
                                                    C.c_void_p(grads_dev_ptr), int(pivot)), ctx.h)


# ---- multi-GPU: last-mode slabs, the exchange inside libcpdgpu.so ----

def slab_bounds(extent: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous last-mode slab (cpdgpu_slab_bounds)."""
    L = _lib.load()
    lo, hi = C.c_int64(), C.c_int64()
    _lib.check(L.cpdgpu_slab_bounds(int(extent), int(world), int(rank), C.byref(lo), C.byref(hi)))
    return int(lo.value), int(hi.value)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 makes it, the caller broadcasts it)."""
    L = _lib.load()
    buf = (C.c_ubyte * _lib.COMM_ID_BYTES)()
    _lib.check(L.cpdgpu_comm_unique_id(buf))
    return bytes(buf)


class Communicator:
    """The context's communicator for cp_gradient_all_sharded: NCCL (one rank per
    GPU, in-place ncclAllReduce on the context stream) or a caller-supplied host
    all-reduce ``fn(np.ndarray) -> None`` that sums a float64 buffer in place
    across the ranks (gloo, MPI, ...)."""

    def __init__(self, ctx: Context, world: int, rank: int, unique_id: Optional[bytes] = None,
                 host_allreduce: Optional[Callable[[np.ndarray], None]] = None) -> None:
        self.ctx, self.world, self.rank = ctx, int(world), int(rank)
        self._cb = None
        L = ctx._L
        if host_allreduce is not None:
            err: list = []

            def _ar(user, buf, count):
                try:
                    host_allreduce(np.ctypeslib.as_array(buf, shape=(int(count),)))
                    return 0
                except BaseException as e:  # noqa: BLE001 - surfaced through the status
                    err.append(e)
                    return 7  # CPDGPU_CUDA_ERROR class: the exchange failed
            self._errors = err
            self._cb = _lib.ALLREDUCE(_ar)
            _lib.check(L.cpdgpu_comm_init_host(ctx.h, self.world, self.rank, self._cb, None), ctx.h)
        else:
            if unique_id is None or len(unique_id) != _lib.COMM_ID_BYTES:
                raise errors.ArgumentError("Communicator: need the 128-byte NCCL unique id or a host all-reduce")
            buf = (C.c_ubyte * _lib.COMM_ID_BYTES).from_buffer_copy(unique_id)
            _lib.check(L.cpdgpu_comm_init(ctx.h, buf, self.world, self.rank), ctx.h)

    def bounds(self, extent: int) -> tuple[int, int]:
        return slab_bounds(extent, self.world, self.rank)

    def close(self) -> None:
        if self.ctx is not None and self.ctx.h:
            _lib.check(self.ctx._L.cpdgpu_comm_destroy(self.ctx.h), self.ctx.h)
        self.ctx = None


def cp_gradient_all_sharded(slab: DenseTensor, global_dims: Sequence[int], factors: list,
                            counter: Optional[CostCounter] = None) -> list[np.ndarray]:
    """Sharded all-mode gradient (mttkrp.hpp:59-69 over a last-mode slab): every
    rank passes its slab and the GLOBAL factors and receives every global G(n).
    The context needs a Communicator; the exchange runs inside the library."""
    gd = [int(d) for d in global_dims]
    bufs = _factor_bufs(factors, gd)
    R = bufs[0].shape[1]
    grads = [np.empty((d, R), dtype=np.float64, order="F") for d in gd]
    mults = (C.c_uint64 * len(gd))()
    ctx = slab.ctx
    _lib.check(ctx._L.cpdgpu_cp_gradient_all_sharded(ctx.h, slab.h, len(gd), _dims_arg(gd), R, _ptr_array(bufs),
                                                     _ptr_array(grads), mults), ctx.h)
    if counter is not None:
        counter.charge(sum(int(m) for m in mults))
    return grads


def cp_gradient_all_sharded_device(slab: DenseTensor, global_dims: Sequence[int], R: int, factors_dev_ptr: int,
                                   out_dev_ptr: int) -> None:
    """Device form, ordered on the context stream: the slab's packed factors in,
    the packed GLOBAL gradients [G(1..N-1) | G(N)] out (every rank)."""
    gd = [int(d) for d in global_dims]
    ctx = slab.ctx
    _lib.check(ctx._L.cpdgpu_cp_gradient_all_sharded_device(ctx.h, slab.h, len(gd), _dims_arg(gd), int(R),
                                                            C.c_void_p(factors_dev_ptr), C.c_void_p(out_dev_ptr)),
               ctx.h)


def als_sweep_sharded(slab: DenseTensor, global_dims: Sequence[int], factors: list, pinv_rtol: float = 1e-12,
                      counter: Optional[CostCounter] = None) -> float:
    """Sharded fast ALS sweep (als.cpp:69-78 over a last-mode slab): every rank
    passes its slab and the GLOBAL factors, which are replaced (list elements)
    by the same updated factors on every rank.  Returns the global cost after
    the sweep (kruskal.cpp:58-77)."""
    gd = [int(d) for d in global_dims]
    bufs = [b.copy(order="F") for b in _factor_bufs(factors, gd)]
    R = bufs[0].shape[1]
    cost, mults = C.c_double(), C.c_uint64()
    ctx = slab.ctx
    _lib.check(ctx._L.cpdgpu_als_sweep_sharded(ctx.h, slab.h, len(gd), _dims_arg(gd), R, _ptr_array(bufs), pinv_rtol,
                                               C.byref(cost), C.byref(mults)), ctx.h)
    for k, b in enumerate(bufs):
        factors[k] = b
    if counter is not None:
        counter.charge(int(mults.value))
    return float(cost.value)


def als_run_sharded(slab: DenseTensor, global_dims: Sequence[int], factors: list, max_iters: int = 20,
                    tol: float = 0.0, pinv_rtol: float = 1e-12) -> "RunTrace":
    """run(..., Algorithm::als_fast) (als.cpp:147-210) over last-mode slabs;
    factors replaced in place (list elements), identical on every rank."""
    gd = [int(d) for d in global_dims]
    bufs = [b.copy(order="F") for b in _factor_bufs(factors, gd)]
    R = bufs[0].shape[1]
    cost, rel, sec = (np.zeros(max_iters) for _ in range(3))
    mults = (C.c_uint64 * max_iters)()
    it = C.c_int()
    ctx = slab.ctx
    dp = lambda a: a.ctypes.data_as(_lib.c_dbl_p)  # noqa: E731
    _lib.check(ctx._L.cpdgpu_als_run_sharded(ctx.h, slab.h, len(gd), _dims_arg(gd), R, _ptr_array(bufs),
                                             int(max_iters), float(tol), float(pinv_rtol), dp(cost), dp(rel),
                                             dp(sec), mults, C.byref(it)), ctx.h)
    for k, b in enumerate(bufs):
        factors[k] = b
    n = it.value
    return RunTrace(cost=list(cost[:n]), rel_error=list(rel[:n]), seconds=list(sec[:n]),
                    mults=[int(m) for m in mults[:n]], iters_run=n)


# ---- direct MTTKRP (mttkrp.hpp:19-20): Algorithm 1's one-pass-per-mode cost ---------

def mttkrp_direct(y: DenseTensor, factors: list, n: int, counter: Optional[CostCounter] = None) -> np.ndarray:
    """M^(n) = Y_(n) (KR_{k != n} A^(k)) for one mode (mttkrp.cpp:29-54), on the device:
    one pass over Y per call (the baseline the all-mode recursion is measured against)."""
    bufs = _factor_bufs(factors, y.dims)
    R = bufs[0].shape[1]
    if not 1 <= n <= len(y.dims):
        raise errors.IndexError(f"mttkrp_direct: mode {n} outside 1..{len(y.dims)}")
    out = np.empty((y.dims[n - 1], R), dtype=np.float64, order="F")
    mults = C.c_uint64()
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_mttkrp_direct(ctx.h, y.h, R, _ptr_array(bufs), int(n),
                                           out.ctypes.data_as(_lib.c_dbl_p), C.byref(mults)), ctx.h)
    if counter is not None:
        counter.charge(int(mults.value))
    return out


def mttkrp_direct_device(y: DenseTensor, R: int, factors_dev_ptr: int, grads_dev_ptr: int, n: int) -> None:
    """Device-buffer form (packed factors in, block n of the packed gradients written)."""
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_mttkrp_direct_device(ctx.h, y.h, int(R), C.c_void_p(factors_dev_ptr), int(n),
                                                  C.c_void_p(grads_dev_ptr)), ctx.h)


def als_sweep_direct(y: DenseTensor, factors: list, order: Sequence[int], pinv_rtol: float = 1e-12,
                     counter: Optional[CostCounter] = None) -> None:
    """One ALS sweep over `order` with direct MTTKRPs (als.cpp:58-67); factors updated in place."""
    bufs = _factor_bufs(factors, y.dims)
    R = bufs[0].shape[1]
    bufs = [np.asfortranarray(b).copy(order="F") for b in bufs]
    arr = (C.c_int * len(order))(*[int(n) for n in order])
    mults = C.c_uint64()
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_als_sweep_direct(ctx.h, y.h, R, _ptr_array(bufs), arr, len(order), pinv_rtol,
                                              C.byref(mults)), ctx.h)
    for k, b in enumerate(bufs):
        factors[k] = b
    if counter is not None:
        counter.charge(int(mults.value))


# ---- ALS (als.hpp:48-93) ---------------------------------------------------------

def pinv_psd(s: np.ndarray, rtol: float = 1e-12, ctx: Optional[Context] = None) -> np.ndarray:
    """Moore-Penrose inverse of a symmetric PSD matrix (als.cpp:34-47), on the device."""
    ctx = ctx or default_context()
    a = np.asfortranarray(np.asarray(s, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise errors.ShapeError("pinv_psd: matrix must be square")
    out = np.empty_like(a, order="F")
    _lib.check(ctx._L.cpdgpu_pinv_psd(ctx.h, a.shape[0], a.ctypes.data_as(_lib.c_dbl_p), rtol,
                                      out.ctypes.data_as(_lib.c_dbl_p)), ctx.h)
    return out


def als_update_mode(m: np.ndarray, factors: list, n: int, pinv_rtol: float = 1e-12,
                    ctx: Optional[Context] = None) -> np.ndarray:
    """A^(n) <- M pinv(hadamard of the skip-mode Grams) (als.cpp:49-56)."""
    ctx = ctx or default_context()
    if n < 1 or n > len(factors):
        raise errors.IndexError(f"als_update_mode: mode {n} outside 1..{len(factors)}")
    dims = [np.asarray(f).shape[0] for f in factors]
    bufs = _factor_bufs(factors, dims)
    R = bufs[0].shape[1]
    mm = np.asfortranarray(np.asarray(m, dtype=np.float64))
    if mm.shape != (dims[n - 1], R):
        raise errors.ShapeError("als_update_mode: mttkrp matrix has the wrong size")
    out = np.empty_like(mm, order="F")
    _lib.check(ctx._L.cpdgpu_als_update_mode(ctx.h, len(dims), _dims_arg(dims), R,
                                             mm.ctypes.data_as(_lib.c_dbl_p), _ptr_array(bufs), n,
                                             pinv_rtol, out.ctypes.data_as(_lib.c_dbl_p)), ctx.h)
    return out


def als_sweep_fast(y: DenseTensor, factors: list, pinv_rtol: float = 1e-12,
                   counter: Optional[CostCounter] = None, stats: Optional[FastStats] = None) -> None:
    """One ALS sweep threaded through the all-mode recursion (als.cpp:69-78);
    factors are replaced in place (list elements)."""
    if y.order() < 2:
        raise errors.ArgumentError("cp_gradient_all: need an order-2 or higher tensor")
    bufs = _factor_bufs(factors, y.dims)
    R = bufs[0].shape[1]
    mults = C.c_uint64()
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_als_sweep(ctx.h, y.h, R, _ptr_array(bufs), pinv_rtol, None,
                                       C.byref(mults)), ctx.h)
    for k, b in enumerate(bufs):
        factors[k] = b
    if counter is not None:
        counter.charge(int(mults.value))


@dataclass
class SolveOptions:
    """als.hpp:21-29 (the fields the fast ALS driver reads)."""
    max_iters: int = 20
    tol: float = 0.0
    pinv_rtol: float = 1e-12
    mu_eps: float = 1e-12
    gd_eta: float = 1e-3
    order: str = "standard"  # UpdateOrder for als_direct: "standard" (1..N) or "pivot"
    seed: int = 0


@dataclass
class RunTrace:
    """als.hpp:31-39; `seconds` are device-timed sweeps (CUDA events)."""
    cost: list = field(default_factory=list)
    rel_error: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    mults: list = field(default_factory=list)
    iters_run: int = 0


@dataclass
class SolveResult:
    factors: list
    trace: RunTrace


def mu_sweep(y: DenseTensor, factors: list, eps: float = 1e-12, counter: Optional[CostCounter] = None) -> None:
    """Multiplicative-update sweep (als.cpp:80-91) on the device; factors updated in place.
    Negative tensor or factor entries raise DomainError."""
    _sweep_call(y, factors, counter, lambda ctx, R, fp, m: ctx._L.cpdgpu_mu_sweep(ctx.h, y.h, R, fp, eps, m))


def gd_step(y: DenseTensor, factors: list, eta: float, counter: Optional[CostCounter] = None) -> None:
    """Gradient-descent step (als.cpp:93-101) on the device; factors updated in place."""
    _sweep_call(y, factors, counter, lambda ctx, R, fp, m: ctx._L.cpdgpu_gd_step(ctx.h, y.h, R, fp, eta, m))


def _sweep_call(y, factors, counter, call):
    bufs = [b.copy(order="F") for b in _factor_bufs(factors, y.dims)]
    R = bufs[0].shape[1]
    mults = C.c_uint64()
    ctx = y.ctx
    _lib.check(call(ctx, R, _ptr_array(bufs), C.byref(mults)), ctx.h)
    for k, b in enumerate(bufs):
        factors[k] = b
    if counter is not None:
        counter.charge(int(mults.value))


def uniform01(seed: int, n: int) -> np.ndarray:
    """The reference's Uniform01 stream (rng.hpp:9-26): mt19937_64 with a splitmix seed."""
    out = np.empty(int(n), dtype=np.float64)
    _lib.check(_lib.load().cpdgpu_uniform01_fill(C.c_uint64(seed), int(n), out.ctypes.data_as(_lib.c_dbl_p)))
    return out


def random_init(dims: Sequence[int], rank: int, seed: int) -> list[np.ndarray]:
    """random_init (als.cpp:122-135): uniform(0,1) factors, column-major per mode in order."""
    if rank < 1:
        raise errors.ArgumentError("random_init: rank must be positive")
    v = uniform01(seed, sum(int(d) for d in dims) * int(rank))
    out, at = [], 0
    for d in dims:
        out.append(v[at:at + int(d) * rank].reshape(int(d), rank, order="F").copy(order="F"))
        at += int(d) * rank
    return out


def generate_problem(dims: Sequence[int], rank: int, seed: int, ctx: Optional[Context] = None):
    """generate_problem (bench.cpp:129-137): tensor from `seed`, init factors from seed + 1."""
    n = int(np.prod([int(d) for d in dims]))
    return DenseTensor.from_values(uniform01(seed, n), dims, ctx=ctx), random_init(dims, rank, seed + 1)


def cost(y: DenseTensor, factors: list) -> float:
    """cost(y, model) (kruskal.cpp:58-77) on the device (Gram identity)."""
    bufs = _factor_bufs(factors, y.dims)
    out = C.c_double()
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_cost(ctx.h, y.h, bufs[0].shape[1], _ptr_array(bufs), C.byref(out)), ctx.h)
    return float(out.value)


def relative_error(y: DenseTensor, factors: list) -> float:
    """relative_error (kruskal.cpp:79-81)."""
    return float(np.sqrt(cost(y, factors)) / np.sqrt(y.norm2()))


def cp_gradient_set(y: DenseTensor, factors: list, mttkrp_results: list) -> tuple:
    """cp_gradient_set (kruskal.cpp:83-101): G(n) = M(n) - A(n) W(n) and the stacked
    derivative g = -2 [vec G(1); ...; vec G(N)] (host epilogue of device gradients)."""
    bufs = _factor_bufs(factors, y.dims)
    if len(mttkrp_results) != len(bufs):
        raise errors.ArgumentError(f"cp_gradient_set: {len(mttkrp_results)} mttkrp matrices for order {len(bufs)}")
    grams = [b.T @ b for b in bufs]
    modes = []
    for n, (M, A) in enumerate(zip(mttkrp_results, bufs)):
        if M.shape != A.shape:
            raise errors.ShapeError(f"cp_gradient_set: mttkrp matrix for mode {n + 1} has wrong size")
        W = np.ones_like(grams[0])
        for k, g in enumerate(grams):
            if k != n:
                W = W * g
        modes.append(M - A @ W)
    return modes, -2.0 * np.concatenate([G.reshape(-1, order="F") for G in modes])


ALGORITHMS = {"als_direct": 0, "als_fast": 1, "mu": 2, "gd": 3}


def run(y: DenseTensor, init: list, opts: Optional[SolveOptions] = None,
        counter: Optional[CostCounter] = None, algo: str = "als_fast") -> SolveResult:
    """run(y, init, algo, opts) (als.cpp:147-210) on the device; algo is one of
    Algorithm's names: als_direct, als_fast (default), mu, gd."""
    opts = opts or SolveOptions()
    if algo not in ALGORITHMS:
        raise errors.ArgumentError(f"run: unknown algorithm {algo!r}")
    if opts.max_iters < 1:
        raise errors.ArgumentError("run: max_iters must be at least 1")
    if opts.tol < 0.0 or opts.pinv_rtol < 0.0 or opts.mu_eps < 0.0:
        raise errors.ArgumentError("run: tolerances must be nonnegative")
    try:
        bufs = _factor_bufs(init, y.dims)
    except errors.ShapeError:
        raise errors.ShapeError("run: init factors do not match the tensor") from None
    bufs = [b.copy(order="F") for b in bufs]
    R = bufs[0].shape[1]
    n = opts.max_iters
    cost = np.zeros(n)
    rel = np.zeros(n)
    sec = np.zeros(n)
    mults = (C.c_uint64 * n)()
    iters = C.c_int()
    ctx = y.ctx
    _lib.check(ctx._L.cpdgpu_run_algo(ctx.h, y.h, R, _ptr_array(bufs), ALGORITHMS[algo],
                                      int(opts.order == "pivot"), n, opts.tol, opts.pinv_rtol, opts.mu_eps,
                                      opts.gd_eta, cost.ctypes.data_as(_lib.c_dbl_p),
                                      rel.ctypes.data_as(_lib.c_dbl_p), sec.ctypes.data_as(_lib.c_dbl_p), mults,
                                      C.byref(iters)), ctx.h)
    k = iters.value
    base = counter.total() if counter is not None else 0
    tr = RunTrace(cost=list(cost[:k]), rel_error=list(rel[:k]), seconds=list(sec[:k]),
                  mults=[base + int(m) for m in list(mults)[:k]] if counter is not None else [0] * k,
                  iters_run=k)
    if counter is not None and k:
        counter.charge(int(mults[k - 1]))
    return SolveResult(factors=bufs, trace=tr)
