"""ctypes wrapper of the CPU oracle (cpd_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference leg — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

c_i64 = C.c_int64
c_dbl_p = C.POINTER(C.c_double)
HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int, c_dbl_p, c_i64, c_i64)

_lib = None


def build() -> Path:
    src = HERE / "cpd_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.ora_select_pivot.restype = C.c_int
        L.ora_fast_count_realized.restype = C.c_uint64
        L.ora_predicted_mult_count.restype = C.c_uint64
        L.ora_cost.restype = C.c_double
        L.ora_hash64.restype = C.c_uint64
        L.ora_hash64.argtypes = [C.c_uint64, C.c_uint64]
        _lib = L
    return _lib


def _dims(dims):
    return (c_i64 * len(dims))(*[int(d) for d in dims])


def _fbufs(factors):
    return [np.asfortranarray(np.asarray(f, dtype=np.float64)).reshape(np.asarray(f).shape[0], -1, order="F")
            for f in factors]


def _ptrs(bufs):
    arr = (c_dbl_p * len(bufs))()
    for i, b in enumerate(bufs):
        arr[i] = b.ctypes.data_as(c_dbl_p)
    return arr


def vec(y):
    """Vectorization-order (column-major) flat float64 copy of an N-d array / flat vector."""
    a = np.asarray(y, dtype=np.float64)
    return np.ascontiguousarray(a.reshape(-1, order="F") if a.ndim > 1 else a)


def select_pivot(dims) -> int:
    return load().ora_select_pivot(len(dims), _dims(dims))


def sort_perm(dims):
    n = len(dims)
    perm, inv = (C.c_int * n)(), (C.c_int * n)()
    load().ora_sort_perm(n, _dims(dims), perm, inv)
    return list(perm), list(inv)


def fast_update_order(dims):
    out = (C.c_int * len(dims))()
    st = load().ora_fast_update_order(len(dims), _dims(dims), out)
    if st:
        raise ValueError(f"oracle status {st}")
    return list(out)


def permute(y, dims, perm):
    yv = vec(y)
    out = np.empty_like(yv)
    load().ora_permute(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), (C.c_int * len(perm))(*perm),
                       out.ctypes.data_as(c_dbl_p))
    return out


def fast_count_realized(dims, R, n) -> int:
    return int(load().ora_fast_count_realized(len(dims), _dims(dims), int(R), int(n)))


def predicted_mult_count(dims, R, n, variant) -> int:
    v = {"direct": 0, "fast": 1, "fast_derived": 2}[variant]
    return int(load().ora_predicted_mult_count(len(dims), _dims(dims), int(R), int(n), v))


def cp_gradient_all(y, dims, factors, hook=None, counter=None, pivot=0, nthreads=0, stats=None):
    """Returns (gradients, mults_total, peak_workspace).  hook(mode, G, factors) may
    assign factors[mode-1] (a python list), as the reference hook does."""
    L = load()
    yv = vec(y)
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    grads = [np.zeros((int(d), R), order="F") for d in dims]
    cnt = C.c_uint64(0)
    peak = C.c_int64(0)
    cb = None
    if hook is not None:
        def _cb(user, mode, g, rows, rank):
            if counter is not None:
                counter["snaps"].append((mode, cnt.value))
            hook(mode, grads[mode - 1].copy(order="F"), factors)
            bufs[mode - 1][...] = np.asarray(factors[mode - 1], dtype=np.float64).reshape(bufs[mode - 1].shape)
        cb = HOOK(_cb)
    st = L.ora_cp_gradient_all(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs),
                               _ptrs(grads), cb, None, C.byref(cnt),
                               C.byref(peak), int(pivot), int(nthreads))
    if st:
        raise ValueError(f"oracle status {st}")
    return grads, int(cnt.value), int(peak.value)


def cp_gradient_all_upm1_f32(dims, seed, factors, offset=0, pivot=0, nthreads=0):
    """All-mode gradient of the generated fp32 U(-1,1) tensor (fill_upm1_f32 values,
    upcast to fp64) without materialising it: the streaming restatement used for
    config 5 at full size (ascending dims)."""
    L = load()
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    grads = [np.zeros((int(d), R), order="F") for d in dims]
    st = L.ora_cp_gradient_all_upm1_f32(len(dims), _dims(dims), C.c_uint64(int(seed)), c_i64(int(offset)),
                                        c_i64(R), _ptrs(bufs), _ptrs(grads), int(pivot), int(nthreads))
    if st:
        raise ValueError(f"oracle status {st}")
    return grads


def brute_mttkrp(y, dims, factors, n):
    yv = vec(y)
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    out = np.zeros((int(dims[n - 1]), R), order="F")
    st = load().ora_brute_mttkrp(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs),
                                 int(n), out.ctypes.data_as(c_dbl_p))
    if st:
        raise ValueError(f"oracle status {st}")
    return out


def gram_hadamard_skip(factors, n):
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    dims = [b.shape[0] for b in bufs]
    w = np.zeros((R, R), order="F")
    load().ora_gram_hadamard_skip(len(dims), _dims(dims), c_i64(R), _ptrs(bufs), int(n), w.ctypes.data_as(c_dbl_p))
    return w


def pinv_psd(s, rtol=1e-12):
    a = np.asfortranarray(np.asarray(s, dtype=np.float64))
    out = np.zeros_like(a, order="F")
    st = load().ora_pinv_psd(c_i64(a.shape[0]), a.ctypes.data_as(c_dbl_p), C.c_double(rtol),
                             out.ctypes.data_as(c_dbl_p))
    if st:
        raise ValueError(f"oracle status {st}")
    return out


def als_update_mode(m, factors, n, rtol=1e-12):
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    dims = [b.shape[0] for b in bufs]
    mm = np.asfortranarray(np.asarray(m, dtype=np.float64))
    out = np.zeros_like(mm, order="F")
    st = load().ora_als_update_mode(len(dims), _dims(dims), c_i64(R), mm.ctypes.data_as(c_dbl_p), _ptrs(bufs),
                                    int(n), C.c_double(rtol), out.ctypes.data_as(c_dbl_p))
    if st:
        raise ValueError(f"oracle status {st}")
    return out


def als_sweep_fast(y, dims, factors, rtol=1e-12, nthreads=0):
    """In place on a list of factors; returns the list."""
    yv = vec(y)
    bufs = [b.copy(order="F") for b in _fbufs(factors)]
    R = bufs[0].shape[1]
    cnt = C.c_uint64(0)
    st = load().ora_als_sweep_fast(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs),
                                   C.c_double(rtol), C.byref(cnt), int(nthreads))
    if st:
        raise ValueError(f"oracle status {st}")
    for k in range(len(factors)):
        factors[k] = bufs[k]
    return factors


def cost(y, dims, factors, materialize_limit=1000000, nthreads=0):
    yv = vec(y)
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    return float(load().ora_cost(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs),
                                 c_i64(materialize_limit), int(nthreads)))


def full(dims, factors):
    bufs = _fbufs(factors)
    R = bufs[0].shape[1]
    out = np.zeros(int(np.prod(dims)))
    load().ora_full(len(dims), _dims(dims), c_i64(R), _ptrs(bufs), out.ctypes.data_as(c_dbl_p))
    return out


def run_als_fast(y, dims, init, max_iters=20, tol=0.0, pinv_rtol=1e-12, nthreads=0):
    yv = vec(y)
    bufs = [b.copy(order="F") for b in _fbufs(init)]
    R = bufs[0].shape[1]
    cost_t, rel_t, sec_t = np.zeros(max_iters), np.zeros(max_iters), np.zeros(max_iters)
    mults = (C.c_uint64 * max_iters)()
    iters = C.c_int(0)
    st = load().ora_run_als_fast(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs),
                                 int(max_iters), C.c_double(tol), C.c_double(pinv_rtol),
                                 cost_t.ctypes.data_as(c_dbl_p), rel_t.ctypes.data_as(c_dbl_p),
                                 sec_t.ctypes.data_as(c_dbl_p), mults, C.byref(iters), int(nthreads))
    if st:
        raise ValueError(f"oracle status {st}")
    k = iters.value
    return bufs, {"cost": cost_t[:k], "rel_error": rel_t[:k], "seconds": sec_t[:k],
                  "mults": [int(m) for m in list(mults)[:k]], "iters_run": k}


ALGOS = {"als_direct": 0, "als_fast": 1, "mu": 2, "gd": 3}


def _fac_run(fn, factors, *args):
    bufs = [b.copy(order="F") for b in _fbufs(factors)]
    st = fn(_ptrs(bufs), *args)
    if st:
        raise ValueError(f"oracle status {st}")
    return bufs


def als_sweep_direct(y, dims, factors, order, rtol=1e-12):
    yv = vec(y)
    R = _fbufs(factors)[0].shape[1]
    cnt = C.c_uint64(0)
    arr = (C.c_int * len(order))(*order)
    bufs = _fac_run(lambda fp: load().ora_als_sweep_direct(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p),
                                                           c_i64(R), fp, arr, len(order), C.c_double(rtol),
                                                           C.byref(cnt)), factors)
    return bufs, int(cnt.value)


def mu_sweep(y, dims, factors, eps=1e-12, nthreads=0):
    yv = vec(y)
    R = _fbufs(factors)[0].shape[1]
    cnt = C.c_uint64(0)
    bufs = _fac_run(lambda fp: load().ora_mu_sweep(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R),
                                                   fp, C.c_double(eps), C.byref(cnt), int(nthreads)), factors)
    return bufs, int(cnt.value)


def gd_step(y, dims, factors, eta, nthreads=0):
    yv = vec(y)
    R = _fbufs(factors)[0].shape[1]
    cnt = C.c_uint64(0)
    bufs = _fac_run(lambda fp: load().ora_gd_step(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R),
                                                  fp, C.c_double(eta), C.byref(cnt), int(nthreads)), factors)
    return bufs, int(cnt.value)


def run(y, dims, init, algo, max_iters=20, tol=0.0, pinv_rtol=1e-12, mu_eps=1e-12, gd_eta=1e-3,
        order_pivot=False, nthreads=0):
    yv = vec(y)
    bufs = [b.copy(order="F") for b in _fbufs(init)]
    R = bufs[0].shape[1]
    cost_t, rel_t = np.zeros(max_iters), np.zeros(max_iters)
    mults = (C.c_uint64 * max_iters)()
    iters = C.c_int(0)
    st = load().ora_run(len(dims), _dims(dims), yv.ctypes.data_as(c_dbl_p), c_i64(R), _ptrs(bufs), ALGOS[algo],
                        int(bool(order_pivot)), int(max_iters), C.c_double(tol), C.c_double(pinv_rtol),
                        C.c_double(mu_eps), C.c_double(gd_eta), cost_t.ctypes.data_as(c_dbl_p),
                        rel_t.ctypes.data_as(c_dbl_p), mults, C.byref(iters), int(nthreads))
    if st:
        raise ValueError(f"oracle status {st}")
    k = iters.value
    return bufs, {"cost": cost_t[:k], "rel_error": rel_t[:k], "mults": [int(m) for m in list(mults)[:k]],
                  "iters_run": k}


# ---- generators -------------------------------------------------------------------

def uniform01(seed, n):
    """The reference fixtures' Uniform01 stream (rng.hpp:16-26)."""
    out = np.empty(int(n))
    load().ora_uniform01_fill(C.c_uint64(seed), c_i64(n), out.ctypes.data_as(c_dbl_p))
    return out


def random_tensor(dims, seed):
    """test_util.hpp:21-28: U(0,1) entries in vectorization order."""
    return uniform01(seed, int(np.prod(dims)))


def random_factors(dims, rank, seed):
    """test_util.hpp:30-41: one Uniform01 stream filling factors column-major in mode order."""
    total = sum(int(d) * int(rank) for d in dims)
    v = uniform01(seed, total)
    out, at = [], 0
    for d in dims:
        n = int(d) * int(rank)
        out.append(np.asfortranarray(v[at:at + n].reshape(int(d), int(rank), order="F")))
        at += n
    return out


def fill_normal(seed, n, offset=0, nthreads=0):
    out = np.empty(int(n))
    load().ora_fill_normal(C.c_uint64(seed), c_i64(offset), c_i64(n), out.ctypes.data_as(c_dbl_p), int(nthreads))
    return out


def fill_upm1_f32(seed, n, offset=0, nthreads=0):
    out = np.empty(int(n), dtype=np.float32)
    load().ora_fill_upm1_f32(C.c_uint64(seed), c_i64(offset), c_i64(n),
                             out.ctypes.data_as(C.POINTER(C.c_float)), int(nthreads))
    return out


def hash64(seed, idx):
    return int(load().ora_hash64(C.c_uint64(seed), C.c_uint64(idx)))


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
