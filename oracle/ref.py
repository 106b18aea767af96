"""ctypes wrapper of the reference itself (oracle/_ref/libcpdref.so).

TEST INFRASTRUCTURE ONLY: the reference's own core sources compiled where they
lie under /root/reference/proj/core (oracle/Makefile target `ref`, Eigen
replaced by oracle/shim) plus the C entry layer oracle/ref_capi.cpp.  Used by
tests/ to pin the C oracle port and the GPU path to the reference's results and
by bench.py's CPU legs (cpu_baseline kind "reference").  The built library
travels to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libcpdref.so"
REFERENCE = Path("/root/reference/proj")

c_i64 = C.c_int64
c_u64 = C.c_uint64
c_dbl_p = C.POINTER(C.c_double)
_lib = None


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"reference status {status}: {msg}")
        self.status = status


def available() -> bool:
    return LIB.exists() or REFERENCE.exists()


def build() -> Path:
    """Compile oracle/_ref (only where /root/reference is present)."""
    if REFERENCE.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref", "-j8"], check=True)
    if not LIB.exists():
        raise FileNotFoundError(f"{LIB} is missing (build it where /root/reference exists)")
    return LIB


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.ref_last_error.restype = C.c_char_p
        L.ref_tensor_new.restype = C.c_void_p
        L.ref_tensor_new.argtypes = [C.c_int, C.POINTER(c_i64), c_dbl_p, C.c_int, C.c_int]
        L.ref_tensor_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _check(st):
    if st:
        raise RefError(st, load().ref_last_error().decode())


def _dims(dims):
    return (c_i64 * len(dims))(*[int(d) for d in dims])


def _ptrs(arrs):
    out = (c_dbl_p * len(arrs))()
    for i, a in enumerate(arrs):
        out[i] = a.ctypes.data_as(c_dbl_p)
    return out


def _fbufs(factors):
    return [np.asfortranarray(np.asarray(f, dtype=np.float64)) for f in factors]


class Tensor:
    """A reference cpd::DenseTensor (values copied in), optionally split into
    `parts` slabs of the first (axis=0) or last (axis=1) mode computed on
    parallel threads (the reference is single-threaded; slab gradients combine
    exactly)."""

    def __init__(self, values, dims, parts=1, axis=1):
        L = load()
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1, order="F"))
        self.dims = [int(d) for d in dims]
        self.h = L.ref_tensor_new(len(self.dims), _dims(self.dims), v.ctypes.data_as(c_dbl_p), int(parts), int(axis))
        if not self.h:
            raise RefError(6, L.ref_last_error().decode())

    def close(self):
        if self.h:
            load().ref_tensor_free(C.c_void_p(self.h))
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def cp_gradient_all(self, factors):
        """(gradients, mults) of cpd::cp_gradient_all (mttkrp.hpp:59-69)."""
        bufs = _fbufs(factors)
        R = bufs[0].shape[1]
        grads = [np.zeros((d, R), order="F") for d in self.dims]
        m = c_u64()
        _check(load().ref_cp_gradient_all(C.c_void_p(self.h), c_i64(R), _ptrs(bufs), _ptrs(grads), C.byref(m)))
        return grads, int(m.value)

    def time_cp_gradient_all(self, factors, reps):
        bufs = _fbufs(factors)
        R = bufs[0].shape[1]
        grads = [np.zeros((d, R), order="F") for d in self.dims]
        sec = C.c_double()
        _check(load().ref_time_cp_gradient_all(C.c_void_p(self.h), c_i64(R), _ptrs(bufs), _ptrs(grads),
                                               C.c_int(reps), C.byref(sec)))
        return float(sec.value)

    def als_sweep_fast(self, factors, rtol=1e-12):
        """In place; returns (mults, seconds of the reference sweep)."""
        R = factors[0].shape[1]
        for f in factors:
            assert f.flags.f_contiguous and f.dtype == np.float64
        m, sec = c_u64(), C.c_double()
        _check(load().ref_als_sweep_fast(C.c_void_p(self.h), c_i64(R), _ptrs(factors), C.c_double(rtol),
                                         C.byref(m), C.byref(sec)))
        return int(m.value), float(sec.value)

    def run(self, factors, algo=1, pivot_order=False, max_iters=10, tol=0.0):
        """cpd::run (als.hpp:88-93): (cost trace, rel trace); factors in place."""
        R = factors[0].shape[1]
        cost, rel, it = np.zeros(max_iters), np.zeros(max_iters), C.c_int()
        _check(load().ref_run(C.c_void_p(self.h), c_i64(R), _ptrs(factors), C.c_int(algo), C.c_int(int(pivot_order)),
                              C.c_int(max_iters), C.c_double(tol), cost.ctypes.data_as(c_dbl_p),
                              rel.ctypes.data_as(c_dbl_p), C.byref(it)))
        return cost[:it.value], rel[:it.value]

    def mttkrp_direct(self, factors, n):
        bufs = _fbufs(factors)
        R = bufs[0].shape[1]
        out = np.zeros((self.dims[n - 1], R), order="F")
        _check(load().ref_mttkrp_direct(C.c_void_p(self.h), c_i64(R), _ptrs(bufs), C.c_int(n),
                                        out.ctypes.data_as(c_dbl_p)))
        return out


def select_pivot(dims):
    p = C.c_int()
    _check(load().ref_select_pivot(len(dims), _dims(dims), C.byref(p)))
    return p.value


def counts(dims, R, n):
    """(direct, fast, fast_derived, realized) of predicted_mult_count / fast_count_realized."""
    v = [c_u64() for _ in range(4)]
    _check(load().ref_counts(len(dims), _dims(dims), c_i64(R), C.c_int(n), *[C.byref(x) for x in v]))
    return tuple(int(x.value) for x in v)


def pinv_psd(s, rtol=1e-12):
    s = np.asfortranarray(np.asarray(s, dtype=np.float64))
    out = np.zeros_like(s, order="F")
    _check(load().ref_pinv_psd(c_i64(s.shape[0]), s.ctypes.data_as(c_dbl_p), C.c_double(rtol),
                               out.ctypes.data_as(c_dbl_p)))
    return out
