"""ctypes loader for oracle/libmpbrute.so (the plain C brute force).  Test infrastructure only.
Built by __graft_entry__.build() or on first use here (gcc is in the image)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mp_brute.c")
_SRCS = [_SRC, os.path.join(_HERE, "mp_tierb.c")]
_LIB = os.path.join(_HERE, "libmpbrute.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_mp_rows.restype = ctypes.c_int
        lib.oracle_mp_rows.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_tierb_selfjoin.restype = ctypes.c_int
        lib.oracle_tierb_selfjoin.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int]
        lib.oracle_window_stats.restype = None
        lib.oracle_window_stats.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def mp_rows(r: np.ndarray, m: int, excl: int, rows: np.ndarray, threads: int = 0):
    lib = _get()
    n = r.shape[0]
    n_sub = n - m + 1
    P = np.empty(len(rows))
    I = np.empty(len(rows), dtype=np.int64)
    flat = np.empty(n_sub, dtype=np.uint8)
    rc = lib.oracle_mp_rows(r.ctypes.data, n, m, excl, rows.ctypes.data, len(rows), P.ctypes.data,
                            I.ctypes.data, flat.ctypes.data, int(threads))
    if rc != 0:
        from .reference import OracleError
        raise OracleError("no_admissible" if rc == -1 else "oom")
    return P, I, flat.astype(bool)


def window_stats(r: np.ndarray, m: int):
    lib = _get()
    r = np.ascontiguousarray(r, dtype=np.float64)
    n_sub = r.shape[0] - m + 1
    mu = np.empty(n_sub)
    sig = np.empty(n_sub)
    flat = np.empty(n_sub, dtype=np.uint8)
    lib.oracle_window_stats(r.ctypes.data, r.shape[0], m, mu.ctypes.data, sig.ctypes.data, flat.ctypes.data)
    return mu, sig, flat.astype(bool)


def tierb_selfjoin(r: np.ndarray, m: int, excl: int, reseed: int = 65536, threads: int = 0):
    lib = _get()
    r = np.ascontiguousarray(r, dtype=np.float64)
    n_sub = r.shape[0] - m + 1
    P = np.empty(n_sub)
    I = np.empty(n_sub, dtype=np.int64)
    rc = lib.oracle_tierb_selfjoin(r.ctypes.data, r.shape[0], m, excl, reseed, P.ctypes.data, I.ctypes.data,
                                   int(threads))
    if rc != 0:
        from .reference import OracleError
        raise OracleError({-1: "no_admissible", -2: "flat_windows_unsupported"}.get(rc, "oom"))
    return P, I

