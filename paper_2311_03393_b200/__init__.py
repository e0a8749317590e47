"""Thin Python binding of the sketch + matrix-profile C-ABI (include/sketchmp.h).

Argument marshalling only: every step of the path runs in libsketchmp.so's CUDA kernels.
PyTorch supplies device memory and the current CUDA stream.  The same names as the C-ABI:

    sketch_hash_plan, sketch_build, sketch_add_dim, sketch_del_dim, sketch_point_update, sketch_view,
    sketch_view64,
    sketch_plan, sketch_refresh, sketch_free, mp_create, mp_join, mp_keys, mp_band, mp_finalize,
    mp_finalize_rows, mp_free,
    mp_selfjoin, mp_abjoin, discord_topk, discord_dims
plus Python-level compositions of those calls: group_rows, detect_dimension, detect.

There is no CPU fallback: if the shared library is missing, `lib()` raises; compute calls
without a GPU return SKMP_E_CUDA (raised as SkmpError).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKMP_LIB") or os.path.join(_HERE, "libsketchmp.so")

F32, F64 = 0, 1
PROJ_COUNT_SKETCH, PROJ_DENSE = 0, 1

STATUS = {
    0: "SKMP_OK", 1: "SKMP_E_INVALID_ARG", 2: "SKMP_E_CONSTANT_SERIES", 3: "SKMP_E_NONFINITE",
    4: "SKMP_E_SERIES_TOO_SHORT", 5: "SKMP_E_NO_ADMISSIBLE", 6: "SKMP_E_DUPLICATE_DIM",
    7: "SKMP_E_UNKNOWN_DIM", 8: "SKMP_E_LENGTH_MISMATCH", 9: "SKMP_E_ALL_GROUPS_INERT",
    10: "SKMP_E_CUDA", 11: "SKMP_E_NCCL", 12: "SKMP_E_OOM",
}


class SkmpError(RuntimeError):
    def __init__(self, status: int, message: str, index: int):
        super().__init__(f"{STATUS.get(status, status)}: {message} (index {index})")
        self.status = status
        self.name = STATUS.get(status, str(status))
        self.message = message
        self.index = index


class SketchCfg(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("dtype", ctypes.c_int32), ("proj", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("groups", ctypes.c_void_p), ("signs", ctypes.c_void_p), ("S", ctypes.c_void_p)]


class Source(ctypes.Structure):
    """skmp_source: one matrix of raw streams for discord_dims_group."""
    _fields_ = [("T", ctypes.c_void_p), ("ld", ctypes.c_int64), ("rows", ctypes.c_int64), ("ids", ctypes.c_void_p)]


class DimResult(ctypes.Structure):
    """skmp_dim_result: Alg. 3's winner (score, id, nn) and how many members were scored."""
    _fields_ = [("score", ctypes.c_double), ("id", ctypes.c_uint64), ("nn", ctypes.c_int64),
                ("n_scored", ctypes.c_int64)]


class MpCfg(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("excl", ctypes.c_int32), ("reseed_rows", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

_SIGS = {
    "skmp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "skmp_last_error": (ctypes.c_char_p, []),
    "skmp_last_error_index": (_I64, []),
    "skmp_abi_version": (_I32, []),
    "skmp_launch_count": (_I64, []),
    "sketch_refresh": (ctypes.c_int, [_P, _P]),
    "sketch_hash_plan": (ctypes.c_int, [_P, _I64, _I32, ctypes.c_uint64, _P, _P]),
    "sketch_build": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, ctypes.POINTER(SketchCfg), _P, ctypes.POINTER(_P)]),
    "sketch_add_dim": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P]),
    "sketch_del_dim": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "sketch_view": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_I32), ctypes.POINTER(_I64),
                                   ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
    "sketch_view64": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "sketch_point_update": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P]),
    "sketch_plan": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "sketch_free": (None, [_P]),
    "mp_create": (ctypes.c_int, [_P, _I32, _I64, _I64, _I32, ctypes.POINTER(MpCfg), _P, ctypes.POINTER(_P)]),
    "mp_join": (ctypes.c_int, [_P, _I64, _I64, _P]),
    "mp_keys": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
    "mp_tile_width": (_I32, [_I32]),
    "mp_band": (ctypes.c_int, [_I64, _I32, _I32, _I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "mp_finalize": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "mp_finalize_rows": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P, _P]),
    "mp_free": (None, [_P]),
    "mp_selfjoin": (ctypes.c_int, [_P, _I32, _I64, _I64, _I32, ctypes.POINTER(MpCfg), _P, _P, _P, _P]),
    "discord_topk": (ctypes.c_int, [_P, _P, _P, _I32, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P,
                                    _P, _P]),
    "mp_abjoin": (ctypes.c_int, [_P, _I64, _I64, _P, _I64, _I64, _I32, _I32, ctypes.POINTER(MpCfg), _P, _P, _P, _P,
                                 _P, _P]),
    "mp_create_ab": (ctypes.c_int, [_P, _I32, _I64, _I64, _I32, ctypes.POINTER(MpCfg), _P, ctypes.POINTER(_P)]),
    "mp_join_ab": (ctypes.c_int, [_P, _P, _I64, _I64, _P]),
    "mp_finalize_ab": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P, _P]),
    "mp_abband": (ctypes.c_int, [_I64, _I64, _I32, _I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                 ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "stream_create": (ctypes.c_int, [_P, ctypes.POINTER(MpCfg), _I64, _P, ctypes.POINTER(_P)]),
    "stream_push": (ctypes.c_int, [_P, _P, _I64, _I64, _P]),
    "stream_view": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P),
                                   ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P]),
    "stream_free": (None, [_P]),
    "skmp_comm_unique_id": (ctypes.c_int, [_P]),
    "skmp_comm_init": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "skmp_comm_free": (None, [_P]),
    "sketch_allreduce": (ctypes.c_int, [_P, _P, _P]),
    "mp_selfjoin_dist": (ctypes.c_int, [_P, _P, _I32, _I64, _I64, _I32, ctypes.POINTER(MpCfg), _P, _P, _P, _P]),
    "discord_dims": (ctypes.c_int, [_P, _I64, _I64, _I32, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _P]),
    "discord_dims_group": (ctypes.c_int, [_P, _I32, _P, _I32, _I64, _I32, _I32, ctypes.POINTER(DimResult), _P]),
    "discord_dims_merge": (ctypes.c_int, [_P, _I32, ctypes.POINTER(DimResult)]),
    "skmp_trim": (ctypes.c_int, []),
    "sketch_free_async": (None, [_P, _P]),
}


def lib():
    """Load libsketchmp.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2311_03393_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        L = lib()
        raise SkmpError(st, L.skmp_last_error().decode(), int(L.skmp_last_error_index()))


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    import torch
    if torch.cuda.is_available():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(0)


def _ptr(x):
    """data pointer of a torch tensor / numpy array / int."""
    if x is None:
        return None
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(x.ctypes.data)


def _dtype_code(t) -> int:
    s = str(getattr(t, "dtype", t))
    if "float32" in s:
        return F32
    if "float64" in s:
        return F64
    raise ValueError(f"unsupported dtype {s} (float32 / float64)")


class _DevArray:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _as_tensor(ptr: int, shape, dtype_code: int):
    import torch
    ts = "<f4" if dtype_code == F32 else "<f8"
    return torch.as_tensor(_DevArray(ptr, shape, ts), device="cuda")


# ----------------------------------------------------------------------------------------------
# host-only
# ----------------------------------------------------------------------------------------------

def sketch_hash_plan(ids, k: int, seed: int):
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    g = np.empty(len(ids), dtype=np.int32)
    s = np.empty(len(ids), dtype=np.int8)
    _check(lib().sketch_hash_plan(_ptr(ids), len(ids), k, seed, _ptr(g), _ptr(s)))
    return g, s


def mp_tile_width(dtype: int) -> int:
    return int(lib().mp_tile_width(dtype))


def mp_band(n_sub: int, excl: int, dtype: int, nbands: int, band: int):
    lo, hi = _I64(), _I64()
    _check(lib().mp_band(n_sub, excl, dtype, nbands, band, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


# ----------------------------------------------------------------------------------------------
# sketch
# ----------------------------------------------------------------------------------------------

class Sketch:
    """Owning wrapper of a skmp_sketch handle."""

    def __init__(self, handle):
        self.handle = handle

    def free(self, stream=None):
        """Free stream-ordered after the handle's own work and everything already enqueued on
        `stream` (default: torch's current stream, where the caller read R)."""
        if self.handle:
            lib().sketch_free_async(self.handle, _stream(stream))
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def R(self):
        return sketch_view(self)[0]

    @property
    def R64(self):
        return sketch_view64(self)


def sketch_build(T, ids, k: int, *, seed: int = 0, proj: int = PROJ_COUNT_SKETCH, groups=None,
                 signs=None, S=None, stream=None, n: int | None = None) -> Sketch:
    """T: d x ld tensor/array (CUDA tensor or host array/tensor, float32/float64)."""
    d = T.shape[0]
    ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
    n = T.shape[1] if n is None else n
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    cfg = SketchCfg()
    cfg.k = k
    cfg.dtype = _dtype_code(T)
    cfg.proj = proj
    cfg.seed = seed
    keep = []
    if groups is not None:
        g = np.ascontiguousarray(groups, dtype=np.int32)
        keep.append(g)
        cfg.groups = g.ctypes.data
    if signs is not None:
        s = np.ascontiguousarray(signs, dtype=np.int8)
        keep.append(s)
        cfg.signs = s.ctypes.data
    if S is not None:
        Sm = np.ascontiguousarray(S, dtype=np.float64)
        keep.append(Sm)
        cfg.S = Sm.ctypes.data
    h = ctypes.c_void_p()
    _check(lib().sketch_build(_ptr(T), d, n, ld, _ptr(ids), ctypes.byref(cfg), _stream(stream), ctypes.byref(h)))
    return Sketch(h)


def sketch_add_dim(sk: Sketch, T, ids, S_cols=None, stream=None):
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
    Sc = None if S_cols is None else np.ascontiguousarray(S_cols, dtype=np.float64)
    _check(lib().sketch_add_dim(sk.handle, _ptr(T), T.shape[0], ld, _ptr(ids), _ptr(Sc), _stream(stream)))


def sketch_del_dim(sk: Sketch, T, ids, stream=None):
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
    _check(lib().sketch_del_dim(sk.handle, _ptr(T), T.shape[0], ld, _ptr(ids), _stream(stream)))


def sketch_point_update(sk: Sketch, ids, t, delta, stream=None):
    """§3.3 point updates: stream ids[q] changes by delta[q] at time t[q] (its own units)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    t = np.ascontiguousarray(t, dtype=np.int64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    assert len(ids) == len(t) == len(delta)
    _check(lib().sketch_point_update(sk.handle, _ptr(ids), _ptr(t), _ptr(delta), len(ids), _stream(stream)))


def sketch_view(sk: Sketch):
    """(R as a zero-copy torch CUDA tensor k x n, k, n, d, dtype)."""
    R, k, n, d, dt = _P(), _I32(), _I64(), _I64(), _I32()
    _check(lib().sketch_view(sk.handle, ctypes.byref(R), ctypes.byref(k), ctypes.byref(n), ctypes.byref(d),
                             ctypes.byref(dt)))
    return _as_tensor(R.value, (k.value, n.value), dt.value), k.value, n.value, d.value, dt.value


def sketch_view64(sk: Sketch):
    p = _P()
    _check(lib().sketch_view64(sk.handle, ctypes.byref(p)))
    _, k, n, _, _ = sketch_view(sk)
    return _as_tensor(p.value, (k, n), F64)


def sketch_plan(sk: Sketch):
    _, k, n, d, _ = sketch_view(sk)
    ids = np.empty(d, np.uint64)
    g = np.empty(d, np.int32)
    s = np.empty(d, np.int8)
    mu = np.empty(d)
    sg = np.empty(d)
    _check(lib().sketch_plan(sk.handle, _ptr(ids), _ptr(g), _ptr(s), _ptr(mu), _ptr(sg)))
    return dict(ids=ids, groups=g, signs=s, mu=mu, sigma=sg)


def group_rows(sk: Sketch, g: int) -> np.ndarray:
    """Plan positions (rows of the sketched T, in input order) of group J_g (Alg. 3's input);
    every position for a dense projection, whose groups are not disjoint."""
    pl = sketch_plan(sk)
    if np.all(pl["groups"] < 0):
        return np.arange(len(pl["groups"]), dtype=np.int64)
    return np.nonzero(pl["groups"] == g)[0].astype(np.int64)


def sketch_refresh(sk: Sketch, stream=None):
    _check(lib().sketch_refresh(sk.handle, _stream(stream)))


def skmp_launch_count() -> int:
    return int(lib().skmp_launch_count())


def skmp_trim():
    """Return the library pools' cached, unused device memory (C-ABI skmp_trim)."""
    _check(lib().skmp_trim())


def sketch_free(sk: Sketch):
    sk.free()


# ----------------------------------------------------------------------------------------------
# matrix profile
# ----------------------------------------------------------------------------------------------

def _mpcfg(m: int, excl: int = -1, reseed_rows: int = 0) -> MpCfg:
    c = MpCfg()
    c.m = m
    c.excl = excl
    c.reseed_rows = reseed_rows
    return c


class MpWorkspace:
    def __init__(self, handle, k: int, n_sub: int, dtype: int):
        self.handle, self.k, self.n_sub, self.dtype = handle, k, n_sub, dtype

    def free(self):
        if self.handle:
            lib().mp_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def mp_create(R, m: int, *, excl: int = -1, reseed_rows: int = 0, n: int | None = None, stream=None) -> MpWorkspace:
    k = R.shape[0]
    n = R.shape[1] if n is None else n
    ld = R.stride(0)
    dt = _dtype_code(R)
    cfg = _mpcfg(m, excl, reseed_rows)
    h = ctypes.c_void_p()
    _check(lib().mp_create(_ptr(R), k, n, ld, dt, ctypes.byref(cfg), _stream(stream), ctypes.byref(h)))
    return MpWorkspace(h, k, n - m + 1, dt)


def mp_join(w: MpWorkspace, diag_lo: int = 0, diag_hi: int = 0, stream=None):
    _check(lib().mp_join(w.handle, diag_lo, diag_hi, _stream(stream)))


def mp_keys(w: MpWorkspace):
    """Zero-copy int64 torch view of the profile keys (k*n_sub*words)."""
    import torch
    p, cnt, words = _P(), _I64(), _I32()
    _check(lib().mp_keys(w.handle, ctypes.byref(p), ctypes.byref(cnt), ctypes.byref(words)))
    arr = _DevArray(p.value, (cnt.value,), "<i8")
    return torch.as_tensor(arr, device="cuda"), words.value


def mp_finalize(w: MpWorkspace, P=None, I=None, stream=None):
    import torch
    tdt = torch.float32 if w.dtype == F32 else torch.float64
    if P is None:
        P = torch.empty((w.k, w.n_sub), dtype=tdt, device="cuda")
    if I is None:
        I = torch.empty((w.k, w.n_sub), dtype=torch.int64, device="cuda")
    inert = np.zeros(w.k, dtype=np.uint8)
    _check(lib().mp_finalize(w.handle, _ptr(P), _ptr(I), _ptr(inert), _stream(stream)))
    return P, I, inert.astype(bool)


def mp_finalize_rows(w: MpWorkspace, row_lo: int, row_hi: int, P=None, I=None, stream=None):
    """Finalize windows [row_lo, row_hi) of every series into P / I (allocated zero-filled when
    not given, so per-rank slices can be sum-reduced)."""
    import torch
    tdt = torch.float32 if w.dtype == F32 else torch.float64
    if P is None:
        P = torch.zeros((w.k, w.n_sub), dtype=tdt, device="cuda")
    if I is None:
        I = torch.zeros((w.k, w.n_sub), dtype=torch.int64, device="cuda")
    inert = np.zeros(w.k, dtype=np.uint8)
    _check(lib().mp_finalize_rows(w.handle, row_lo, row_hi, _ptr(P), _ptr(I), _ptr(inert), _stream(stream)))
    return P, I, inert.astype(bool)


def mp_abband(n_subA: int, n_subB: int, dtype: int, nbands: int, band: int):
    """Band `band` of `nbands` equal-cell bands of the AB-join's two passes: ((lo1, hi1) of pass 1,
    (lo2, hi2) of pass 2), diagonal ranges (empty as lo == hi)."""
    v = [_I64() for _ in range(4)]
    _check(lib().mp_abband(n_subA, n_subB, dtype, nbands, band, *[ctypes.byref(x) for x in v]))
    return (v[0].value, v[1].value), (v[2].value, v[3].value)


def mp_create_ab(R, m: int, *, reseed_rows: int = 0, stream=None) -> MpWorkspace:
    """AB workspace of one side (k x n CUDA tensor) for the staged AB-join."""
    k, n = R.shape
    dt = _dtype_code(R)
    cfg = _mpcfg(m, -1, reseed_rows)
    h = ctypes.c_void_p()
    _check(lib().mp_create_ab(_ptr(R), k, n, R.stride(0), dt, ctypes.byref(cfg), _stream(stream), ctypes.byref(h)))
    return MpWorkspace(h, k, n - m + 1, dt)


def mp_join_ab(rows: MpWorkspace, cols: MpWorkspace, diag_lo: int, diag_hi: int, stream=None):
    """Cells (i, i + delta), delta in [diag_lo, diag_hi): pass 1 = (test, train), pass 2 = (train, test)
    with delta >= 1."""
    _check(lib().mp_join_ab(rows.handle, cols.handle, diag_lo, diag_hi, _stream(stream)))


def mp_finalize_ab(w: MpWorkspace, other: MpWorkspace, row_lo: int = 0, row_hi: int = 0, P=None, I=None,
                   stream=None):
    """Profile of w's windows [row_lo, row_hi) (0, 0 -> all) against other's windows; P / I are
    allocated zero-filled when not given (per-rank slices sum-reduce)."""
    import torch
    tdt = torch.float32 if w.dtype == F32 else torch.float64
    if P is None:
        P = torch.zeros((w.k, w.n_sub), dtype=tdt, device="cuda")
    if I is None:
        I = torch.zeros((w.k, w.n_sub), dtype=torch.int64, device="cuda")
    inert = np.zeros(w.k, dtype=np.uint8)
    _check(lib().mp_finalize_ab(w.handle, other.handle, row_lo, row_hi, _ptr(P), _ptr(I), _ptr(inert),
                                _stream(stream)))
    return P, I, inert.astype(bool)


def mp_free(w: MpWorkspace):
    w.free()


def mp_selfjoin(R, m: int, *, excl: int = -1, reseed_rows: int = 0, n: int | None = None, P=None, I=None,
                stream=None):
    """R: k x ld CUDA tensor.  Returns (P k x n_sub, I k x n_sub int64, inert bool[k])."""
    import torch
    k = R.shape[0]
    n = R.shape[1] if n is None else n
    n_sub = n - m + 1
    dt = _dtype_code(R)
    tdt = torch.float32 if dt == F32 else torch.float64
    if P is None:
        P = torch.empty((k, max(n_sub, 1)), dtype=tdt, device=R.device)
    if I is None:
        I = torch.empty((k, max(n_sub, 1)), dtype=torch.int64, device=R.device)
    inert = np.zeros(k, dtype=np.uint8)
    cfg = _mpcfg(m, excl, reseed_rows)
    _check(lib().mp_selfjoin(_ptr(R), k, n, R.stride(0), dt, ctypes.byref(cfg), _ptr(P), _ptr(I), _ptr(inert),
                             _stream(stream)))
    return P, I, inert.astype(bool)


# ----------------------------------------------------------------------------------------------
# detection
# ----------------------------------------------------------------------------------------------

@dataclass
class Discord:
    t: int
    g: int
    nn: int
    score: float


def mp_abjoin(RA, RB, m: int, *, reseed_rows: int = 0, both: bool = False, stream=None):
    """AB-join (Def. 6): profile of the test series RA (k x nA) against the train series RB
    (k x nB), same dtype, CUDA tensors.  Returns (PA, IA, inert) or, with both=True,
    (PA, IA, PB, IB, inert)."""
    import torch
    k, nA = RA.shape
    nB = RB.shape[1]
    assert RB.shape[0] == k and RA.dtype == RB.dtype
    PA = torch.empty((k, nA - m + 1), dtype=RA.dtype, device=RA.device)
    IA = torch.empty((k, nA - m + 1), dtype=torch.int64, device=RA.device)
    PB = torch.empty((k, nB - m + 1), dtype=RA.dtype, device=RA.device) if both else None
    IB = torch.empty((k, nB - m + 1), dtype=torch.int64, device=RA.device) if both else None
    inert = np.zeros(k, dtype=np.uint8)
    cfg = _mpcfg(m, -1, reseed_rows)
    _check(lib().mp_abjoin(_ptr(RA), nA, RA.stride(0), _ptr(RB), nB, RB.stride(0), k, _dtype_code(RA),
                           ctypes.byref(cfg), _ptr(PA), _ptr(IA), _ptr(PB), _ptr(IB), _ptr(inert), _stream(stream)))
    if both:
        return PA, IA, PB, IB, inert.astype(bool)
    return PA, IA, inert.astype(bool)


class Comm:
    """Native NCCL communicator of the C-ABI (skmp_comm_*): one per process / GPU.  The 128-byte
    id comes from Comm.unique_id() on rank 0 and is shipped to the other ranks by the caller."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().skmp_comm_unique_id(ctypes.cast(buf, _P)))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = _P()
        _check(lib().skmp_comm_init(ctypes.cast(buf, _P), nranks, rank, ctypes.byref(h)))
        self.handle, self.nranks, self.rank = h, nranks, rank

    def free(self):
        if self.handle:
            lib().skmp_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sketch_allreduce(comm: Comm, sk: Sketch, stream=None):
    """NC1 through the native communicator: sum the per-rank partial sketches, refresh R."""
    _check(lib().sketch_allreduce(comm.handle, sk.handle, _stream(stream)))


def mp_selfjoin_dist(comm: Comm, R, m: int, *, excl: int = -1, reseed_rows: int = 0, stream=None):
    """mp_selfjoin split over the communicator's ranks (C-ABI mp_selfjoin_dist): every rank gets
    the full (P, I, inert)."""
    import torch
    k, n = R.shape
    dt = _dtype_code(R)
    tdt = torch.float32 if dt == F32 else torch.float64
    P = torch.empty((k, n - m + 1), dtype=tdt, device=R.device)
    I = torch.empty((k, n - m + 1), dtype=torch.int64, device=R.device)
    inert = np.zeros(k, dtype=np.uint8)
    cfg = _mpcfg(m, excl, reseed_rows)
    _check(lib().mp_selfjoin_dist(comm.handle, _ptr(R), k, n, R.stride(0), dt, ctypes.byref(cfg), _ptr(P), _ptr(I),
                                  _ptr(inert), _stream(stream)))
    return P, I, inert.astype(bool)


class Stream:
    """Streaming test data (f4): new time points are sketched with the train plan and
    statistics and every completed test window is AB-joined against the train sketch."""

    def __init__(self, train: Sketch, m: int, capacity: int, *, reseed_rows: int = 0, stream=None):
        cfg = _mpcfg(m, -1, reseed_rows)
        h = ctypes.c_void_p()
        _check(lib().stream_create(train.handle, ctypes.byref(cfg), capacity, _stream(stream), ctypes.byref(h)))
        _, k, _, d, dt = sketch_view(train)
        self.handle, self.m, self.k, self.cap, self.dtype, self.d = h, m, k, capacity, dt, d

    def push(self, T, stream=None):
        """T: d x n_new (torch CUDA tensor or numpy array, train dtype), rows in the plan order."""
        try:
            dc = _dtype_code(T)
        except ValueError:
            dc = -1
        if T.ndim != 2 or T.shape[0] != self.d or dc != self.dtype:
            raise SkmpError(1, f"Stream.push: T must be {self.d} x n_new of the train sketch's dtype "
                               f"({'float32' if self.dtype == F32 else 'float64'}), got {tuple(T.shape)} {T.dtype}", -1)
        n_new = T.shape[1]
        ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
        _check(lib().stream_push(self.handle, _ptr(T), n_new, ld, _stream(stream)))

    def view(self):
        """(R k x n_test, P k x n_sub, I k x n_sub, inert) — zero-copy views of library memory
        (valid until the next push or free)."""
        import torch
        R, P, I = _P(), _P(), _P()
        nt, ns, ld = _I64(), _I64(), _I64()
        inert = np.zeros(self.k, dtype=np.uint8)
        _check(lib().stream_view(self.handle, ctypes.byref(R), ctypes.byref(P), ctypes.byref(I), ctypes.byref(nt),
                                 ctypes.byref(ns), ctypes.byref(ld), _ptr(inert)))
        Rt = _as_tensor(R.value, (self.k, ld.value), self.dtype)[:, :nt.value]
        Pt = _as_tensor(P.value, (self.k, ld.value), self.dtype)[:, :ns.value]
        It = torch.as_tensor(_DevArray(I.value, (self.k, ld.value), "<i8"), device="cuda")[:, :ns.value]
        return Rt, Pt, It, inert.astype(bool)

    def topk(self, top: int, radius: int = -1, stream=None) -> list[Discord]:
        """Alg. 2's ordered discord list over the test windows seen so far."""
        _, P, I, inert = self.view()
        return discord_topk(P, I, inert, self.m, top, radius, stream)

    def free(self):
        if self.handle:
            lib().stream_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def discord_topk(P, I, inert, m: int, top: int, radius: int = -1, stream=None) -> list[Discord]:
    k, n_sub = P.shape
    inert_a = None if inert is None else np.ascontiguousarray(inert, dtype=np.uint8)
    t = np.empty(top, np.int64)
    g = np.empty(top, np.int32)
    nn = np.empty(top, np.int64)
    sc = np.empty(top, np.float64)
    nf = _I32()
    _check(lib().discord_topk(_ptr(P), _ptr(I), _ptr(inert_a), k, n_sub, P.stride(0), m, _dtype_code(P), top,
                              radius, _ptr(t), _ptr(g), _ptr(nn), _ptr(sc), ctypes.byref(nf), _stream(stream)))
    return [Discord(int(t[q]), int(g[q]), int(nn[q]), float(sc[q])) for q in range(nf.value)]


def discord_dims(T, rows, t_star: int, m: int, excl: int = -1, n: int | None = None, stream=None):
    """Alg. 3 Dimension-Detection (self-join mode): (scores, nn, j_star) for the streams `rows`
    of T (d x ld tensor / array), j_star indexing `rows`."""
    rows_a = np.ascontiguousarray(rows, dtype=np.int64)
    n = T.shape[1] if n is None else n
    sc = np.empty(len(rows_a), np.float64)
    nn = np.empty(len(rows_a), np.int64)
    js = _I64()
    ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
    _check(lib().discord_dims(_ptr(T), ld, n, _dtype_code(T), _ptr(rows_a), len(rows_a), t_star, m, excl,
                              _ptr(sc), _ptr(nn), ctypes.byref(js), _stream(stream)))
    return sc, nn, int(js.value)


def discord_dims_group(sk: Sketch, g: int, sources, t_star: int, m: int, excl: int = -1, stream=None) -> DimResult:
    """Alg. 3 over J_g of the sketch plan with the raw streams spread over several matrices
    (C-ABI discord_dims_group): `sources` = [(T, ids), ...] (rows of T hold the streams with
    those ids; T a CUDA tensor or a host array, None / empty skipped).  Returns the DimResult
    (n_scored == 0: no member of J_g in `sources`)."""
    keep, arr = [], []
    for T, ids in sources:
        if T is None or ids is None or len(ids) == 0:
            continue
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        assert T.shape[0] == len(ids), "one id per row of T"
        ld = T.stride(0) if hasattr(T, "stride") and callable(T.stride) else T.strides[0] // T.itemsize
        keep.append(ids)
        arr.append(Source(_ptr(T).value, ld, len(ids), ids.ctypes.data))
    src = (Source * max(1, len(arr)))(*arr)
    out = DimResult()
    _check(lib().discord_dims_group(sk.handle, g, ctypes.cast(src, _P), len(arr), t_star, m, excl, ctypes.byref(out),
                                    _stream(stream)))
    return out


def discord_dims_merge(parts) -> DimResult:
    """Host-only: the first strict maximum over per-part winners in J_g order (C-ABI)."""
    arr = (DimResult * len(parts))(*parts)
    out = DimResult()
    _check(lib().discord_dims_merge(ctypes.cast(arr, _P), len(parts), ctypes.byref(out)))
    return out


def detect_dimension(sk: Sketch, sources, t: int, g: int, m: int, excl: int = -1, stream=None):
    """Alg. 3 over J_g for the discord at time t (discord_dims_group).  Returns (id*, score, nn)
    with Alg. 3's tie rule (first strict maximiser in plan order), or None when no stream of J_g
    is in `sources`."""
    r = discord_dims_group(sk, g, sources, t, m, excl, stream)
    return None if r.n_scored == 0 else (int(r.id), float(r.score), int(r.nn))


@dataclass
class DiscordReport:
    """The paper's detection output (Alg. 2 + Alg. 3 + optional refinement)."""
    t: int                 # discord time i* (Alg. 2, combined sketch profile)
    g: int                 # discord group g*
    score: float           # sketched discord score C[i*]
    j_id: int              # dimension j* (stream id, Alg. 3)
    j_score: float         # 1NN distance of T_{j*, i*, m} in its own stream
    j_nn: int              # its nearest neighbour's time
    refined_t: int | None  # top-1 discord of the full profile of stream j*
    refined_score: float | None
    ms: dict               # per-phase device times


def detect(T, ids, k: int, m: int, *, seed: int = 0, proj: int = PROJ_COUNT_SKETCH, S=None,
           refine: bool = True, stream=None) -> DiscordReport:
    """End-to-end single-series mode over the C-ABI: Alg. 1 sketch -> self-join of every
    sketch series -> Alg. 2 combine / top-1 -> Alg. 3 over J_g* -> optional refinement join.
    T: d x n CUDA tensor (rows = streams with `ids`)."""
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    if proj == PROJ_DENSE:
        sk = sketch_build(T, ids, k, proj=PROJ_DENSE, S=S, stream=stream)
    else:
        sk = sketch_build(T, ids, k, seed=seed, stream=stream)
    ev[1].record()
    P, I, inert = mp_selfjoin(sk.R, m, stream=stream)
    top = discord_topk(P, I, inert, m=m, top=1, stream=stream)[0]
    ev[2].record()
    ids_a = np.ascontiguousarray(ids, dtype=np.uint64)
    dim = discord_dims_group(sk, top.g, [(T, ids_a)], top.t, m, stream=stream)
    ev[3].record()
    rt = rs = None
    if refine:  # the full profile of stream j* and its top-1 discord (discord_topk)
        j = int(np.nonzero(ids_a == dim.id)[0][0])
        Pj, Ij, inj = mp_selfjoin(T[j:j + 1], m, stream=stream)
        d1 = discord_topk(Pj, Ij, inj, m, 1, stream=stream)[0]
        rt, rs = d1.t, d1.score
    ev[4].record()
    torch.cuda.synchronize()
    sk.free()
    ms = {"sketch": ev[0].elapsed_time(ev[1]), "time_detection": ev[1].elapsed_time(ev[2]),
          "dimension_detection": ev[2].elapsed_time(ev[3]), "refine": ev[3].elapsed_time(ev[4])}
    return DiscordReport(top.t, top.g, top.score, int(dim.id), float(dim.score), int(dim.nn), rt, rs, ms)

