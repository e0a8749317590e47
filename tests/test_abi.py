"""CPU-only checks of the C-ABI library: it loads, exports every function include/sketchmp.h
declares, and its host-only entry points (hash plan, band partition, errors) work without a
GPU; compute entry points fail loudly (no CPU fallback)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2311_03393_b200 as skmp
from oracle.hashplan import plan_count_sketch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sketchmp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(?:skmp_status|void|const char\*|int64_t|int32_t)\s+\**(\w+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = skmp.lib()
    names = _declared()
    assert len(names) >= 20, names
    for n in names:
        assert hasattr(L, n), f"missing export {n}"
    assert set(names) >= set(skmp._SIGS), set(skmp._SIGS) - set(names)
    assert L.skmp_abi_version() == 1


def test_status_strings():
    L = skmp.lib()
    for code, name in skmp.STATUS.items():
        assert L.skmp_status_string(code).decode() == name


@pytest.mark.parametrize("k,seed", [(1, 0), (7, 2311033932), (64, 12345), (100, 2**63 + 5)])
def test_hash_plan_matches_oracle(k, seed):
    """C++ Carter-Wegman plan (128-bit products) == the oracle's Python-integer plan, bit-equal."""
    edge = [2**61 - 2, 2**61 - 1, 2**61, 2**61 + 1, 2**62, 2**63, 2**64 - 2, 2**64 - 1]
    ids = np.concatenate([np.arange(0, 3000, dtype=np.uint64), np.array(edge, dtype=np.uint64)])
    assert ids.dtype == np.uint64 and [int(x) for x in ids[3000:]] == edge   # no float promotion
    g, s = skmp.sketch_hash_plan(ids, k, seed)
    go, so = plan_count_sketch([int(x) for x in ids], k, seed)
    assert np.array_equal(g, np.array(go, dtype=np.int32))
    assert np.array_equal(s, np.array(so, dtype=np.int8))


def test_hash_plan_invalid():
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_hash_plan(np.arange(3), 0, 1)
    assert e.value.name == "SKMP_E_INVALID_ARG"


@pytest.mark.parametrize("n_sub,excl,dtype", [(1999745, 128, 0), (199745, 128, 0), (19901, 50, 1), (1951, 25, 1)])
def test_band_partition(n_sub, excl, dtype):
    W = skmp.mp_tile_width(dtype)
    for nb in (1, 2, 4, 8):
        edges = []
        for b in range(nb):
            lo, hi = skmp.mp_band(n_sub, excl, dtype, nb, b)
            edges.append((lo, hi))
        # contiguous cover of [0, n_sub), interior edges on the tile grid
        assert edges[0][0] == 0 and edges[-1][1] == n_sub
        for (a, b_), (c, d) in zip(edges, edges[1:]):
            assert b_ == c and c % W == 0 and a <= b_
        # balance: each band within one tile-width of diagonals of the ideal share of the cost
        # (cells + 5 W per diagonal, the per-tile work that does not scale with rows)
        lo0 = excl + 1
        def cum(x):  # cost of diagonals [lo0, x): cells + 5 W each, first W diagonals' cells x 4.5
            A = max(x, lo0) - lo0
            F = min(A, W)
            return (A * (n_sub - lo0) - A * (A - 1) // 2 + 5 * W * A + 3.5 * (F * (n_sub - lo0) - F * (F - 1) // 2))
        tot = cum(n_sub)
        for a, b in edges:
            assert abs((cum(b) - cum(a)) - tot / nb) <= 4.5 * W * (n_sub + 5 * W) + 1


@pytest.mark.parametrize("nA,nB,dtype", [(199745, 199745, 0), (9901, 99873, 0), (99873, 9901, 0), (1951, 1951, 1),
                                         (300, 5000, 1), (5000, 300, 0), (1, 1, 0), (7, 1, 1)])
def test_abband_partition(nA, nB, dtype):
    """The AB-join's two passes (pass 1 diagonals [0, nB), pass 2 diagonals [1, nA)) split into
    equal-cell bands: every diagonal in exactly one band, interior edges on the tile grid,
    balanced to within a tile width of cells."""
    W = skmp.mp_tile_width(dtype)

    def c1(a, b):  # cells of pass-1 diagonals [a, b): sum min(nA, nB - delta)
        x = np.arange(a, b, dtype=np.float64)
        return float(np.minimum(nA, nB - x).sum())

    def c2(a, b):
        x = np.arange(a, b, dtype=np.float64)
        return float(np.minimum(nB, nA - x).sum())

    assert c1(0, nB) + c2(1, nA) == float(nA) * nB
    for nb in (1, 2, 3, 8):
        bands = [skmp.mp_abband(nA, nB, dtype, nb, b) for b in range(nb)]
        p1 = [bd[0] for bd in bands if bd[0][0] < bd[0][1]]
        p2 = [bd[1] for bd in bands if bd[1][0] < bd[1][1]]
        # contiguous, disjoint cover of each pass
        assert p1[0][0] == 0 and p1[-1][1] == nB
        assert all(a[1] == b[0] and b[0] % W == 0 for a, b in zip(p1, p1[1:]))
        if nA > 1:
            assert p2[0][0] == 1 and p2[-1][1] == nA
            assert all(a[1] == b[0] and b[0] % W == 0 for a, b in zip(p2, p2[1:]))
        else:
            assert not p2
        # bands are consecutive in the pass-1-then-pass-2 order
        order = []
        for (a1, b1), (a2, b2) in bands:
            if a1 < b1:
                order.append((1, a1, b1))
            if a2 < b2:
                order.append((2, a2, b2))
        assert order == sorted(order)
        tot = float(nA) * nB
        for (a1, b1), (a2, b2) in bands:
            got = (c1(a1, b1) if a1 < b1 else 0.0) + (c2(a2, b2) if a2 < b2 else 0.0)
            assert abs(got - tot / nb) <= 2 * W * max(nA, nB) + 1


def test_abband_invalid():
    with pytest.raises(skmp.SkmpError):
        skmp.mp_abband(0, 10, 0, 2, 0)
    with pytest.raises(skmp.SkmpError):
        skmp.mp_abband(10, 10, 0, 2, 2)


def test_compute_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    T = np.random.default_rng(0).standard_normal((3, 100))
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_build(T, np.arange(3), 2, seed=1)
    assert e.value.name == "SKMP_E_CUDA"


def test_argument_validation_before_any_device_work():
    """Validation precedes the device check (ABI rule: errors before any launch): these fail with
    the argument error, not SKMP_E_CUDA, even without a GPU."""
    import torch
    T = np.random.default_rng(1).standard_normal((3, 100))
    cases = [
        (lambda: skmp.discord_dims(T, [0], 100 - 16 + 1, 16), "SKMP_E_INVALID_ARG"),    # t* past the end
        (lambda: skmp.discord_dims(T, [-1], 0, 16), "SKMP_E_INVALID_ARG"),              # negative row
        (lambda: skmp.discord_dims(T, [0], 40, 16, 60), "SKMP_E_NO_ADMISSIBLE"),        # excl too wide
        (lambda: skmp.discord_dims(T[:, :10].copy(), [0], 0, 16), "SKMP_E_SERIES_TOO_SHORT"),
    ]
    for fn, name in cases:
        with pytest.raises(skmp.SkmpError) as e:
            fn()
        assert e.value.name == name
    if not torch.cuda.is_available():
        with pytest.raises(skmp.SkmpError) as e:
            skmp.discord_dims(T, [0, 2], 10, 16)
        assert e.value.name == "SKMP_E_CUDA"   # valid arguments: then no device -> loud failure


def test_abjoin_argument_validation():
    L = skmp.lib()
    cfg = skmp._mpcfg(16)
    buf = (ctypes.c_double * 4)()
    i64 = (ctypes.c_int64 * 4)()
    # NULL outputs / too-short series rejected before any device work
    assert L.mp_abjoin(ctypes.cast(buf, ctypes.c_void_p), 100, 100, ctypes.cast(buf, ctypes.c_void_p), 100, 100, 1, 1,
                       ctypes.byref(cfg), None, None, None, None, None, None) == 1
    assert L.mp_abjoin(ctypes.cast(buf, ctypes.c_void_p), 10, 10, ctypes.cast(buf, ctypes.c_void_p), 100, 100, 1, 1,
                       ctypes.byref(cfg), ctypes.cast(buf, ctypes.c_void_p), ctypes.cast(i64, ctypes.c_void_p),
                       None, None, None, None) == 4


def test_stream_and_staged_ab_null_handles():
    """The f4 stream and staged AB-join entry points reject NULL handles / bad arguments with
    SKMP_E_INVALID_ARG before touching a device (called through the raw ctypes symbols)."""
    import ctypes
    L = skmp.lib()
    cfg = skmp._mpcfg(16)
    out = ctypes.c_void_p()
    assert L.stream_create(None, ctypes.byref(cfg), 100, None, ctypes.byref(out)) == 1
    assert L.stream_push(None, None, 1, 1, None) == 1
    assert L.stream_view(None, None, None, None, None, None, None, None) == 1
    L.stream_free(None)                                   # no-op
    assert L.mp_join_ab(None, None, 0, 1, None) == 1
    assert L.mp_finalize_ab(None, None, 0, 0, None, None, None, None) == 1
    assert L.mp_create_ab(None, 1, 100, 100, 0, ctypes.byref(cfg), None, ctypes.byref(out)) == 1


def _c_compile(args, tmp_path):
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    return subprocess.run(["gcc", *args], capture_output=True, text=True, cwd=str(tmp_path))


def test_header_is_plain_c99(tmp_path):
    """include/sketchmp.h is a C header (no C++ constructs): a C99 translation unit that only
    includes it compiles warning-free under -pedantic -Werror."""
    src = tmp_path / "h.c"
    src.write_text('#include "sketchmp.h"\nint main(void) { return (int)SKMP_OK; }\n')
    r = _c_compile(["-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror",
                    f"-I{os.path.join(ROOT, 'include')}", str(src), "-o", str(tmp_path / "h")], tmp_path)
    assert r.returncode == 0, r.stderr


def test_c_demo_links_against_the_library(tmp_path):
    """examples/abi_demo.c (a plain-C user of the ABI) compiles and links against libsketchmp.so;
    tests/test_gpu_c_abi.py runs it on a B200."""
    r = _c_compile(["-std=c99", "-O2", os.path.join(ROOT, "examples", "abi_demo.c"),
                    f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include",
                    f"-L{os.path.join(ROOT, 'paper_2311_03393_b200')}", "-lsketchmp",
                    "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-o", str(tmp_path / "abi_demo")], tmp_path)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("n_sub,excl,dtype", [(199745, 128, 0), (1999745, 128, 0), (19901, 50, 1), (700, 8, 0)])
def test_rank_diagonals_tile_the_join(n_sub, excl, dtype):
    """dist.rank_diagonals: the ranks' bands tile [0, n_sub) contiguously on the tile grid."""
    from paper_2311_03393_b200 import dist as sdist
    W = skmp.mp_tile_width(dtype)
    assert sdist.rank_diagonals(n_sub, excl, dtype, 1, 0) == [(0, n_sub)]
    for world in (2, 4, 8):
        bands = [sdist.rank_diagonals(n_sub, excl, dtype, world, r)[0] for r in range(world)]
        assert bands[0][0] == 0 and bands[-1][1] == n_sub
        for (a, b), (c, d) in zip(bands, bands[1:]):
            assert b == c and c % W == 0 and a <= b


def test_native_comm_argument_validation():
    """skmp_comm_* / sketch_allreduce / mp_selfjoin_dist reject NULL / bad arguments before any
    NCCL or device work."""
    import ctypes
    L = skmp.lib()
    out = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 128)()
    assert L.skmp_comm_unique_id(None) == 1
    assert L.skmp_comm_init(None, 1, 0, ctypes.byref(out)) == 1
    assert L.skmp_comm_init(ctypes.cast(buf, ctypes.c_void_p), 2, 2, ctypes.byref(out)) == 1
    assert L.sketch_allreduce(None, None, None) == 1
    cfg = skmp._mpcfg(16)
    assert L.mp_selfjoin_dist(None, None, 1, 100, 100, 0, ctypes.byref(cfg), None, None, None, None) == 1
    L.skmp_comm_free(None)


def test_dims_merge_host_only():
    """discord_dims_merge (host-only): the first strict maximum over parts in J_g order; parts
    with nothing scored are skipped; ids keep all 64 bits."""
    D = skmp.DimResult
    r = skmp.discord_dims_merge([D(1.0, 7, 3, 2), D(2.0, 2**64 - 1, 9, 4), D(2.0, 5, 1, 1), D(9.0, 3, 3, 0)])
    assert (r.score, r.id, r.nn, r.n_scored) == (2.0, 2**64 - 1, 9, 7)
    r = skmp.discord_dims_merge([D(0.0, 0, 0, 0), D(0.0, 0, 0, 0)])
    assert r.n_scored == 0
    L = skmp.lib()
    assert L.discord_dims_merge(None, 1, None) == 1
    parts = (D * 1)(D(1.0, 1, 1, -1))
    out = D()
    assert L.discord_dims_merge(ctypes.cast(parts, ctypes.c_void_p), 1, ctypes.byref(out)) == 1


def test_dims_group_argument_validation():
    """discord_dims_group rejects a NULL handle / output before any device work."""
    L = skmp.lib()
    out = skmp.DimResult()
    assert L.discord_dims_group(None, 0, None, 0, 0, 16, -1, ctypes.byref(out), None) == 1
    assert L.discord_dims_group(None, 0, None, -1, 0, 16, -1, None, None) == 1


def test_trim_and_free_without_gpu():
    """skmp_trim is callable without a device (no pools yet: a no-op); sketch_free[_async] of
    NULL is a no-op."""
    skmp.skmp_trim()
    L = skmp.lib()
    L.sketch_free(None)
    L.sketch_free_async(None, None)
