"""GPU parity: mp_selfjoin (K4-K7) through the C-ABI vs the oracle's brute-force self-join.

Inputs come from synthgen (sketch-like series) and are handed byte-identical to both sides;
nothing the CUDA path computes is fed to the oracle.  Sizes span several W-diagonal blocks,
several L-row tiles (small reseed_rows), and ragged tails.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from tests._parity import TOL, check_profile

pytestmark = pytest.mark.gpu


def _run(cuda, X: np.ndarray, m: int, dtype: str, excl=None, reseed=0, label=""):
    import torch
    import paper_2311_03393_b200 as skmp
    tdt = torch.float32 if dtype == "f32" else torch.float64
    R = torch.from_numpy(X).to(cuda, tdt)
    e = (m + 1) // 2 if excl is None else excl
    P, I, inert = skmp.mp_selfjoin(R, m, excl=e, reseed_rows=reseed)
    torch.cuda.synchronize()
    P, I = P.cpu().numpy(), I.cpu().numpy()
    Xo = R.double().cpu().numpy()  # the exact values both sides see (fp32 upcast is exact)
    ties = 0
    for g in range(X.shape[0]):
        Po, Io, Fo = ref.selfjoin_rows(Xo[g], m, e)
        ties += check_profile(Xo[g], m, e, P[g], I[g], Po, Io, Fo, TOL[dtype], label=f"{label} g={g}")
        assert bool(inert[g]) == bool(np.all(Fo))
    return ties


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,m,k,kind,reseed", [
    (300, 16, 2, "mix", 0),          # single tile, triangle boundary
    (2500, 50, 3, "randwalk", 128),  # 3 diagonal blocks, many row tiles, ragged tail
    (4099, 33, 2, "noise", 64),      # odd m, ragged everything
    (1100, 8, 1, "seasonal", 0),     # tiny m
])
def test_mp_selfjoin_parity(cuda, dtype, n, m, k, kind, reseed):
    X = synthgen.mp_series(k, n, seed=1000 + n + m, kind=kind)
    _run(cuda, X, m, dtype, reseed=reseed, label=f"{dtype} n={n} m={m}")


def test_mp_f64_large_grid_instance(cuda):
    """FP64 joins above 16 waves of CTAs run the 114-register kernel instance, smaller ones the
    96-register instance (mp_join.cu kJoinSmallGrid): 64-row tiles give this n = 20,000 pair of
    series ~49k CTAs, so the large instance is checked against the brute force too."""
    X = synthgen.mp_series(2, 20000, seed=77, kind="mix")
    _run(cuda, X, 50, "f64", reseed=64, label="f64 large grid")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_exclusion_zone_variants(cuda, dtype):
    X = synthgen.mp_series(1, 1500, seed=77, kind="mix")
    for excl in (0, 1, 40, 200):
        _run(cuda, X, 32, dtype, excl=excl, reseed=256, label=f"excl={excl}")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_planted_motif(cuda, dtype):
    """Two exact copies more than r apart -> P ~ 0 at both (SPEC self_join example)."""
    import torch
    import paper_2311_03393_b200 as skmp
    X = synthgen.mp_series(1, 3000, seed=5, kind="noise")
    m = 64
    X[0, 2000:2000 + m] = X[0, 300:300 + m]
    R = torch.from_numpy(X).to(cuda, torch.float32 if dtype == "f32" else torch.float64)
    P, I, _ = skmp.mp_selfjoin(R, m)
    P, I = P.cpu().numpy()[0], I.cpu().numpy()[0]
    assert I[300] == 2000 and I[2000] == 300
    assert P[300] < 1e-3 and P[2000] < 1e-3


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_flat_and_inert(cuda, dtype):
    """Flat windows (reading 5) and an all-flat (inert, reading 6) series."""
    n, m = 1600, 40
    X = synthgen.mp_series(3, n, seed=9, kind="mix")
    X[0, 200:400] = 1.5            # flat windows inside series 0
    X[0, 900:1000] = -2.0          # a second flat run, > excl away
    X[1, :] = 0.0                  # empty group -> inert
    X[2, 1200:1300] = 0.25
    _run(cuda, X, m, dtype, reseed=128, label="flat")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_band_invariance(cuda, dtype):
    """Any diagonal-band split accumulates bit-identical keys (multi-GPU invariant, one GPU)."""
    import torch
    import paper_2311_03393_b200 as skmp
    X = synthgen.mp_series(2, 6000, seed=31, kind="randwalk")
    m = 48
    R = torch.from_numpy(X).to(cuda, torch.float32 if dtype == "f32" else torch.float64)
    ref_w = skmp.mp_create(R, m, reseed_rows=512)
    skmp.mp_join(ref_w)
    k0, _ = skmp.mp_keys(ref_w)
    k0 = k0.clone()
    n_sub = 6000 - m + 1
    excl = (m + 1) // 2
    for nb in (2, 3, 4, 8):
        w = skmp.mp_create(R, m, reseed_rows=512)
        for b in range(nb):
            lo, hi = skmp.mp_band(n_sub, excl, skmp.F32 if dtype == "f32" else skmp.F64, nb, b)
            skmp.mp_join(w, lo, hi)
        kb, _ = skmp.mp_keys(w)
        torch.cuda.synchronize()
        assert torch.equal(kb, k0), f"{nb} bands differ"
        w.free()
    ref_w.free()


def test_mp_errors(cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    R = torch.zeros((1, 10), device=cuda, dtype=torch.float64)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.mp_selfjoin(R, 16)
    assert e.value.name == "SKMP_E_SERIES_TOO_SHORT"
    R = torch.randn((1, 20), device=cuda, dtype=torch.float64)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.mp_selfjoin(R, 16)  # n_sub = 5 < 2*8+2
    assert e.value.name == "SKMP_E_NO_ADMISSIBLE"
    with pytest.raises(skmp.SkmpError) as e:
        skmp.mp_selfjoin(R, 1)
    assert e.value.name == "SKMP_E_INVALID_ARG"


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_finalize_rows_slices(cuda, dtype):
    """mp_finalize_rows over disjoint window slices (the multi-GPU sharded finalize) reproduces
    mp_finalize exactly."""
    import torch
    import paper_2311_03393_b200 as skmp
    X = synthgen.mp_series(3, 3000, seed=71, kind="mix")
    R = torch.from_numpy(X).to(cuda, torch.float32 if dtype == "f32" else torch.float64)
    w = skmp.mp_create(R, 40, reseed_rows=256)
    skmp.mp_join(w)
    P, I, inert = skmp.mp_finalize(w)
    n_sub = 3000 - 40 + 1
    Ps = torch.zeros_like(P)
    Is = torch.zeros_like(I)
    for lo, hi in ((0, 1), (1, 777), (777, 778), (778, n_sub)):
        Pp, Ip, _ = skmp.mp_finalize_rows(w, lo, hi)
        Ps += Pp
        Is += Ip
    torch.cuda.synchronize()
    assert torch.equal(Ps, P) and torch.equal(Is, I)
    with pytest.raises(skmp.SkmpError):
        skmp.mp_finalize_rows(w, 5, n_sub + 1)
    w.free()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_long_windows(cuda, dtype):
    """m larger than the finalize staging chunk (256 windows positions): the set resolution and
    the explicit-difference distance run over several staged chunks / from global memory."""
    X = synthgen.mp_series(2, 3000, seed=81, kind="mix")
    _run(cuda, X, 600, dtype, reseed=256, label=f"m=600 {dtype}")
    X = synthgen.mp_series(1, 2200, seed=82, kind="randwalk")
    _run(cuda, X, 257, dtype, label=f"m=257 {dtype}")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_minimal_admissible_size(cuda, dtype):
    """n_sub = 2 excl + 2: the two end rows have exactly one admissible neighbour each (each
    other) and every row has at least one (reading 16)."""
    for m in (8, 33):
        excl = (m + 1) // 2
        n = 2 * excl + 2 + m - 1
        X = synthgen.mp_series(2, n, seed=100 + m, kind="noise")
        _run(cuda, X, m, dtype, label=f"minimal m={m}")


def test_oom_is_reported_and_the_context_stays_usable(cuda):
    """A workspace larger than the device (64 series x 2^30 windows ~ 2.8 TB) fails with
    SKMP_E_OOM before any kernel touches the (tiny) input, and the library keeps working."""
    import ctypes
    import torch
    import paper_2311_03393_b200 as skmp
    R = torch.zeros(64, 64, device=cuda)
    L = skmp.lib()
    cfg = skmp._mpcfg(16)
    h = ctypes.c_void_p()
    n = 1 << 30
    st = L.mp_create(skmp._ptr(R), 64, n, n, skmp.F32, ctypes.byref(cfg), skmp._stream(None), ctypes.byref(h))
    assert st == 12, L.skmp_last_error()              # SKMP_E_OOM
    # stream_create with an impossible capacity (64 groups x 2^30 samples ~ 1.6 TB of buffers)
    R2 = torch.from_numpy(synthgen.mp_series(2, 3000, seed=2, kind="mix")).to(cuda, torch.float32)
    T = torch.from_numpy(synthgen.mp_series(80, 3000, seed=3, kind="mix")).to(cuda, torch.float32)
    skt = skmp.sketch_build(T, np.arange(80, dtype=np.uint64), 64, seed=1)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.Stream(skt, 32, capacity=1 << 30)
    assert e.value.name == "SKMP_E_OOM"
    P, I, _ = skmp.mp_selfjoin(R2, 32)                 # still fine afterwards
    torch.cuda.synchronize()
    assert torch.isfinite(P).all()
