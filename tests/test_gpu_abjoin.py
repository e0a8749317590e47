"""GPU parity: mp_abjoin (Def. 6 ab-join, P:L166-169 — the join Alg. 2 calls as written,
P:L249-269) through the C-ABI vs the oracle's brute force, and Alg. 2 end to end on a
train/test split."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch
from tests._parity import TOL, check_topk

pytestmark = pytest.mark.gpu


def _check_ab(a, b, m, P, I, tol, rows=None, label=""):
    """Compare one AB profile (rows of a against all windows of b) with the oracle."""
    Po, Io = ref.abjoin_brute(a, b, m, rows=rows)
    rows = np.arange(len(Po)) if rows is None else np.asarray(rows)
    P = np.asarray(P, dtype=np.float64)[rows]
    I = np.asarray(I)[rows]
    floor = 1e-3 * math.sqrt(m)
    err = np.abs(P - Po) / np.maximum(Po, floor)
    assert err.max() <= tol, f"{label}: rel err {err.max():.3e} at row {rows[int(np.argmax(err))]}"
    mism = np.where(I != Io)[0]
    if len(mism):
        Za, fa = ref.znorm_windows(a, m)
        Zb, fb = ref.znorm_windows(b, m)
        for q in mism:
            i, j = int(rows[q]), int(I[q])
            assert 0 <= j < Zb.shape[0], f"{label}: row {i}: index {j} out of range"
            dj = 0.0 if (fa[i] and fb[j]) else (math.sqrt(m) if (fa[i] or fb[j]) else
                                                float(np.sqrt(((Za[i] - Zb[j]) ** 2).sum())))
            assert dj <= Po[q] + tol * max(Po[q], floor), f"{label}: row {i}: {j} ({dj}) vs {Io[q]} ({Po[q]})"
    return len(mism)


def _run(cuda, A, B, m, dtype, reseed=0, label=""):
    import torch
    import paper_2311_03393_b200 as skmp
    tdt = torch.float32 if dtype == "f32" else torch.float64
    RA = torch.from_numpy(A).to(cuda, tdt)
    RB = torch.from_numpy(B).to(cuda, tdt)
    PA, IA, PB, IB, inert = skmp.mp_abjoin(RA, RB, m, reseed_rows=reseed, both=True)
    torch.cuda.synchronize()
    Ao, Bo = RA.double().cpu().numpy(), RB.double().cpu().numpy()
    PA, IA, PB, IB = PA.cpu().numpy(), IA.cpu().numpy(), PB.cpu().numpy(), IB.cpu().numpy()
    for g in range(A.shape[0]):
        _check_ab(Ao[g], Bo[g], m, PA[g], IA[g], TOL[dtype], label=f"{label} AB g={g}")
        _check_ab(Bo[g], Ao[g], m, PB[g], IB[g], TOL[dtype], label=f"{label} BA g={g}")
    return inert


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("nA,nB,m,k,reseed", [
    (900, 700, 32, 2, 0),        # test longer than train
    (600, 2500, 50, 3, 128),     # train longer: several diagonal blocks, many row tiles
    (1501, 1501, 33, 1, 64),     # equal lengths, odd m
    (300, 4099, 16, 2, 0),       # very unequal, ragged
    (120, 90, 8, 2, 0),          # tiny
])
def test_mp_abjoin_parity(cuda, dtype, nA, nB, m, k, reseed):
    A = synthgen.mp_series(k, nA, seed=7000 + nA, kind="mix")
    B = synthgen.mp_series(k, nB, seed=8000 + nB, kind="mix")
    _run(cuda, A, B, m, dtype, reseed, label=f"{dtype} nA={nA} nB={nB} m={m}")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_abjoin_flat_empty_and_planted(cuda, dtype):
    import torch
    import paper_2311_03393_b200 as skmp
    m = 24
    A = synthgen.mp_series(3, 1300, seed=51, kind="mix")
    B = synthgen.mp_series(3, 1700, seed=52, kind="noise")
    A[0, 100:200] = 1.0          # flat test windows ...
    B[0, 900:960] = -3.0         # ... with flat train partners
    A[1, 400:470] = 2.0          # flat test windows, train series 1 has none
    A[2], B[2] = 0.0, 0.0        # empty group: both flat -> inert
    B[1, 1000:1000 + m] = 5 * A[1, 700:700 + m] + 1   # planted affine copy -> 0
    inert = _run(cuda, A, B, m, dtype, label="flat")
    assert list(inert) == [False, False, True]
    RA = torch.from_numpy(A).to(cuda, torch.float32 if dtype == "f32" else torch.float64)
    RB = torch.from_numpy(B).to(cuda, RA.dtype)
    PA, IA, _ = skmp.mp_abjoin(RA, RB, m)
    assert float(PA[1, 700]) < 1e-3 and int(IA[1, 700]) == 1000


def test_mp_abjoin_c3_lengths_sampled(cuda):
    """C3 scale (FP32, m = 128): train n = 100,000, test n = 40,000, sampled rows."""
    import torch
    import paper_2311_03393_b200 as skmp
    A = synthgen.mp_series(2, 40_000, seed=61, kind="mix")
    B = synthgen.mp_series(2, 100_000, seed=62, kind="randwalk")
    RA = torch.from_numpy(A).to(cuda, torch.float32)
    RB = torch.from_numpy(B).to(cuda, torch.float32)
    PA, IA, PB, IB, _ = skmp.mp_abjoin(RA, RB, 128, both=True)
    rng = np.random.default_rng(63)
    Ao, Bo = RA.double().cpu().numpy(), RB.double().cpu().numpy()
    for g in range(2):
        ra = np.sort(rng.choice(40_000 - 127, 48, replace=False))
        rb = np.sort(rng.choice(100_000 - 127, 24, replace=False))
        _check_ab(Ao[g], Bo[g], 128, PA[g].cpu().numpy(), IA[g].cpu().numpy(), TOL["f32"], rows=ra, label="c3 AB")
        _check_ab(Bo[g], Ao[g], 128, PB[g].cpu().numpy(), IB[g].cpu().numpy(), TOL["f32"], rows=rb, label="c3 BA")


def test_alg2_time_detection_train_test(cuda):
    """Alg. 2 as written: both halves of a C2-recipe dataset sketched with the same
    id-keyed plan (each half z-normalised by its own statistics, reading 21), the test sketch
    AB-joined against the train sketch per group, then the combine + ordered top-K."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], n=6000)   # C2 recipe; oracle-sized
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    cut = 3500
    Ttr, Tte = np.ascontiguousarray(T[:, :cut]), np.ascontiguousarray(T[:, cut:])
    d = lambda x: torch.from_numpy(x).to(cuda, torch.float64)  # noqa: E731
    sk_tr = skmp.sketch_build(d(Ttr), ids, cfg.k, seed=cfg.seed)
    sk_te = skmp.sketch_build(d(Tte), ids, cfg.k, seed=cfg.seed)
    PA, IA, inert = skmp.mp_abjoin(sk_te.R, sk_tr.R, cfg.m)
    top = skmp.discord_topk(PA, IA, inert, m=cfg.m, top=6)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    Rtr, _, _ = ref.sketch(Ttr, cfg.k, g, s)
    Rte, _, _ = ref.sketch(Tte, cfg.k, g, s)
    Po, Io = zip(*(ref.abjoin_brute(Rte[q], Rtr[q], cfg.m) for q in range(cfg.k)))
    Po, Io = np.stack(Po), np.stack(Io)
    inert_o = np.array([np.all(ref.window_stats(Rte[q], cfg.m)[2]) and np.all(ref.window_stats(Rtr[q], cfg.m)[2])
                        for q in range(cfg.k)])
    assert np.array_equal(inert, inert_o)
    Pg = PA.cpu().numpy()
    err = np.abs(Pg - Po) / np.maximum(Po, 1e-3 * math.sqrt(cfg.m))
    assert err[~inert_o].max() <= TOL["f64"]
    C, G = ref.combine(Po, inert_o)
    want = ref.topk_greedy(C, G, Io, 6, (cfg.m + 1) // 2)
    check_topk(top, want, C, TOL["f64"], label="alg2 train/test")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mp_abjoin_long_windows(cuda, dtype):
    A = synthgen.mp_series(1, 1800, seed=91, kind="mix")
    B = synthgen.mp_series(1, 2500, seed=92, kind="seasonal")
    _run(cuda, A, B, 300, dtype, label=f"m=300 {dtype}")


def _combine(keys_list, words):
    """On-device stand-in for dist.reduce_keys over band workspaces: FP32 keys max; FP64 keys
    max on the value word, then max on the index word among the holders of that value."""
    import torch
    K = torch.stack([k.view(-1, words) for k in keys_list])
    if words == 1:
        return K.max(dim=0).values.view(-1)
    v = K[:, :, 0].max(dim=0).values
    idx = torch.where(K[:, :, 0] == v, K[:, :, 1], torch.full_like(K[:, :, 1], -(1 << 63))).max(dim=0).values
    return torch.stack([v, idx], dim=1).view(-1)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("nA,nB,m,k", [(3000, 9000, 64, 3), (9000, 2500, 33, 2), (40000, 40000, 100, 1)])
def test_staged_abjoin_band_invariance(cuda, dtype, nA, nB, m, k):
    """The staged AB-join (mp_create_ab / mp_join_ab / mp_finalize_ab) split into 1, 2, 3 and 5
    mp_abband bands, keys combined like the multi-GPU reduce: keys bit-identical to the
    one-band join and profiles identical to mp_abjoin (SURVEY §8(e) applied to f1)."""
    import torch
    import paper_2311_03393_b200 as skmp
    tdt = torch.float32 if dtype == "f32" else torch.float64
    RA = torch.from_numpy(synthgen.mp_series(k, nA, seed=21, kind="mix")).to(cuda, tdt)
    RB = torch.from_numpy(synthgen.mp_series(k, nB, seed=22, kind="mix")).to(cuda, tdt)
    PA0, IA0, PB0, IB0, inert0 = skmp.mp_abjoin(RA, RB, m, both=True)
    ref_keys = None
    for nb in (1, 2, 3, 5):
        parts = []
        for band in range(nb):
            a, b = skmp.mp_create_ab(RA, m), skmp.mp_create_ab(RB, m)
            (l1, h1), (l2, h2) = skmp.mp_abband(a.n_sub, b.n_sub, a.dtype, nb, band)
            if l1 < h1:
                skmp.mp_join_ab(a, b, l1, h1)
            if l2 < h2:
                skmp.mp_join_ab(b, a, l2, h2)
            parts.append((a, b))
        words = skmp.mp_keys(parts[0][0])[1]
        ka = _combine([skmp.mp_keys(a)[0] for a, _ in parts], words)
        kb = _combine([skmp.mp_keys(b)[0] for _, b in parts], words)
        if ref_keys is None:
            ref_keys = (ka.clone(), kb.clone())
        assert torch.equal(ka, ref_keys[0]) and torch.equal(kb, ref_keys[1]), f"{nb} bands: keys differ"
        a, b = parts[0]
        skmp.mp_keys(a)[0].copy_(ka)
        skmp.mp_keys(b)[0].copy_(kb)
        # sharded finalize: row slices into zero-filled profiles, summed (the dist path)
        PA = torch.zeros_like(PA0)
        IA = torch.zeros_like(IA0)
        edges = np.linspace(0, a.n_sub, nb + 1).astype(np.int64)
        for r in range(nb):
            if edges[r + 1] > edges[r]:
                p, i, inert = skmp.mp_finalize_ab(a, b, int(edges[r]), int(edges[r + 1]))
                PA += p
                IA += i
        PB, IB, _ = skmp.mp_finalize_ab(b, a)
        torch.cuda.synchronize()
        assert torch.equal(PA, PA0) and torch.equal(IA, IA0) and torch.equal(PB, PB0) and torch.equal(IB, IB0)
        assert np.array_equal(inert, inert0)
        for a, b in parts:
            a.free()
            b.free()


def test_staged_abjoin_rejects_mixed_workspaces(cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    R = torch.from_numpy(synthgen.mp_series(2, 500, seed=3, kind="mix")).to(cuda, torch.float32)
    a, b = skmp.mp_create_ab(R, 32), skmp.mp_create_ab(R[:, :400].contiguous(), 32)
    s = skmp.mp_create(R, 32)
    with pytest.raises(skmp.SkmpError):
        skmp.mp_join(a)                       # AB workspace through the self-join entry
    with pytest.raises(skmp.SkmpError):
        skmp.mp_finalize(a)
    with pytest.raises(skmp.SkmpError):
        skmp.mp_join_ab(a, s, 0, 10)          # self-join workspace through the AB entry
    with pytest.raises(skmp.SkmpError):
        skmp.mp_join_ab(a, skmp.mp_create_ab(R.double(), 32), 0, 10)   # dtype differs
    with pytest.raises(skmp.SkmpError):
        skmp.mp_finalize_ab(a, b, 5, 3)
    for w in (a, b, s):
        w.free()
