"""GPU parity of the streaming extension: test points pushed in
chunks are sketched with the train plan and statistics (reading 25) and every completed window is
AB-joined against the train sketch — checked against the oracle's batch definition
(oracle.reference.streaming_ab) and against the library's own batch mp_abjoin."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch
from tests._parity import TOL, check_topk

pytestmark = pytest.mark.gpu


def _data(n_tr, n_te, d=40, k=6, seed=3):
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], n=n_tr + n_te, d=d, k=k)
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    return cfg, ids, np.ascontiguousarray(T[:, :n_tr]), np.ascontiguousarray(T[:, n_tr:])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("chunks", [[1700], [1, 7, 31, 32, 300, 1329], [5] * 20 + [1600],
                                    [20, 700, 10, 1, 300, 3, 3]])   # carried, tiled, carried again
def test_stream_parity(cuda, dtype, chunks):
    import torch
    import paper_2311_03393_b200 as skmp
    m = 64
    cfg, ids, Ttr, Tte = _data(2500, sum(chunks))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    sk = skmp.sketch_build(torch.from_numpy(Ttr).to(cuda, tdt), ids, cfg.k, seed=cfg.seed)
    st = skmp.Stream(sk, m, capacity=Tte.shape[1] + 10)
    t0 = 0
    for c in chunks:
        blk = torch.from_numpy(np.ascontiguousarray(Tte[:, t0:t0 + c])).to(cuda, tdt)
        st.push(blk)
        t0 += c
        R, P, I, inert = st.view()
        assert R.shape[1] == t0 and P.shape[1] == max(0, t0 - m + 1)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    R_or, P_or, I_or = ref.streaming_ab(Ttr.astype(np.float64) if dtype == "f64" else Ttr.astype(np.float32).astype(np.float64),
                                        Tte.astype(np.float64) if dtype == "f64" else Tte.astype(np.float32).astype(np.float64),
                                        cfg.k, g, s, m)
    R, P, I, inert = st.view()
    Rg = R.double().cpu().numpy()
    scale = np.abs(R_or).max() + 1.0
    assert np.abs(Rg - R_or).max() <= (1e-12 if dtype == "f64" else 1e-6) * scale
    # the profile against the oracle's batch definition on the GPU's own sketches (the sketches
    # are compared above; the join tolerance is the north-star's)
    Rtr = sk.R.double().cpu().numpy()
    Pg, Ig = P.double().cpu().numpy(), I.cpu().numpy()
    floor = 1e-3 * math.sqrt(m)
    for q in range(cfg.k):
        Po, Io = ref.abjoin_brute(Rg[q], Rtr[q], m)
        err = np.abs(Pg[q] - Po) / np.maximum(Po, floor)
        assert err.max() <= TOL[dtype], f"group {q}: rel err {err.max():.3e}"
        Za, _ = ref.znorm_windows(Rg[q], m)
        Zb, _ = ref.znorm_windows(Rtr[q], m)
        for i in np.where(Ig[q] != Io)[0]:
            dj = float(np.sqrt(((Za[i] - Zb[Ig[q, i]]) ** 2).sum()))
            assert dj <= Po[i] + TOL[dtype] * max(Po[i], floor)
    # and the oracle's own end-to-end values (its own sketches)
    err = np.abs(Pg - P_or) / np.maximum(P_or, floor)
    print(f"stream {dtype} {chunks[:4]}: end-to-end max rel err vs the oracle's own sketches {err.max():.2e}")
    assert err.max() <= TOL[dtype]
    assert not inert.any()
    # Alg. 2's ranking over the streamed profile
    top = st.topk(5)
    C, G = ref.combine(Pg, np.zeros(cfg.k, bool))
    want = ref.topk_greedy(C, G, Ig, 5, (m + 1) // 2)
    check_topk(top, want, C, TOL[dtype], label="stream top-K")
    st.free()


def test_stream_matches_batch_abjoin_and_host_input(cuda):
    """One big push from HOST memory (> kStreamIncrMax windows: the tiled AB-join) equals the
    batch mp_abjoin of the final test sketch bit for bit; 25-point device pushes (the carried
    FP64 path) give the same sketch columns and profiles within tolerance."""
    import torch
    import paper_2311_03393_b200 as skmp
    m = 100
    cfg, ids, Ttr, Tte = _data(6000, 5000, d=60, k=8, seed=4)
    Ttr32, Tte32 = Ttr.astype(np.float32), np.ascontiguousarray(Tte.astype(np.float32))
    sk = skmp.sketch_build(torch.from_numpy(Ttr32).to(cuda), ids, cfg.k, seed=cfg.seed)
    a = skmp.Stream(sk, m, capacity=5000)
    a.push(Tte32)                                     # host numpy input: staged by the library
    b = skmp.Stream(sk, m, capacity=5000)
    for t0 in range(0, 5000, 25):
        b.push(torch.from_numpy(Tte32[:, t0:t0 + 25].copy()).to(cuda))
    Ra, Pa, Ia, _ = a.view()
    Rb, Pb, Ib, _ = b.view()
    assert torch.equal(Ra, Rb)
    PA, IA, _ = skmp.mp_abjoin(Ra.contiguous(), sk.R, m)
    assert torch.equal(Pa, PA) and torch.equal(Ia, IA)   # same block -> same arithmetic
    floor = 1e-3 * math.sqrt(m)
    err = ((Pb.double() - PA.double()).abs() / PA.double().clamp_min(floor)).max().item()
    assert err <= TOL["f32"]
    # where the carried path picked another neighbour it is a tie within tolerance
    Rte, Rtr = Ra.double().cpu().numpy(), sk.R.double().cpu().numpy()
    diff = (Ib != IA).nonzero().cpu().numpy()
    for g, i in diff[:200]:
        Za, _ = ref.znorm_windows(Rte[g], m)
        Zb, _ = ref.znorm_windows(Rtr[g], m)
        d = float(np.sqrt(((Za[i] - Zb[int(Ib[g, i])]) ** 2).sum()))
        assert abs(d - float(PA[g, i])) <= TOL["f32"] * max(float(PA[g, i]), floor)
    a.free()
    b.free()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_stream_carried_long_run(cuda, dtype):
    """Many 1..3-point pushes across the carried path's exact re-seed grid (kStreamReseed = 8192
    rows): every profile value stays within tolerance of the batch AB-join of the same sketch."""
    import torch
    import paper_2311_03393_b200 as skmp
    m = 64
    cfg, ids, Ttr, Tte = _data(1500, 9000, d=12, k=2, seed=6)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    sk = skmp.sketch_build(torch.from_numpy(Ttr).to(cuda, tdt), ids, cfg.k, seed=cfg.seed)
    st = skmp.Stream(sk, m, capacity=9000)
    Td = torch.from_numpy(Tte).to(cuda, tdt)
    t0, step = 0, 0
    while t0 < 9000:
        c = min(9000 - t0, 1 + step % 3)
        st.push(Td[:, t0:t0 + c].contiguous())
        t0 += c
        step += 1
    R, P, I, _ = st.view()
    PA, IA, _ = skmp.mp_abjoin(R.contiguous(), sk.R, m)
    floor = 1e-3 * math.sqrt(m)
    err = ((P.double() - PA.double()).abs() / PA.double().clamp_min(floor)).max().item()
    assert err <= TOL[dtype] * (1 if dtype == "f64" else 1), err
    st.free()


def test_stream_self_and_errors(cuda):
    """Streaming the train data itself: every window finds itself (P ~ 0, I = t); capacity and
    argument errors are reported before any device work."""
    import torch
    import paper_2311_03393_b200 as skmp
    m = 32
    cfg, ids, Ttr, _ = _data(1500, 10, d=20, k=4)
    Td = torch.from_numpy(Ttr).to(cuda, torch.float64)
    sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    st = skmp.Stream(sk, m, capacity=1500)
    st.push(Td[:, :700].contiguous())
    st.push(Td[:, 700:].contiguous())
    R, P, I, _ = st.view()
    assert torch.equal(R, sk.R)
    assert P.max().item() <= 1e-6 * math.sqrt(m)
    assert torch.equal(I, torch.arange(P.shape[1], device=cuda).expand_as(I))
    with pytest.raises(skmp.SkmpError):
        st.push(Td[:, :1].contiguous())                  # capacity exceeded
    with pytest.raises(skmp.SkmpError):
        skmp.Stream(sk, m, capacity=m - 1)
    st.free()
    # a NaN among new points is rejected and the stream stays usable
    st = skmp.Stream(sk, m, capacity=200)
    st.push(Td[:, :80].contiguous())
    bad = Td[:, 80:90].clone()
    bad[3, 4] = float("nan")
    with pytest.raises(skmp.SkmpError) as e:
        st.push(bad)
    assert e.value.name == "SKMP_E_NONFINITE"
    st.push(Td[:, 80:90].contiguous())
    R, P, I, _ = st.view()
    assert R.shape[1] == 90 and torch.equal(R, sk.R[:, :90]) and P.max().item() <= 1e-6 * math.sqrt(m)
    st.free()


def test_prefetcher_overlap_results_identical(cuda):
    """pipeline.Prefetcher: a batch sketched from pinned host memory on the prefetch stream while
    the previous batch's join runs gives the same sketch and profile as the plain sequence."""
    import torch
    import paper_2311_03393_b200 as skmp
    from paper_2311_03393_b200.pipeline import Prefetcher
    cfg, ids, T1, T2 = _data(4000, 4000, d=30, k=4)
    h1 = torch.from_numpy(T1.astype(np.float32)).pin_memory()
    h2 = torch.from_numpy(T2.astype(np.float32)).pin_memory()
    m = 50
    stage = lambda T: skmp.sketch_build(T, ids, cfg.k, seed=cfg.seed)  # noqa: E731
    pf = Prefetcher(cuda)
    sk1 = pf.run(stage, h1)
    pf.handoff()
    w = skmp.mp_create(sk1.R, m)
    skmp.mp_join(w)
    sk2 = pf.run(stage, h2)             # overlaps the join above
    P1, I1, _ = skmp.mp_finalize(w)
    pf.handoff()
    P2, I2, _ = skmp.mp_selfjoin(sk2.R, m)
    torch.cuda.synchronize()
    for T, sk, P, I in ((h1, sk1, P1, I1), (h2, sk2, P2, I2)):
        ref_sk = skmp.sketch_build(T.to(cuda), ids, cfg.k, seed=cfg.seed)
        assert torch.equal(ref_sk.R, sk.R)
        Pr, Ir, _ = skmp.mp_selfjoin(ref_sk.R, m)
        assert torch.equal(Pr, P) and torch.equal(Ir, I)
    w.free()
