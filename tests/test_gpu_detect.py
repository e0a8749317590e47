"""GPU parity: discord_topk (K8) and the end-to-end pipeline sketch -> self-join -> combine ->
top-K against the oracle's own pipeline (its own sketch) on the same synthgen streams."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch
from tests._parity import TOL, check_profile, check_topk

pytestmark = pytest.mark.gpu


def _profiles(k, n_sub, seed, ties=True):
    rng = np.random.default_rng([seed, 0x70B])
    P = rng.uniform(0.5, 6.0, size=(k, n_sub))
    if ties:  # exact ties across groups and within a group
        a = n_sub // 3
        P[1, a:a + 10] = P[0, a:a + 10]
        P[:, n_sub // 2] = 9.0
        P[0, n_sub // 5] = P[0, (4 * n_sub) // 5] = 9.0
    I = rng.integers(0, n_sub, size=(k, n_sub))
    return P, I


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("k,n_sub,top,radius", [(4, 2000, 10, 25), (3, 257, 40, 30), (16, 50000, 25, 64)])
def test_discord_topk_parity(cuda, dtype, k, n_sub, top, radius):
    import torch
    import paper_2311_03393_b200 as skmp
    P, I = _profiles(k, n_sub, n_sub + k)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Pt = torch.from_numpy(P).to(cuda, tdt)
    Pn = Pt.double().cpu().numpy()
    It = torch.from_numpy(I).to(cuda)
    inert = np.zeros(k, dtype=bool)
    inert[k - 1] = True
    got = skmp.discord_topk(Pt, It, inert, m=2 * radius, top=top, radius=radius)
    C, G = ref.combine(Pn, inert)
    want = ref.topk_greedy(C, G, I, top, radius)
    assert [(d.t, d.g, d.nn) for d in got] == [(t, g, nn) for t, g, nn, _ in want]
    assert [d.score for d in got] == [s for *_, s in want]


@pytest.mark.parametrize("dtype,k,n_sub,top,radius", [
    ("f32", 64, 2_000_000, 64, 128),     # > 296 CTAs x 256 windows: the grid-stride argmax path
    ("f32", 32, 1_999_745, 100, 128),    # C5's shape and bench.py's top-100
    ("f64", 16, 1_000_003, 40, 77),      # ragged, odd radius
])
def test_discord_topk_parity_grid_stride(cuda, dtype, k, n_sub, top, radius):
    """discord_topk above 296 x 256 = 75,776 windows (detect.cu's capped grid walks the profile
    with a grid stride) against the oracle's combine + greedy top-K (Alg. 2; the
    ordered list of P:L445), with exact ties across groups, within a group and at the maxima."""
    import torch
    import paper_2311_03393_b200 as skmp
    rng = np.random.default_rng([n_sub, k, 0x70B])
    P = rng.uniform(0.5, 6.0, size=(k, n_sub)).astype(np.float32 if dtype == "f32" else np.float64)
    # exact ties at the top: plateaus of equal maxima far apart, across groups, and repeated
    # values inside one mask radius (the smallest index must win every time)
    for q, t in enumerate(rng.choice(n_sub, size=3 * top, replace=False)):
        P[q % k, t] = 7.0 + (q % 5) * 0.25
    P[:, n_sub // 2] = 9.0
    P[3, n_sub - 1] = 9.0
    P[5, 0] = 9.0
    I = rng.integers(0, n_sub, size=(k, n_sub))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Pt = torch.from_numpy(P).to(cuda, tdt)
    It = torch.from_numpy(I).to(cuda)
    inert = np.zeros(k, dtype=bool)
    inert[1] = True
    got = skmp.discord_topk(Pt, It, inert, m=2 * radius, top=top, radius=radius)
    C, G = ref.combine(P.astype(np.float64), inert)
    want = ref.topk_greedy(C, G, I, top, radius)
    assert len(got) == len(want) == top
    assert [(d.t, d.g, d.nn) for d in got] == [(t, g, nn) for t, g, nn, _ in want]
    assert [d.score for d in got] == [s for *_, s in want]


def test_discord_topk_all_inert(cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    P = torch.zeros((2, 100), device=cuda, dtype=torch.float64)
    I = torch.zeros((2, 100), device=cuda, dtype=torch.int64)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.discord_topk(P, I, np.ones(2, dtype=bool), m=10, top=3)
    assert e.value.name == "SKMP_E_ALL_GROUPS_INERT"


def _gpu_pipeline(cfg, T, ids, top, cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    Td = torch.from_numpy(T).to(cuda, tdt)
    if cfg.proj == "dense":
        sk = skmp.sketch_build(Td, ids, cfg.k, proj=skmp.PROJ_DENSE, S=synthgen.dense_S(cfg))
    else:
        sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    P, I, inert = skmp.mp_selfjoin(sk.R, cfg.m)
    top_gpu = skmp.discord_topk(P, I, inert, m=cfg.m, top=top)
    return sk, P.cpu().numpy(), I.cpu().numpy(), inert, top_gpu


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_end_to_end_small_configs(cuda, name):
    """C1 (dense Gaussian S, FP64) and C2 (count sketch, FP64) in full: the oracle runs its own
    sketch and brute-force joins; profiles and top-K must agree."""
    cfg = synthgen.CONFIGS[name]
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    top = 2 * cfg.n_discords + 2
    sk, P, I, inert, top_gpu = _gpu_pipeline(cfg, T, ids, top, cuda)
    if cfg.proj == "dense":
        o = ref.detect(T, cfg.k, cfg.m, top, S=synthgen.dense_S(cfg))
    else:
        g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
        o = ref.detect(T, cfg.k, cfg.m, top, groups=g, signs=s)
    excl = cfg.excl
    for gi in range(cfg.k):
        check_profile(o["R"][gi], cfg.m, excl, P[gi], I[gi], o["P"][gi], o["I"][gi], o["flat"][gi],
                      TOL[cfg.dtype], label=f"{name} g={gi}")
    assert np.array_equal(inert, o["inert"])
    check_topk(top_gpu, o["top"], o["C"], TOL[cfg.dtype], label=name)


def test_end_to_end_c3_scaled(cuda):
    """C3 recipe (AR(1) + daily period, level shifts/spikes, FP32 count sketch) at reduced n."""
    cfg = synthgen.scaled(synthgen.CONFIGS["c3"], d=200, n=6000, k=8)
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    sk, P, I, inert, top_gpu = _gpu_pipeline(cfg, T, ids, 12, cuda)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    o = ref.detect(T.astype(np.float64), cfg.k, cfg.m, 12, groups=g, signs=s)
    for gi in range(cfg.k):
        check_profile(o["R"][gi], cfg.m, cfg.excl, P[gi], I[gi], o["P"][gi], o["I"][gi], o["flat"][gi],
                      TOL["f32"], label=f"c3s g={gi}")
    check_topk(top_gpu, o["top"], o["C"], TOL["f32"], label="c3s")


def test_c1_injected_discord_recovery_reported(cuda):
    """Reported, not asserted beyond the oracle pin: where the sketched top-3 lands vs the burst."""
    cfg = synthgen.CONFIGS["c1"]
    T = synthgen.streams(cfg)
    _, _, _, _, top_gpu = _gpu_pipeline(cfg, T, synthgen.stream_ids(cfg), 3, cuda)
    hits = [d.t for d in top_gpu if 1200 - cfg.m < d.t < 1250]
    print(f"C1 sketched top-3 {[d.t for d in top_gpu]}; burst hits {hits}")
