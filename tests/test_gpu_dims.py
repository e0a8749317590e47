"""GPU parity: discord_dims (K9, Alg. 3 Dimension-Detection in self-join mode, P:L272-292 and
P:L322) and the refinement join through the C-ABI vs the oracle on the same
synthgen streams."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch
from tests._parity import TOL, check_profile

pytestmark = pytest.mark.gpu


def _check_dims(T, rows, t_star, m, excl, got, tol, label=""):
    sc, nn, js = got
    so, no, jo = ref.dimension_detection(T, rows, t_star, m, excl)
    floor = 1e-3 * math.sqrt(m)
    err = np.abs(sc - so) / np.maximum(so, floor)
    assert err.max() <= tol, f"{label}: score rel err {err.max():.3e}"
    for q in np.where(nn != no)[0]:  # documented tie: the GPU neighbour is as near
        Z, fl = ref.znorm_windows(T[rows[q]], m)
        j = int(nn[q])
        assert abs(j - t_star) > excl
        dj = 0.0 if (fl[j] and fl[t_star]) else (math.sqrt(m) if (fl[j] or fl[t_star]) else
                                                  float(np.sqrt(((Z[j] - Z[t_star]) ** 2).sum())))
        assert dj <= so[q] + tol * max(so[q], floor), f"{label}: row {rows[q]} nn {j} vs {no[q]}"
    if js != jo:
        assert abs(so[js] - so[jo]) <= tol * max(so[jo], floor), f"{label}: j* {js} vs {jo}"


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,m,t_star", [(2000, 50, 1200), (3001, 33, 0), (1500, 64, 1500 - 64), (700, 7, 350)])
def test_discord_dims_parity(cuda, dtype, n, m, t_star):
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c1"], d=12, n=n)
    T = synthgen.streams(cfg)
    T[5, t_star:t_star + m] += 3.0 * T[5].std() * np.sin(2 * np.pi * np.arange(m) / 10)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Td = torch.from_numpy(T).to(cuda, tdt)
    To = Td.double().cpu().numpy()  # the exact values both sides see
    rows = [7, 5, 0, 11, 3]
    excl = (m + 1) // 2
    got = skmp.discord_dims(Td, rows, t_star, m)
    _check_dims(To, rows, t_star, m, excl, got, TOL["f64"], label=f"{dtype} n={n} m={m}")
    # host input (staged by the library) gives the identical answer
    got_h = skmp.discord_dims(np.ascontiguousarray(Td.cpu().numpy()), rows, t_star, m)
    assert np.array_equal(got_h[0], got[0]) and np.array_equal(got_h[1], got[1]) and got_h[2] == got[2]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_discord_dims_flat_and_exclusion(cuda, dtype):
    import torch
    import paper_2311_03393_b200 as skmp
    m = 20
    T = synthgen.mp_series(4, 1200, seed=41, kind="mix")
    T[0, 300:360] = 2.0            # flat windows around t* = 310 in stream 0
    T[1, 800:850] = -1.0           # flat windows elsewhere in stream 1
    T[2, 290:350] = 0.5            # flat at t* in stream 2, and ...
    T[2, 900:950] = 0.5            # ... an admissible flat partner
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Td = torch.from_numpy(T).to(cuda, tdt)
    To = Td.double().cpu().numpy()
    for excl in (-1, 0, 100):
        e = (m + 1) // 2 if excl < 0 else excl
        for t_star in (310, 5, 1180):
            got = skmp.discord_dims(Td, [0, 1, 2, 3], t_star, m, excl=excl)
            _check_dims(To, [0, 1, 2, 3], t_star, m, e, got, TOL["f64"], label=f"flat excl={excl} t*={t_star}")
    sc, nn, _ = skmp.discord_dims(Td, [2], 310, m)
    assert sc[0] == 0.0 and nn[0] == 290  # flat-flat = 0, smallest admissible flat partner (same run)
    sc, nn, _ = skmp.discord_dims(Td, [2], 310, m, excl=100)
    assert sc[0] == 0.0 and nn[0] == 900  # the run's own windows now inside the exclusion zone


def test_discord_dims_errors(cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    T = torch.randn((3, 100), device=cuda, dtype=torch.float64)
    for args, name in (((T, [0], 100 - 16 + 1, 16), "SKMP_E_INVALID_ARG"),
                       ((T, [0], -1, 16), "SKMP_E_INVALID_ARG"),
                       ((T, [-1], 0, 16), "SKMP_E_INVALID_ARG"),
                       ((T, [0], 40, 16, 60), "SKMP_E_NO_ADMISSIBLE")):
        with pytest.raises(skmp.SkmpError) as e:
            skmp.discord_dims(*args)
        assert e.value.name == name, args


def test_discord_dims_c3_size_sampled(cuda):
    """BASELINE C3 lengths (n = 1e5, m = 128, FP32) for 6 streams of one group."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS["c3"]
    ids = np.arange(6)
    T = synthgen.streams(cfg, ids)
    Td = torch.from_numpy(T).to(cuda, torch.float32)
    To = Td.double().cpu().numpy()
    t_star = int(synthgen.injections(cfg)[0].t)
    rows = list(range(6))
    got = skmp.discord_dims(Td, rows, t_star, cfg.m)
    _check_dims(To, rows, t_star, cfg.m, cfg.excl, got, TOL["f64"], label="c3")


def test_alg2_alg3_refine_end_to_end_c2(cuda):
    """C2 (count sketch, FP64): Alg. 2 top-1 (t*, g*) -> Alg. 3 over J_{g*} -> refinement join of
    stream j* (P:L303-304), against the oracle's own pipeline."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS["c2"]
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    Td = torch.from_numpy(T).to(cuda, torch.float64)
    sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    P, I, inert = skmp.mp_selfjoin(sk.R, cfg.m)
    top = skmp.discord_topk(P, I, inert, m=cfg.m, top=1)[0]
    rows = skmp.group_rows(sk, top.g)
    sc, nn, js = skmp.discord_dims(Td, rows, top.t, cfg.m)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    o = ref.detect(T, cfg.k, cfg.m, 1, groups=g, signs=s)
    t_o, g_o = o["top"][0][0], o["top"][0][1]
    assert (top.t, top.g) == (t_o, g_o)
    rows_o = [j for j in range(cfg.d) if g[j] == g_o]
    assert list(rows) == rows_o
    _check_dims(T, rows_o, t_o, cfg.m, cfg.excl, (sc, nn, js), TOL["f64"], label="c2 alg3")
    jstar = rows[js]
    # refinement: full self-join of stream j*
    Pj, Ij, _ = skmp.mp_selfjoin(Td[jstar:jstar + 1], cfg.m)
    t_r, nn_r, s_r, Po, Io = ref.refine(T[jstar], cfg.m, cfg.excl)
    check_profile(T[jstar], cfg.m, cfg.excl, Pj.cpu().numpy()[0], Ij.cpu().numpy()[0], Po, Io,
                  ref.window_stats(T[jstar], cfg.m)[2], TOL["f64"], label="c2 refine")
    assert int(torch.argmax(Pj[0])) == t_r
    print(f"C2: Alg. 2 (t*={top.t}, g*={top.g}), Alg. 3 j*={jstar} (score {sc[js]:.4f}), "
          f"refined discord t={t_r} score {s_r:.4f}")


def test_detect_dimension_after_add_delete(cuda):
    """Alg. 3 over a group whose members come from two device matrices (original streams with
    some deleted, plus added streams), as bench.py calls it, against the oracle on the final
    member set in plan order."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c4"], d=60, n=3000, k=4, m=64)
    ids = np.arange(60, dtype=np.uint64)
    add = np.arange(60, 72, dtype=np.uint64)
    dele = np.array([3, 7, 22, 41], dtype=np.uint64)
    T = synthgen.streams(cfg, ids)
    Ta = synthgen.streams(cfg, add)
    Td = torch.from_numpy(T).to(cuda, torch.float64)
    Tad = torch.from_numpy(Ta).to(cuda, torch.float64)
    sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    skmp.sketch_add_dim(sk, Tad, add)
    skmp.sketch_del_dim(sk, Td[dele.astype(np.int64)].contiguous(), dele)
    t_star, g = 1234, 2
    got = skmp.detect_dimension(sk, [(Td, ids), (Tad, add)], t_star, g, cfg.m)
    plan = skmp.sketch_plan(sk)
    members = [int(j) for j, gg in zip(plan["ids"], plan["groups"]) if gg == g]
    allT = {int(j): T[q] for q, j in enumerate(ids)}
    allT.update({int(j): Ta[q] for q, j in enumerate(add)})
    M = np.stack([allT[j] for j in members])
    sc, nn, js = ref.dimension_detection(M, list(range(len(members))), t_star, cfg.m)
    assert got[0] == members[js] and abs(got[1] - sc[js]) <= 1e-9 * sc[js] and got[2] == nn[js]
    assert all(j not in members for j in dele.tolist())


def test_detect_report_matches_oracle_pipeline(cuda):
    """skmp.detect (Alg. 1 -> Alg. 2 -> Alg. 3 -> refinement, single-series mode
    P:L322) on C2 against the oracle's pipeline."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS["c2"]
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    rep = skmp.detect(torch.from_numpy(T).to(cuda), ids, cfg.k, cfg.m, seed=cfg.seed)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    o = ref.detect(T, cfg.k, cfg.m, 1, groups=g, signs=s)
    t_o, g_o, _, c_o = o["top"][0]
    assert (rep.t, rep.g) == (t_o, g_o) and abs(rep.score - c_o) <= 1e-9 * c_o
    rows = [q for q in range(cfg.d) if g[q] == g_o]
    so, no, jo = ref.dimension_detection(T, rows, t_o, cfg.m)
    assert rep.j_id == int(ids[rows[jo]]) and abs(rep.j_score - so[jo]) <= 1e-9 * so[jo]
    t_r, _, s_r, _, _ = ref.refine(T[rows[jo]], cfg.m)
    assert rep.refined_t == t_r and abs(rep.refined_score - s_r) <= 1e-9 * s_r
    assert set(rep.ms) == {"sketch", "time_detection", "dimension_detection", "refine"}
