"""GPU parity: sketch_build / sketch_add_dim / sketch_del_dim (K1-K3) through the C-ABI vs the
oracle's Alg. 1 on the same synthgen streams."""
from __future__ import annotations

import numpy as np
import pytest

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch

pytestmark = pytest.mark.gpu


def _terms_bound(T, mu, sigma, groups, signs, k, S=None):
    """sum_j |c_j (T_jt - mu_j)| per (g, t): the FP64 sketch tolerance scale."""
    T = np.asarray(T, dtype=np.float64)
    B = np.zeros((k, T.shape[1]))
    for j in range(T.shape[0]):
        z = np.abs((T[j] - mu[j]) / sigma[j])
        if S is None:
            B[groups[j]] += z
        else:
            B += np.abs(S[:, j])[:, None] * z[None, :]
    return B


def _check_R(R_gpu64, R_gpu, R_or, bound, dtype):
    R_gpu64 = np.asarray(R_gpu64)
    assert np.all(np.abs(R_gpu64 - R_or) <= 1e-12 * bound + 1e-300), \
        f"FP64 sketch off by {np.max(np.abs(R_gpu64 - R_or) / np.maximum(bound, 1e-300)):.3e} x bound"
    if dtype == "f32":
        want = R_or.astype(np.float32)
        got = np.asarray(R_gpu, dtype=np.float32)
        # one rounding of a value within 1e-12 of the oracle's: at most 1 ulp apart
        gap = np.abs(got.astype(np.float64) - want.astype(np.float64))
        assert np.all(gap <= np.spacing(np.abs(want)).astype(np.float64)), "FP32 sketch differs by > 1 ulp"


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_sketch_small_configs(cuda, name):
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS[name]
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    Td = torch.from_numpy(T).to(cuda, tdt)
    if cfg.proj == "dense":
        S = synthgen.dense_S(cfg)
        sk = skmp.sketch_build(Td, ids, cfg.k, proj=skmp.PROJ_DENSE, S=S)
        R_or, mu, sg = ref.sketch(T, cfg.k, S=S)
        bound = _terms_bound(T, mu, sg, None, None, cfg.k, S=S)
    else:
        sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
        g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
        R_or, mu, sg = ref.sketch(T, cfg.k, g, s)
        bound = _terms_bound(T, mu, sg, g, s, cfg.k)
        plan = skmp.sketch_plan(sk)
        assert np.array_equal(plan["groups"], np.array(g)) and np.array_equal(plan["signs"], np.array(s))
    torch.cuda.synchronize()
    plan = skmp.sketch_plan(sk)
    assert np.allclose(plan["mu"], mu, rtol=1e-13, atol=1e-13 * np.abs(T).max())
    assert np.allclose(plan["sigma"], sg, rtol=1e-12)
    _check_R(sk.R64.cpu().numpy(), sk.R.cpu().numpy(), R_or, bound, cfg.dtype)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_sketch_c3_like_and_host_input(cuda, dtype):
    """C3 recipe at reduced d (count sketch, FP32/FP64), device and host (pinned) inputs."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c3"], d=120, n=30011, k=12)
    T = synthgen.streams(cfg)
    ids = synthgen.stream_ids(cfg)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Tn = T.astype(np.float32 if dtype == "f32" else np.float64)
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    R_or, mu, sg = ref.sketch(Tn, cfg.k, g, s)
    bound = _terms_bound(Tn, mu, sg, g, s, cfg.k)
    for src in ("device", "host_pinned", "host_pageable"):
        if src == "device":
            Tin = torch.from_numpy(Tn).to(cuda)
        elif src == "host_pinned":
            Tin = torch.from_numpy(Tn).pin_memory()
        else:
            Tin = torch.from_numpy(Tn)
        sk = skmp.sketch_build(Tin, ids, cfg.k, seed=cfg.seed)
        torch.cuda.synchronize()
        _check_R(sk.R64.cpu().numpy(), sk.R.cpu().numpy(), R_or, bound, "f32" if tdt == torch.float32 else "f64")
        sk.free()


def test_identity_plan_and_fig1(cuda):
    """Identity plan (k = d, s = +1) gives each stream's own z-normalisation; Fig. 1 (k = 1,
    all s = +1) gives the plain sum of z-normalised streams."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS["c1"]
    T = synthgen.streams(cfg)
    d = T.shape[0]
    ids = np.arange(d, dtype=np.uint64)
    Td = torch.from_numpy(T).to(cuda)
    sk = skmp.sketch_build(Td, ids, d, groups=np.arange(d), signs=np.ones(d))
    R = sk.R.cpu().numpy()
    for j in range(d):
        np.testing.assert_allclose(R[j], ref.znormalize(T[j]), rtol=0, atol=1e-13)
    sk1 = skmp.sketch_build(Td, ids, 1, groups=np.zeros(d), signs=np.ones(d))
    want = sum(ref.znormalize(T[j]) for j in range(d))
    np.testing.assert_allclose(sk1.R.cpu().numpy()[0], want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_add_delete_dimensions(cuda, dtype):
    """§3.3: build(A), add(B), delete(C subset of A) == oracle sketch of A+B-C;
    add-then-delete is the identity; add after build == one-shot build of the union."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c4"], d=300, n=8000, k=16)
    tnp = np.float32 if dtype == "f32" else np.float64
    A_ids = np.arange(300, dtype=np.uint64)
    B_ids = np.arange(300, 360, dtype=np.uint64)
    A = synthgen.streams(cfg, A_ids).astype(tnp)
    B = synthgen.streams(cfg, B_ids).astype(tnp)
    del_ids = np.array([3, 50, 51, 120, 299], dtype=np.uint64)
    Ad, Bd = torch.from_numpy(A).to(cuda), torch.from_numpy(B).to(cuda)
    sk = skmp.sketch_build(Ad, A_ids, cfg.k, seed=cfg.seed)
    R0 = sk.R64.clone()
    skmp.sketch_add_dim(sk, Bd, B_ids)
    # add after build == one-shot of the union (appended in input order): bit-identical FP64
    both = skmp.sketch_build(torch.cat([Ad, Bd]), np.concatenate([A_ids, B_ids]), cfg.k, seed=cfg.seed)
    assert torch.equal(sk.R64, both.R64)
    Cd = Ad[del_ids.astype(np.int64)]
    skmp.sketch_del_dim(sk, Cd, del_ids)
    keep = np.array([j for j in range(300) if j not in set(del_ids.tolist())])
    final_T = np.concatenate([A[keep], B])
    final_ids = np.concatenate([A_ids[keep], B_ids])
    g, s = plan_count_sketch(final_ids, cfg.k, cfg.seed)
    R_or, mu, sg = ref.sketch(final_T, cfg.k, g, s)
    bound = _terms_bound(final_T, mu, sg, g, s, cfg.k)
    # incremental order differs from the oracle's one-shot order: a few FP64 roundings
    d64 = np.abs(sk.R64.cpu().numpy() - R_or)
    assert np.all(d64 <= 1e-12 * bound), f"{(d64 / bound).max():.3e}"
    plan = skmp.sketch_plan(sk)
    assert sorted(plan["ids"].tolist()) == sorted(final_ids.tolist())
    # add then delete the same streams -> original within one FP64 rounding per step
    skmp.sketch_add_dim(sk, Cd, del_ids)
    skmp.sketch_del_dim(sk, Cd, del_ids)
    skmp.sketch_del_dim(sk, Bd, B_ids)
    skmp.sketch_add_dim(sk, Cd, del_ids)
    R_back = sk.R64.cpu().numpy()
    bA = _terms_bound(A, *ref.stream_stats(A), *plan_count_sketch(A_ids, cfg.k, cfg.seed), cfg.k)
    assert np.all(np.abs(R_back - R0.cpu().numpy()) <= 1e-12 * bA)


def test_sketch_errors(cuda):
    import torch
    import paper_2311_03393_b200 as skmp
    T = torch.randn((4, 100), device=cuda, dtype=torch.float64)
    T[2] = 3.0
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_build(T, np.arange(4), 2, seed=1)
    assert e.value.name == "SKMP_E_CONSTANT_SERIES" and e.value.index == 2
    T = torch.randn((4, 100), device=cuda, dtype=torch.float32)
    T[1, 17] = float("nan")
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_build(T, np.arange(4), 2, seed=1)
    assert e.value.name == "SKMP_E_NONFINITE" and e.value.index == 1
    T = torch.randn((4, 100), device=cuda, dtype=torch.float32)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_build(T, np.array([0, 1, 1, 2]), 2, seed=1)
    assert e.value.name == "SKMP_E_DUPLICATE_DIM"
    sk = skmp.sketch_build(T, np.arange(4), 2, seed=1)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_add_dim(sk, T[:1], np.array([3]))
    assert e.value.name == "SKMP_E_DUPLICATE_DIM"
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_del_dim(sk, T[:1], np.array([9]))
    assert e.value.name == "SKMP_E_UNKNOWN_DIM"


@pytest.mark.parametrize("dtype,proj", [("f64", "count"), ("f32", "count"), ("f64", "dense")])
def test_point_updates(cuda, dtype, proj):
    """§3.3 point updates (reading 24) vs the oracle's Alg. 1 on the modified data
    with the stored statistics; repeated (id, t) pairs accumulate."""
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=30, n=3000, k=5)
    T = synthgen.streams(cfg)
    ids = np.arange(100, 130, dtype=np.uint64)          # ids need not equal rows
    tdt = torch.float32 if dtype == "f32" else torch.float64
    Td = torch.from_numpy(T).to(cuda, tdt)
    To = Td.double().cpu().numpy()
    S = np.random.default_rng(5).standard_normal((cfg.k, cfg.d)) if proj == "dense" else None
    if proj == "dense":
        sk = skmp.sketch_build(Td, ids, cfg.k, proj=skmp.PROJ_DENSE, S=S)
    else:
        sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    rng = np.random.default_rng(9)
    rows = rng.integers(0, cfg.d, 400)
    ts = rng.integers(0, cfg.n, 400)
    rows[-5:], ts[-5:] = rows[0], ts[0]                  # repeats of one (id, t)
    dl = rng.standard_normal(400) * 3.0
    skmp.sketch_point_update(sk, ids[rows], ts, dl)
    torch.cuda.synchronize()
    T2 = To.copy()
    np.add.at(T2, (rows, ts), dl)
    plan = skmp.sketch_plan(sk)
    if proj == "dense":
        R_or, _, _ = ref.sketch(T2, cfg.k, S=S, stats=(plan["mu"], plan["sigma"]))
        bound = _terms_bound(T2, plan["mu"], plan["sigma"], None, None, cfg.k, S=S)
    else:
        g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
        R_or, _, _ = ref.sketch(T2, cfg.k, g, s, stats=(plan["mu"], plan["sigma"]))
        bound = _terms_bound(T2, plan["mu"], plan["sigma"], g, s, cfg.k)
    _check_R(sk.R64.cpu().numpy(), sk.R.cpu().numpy(), R_or, bound, dtype)
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_point_update(sk, [999], [0], [1.0])
    assert e.value.name == "SKMP_E_UNKNOWN_DIM"
    with pytest.raises(skmp.SkmpError) as e:
        skmp.sketch_point_update(sk, [ids[0]], [cfg.n], [1.0])
    assert e.value.name == "SKMP_E_INVALID_ARG"


def test_sketch_refresh_rerounds_the_master_copy(cuda):
    """sketch_refresh (used after the multi-GPU sum-reduce of the FP64 master sketch) re-rounds R
    from R64; sketch_view64 is a live view of the master."""
    import torch
    import paper_2311_03393_b200 as skmp
    T = torch.from_numpy(np.random.default_rng(4).standard_normal((6, 500)).cumsum(axis=1)).to(cuda, torch.float32)
    sk = skmp.sketch_build(T, np.arange(6, dtype=np.uint64), 3, seed=2)
    R64 = skmp.sketch_view64(sk)
    assert torch.equal(sk.R, R64.float())
    R64 += 0.1234567891
    skmp.sketch_refresh(sk)
    torch.cuda.synchronize()
    assert torch.equal(sk.R, R64.float())
    skmp.sketch_free(sk)
    assert sk.handle is None
