"""Pins of the oracle to things other than itself (CPU only): worked values, closed forms,
library routines (scipy cdist, numpy BLAS / corrcoef), invariants, brute force on tiny inputs,
and the paper's Lemma 1.  A plausible mistake anywhere in oracle/ (dropped term, wrong sign or
index, transposed operand, wrong tie rule) fails at least one of these."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist

import synthgen
from oracle import reference as ref
from oracle.hashplan import cw_params, plan_count_sketch, splitmix64_stream

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold_lines(name):
    return [l.strip() for l in open(os.path.join(GOLD, name)) if l.strip() and not l.startswith("#")]


# ---------------------------------------------------------------------------------- z-norm
def test_znorm_worked_example():
    lines = dict(l.split(":", 1) for l in _gold_lines("znorm_1234.txt"))
    x = np.array([float(v) for v in lines["input"].split()])
    want = np.array([float(v) for v in lines["output"].split()])
    np.testing.assert_allclose(ref.znormalize(x), want, atol=float(lines["tolerance"]))
    np.testing.assert_allclose(ref.znormalize(x), (x - 2.5) / math.sqrt(1.25), atol=1e-15)


def test_znorm_closed_form_and_errors():
    x = np.random.default_rng(1).standard_normal(1000) * 7 + 3
    z = ref.znormalize(x)
    assert abs(z.mean()) < 1e-12 and abs(z.std() - 1) < 1e-12  # population convention
    np.testing.assert_allclose(ref.znormalize(z), z, atol=1e-12)  # idempotent
    with pytest.raises(ref.OracleError) as e:
        ref.stream_stats(np.array([[1.0, 2.0, 3.0], [5.0, 5.0, 5.0]]))
    assert e.value.kind == "constant" and e.value.index == 1
    with pytest.raises(ref.OracleError) as e:
        ref.stream_stats(np.array([[1.0, np.nan, 3.0]]))
    assert e.value.kind == "nonfinite" and e.value.index == 0


# ---------------------------------------------------------------------------------- dist
def test_dist_invariants_and_closed_form():
    rng = np.random.default_rng(2)
    for m in (8, 33, 100):
        a = rng.standard_normal(m)
        b = rng.standard_normal(m)
        assert ref.dist(a, a) == 0.0
        assert ref.dist(a, 3 * a + 5) < 1e-9
        assert abs(ref.dist(a, b) - ref.dist(b, a)) < 1e-12
        assert abs(ref.dist(-a, -b) - ref.dist(a, b)) < 1e-12
        assert abs(ref.dist(2 * a - 1, 0.5 * b + 7) - ref.dist(a, b)) < 1e-9
        rho = np.corrcoef(a, b)[0, 1]                      # library Pearson correlation
        assert abs(ref.dist(a, b) ** 2 - 2 * m * (1 - rho)) < 1e-9 * m
        # flat convention (reading 5)
        assert ref.dist(np.full(m, 2.0), np.full(m, -1.0)) == 0.0
        assert ref.dist(np.full(m, 2.0), b) == math.sqrt(m)


# ---------------------------------------------------------------------------------- self-join
def _cdist_profile(r, m, excl):
    Z, flat = ref.znorm_windows(r, m)
    D = cdist(Z, Z)                                        # library Euclidean distances
    n_sub = Z.shape[0]
    ii = np.arange(n_sub)
    D[np.abs(ii[:, None] - ii[None, :]) <= excl] = np.inf
    return D.min(axis=1), D.argmin(axis=1)


@pytest.mark.parametrize("seed", range(40))
def test_selfjoin_brute_vs_scipy_cdist(seed):
    rng = np.random.default_rng([seed, 11])
    m = [8, 16, 32][seed % 3]
    n = int(rng.integers(3 * m, 300))
    kind = ["mix", "randwalk", "noise", "seasonal"][seed % 4]
    r = synthgen.mp_series(1, n, seed=seed, kind=kind)[0]
    excl = (m + 1) // 2
    P, I, F = ref.selfjoin_brute(r, m, excl)
    Pc, Ic = _cdist_profile(r, m, excl)
    np.testing.assert_allclose(P, Pc, rtol=1e-12, atol=1e-12)
    # identical argmin except where cdist and explicit sums tie within rounding
    diff = np.where(I != Ic)[0]
    for i in diff:
        assert abs(Pc[i] - P[i]) < 1e-12
    assert len(diff) <= 1
    # plain-C brute force agrees with the numpy brute force exactly on the index
    Pr, Ir, Fr = ref.selfjoin_rows(r, m, excl)
    np.testing.assert_allclose(Pr, P, rtol=1e-13, atol=1e-13)
    assert np.array_equal(Ir, I)
    assert np.array_equal(Fr, F)
    # bounds: 0 <= P <= 2 sqrt(m) (triangle inequality with ||z|| = sqrt(m))
    assert P.min() >= 0 and P.max() <= 2 * math.sqrt(m) + 1e-12


def test_selfjoin_consistency_and_motif():
    r = synthgen.mp_series(1, 1200, seed=3, kind="noise")[0]
    m = 40
    r[900:900 + m] = r[100:100 + m]                        # planted exact motif
    P, I, _ = ref.selfjoin_rows(r, m)
    assert I[100] == 900 and I[900] == 100 and P[100] < 1e-6 and P[900] < 1e-6
    rng = np.random.default_rng(4)
    Z, _ = ref.znorm_windows(r, m)
    excl = (m + 1) // 2
    for i in rng.integers(0, len(P), 30):
        assert abs(i - I[i]) > excl
        assert abs(P[i] - ref.dist(r[i:i + m], r[I[i]:I[i] + m])) < 1e-9
        for j in rng.integers(0, len(P), 100):
            if abs(int(i) - int(j)) > excl:
                assert P[i] <= np.sqrt(((Z[i] - Z[j]) ** 2).sum()) + 1e-12


def test_selfjoin_flat_windows_convention():
    """Hand-derived expectations for flat windows (reading 5)."""
    m = 10
    r = synthgen.mp_series(1, 400, seed=5, kind="noise")[0]
    r[50:80] = 4.0          # windows 50..70 flat
    r[300:320] = -1.0       # windows 300..310 flat
    P, I, F = ref.selfjoin_rows(r, m)
    assert F[50] and F[70] and not F[71] and F[305]
    excl = (m + 1) // 2
    assert P[50] == 0.0 and I[50] == 56                   # smallest admissible flat: 50+excl+1
    assert P[300] == 0.0 and I[300] == 50
    assert P[60] == 0.0 and I[60] == 50                   # |60-50| > excl
    assert P[68] == 0.0 and I[68] == 50
    nonflat = [i for i in range(len(P)) if not F[i]]
    assert all(P[i] <= math.sqrt(m) for i in nonflat)     # a flat window is always admissible
    Pb, Ib, _ = ref.selfjoin_brute(r, m)
    np.testing.assert_allclose(Pb, P, atol=1e-12)
    assert np.array_equal(Ib, I)


def test_no_admissible():
    with pytest.raises(ref.OracleError) as e:
        ref.selfjoin_brute(np.arange(20.0) ** 2, 16)
    assert e.value.kind == "no_admissible"


# ---------------------------------------------------------------------------------- sketch
def test_sketch_matches_blas_dense_and_count():
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=30, n=3000, k=5)
    T = synthgen.streams(cfg)
    ids = np.arange(30)
    # dense S: numpy BLAS S @ Z
    S = synthgen.dense_S(cfg)
    R, mu, sg = ref.sketch(T, cfg.k, S=S)
    Z = (T - T.mean(axis=1, keepdims=True)) / T.std(axis=1, keepdims=True)
    bound = np.abs(S) @ np.abs(Z)
    assert np.all(np.abs(R - S @ Z) <= 1e-12 * bound)
    # count sketch as the equivalent sparse +-1 matrix (S_gj = s_j [h_j = g])
    g, s = plan_count_sketch(ids, cfg.k, cfg.seed)
    Sc = np.zeros((cfg.k, 30))
    Sc[g, np.arange(30)] = s
    Rc, _, _ = ref.sketch(T, cfg.k, g, s)
    assert np.all(np.abs(Rc - Sc @ Z) <= 1e-12 * (np.abs(Sc) @ np.abs(Z)))


def test_fig1_sum_and_linearity():
    cfg = synthgen.scaled(synthgen.CONFIGS["c1"], d=5)
    T = synthgen.streams(cfg)
    R, _, _ = ref.sketch(T, 1, [0] * 5, [1] * 5)     # Fig. 1: T_sum of z-normalised dims
    np.testing.assert_allclose(R[0], sum(ref.znormalize(T[j]) for j in range(5)), atol=1e-13)
    g, s = plan_count_sketch(range(5), 3, 99)
    RA, _, _ = ref.sketch(T[:2], 3, g[:2], s[:2])
    RB, _, _ = ref.sketch(T[2:], 3, g[2:], s[2:])
    RAB, _, _ = ref.sketch(T, 3, g, s)
    np.testing.assert_allclose(RAB, RA + RB, atol=1e-12)


def test_identity_plan_is_exact_multidim_discord():
    """k = d, identity plan: each group profile is the exact profile of its stream (Def. 5 via
    d per-dimension MPs); top-1 of C is the exact multidimensional discord."""
    cfg = synthgen.CONFIGS["c1"]
    T = synthgen.streams(cfg)
    d, m = T.shape[0], cfg.m
    o = ref.detect(T, d, m, 1, groups=list(range(d)), signs=[1] * d)
    exact = np.stack([ref.selfjoin_rows(T[j], m)[0] for j in range(d)])  # raw streams, not sketched
    np.testing.assert_allclose(o["P"], exact, rtol=1e-9, atol=1e-9)
    jstar, istar = np.unravel_index(np.argmax(exact), exact.shape)
    assert o["top"][0][0] == istar and o["top"][0][1] == jstar
    # joint negation invariance: flipping every sign leaves the profiles unchanged
    o2 = ref.detect(T, d, m, 1, groups=list(range(d)), signs=[-1] * d)
    np.testing.assert_allclose(o2["P"], o["P"], atol=1e-9)


# ---------------------------------------------------------------------------------- hash
def test_splitmix64_reference_vectors():
    want = [int(v, 16) for v in _gold_lines("splitmix64_seed0.txt")]
    assert splitmix64_stream(0, 3) == want


def test_hash_family_properties():
    a, b, c, e = cw_params(7)
    assert 0 < a < 2**61 - 1 and 0 < c < 2**61 - 1 and 0 <= b < 2**61 - 1 and 0 <= e < 2**61 - 1
    ids = list(range(200))
    assert plan_count_sketch(ids, 10, 5) == plan_count_sketch(ids, 10, 5)      # deterministic
    g5, _ = plan_count_sketch(ids + [10**12], 10, 5)
    assert g5[:200] == plan_count_sketch(ids, 10, 5)[0]                        # keyed by id
    # pairwise collision probability ~ 1/k over random seeds (2-universality)
    k, trials, hits, sflip = 10, 3000, 0, 0
    for sd in range(trials):
        g, s = plan_count_sketch([17, 912], k, 1000 + sd)
        hits += g[0] == g[1]
        sflip += s[0] != s[1]
    se = math.sqrt(trials * (1 / k) * (1 - 1 / k))
    assert abs(hits - trials / k) < 4 * se
    assert abs(sflip - trials / 2) < 4 * math.sqrt(trials / 4)


def test_lemma1_unbiased_estimate():
    """Lemma 1: s(j) R^(h(j))_i is an unbiased estimate of T_bar_{j,i} with variance
    (1/k) sum_{j' != j} T_bar_{j',i}^2; Monte-Carlo over seeds of the hash family."""
    rng = np.random.default_rng(8)
    T = rng.standard_normal((12, 6)) * 3
    Tb = (T - T.mean(1, keepdims=True)) / T.std(1, keepdims=True)
    k, j, i, trials = 4, 3, 2, 4000
    est = []
    for sd in range(trials):
        g, s = plan_count_sketch(range(12), k, 50_000 + sd)
        R, _, _ = ref.sketch(T, k, g, s)
        est.append(s[j] * R[g[j], i])
    est = np.array(est)
    var = (Tb[:, i] ** 2).sum() - Tb[j, i] ** 2
    var /= k
    assert abs(est.mean() - Tb[j, i]) < 4 * math.sqrt(var / trials)
    assert abs(est.var() / var - 1) < 0.2


# ---------------------------------------------------------------------------------- detection
def _topk_sorted(C, G, I, K, radius):
    """Independent reimplementation: sort by (C desc, i asc), accept i unless within radius of an
    accepted discord (equivalent to greedy argmax-and-mask)."""
    order = sorted(range(len(C)), key=lambda i: (-C[i], i))
    acc = []
    for i in order:
        if len(acc) == K:
            break
        if all(abs(i - a) > radius for a in acc):
            acc.append(i)
    return [(i, int(G[i]), int(I[G[i]][i]), float(C[i])) for i in acc]


@pytest.mark.parametrize("seed", range(6))
def test_combine_topk_vs_sorted_reimplementation(seed):
    rng = np.random.default_rng([seed, 9])
    k, n_sub = 5, 400
    P = np.round(rng.uniform(0, 5, (k, n_sub)), 1)          # many exact ties
    I = rng.integers(0, n_sub, (k, n_sub))
    inert = np.zeros(k, dtype=bool)
    inert[seed % k] = True
    C, G = ref.combine(P, inert)
    live = [g for g in range(k) if not inert[g]]
    np.testing.assert_array_equal(C, P[live].max(0))
    for i in range(n_sub):
        assert G[i] == min(g for g in live if P[g, i] == C[i])
    for K, rad in ((1, 3), (12, 7), (200, 20)):
        assert ref.topk_greedy(C, G, I, K, rad) == _topk_sorted(C, G, I, K, rad)
    with pytest.raises(ref.OracleError):
        ref.combine(P, np.ones(k, dtype=bool))


def test_injected_discord_recovery():
    """An injected anomaly is recovered: (a) a clean periodic series with one window replaced by
    noise -> the top-1 discord lies on it; (b) C1's stream 0 (random walk + 3-sigma sine burst at
    t=1200, BASELINE configs[0]) -> the burst is in the greedy top-3 of its exact profile."""
    n, m = 3000, 50
    t = np.arange(n)
    x = np.sin(2 * np.pi * t / 50) + 0.01 * np.random.default_rng(1).standard_normal(n)
    x[1700:1750] = np.random.default_rng(2).standard_normal(50)
    P, I, _ = ref.selfjoin_rows(x, m)
    assert 1700 - m < int(np.argmax(P)) < 1750
    cfg = synthgen.CONFIGS["c1"]
    T = synthgen.streams(cfg)
    P0, I0, _ = ref.selfjoin_rows(T[0], cfg.m)
    top = ref.topk_greedy(P0, np.zeros(len(P0), int), I0[None], 3, cfg.excl)
    assert any(1200 - cfg.m < tt < 1250 for tt, *_ in top), top


# ---------------------------------------------------------------------------------- Alg. 3
def test_dimension_detection_vs_cdist_and_planted():
    """Alg. 3 (self-join mode P:L322): per-stream 1NN distance of window t* pinned to
    scipy cdist; an exactly periodic stream scores 0 (its window repeats one period later); a
    burst planted in one stream of the group makes that stream j*."""
    m, n = 32, 900
    rng = np.random.default_rng(21)
    t = np.arange(n)
    T = np.stack([np.sin(2 * np.pi * t / p) + 0.05 * rng.standard_normal(n) for p in (60, 75, 90, 110)])
    T = np.concatenate([T, np.sin(2 * np.pi * t / 50)[None, :]])   # exact period 50
    t_star = 400
    T[2, t_star:t_star + m] += 3.0 * np.sin(2 * np.pi * np.arange(m) / 7)   # burst in stream 2
    rows = [4, 0, 2, 3, 1]
    excl = (m + 1) // 2
    scores, nn, js = ref.dimension_detection(T, rows, t_star, m, excl)
    for q, j in enumerate(rows):
        Z, _ = ref.znorm_windows(T[j], m)
        D = cdist(Z[t_star][None, :], Z)[0]                     # library Euclidean distances
        D[np.abs(np.arange(len(D)) - t_star) <= excl] = np.inf
        assert abs(scores[q] - D.min()) < 1e-12 and nn[q] == int(np.argmin(D))
    assert scores[0] < 1e-6 and (t_star - nn[0]) % 50 == 0     # an exact repeat, whole periods away
    assert rows[js] == 2                                        # the planted stream
    # Alg. 3's strict '>' in group order: equal scores keep the first member
    T2 = np.stack([T[1], T[1], T[3]])
    s2, _, j2 = ref.dimension_detection(T2, [0, 1, 2], t_star, m, excl)
    assert s2[0] == s2[1]
    assert j2 == (0 if s2[0] >= s2[2] else 2)


def test_refine_is_top1_of_the_stream_profile():
    """Refinement: the top-1 discord of the identified stream's full profile,
    against the cdist profile."""
    r = synthgen.mp_series(1, 700, seed=23, kind="seasonal")[0]
    m = 24
    excl = (m + 1) // 2
    t, nn, score, P, I = ref.refine(r, m, excl)
    Pc, Ic = _cdist_profile(r, m, excl)
    assert t == int(np.argmax(Pc)) and abs(score - Pc.max()) < 1e-12 and nn == Ic[t]


# ---------------------------------------------------------------------------------- AB-join
@pytest.mark.parametrize("seed", range(6))
def test_abjoin_brute_vs_cdist_and_planted(seed):
    """Def. 6 ab-join: pinned to scipy cdist on the two window sets; both
    directions (A against B is the transpose of B against A); a window of A copied into B
    scores 0 at its copy."""
    rng = np.random.default_rng([seed, 31])
    m = [8, 16, 32][seed % 3]
    a = synthgen.mp_series(1, int(rng.integers(3 * m, 260)), seed=seed, kind="mix")[0]
    b = synthgen.mp_series(1, int(rng.integers(3 * m, 260)), seed=seed + 100, kind="randwalk")[0]
    t = int(rng.integers(0, len(a) - m + 1))
    u = int(rng.integers(0, len(b) - m + 1))
    b[u:u + m] = 2.0 * a[t:t + m] - 1.0                    # affine copy: z-normalised identical
    P, I = ref.abjoin_brute(a, b, m)
    Za, _ = ref.znorm_windows(a, m)
    Zb, _ = ref.znorm_windows(b, m)
    D = cdist(Za, Zb)                                       # library Euclidean distances
    np.testing.assert_allclose(P, D.min(axis=1), rtol=1e-12, atol=1e-12)
    for i in np.where(I != D.argmin(axis=1))[0]:
        assert abs(D[i, I[i]] - D[i].min()) < 1e-12
    Pt, It = ref.abjoin_brute(b, a, m)
    np.testing.assert_allclose(Pt, D.min(axis=0), rtol=1e-12, atol=1e-12)
    assert P[t] < 1e-6 and Pt[u] < 1e-6


def test_sketch_with_stored_stats_point_update_closed_form():
    """§3.3 point update under reading 24: the plain Alg. 1 loop on the modified data
    with the STORED statistics moves exactly one entry per update by s(j) delta / sigma_j (dense:
    S_gj delta / sigma_j in every group); with the data's own statistics it equals sketch()."""
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=9, n=400, k=3)
    T = synthgen.streams(cfg)
    g, s = plan_count_sketch(np.arange(cfg.d), cfg.k, cfg.seed)
    R, mu, sig = ref.sketch(T, cfg.k, g, s)
    R2, _, _ = ref.sketch(T, cfg.k, g, s, stats=(mu, sig))
    np.testing.assert_array_equal(R, R2)
    T2 = T.copy()
    T2[4, 123] += 2.5
    T2[7, 5] -= 1.25
    Ru, _, _ = ref.sketch(T2, cfg.k, g, s, stats=(mu, sig))
    want = R.copy()
    want[g[4], 123] += s[4] * 2.5 / sig[4]
    want[g[7], 5] += s[7] * -1.25 / sig[7]
    np.testing.assert_allclose(Ru, want, rtol=0, atol=1e-12 * np.abs(R).max())
    S = np.random.default_rng(3).standard_normal((cfg.k, cfg.d))
    Rd, mu_d, sig_d = ref.sketch(T, cfg.k, S=S)
    Rdu, _, _ = ref.sketch(T2, cfg.k, S=S, stats=(mu_d, sig_d))
    want = Rd.copy()
    want[:, 123] += S[:, 4] * 2.5 / sig_d[4]
    want[:, 5] += S[:, 7] * -1.25 / sig_d[7]
    np.testing.assert_allclose(Rdu, want, rtol=0, atol=1e-12 * np.abs(Rd).max())


@pytest.mark.parametrize("seed", range(6))
def test_tierb_recurrence_matches_brute_force(seed):
    """Tier B: the FP64 diagonal recurrence with exact re-seeds equals the
    explicit-difference brute force to 1e-10 relative, also across re-seed boundaries (a short
    re-seed interval) and for several exclusion radii; indices equal up to exact-rho ties."""
    rng = np.random.default_rng([seed, 41])
    m = [16, 32, 50][seed % 3]
    n = int(rng.integers(600, 1500))
    r = synthgen.mp_series(1, n, seed=400 + seed, kind=["mix", "randwalk", "seasonal"][seed % 3])[0]
    for excl, reseed in (((m + 1) // 2, 65536), ((m + 1) // 2, 37), (0, 100), (3 * m, 1)):
        Pb, Ib, _ = ref.selfjoin_rows(r, m, excl)
        Pt, It = ref.selfjoin_tierb(r, m, excl, reseed=reseed, threads=3)
        np.testing.assert_allclose(Pt, Pb, rtol=1e-10, atol=0)
        Z, _ = ref.znorm_windows(r, m)
        for i in np.where(It != Ib)[0]:
            assert abs(np.sqrt(((Z[i] - Z[It[i]]) ** 2).sum()) - Pb[i]) <= 1e-10 * Pb[i]


def test_streaming_ab_invariants():
    """f4 oracle (reading 25) pinned by what the mathematics fixes: (1) streaming the
    train data itself reproduces the train sketch exactly and every window finds itself (P = 0,
    I = t); (2) with one stream the sketch is an affine map of it, which window z-normalisation
    (Def. 3) removes, so P / I equal the raw streams' AB profile; (3) a planted test-only shape
    is the top discord."""
    rng = np.random.default_rng(5)
    m = 24
    Ttr = np.cumsum(rng.standard_normal((7, 400)), axis=1)
    g = np.array([0, 1, 2, 0, 1, 2, 0])
    s = np.array([1, -1, 1, 1, -1, -1, 1])
    R_tr, _, _ = ref.sketch(Ttr, 3, g, s)
    R_te, P, I = ref.streaming_ab(Ttr, Ttr, 3, g, s, m)
    assert np.array_equal(R_te, R_tr)
    assert np.all(P <= 1e-6) and np.all(I == np.arange(P.shape[1])[None, :])
    # (2) one stream, sign -1: P equals the raw AB profile
    x_tr = np.cumsum(rng.standard_normal(300))
    x_te = np.cumsum(rng.standard_normal(260)) + 40.0
    _, P1, I1 = ref.streaming_ab(x_tr[None], x_te[None], 1, [0], [-1], m)
    Pr, Ir = ref.abjoin_brute(x_te, x_tr, m)
    np.testing.assert_allclose(P1[0], Pr, rtol=1e-9, atol=1e-9)
    assert np.array_equal(I1[0], Ir)
    # (3) a sine burst only in the test data of stream 4 (group 1) is the top discord
    Tte = Ttr[:, 50:350] + 0.01 * rng.standard_normal((7, 300))   # seen behaviour plus noise
    Tte[4, 150:150 + m] += 6.0 * np.sin(np.linspace(0, 4 * np.pi, m))
    _, P3, _ = ref.streaming_ab(Ttr, Tte, 3, g, s, m)
    C, _ = ref.combine(P3, np.zeros(3, bool))
    assert abs(int(np.argmax(C)) - 150) <= m
