"""Oracle: the method step by step, by the plain definitions, in FP64 (numpy).

Test infrastructure only (see oracle/__init__.py).  Each function cites the passage it
follows.  Where the paper is silent the reading taken is SURVEY §8(c)'s, listed in
DESIGN.md §3 (numbered "reading N" below).  No recurrence, no blocking beyond row chunks
of an explicit double loop, no shared code with the CUDA path.

Function pins (tests/test_oracle_pins.py):
  stream_stats / znormalize  -> SPEC worked example [1,2,3,4], mean 0 / std 1 closed form
  sketch                     -> numpy BLAS S @ Z; Fig. 1 toy (k=1, s=+1 gives the plain sum);
                                linearity over disjoint stream sets
  window_stats/znorm_windows -> per-window closed form mean 0 / norm sqrt(m)
  dist                       -> affine invariance, symmetry, joint negation, dist^2 = 2m(1-rho)
  selfjoin_brute             -> scipy.spatial.distance.cdist on the same z-windows;
                                planted motif -> 0; bounds 0 <= P <= 2 sqrt(m)
  selfjoin_rows (C)          -> selfjoin_brute on tiny inputs
  selfjoin_tierb (C, tier B) -> selfjoin_brute to 1e-10 relative (incl. re-seed boundaries)
  combine / topk_greedy      -> an independent sort-then-scan reimplementation
  detect (identity plan)     -> per-stream exact profiles of Def. 5
  dimension_detection        -> scipy cdist distance profile; exact repeat (periodic stream)
                                -> score 0; planted single-stream burst -> j* on it
  sketch(stats=...)          -> own statistics reproduce sketch(); a point change of one sample
                                moves one sketch entry by s(j) delta / sigma_j (closed form)
  abjoin_brute               -> scipy cdist between the two window sets (rows and columns);
                                a window copied into the other series -> 0 at its copy
"""
from __future__ import annotations

import math

import numpy as np

FLAT_EPS = 1e-12  # reading 4/5: sigma <= 1e-12 (max|x| + 1) is "constant"/"flat"


class OracleError(Exception):
    def __init__(self, kind: str, index: int = -1):
        super().__init__(f"{kind} (index {index})")
        self.kind = kind
        self.index = index


# ------------------------------------------------------------------------------------------
# a2: whole-stream z-normalisation statistics (§1, §3.1; reading 3: each
# stream's own statistics, population sigma S:L56, L90)
# ------------------------------------------------------------------------------------------

def stream_stats(T: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Two-pass FP64 mean and population standard deviation of every row of T (d x n)."""
    T = np.asarray(T, dtype=np.float64)
    d, n = T.shape
    mu = np.empty(d)
    sigma = np.empty(d)
    for j in range(d):
        x = T[j]
        if not np.all(np.isfinite(x)):
            raise OracleError("nonfinite", j)
        mu[j] = x.sum() / n
        sigma[j] = math.sqrt(((x - mu[j]) ** 2).sum() / n)
        if sigma[j] <= FLAT_EPS * (np.abs(x).max() + 1.0):
            raise OracleError("constant", j)
    return mu, sigma


def znormalize(x: np.ndarray) -> np.ndarray:
    """T_bar = (T - mu) / sigma for one stream (P:L210 'z-normalized multidimensional time series')."""
    mu, sigma = stream_stats(np.asarray(x, dtype=np.float64)[None, :])
    return (np.asarray(x, dtype=np.float64) - mu[0]) / sigma[0]


# ------------------------------------------------------------------------------------------
# a3/a4: Alg. 1: R^(g) = sum_{j in J_g} s(j) T_bar^(j), J_g = {j : h(j) = g}
# ------------------------------------------------------------------------------------------

def sketch(T: np.ndarray, k: int, groups=None, signs=None, S: np.ndarray | None = None, stats=None):
    """Returns (R (k x n, FP64), mu, sigma).  Count sketch when `groups`/`signs` are given
    (one entry per row of T, in input order); dense projection R = S T_bar when S (k x d) is
    given (reading 1).  Sums run sequentially over j in ascending input order, exactly as the
    loop of Alg. 1 lines 3-5.  `stats` = (mu, sigma) z-normalises with given (stored)
    statistics instead of the data's own (§3.3 point updates, reading 24)."""
    T = np.asarray(T, dtype=np.float64)
    d, n = T.shape
    mu, sigma = stream_stats(T) if stats is None else (np.asarray(stats[0], float), np.asarray(stats[1], float))
    R = np.zeros((k, n))
    for j in range(d):                      # Alg. 1 line 3: for j in [0, ..., d-1]
        z = (T[j] - mu[j]) / sigma[j]       # T_bar^(j)
        if S is None:
            g = int(groups[j])              # line 4: i = h(j)
            R[g] = R[g] + float(signs[j]) * z   # line 5: R^(i) = R^(i) + s(j) T^(j)
        else:
            for g in range(k):
                R[g] = R[g] + float(S[g, j]) * z
    return R, mu, sigma


# ------------------------------------------------------------------------------------------
# a6: subsequences and their z-normalisation (Defs. 2-3); reading 5: a window
# with sigma <= 1e-12 (max|R_g| + 1) is flat and z-normalises to the zero vector
# ------------------------------------------------------------------------------------------

def window_stats(r: np.ndarray, m: int):
    """Direct two-pass mean / population std of every length-m window T_{i,m} of r."""
    r = np.asarray(r, dtype=np.float64)
    n_sub = r.shape[0] - m + 1
    W = np.lib.stride_tricks.sliding_window_view(r, m)      # n_sub x m view
    mu = W.sum(axis=1) / m
    sig = np.sqrt(((W - mu[:, None]) ** 2).sum(axis=1) / m)
    flat = sig <= FLAT_EPS * (np.abs(r).max() + 1.0)
    assert mu.shape[0] == n_sub
    return mu, sig, flat


def znorm_windows(r: np.ndarray, m: int):
    """Matrix of z-normalised windows z_hat_i = (T_{i,m} - mu_i) / sigma_i (zero if flat)."""
    mu, sig, flat = window_stats(r, m)
    W = np.lib.stride_tricks.sliding_window_view(np.asarray(r, dtype=np.float64), m)
    Z = np.zeros(W.shape)
    ok = ~flat
    Z[ok] = (W[ok] - mu[ok, None]) / sig[ok, None]
    return Z, flat


def dist(a: np.ndarray, b: np.ndarray) -> float:
    """z-normalised Euclidean distance of two equal-length windows (Def. 3), with the
    flat-window convention of reading 5 (flat-flat 0, flat vs non-flat sqrt(m))."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m = a.shape[0]
    za, fa = znorm_windows(a, m)
    zb, fb = znorm_windows(b, m)
    # a single window: the flat threshold is relative to that window's own max|x|
    if fa[0] and fb[0]:
        return 0.0
    if fa[0] or fb[0]:
        return math.sqrt(m)
    return float(math.sqrt(((za[0] - zb[0]) ** 2).sum()))


def selfjoin_brute(r: np.ndarray, m: int, excl: int | None = None, rows=None):
    """Self-join matrix profile (Def. 6; self-join variant P:L322) by explicit
    differences of z-normalised windows: P[i] = min_{j : |i-j| > excl} ||z_i - z_j||_2 and
    I[i] = the smallest such argmin (reading 8).  excl defaults to ceil(m/2) (reading 7).
    O(n_sub^2 m): small inputs only.  Returns (P, I, flat)."""
    r = np.asarray(r, dtype=np.float64)
    excl = (m + 1) // 2 if excl is None else excl
    Z, flat = znorm_windows(r, m)
    n_sub = Z.shape[0]
    if n_sub < 2 * excl + 2:
        raise OracleError("no_admissible", n_sub)
    rows = np.arange(n_sub) if rows is None else np.asarray(rows)
    P = np.empty(len(rows))
    I = np.empty(len(rows), dtype=np.int64)
    jj = np.arange(n_sub)
    B = max(1, 4_000_000 // max(1, n_sub * m))
    for s in range(0, len(rows), B):
        blk = rows[s:s + B]
        diff = Z[blk][:, None, :] - Z[None, :, :]
        d2 = (diff * diff).sum(axis=2)
        fi = flat[blk][:, None]
        fj = flat[None, :]
        d2 = np.where(fi & fj, 0.0, np.where(fi ^ fj, float(m), d2))
        adm = np.abs(blk[:, None] - jj[None, :]) > excl
        d2 = np.where(adm, d2, np.inf)
        idx = np.argmin(d2, axis=1)                 # first occurrence = smallest j
        P[s:s + len(blk)] = np.sqrt(d2[np.arange(len(blk)), idx])
        I[s:s + len(blk)] = idx
    return P, I, flat


def selfjoin_rows(r: np.ndarray, m: int, excl: int | None = None, rows=None, threads: int = 0):
    """Same definition as selfjoin_brute, computed for the requested rows by the plain C
    double loop in oracle/mp_brute.c (OpenMP over rows).  Returns (P, I, flat)."""
    from ._clib import mp_rows
    excl = (m + 1) // 2 if excl is None else excl
    r = np.ascontiguousarray(r, dtype=np.float64)
    n_sub = r.shape[0] - m + 1
    if n_sub < 2 * excl + 2:
        raise OracleError("no_admissible", n_sub)
    rows = np.arange(n_sub, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    return mp_rows(r, m, excl, rows, threads)


def selfjoin_tierb(r: np.ndarray, m: int, excl: int | None = None, reseed: int = 65536, threads: int = 0):
    """TIER-B reference: the same self-join profile as selfjoin_brute for FULL
    C3/C4-size series, by a plain multithreaded FP64 diagonal recurrence with exact re-seeding
    every `reseed` rows (oracle/mp_tierb.c).  Pinned to selfjoin_brute; series with flat windows
    are not supported.  Returns (P, I)."""
    from ._clib import tierb_selfjoin
    excl = (m + 1) // 2 if excl is None else excl
    return tierb_selfjoin(r, m, excl, reseed, threads)


# ------------------------------------------------------------------------------------------
# a10/a11: Alg. 2 Time-Detection over the sketch + ordered top-K list
# (reading 12)
# ------------------------------------------------------------------------------------------

def inert_groups(flats) -> np.ndarray:
    """Reading 6: a group whose every window is flat (incl. an empty group) is inert."""
    return np.array([bool(np.all(f)) for f in flats])


def combine(P: np.ndarray, inert: np.ndarray):
    """C[i] = max over non-inert g of P_g[i]; G[i] = smallest maximising g (Alg. 2's strict '>'
    over ascending g).  All groups inert -> error (reading 10)."""
    P = np.asarray(P, dtype=np.float64)
    k, n_sub = P.shape
    live = [g for g in range(k) if not inert[g]]
    if not live:
        raise OracleError("all_groups_inert")
    C = np.full(n_sub, -np.inf)
    G = np.full(n_sub, -1, dtype=np.int64)
    for g in live:                      # ascending g, strict '>' keeps the smallest g on ties
        better = P[g] > C
        C = np.where(better, P[g], C)
        G = np.where(better, g, G)
    return C, G


def topk_greedy(C: np.ndarray, G: np.ndarray, I: np.ndarray, K: int, radius: int):
    """Greedy ordered discord list: repeatedly take the smallest-index argmax of C over
    unmasked windows, emit (t, g, nn, score), mask [t - radius, t + radius]; stop early when
    everything is masked."""
    C = np.asarray(C, dtype=np.float64)
    masked = np.zeros(C.shape[0], dtype=bool)
    out = []
    for _ in range(K):
        if masked.all():
            break
        vals = np.where(masked, -np.inf, C)
        t = int(np.argmax(vals))
        g = int(G[t])
        out.append((t, g, int(I[g][t]), float(C[t])))
        masked[max(0, t - radius):t + radius + 1] = True
    return out


def detect(T: np.ndarray, k: int, m: int, K: int, *, groups=None, signs=None, S=None,
           excl: int | None = None, radius: int | None = None, rows_impl: str = "c"):
    """End-to-end oracle pipeline: Alg. 1 sketch -> per-group self-join -> Alg. 2
    combine -> ordered top-K.  Returns dict(R, P, I, flat, inert, C, G, top)."""
    excl = (m + 1) // 2 if excl is None else excl
    radius = (m + 1) // 2 if radius is None else radius
    R, mu, sigma = sketch(T, k, groups, signs, S)
    Ps, Is, Fs = [], [], []
    for g in range(k):
        if rows_impl == "c":
            P, I, F = selfjoin_rows(R[g], m, excl)
        else:
            P, I, F = selfjoin_brute(R[g], m, excl)
        Ps.append(P)
        Is.append(I)
        Fs.append(F)
    P = np.stack(Ps)
    I = np.stack(Is)
    inert = inert_groups(Fs)
    C, G = combine(P, inert)
    top = topk_greedy(C, G, I, K, radius)
    return dict(R=R, mu=mu, sigma=sigma, P=P, I=I, flat=np.stack(Fs), inert=inert, C=C, G=G, top=top)


# ------------------------------------------------------------------------------------------
# f2: Alg. 3 Dimension-Detection in the single-series mode of P:L322,
# and the optional refinement join on j*
# ------------------------------------------------------------------------------------------

def dimension_detection(T: np.ndarray, rows, t_star: int, m: int, excl: int | None = None):
    """Alg. 3 with the self-join variant: for every stream j of J_{g*} (given as the
    rows of T, in the group's order) s^(j) = 1NN_dist(T_{j, t*, m}, T_j) (Def. 4/6: the nearest
    admissible window |t - t*| > excl, reading 7; smallest t on ties, reading 8; flat
    convention reading 5 on the stream as given), then j* = the first strict maximiser
    (lines 3-7; starting from -inf instead of s_bsf = 0 so an all-zero group still names its
    first member, reading 20).  Returns (scores, nn, j_star) with j_star an index into rows."""
    T = np.asarray(T, dtype=np.float64)
    excl = (m + 1) // 2 if excl is None else excl
    scores = np.empty(len(rows))
    nns = np.empty(len(rows), dtype=np.int64)
    for q, j in enumerate(rows):
        Z, flat = znorm_windows(T[j], m)
        n_sub = Z.shape[0]
        diff = Z - Z[t_star][None, :]
        d2 = (diff * diff).sum(axis=1)
        d2 = np.where(flat & flat[t_star], 0.0, np.where(flat ^ flat[t_star], float(m), d2))
        adm = np.abs(np.arange(n_sub) - t_star) > excl
        d2 = np.where(adm, d2, np.inf)
        t = int(np.argmin(d2))                          # first occurrence = smallest t
        nns[q] = t
        scores[q] = math.sqrt(d2[t])
    best, j_star = -np.inf, -1
    for q in range(len(rows)):                          # Alg. 3 line 5: strict '>' in J_g* order
        if scores[q] > best:
            best, j_star = scores[q], q
    return scores, nns, j_star


def refine(r: np.ndarray, m: int, excl: int | None = None):
    """Refinement: the full self-join profile of the identified stream and its
    top-1 discord (smallest-index argmax, reading 8).  Returns (t, nn, score, P, I)."""
    P, I, _ = selfjoin_rows(r, m, excl)
    t = int(np.argmax(P))
    return t, int(I[t]), float(P[t]), P, I


# ------------------------------------------------------------------------------------------
# f1: AB-join matrix profile (Def. 6 ab-join) as Alg. 2 uses it:
# the test series' windows against the training series' windows
# ------------------------------------------------------------------------------------------

def streaming_ab(T_train: np.ndarray, T_test: np.ndarray, k: int, groups, signs, m: int, S=None):
    """f4: Alg. 2 on test data that arrives over time.  The streaming method sketches
    each new test point with Alg. 1 lines 4-5 using the TRAIN statistics (reading 25: the test
    series' own statistics are unknown while it streams) and joins each completed test window
    against every train window (Def. 6 ab-join).  Its result does not depend on how
    the points arrive, so the oracle is the batch definition: R_train = Alg. 1 on T_train,
    R_test = Alg. 1 on T_test with the train (mu, sigma), then the brute-force AB profile per
    group.  Returns (R_test, P, I) with P, I of shape k x (n_test - m + 1)."""
    R_tr, mu, sigma = sketch(T_train, k, groups, signs, S)
    R_te, _, _ = sketch(T_test, k, groups, signs, S, stats=(mu, sigma))
    PI = [abjoin_brute(R_te[q], R_tr[q], m) for q in range(k)]
    return R_te, np.stack([p for p, _ in PI]), np.stack([i for _, i in PI])


def abjoin_brute(a: np.ndarray, b: np.ndarray, m: int, rows=None):
    """P[i] = min_j ||z(A_i) - z(B_j)||_2 over ALL windows j of B (no exclusion zone: the two
    series are different, Def. 6), I[i] = the smallest argmin (reading 8); flat windows per
    reading 5, each series' flat threshold relative to its own max|x|.  Returns (P, I)."""
    Za, fa = znorm_windows(a, m)
    Zb, fb = znorm_windows(b, m)
    rows = np.arange(Za.shape[0]) if rows is None else np.asarray(rows)
    P = np.empty(len(rows))
    I = np.empty(len(rows), dtype=np.int64)
    B = max(1, 4_000_000 // max(1, Zb.shape[0] * m))
    for s in range(0, len(rows), B):
        blk = rows[s:s + B]
        diff = Za[blk][:, None, :] - Zb[None, :, :]
        d2 = (diff * diff).sum(axis=2)
        fi = fa[blk][:, None]
        fj = fb[None, :]
        d2 = np.where(fi & fj, 0.0, np.where(fi ^ fj, float(m), d2))
        idx = np.argmin(d2, axis=1)                 # first occurrence = smallest j
        P[s:s + len(blk)] = np.sqrt(d2[np.arange(len(blk)), idx])
        I[s:s + len(blk)] = idx
    return P, I
