"""Shared parity checks (test-side).  Tolerances follow BASELINE.json north_star:
profile values within 1e-9 relative (FP64) / 1e-3 relative (FP32), with the floor
max(P_or, 1e-3 sqrt(m)) of SURVEY §8(c); indices equal except at documented ties."""
from __future__ import annotations

import math

import numpy as np

from oracle import reference as ref

TOL = {"f64": 1e-9, "f32": 1e-3}


def check_profile(r_or: np.ndarray, m: int, excl: int, P_gpu, I_gpu, P_or, I_or, flat_or, tol: float,
                  rows=None, label: str = ""):
    """Compare GPU (P, I) with the oracle's on the given rows (default all).  Returns #ties."""
    P_gpu = np.asarray(P_gpu, dtype=np.float64)
    I_gpu = np.asarray(I_gpu, dtype=np.int64)
    rows = np.arange(len(P_or)) if rows is None else np.asarray(rows)
    n_sub = r_or.shape[0] - m + 1
    floor = 1e-3 * math.sqrt(m)
    err = np.abs(P_gpu - P_or) / np.maximum(np.abs(P_or), floor)
    bad = np.where(err > tol)[0]
    assert len(bad) == 0, (f"{label}: {len(bad)} profile values out of tolerance {tol}; worst rel err "
                           f"{err.max():.3e} at row {rows[int(np.argmax(err))]} (gpu {P_gpu[int(np.argmax(err))]!r}, "
                           f"oracle {P_or[int(np.argmax(err))]!r})")
    # indices: equal, or a documented tie (admissible and its distance within tol of the optimum)
    mism = np.where(I_gpu != I_or)[0]
    ties = 0
    if len(mism):
        Z, fl = ref.znorm_windows(r_or, m)
        for q in mism:
            i = int(rows[q])
            j = int(I_gpu[q])
            assert 0 <= j < n_sub and abs(i - j) > excl, f"{label}: row {i}: inadmissible index {j}"
            if fl[i] and fl[j]:
                dj = 0.0
            elif fl[i] or fl[j]:
                dj = math.sqrt(m)
            else:
                dj = float(np.sqrt(((Z[i] - Z[j]) ** 2).sum()))
            assert dj <= P_or[q] + tol * max(P_or[q], floor), (
                f"{label}: row {i}: gpu index {j} has dist {dj} > oracle optimum {P_or[q]} (index {I_or[q]})")
            ties += 1
    return ties


def check_topk(top_gpu, top_or, C_or: np.ndarray, tol: float, label: str = ""):
    """Identical (t, g) lists; a differing entry is accepted only when the oracle's combined
    scores of the two candidates are within tol (a documented tie)."""
    assert len(top_gpu) == len(top_or), f"{label}: {len(top_gpu)} vs {len(top_or)} discords"
    ties = 0
    for q, (a, b) in enumerate(zip(top_gpu, top_or)):
        if (a.t, a.g) == (b[0], b[1]):
            continue
        ca, cb = C_or[a.t], C_or[b[0]]
        assert abs(ca - cb) <= tol * max(abs(cb), 1e-12), (
            f"{label}: entry {q}: gpu (t={a.t}, g={a.g}, C_or={ca}) vs oracle (t={b[0]}, g={b[1]}, C={cb})")
        ties += 1
    return ties
