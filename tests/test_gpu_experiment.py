"""GPU: the §4.1 synthetic experiment harness (tools/exp_synthetic.py) at a reduced
size, checked against the oracle's pipeline on the same random walks: the identified discord
(t*, g*, j*) and its rank in the exact (dimension, time) list."""
from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

from oracle import reference as ref
from oracle.hashplan import plan_count_sketch

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_exp41_one_trial_matches_oracle(cuda):
    import torch
    import exp_synthetic as ex
    d, n, m = 16, 1500, 50
    k = math.ceil(math.sqrt(d))
    T = ex.random_walks(d, n, 7, torch.float64)
    P, top_ex = ex.exact(T, m)
    t, g, j, t_ref = ex.sketched(T, m, k, 11, True)
    Tn = T.cpu().numpy()
    # oracle: exact per-stream profiles (Def. 5) and the sketched pipeline (Algs. 1-3)
    Pex = np.stack([ref.selfjoin_rows(Tn[q], m)[0] for q in range(d)])
    np.testing.assert_allclose(P.cpu().numpy(), Pex, rtol=1e-9)
    gs, ss = plan_count_sketch(np.arange(d), k, 11)
    o = ref.detect(Tn, k, m, 1, groups=gs, signs=ss)
    to, go = o["top"][0][0], o["top"][0][1]
    assert (t, g) == (to, go)
    rows = [q for q in range(d) if gs[q] == go]
    _, _, jo = ref.dimension_detection(Tn, rows, to, m)
    assert j == rows[jo]
    rank_gpu = 1 + int((P > P[j, t]).sum())
    rank_or = 1 + int((Pex > Pex[rows[jo], to]).sum())
    assert rank_gpu == rank_or
    assert t_ref == int(np.argmax(Pex[j]))
    # the exact multidimensional discord = the top of the exact list
    flat_max = np.unravel_index(np.argmax(Pex), Pex.shape)
    assert (top_ex.t, top_ex.g) == (int(flat_max[1]), int(flat_max[0]))


def test_exp41_harness_runs(cuda, capsys):
    import exp_synthetic as ex

    class A:
        m, n, dtype, trials, no_refine = 50, 2000, "f32", 2, False
    rec = ex.run_d(64, A)
    assert rec["k"] == 8 and 0.0 <= rec["success_rate"] <= 1.0 and rec["speedup"] > 0
    assert rec["rank_cut"] == max(1, int(1e-4 * 64 * (2000 - 50 + 1)))
