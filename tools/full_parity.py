#!/usr/bin/env python
"""Full-profile parity of a whole BASELINE config against the tier-B reference (test
infrastructure; a one-off evidence run, too slow for the regular GPU suite at C4 size).

    python tools/full_parity.py --config c4     # all 64 series x 199,745 rows (C4 dynamic pipeline)
    python tools/full_parity.py --config c3     # all 32 series x 99,873 rows

The GPU runs the bench pipeline through the C-ABI (sketch_build, add / delete for C4,
mp_selfjoin); the oracle builds its OWN FP64 sketch of the final stream set (Alg. 1) and the
tier-B FP64 diagonal recurrence (oracle/mp_tierb.c, pinned to the brute force) gives every row's
profile.  Checks: |P_gpu - P_tierB| <= 1e-3 max(P, 1e-3 sqrt(m)) for EVERY row; an index that
differs must be a documented tie (the GPU's neighbour as near within the tolerance); the GPU's
top-K discords (discord_topk, K = 2 x injected as bench.py ranks) against the oracle's Alg. 2
combine + greedy top-K over the tier-B profiles: identical (t, g) lists, a differing entry only
where the oracle's combined scores of the two candidates agree within the tolerance.  Prints one
JSON summary line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthgen  # noqa: E402
from oracle import reference as ref  # noqa: E402
from oracle.hashplan import plan_count_sketch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--tol", type=float, default=1e-3)
    args = ap.parse_args()
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS[args.config]
    dev = torch.device("cuda:0")
    t0 = time.time()
    ids = synthgen.stream_ids(cfg)
    T = synthgen.streams(cfg)
    Td = torch.from_numpy(T).to(dev)
    sk = skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed)
    final_T, final_ids = T, ids
    if cfg.extra.get("n_add"):
        add_ids, del_ids = synthgen.dynamic_ids(cfg)
        Ta = synthgen.streams(cfg, add_ids)
        skmp.sketch_add_dim(sk, torch.from_numpy(Ta).to(dev), add_ids)
        skmp.sketch_del_dim(sk, Td[del_ids.astype(np.int64)].contiguous(), del_ids)
        keep = np.setdiff1d(np.arange(cfg.d), del_ids.astype(np.int64))
        final_T = np.concatenate([T[keep], Ta])
        final_ids = np.concatenate([ids[keep], add_ids])
    P, I, inert = skmp.mp_selfjoin(sk.R, cfg.m)
    K = 2 * cfg.n_discords
    top = skmp.discord_topk(P, I, inert, m=cfg.m, top=K)
    P, I = P.cpu().numpy().astype(np.float64), I.cpu().numpy()
    del Td
    t_gpu = time.time() - t0
    g, s = plan_count_sketch(final_ids, cfg.k, cfg.seed)
    # the oracle's own FP64 sketch (Alg. 1), summed over blocks of streams (linearity) so
    # the FP64 copy of the inputs stays small
    R_or = np.zeros((cfg.k, cfg.n))
    for j0 in range(0, final_T.shape[0], 500):
        Rb, _, _ = ref.sketch(final_T[j0:j0 + 500], cfg.k, g[j0:j0 + 500], s[j0:j0 + 500])
        R_or += Rb
    m, excl = cfg.m, cfg.excl
    floor = 1e-3 * math.sqrt(m)
    worst, ties, rows = 0.0, 0, 0
    t1 = time.time()
    P_or = np.empty_like(P)
    I_or = np.empty_like(I)
    for q in range(cfg.k):
        Pt, It = ref.selfjoin_tierb(R_or[q], m, excl)
        P_or[q], I_or[q] = Pt, It
        err = np.abs(P[q] - Pt) / np.maximum(Pt, floor)
        worst = max(worst, float(err.max()))
        assert err.max() <= args.tol, f"series {q}: rel err {err.max():.3e} at row {int(np.argmax(err))}"
        mism = np.where(I[q] != It)[0]
        if len(mism):
            mu, sig, _ = ref.window_stats(R_or[q], m)
            for i in mism:
                j = int(I[q, i])
                assert abs(int(i) - j) > excl
                zi = (R_or[q, i:i + m] - mu[i]) / sig[i]
                zj = (R_or[q, j:j + m] - mu[j]) / sig[j]
                d = float(np.sqrt(((zi - zj) ** 2).sum()))
                assert d <= Pt[i] * (1 + args.tol) + floor * args.tol, (q, int(i), j, int(It[i]), d, float(Pt[i]))
        ties += len(mism)
        rows += len(Pt)
    # identical top-K discord locations (north_star), the oracle's own combined profile
    inert_or = ref.inert_groups([ref.window_stats(R_or[q], m)[2] for q in range(cfg.k)])
    assert np.array_equal(inert, inert_or)
    C_or, G_or = ref.combine(P_or, inert_or)
    want = ref.topk_greedy(C_or, G_or, I_or, K, excl)
    assert len(want) == len(top)
    top_ties = 0
    for q, (a, b) in enumerate(zip(top, want)):
        if (a.t, a.g) != (b[0], b[1]):
            assert abs(C_or[a.t] - C_or[b[0]]) <= args.tol * C_or[b[0]], (q, a, b)
            top_ties += 1
    print(json.dumps({"config": args.config, "series": cfg.k, "rows_checked": rows, "documented_ties": ties,
                      "top_k": K, "top_k_identical": K - top_ties, "top_k_documented_ties": top_ties,
                      "max_rel_err": worst, "tolerance": args.tol, "reference": "tier B (oracle/mp_tierb.c)",
                      "gpu_pipeline_s": round(t_gpu, 1), "tierb_s": round(time.time() - t1, 1),
                      "cores": len(os.sched_getaffinity(0))}), flush=True)


if __name__ == "__main__":
    main()
