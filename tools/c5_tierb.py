#!/usr/bin/env python
"""Full-profile parity of whole C5 series (d=2,000, n=2e6, m=256, k=32, FP32) against the tier-B
reference (test infrastructure; a one-off evidence run: tier B costs ~2e12 cells per series,
minutes on 16 host cores, so only a few series are checked).

    python tools/c5_tierb.py --series 19 0

The GPU runs bench.py's C5 pipeline through the C-ABI (device-generated streams
synthgen.streams_torch -> sketch_build -> mp_selfjoin -> discord_topk); the oracle builds its OWN
FP64 sketch of the same streams (copied to the host block by block, Alg. 1) and the tier-B FP64
diagonal recurrence (oracle/mp_tierb.c, pinned to the brute force) gives every row of the listed
series.  Checks: |P_gpu - P_tierB| <= 1e-3 max(P, 1e-3 sqrt(m)) for EVERY row of those series; an
index that differs must be a documented tie.  Default series: the top discord's group and group
0.  Prints one JSON line.
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
    ap.add_argument("--series", type=int, nargs="*", default=None)
    ap.add_argument("--tol", type=float, default=1e-3)
    args = ap.parse_args()
    import torch
    import paper_2311_03393_b200 as skmp
    cfg = synthgen.CONFIGS["c5"]
    k, n, m = cfg.k, cfg.n, cfg.m
    dev = torch.device("cuda:0")
    t0 = time.time()
    ids = synthgen.stream_ids(cfg)
    T = synthgen.streams_torch(cfg, dev)
    sk = skmp.sketch_build(T, ids, k, seed=cfg.seed)
    P, I, inert = skmp.mp_selfjoin(sk.R, m)
    top = skmp.discord_topk(P, I, inert, m=m, top=2 * cfg.n_discords)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    series = args.series if args.series else sorted({top[0].g, 0})
    # the oracle's own FP64 sketch rows of the listed groups (Alg. 1, ascending j per group)
    g, s = plan_count_sketch(ids, k, cfg.seed)
    R_or = {q: np.zeros(n) for q in series}
    for j0 in range(0, cfg.d, 50):
        blk = T[j0:j0 + 50].cpu().numpy()
        for q in range(blk.shape[0]):
            j = j0 + q
            if g[j] in R_or:
                x = blk[q].astype(np.float64)
                mu = x.sum() / n
                sg = math.sqrt(((x - mu) ** 2).sum() / n)
                R_or[g[j]] += s[j] * ((x - mu) / sg)
    del T
    Pn, In = P.cpu().numpy().astype(np.float64), I.cpu().numpy()
    excl = cfg.excl
    floor = 1e-3 * math.sqrt(m)
    worst, ties, rows = 0.0, 0, 0
    t1 = time.time()
    for q in series:
        Pt, It = ref.selfjoin_tierb(R_or[q], m, excl)
        err = np.abs(Pn[q] - Pt) / np.maximum(Pt, floor)
        worst = max(worst, float(err.max()))
        assert err.max() <= args.tol, f"series {q}: rel err {err.max():.3e} at row {int(np.argmax(err))}"
        mism = np.where(In[q] != It)[0]
        if len(mism):
            mu, sig, _ = ref.window_stats(R_or[q], m)
            for i in mism:
                j = int(In[q, i])
                assert abs(int(i) - j) > excl
                zi = (R_or[q][i:i + m] - mu[i]) / sig[i]
                zj = (R_or[q][j:j + m] - mu[j]) / sig[j]
                d = float(np.sqrt(((zi - zj) ** 2).sum()))
                assert d <= Pt[i] * (1 + args.tol) + floor * args.tol, (q, int(i), j, int(It[i]), d, float(Pt[i]))
        ties += len(mism)
        rows += len(Pt)
    print(json.dumps({"config": "c5", "series_checked": series, "rows_checked": rows, "documented_ties": ties,
                      "max_rel_err": worst, "tolerance": args.tol, "reference": "tier B (oracle/mp_tierb.c)",
                      "gpu_pipeline_s": round(t_gpu, 1), "tierb_s": round(time.time() - t1, 1),
                      "cores": len(os.sched_getaffinity(0))}), flush=True)


if __name__ == "__main__":
    main()
