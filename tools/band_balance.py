"""Multi-GPU load balance of the banded self-join, measured on ONE GPU (no collectives, no
concurrency: each rank's join work is timed alone, as that rank of an N-GPU run executes it).

For N in (2, 4, 8) the C4 join (k = 64, n = 200,000, m = 256, FP32) is split as bench.py splits it
(dist.rank_diagonals = mp_band's equal-cost bands), and each rank's joins are timed with CUDA
events in a fresh workspace.  The strong-scaling bound of the join is t(1 rank) / (N * max_rank
t).  Prints one JSON line per N.  (--plain calls mp_band directly: the same split.)

    python tools/band_balance.py [--k 64] [--n 200000] [--m 256] [--plain]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_03393_b200 as skmp  # noqa: E402
from paper_2311_03393_b200 import dist as sdist  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--plain", action="store_true")
a = ap.parse_args()
R = synthgen.mp_series_torch(a.k, a.n, 7, "cuda", torch.float32)
n_sub = a.n - a.m + 1
excl = (a.m + 1) // 2


def timed(ranges):
    best = None
    for _ in range(a.reps):
        w = skmp.mp_create(R, a.m)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for lo, hi in ranges:
            if hi > lo:
                skmp.mp_join(w, lo, hi)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
        w.free()
    return best


t1 = timed([(0, n_sub)])
print(json.dumps({"ranks": 1, "join_ms": round(t1, 2)}), flush=True)
for N in (2, 4, 8):
    if a.plain:
        rr = [[skmp.mp_band(n_sub, excl, skmp.F32, N, r)] for r in range(N)]
    else:
        rr = [sdist.rank_diagonals(n_sub, excl, skmp.F32, N, r) for r in range(N)]
    ts = [timed(x) for x in rr]
    print(json.dumps({"ranks": N, "scheme": "equal-cost bands (dist.rank_diagonals)" if not a.plain else "mp_band",
                      "rank_ms": [round(x, 2) for x in ts], "max_ms": round(max(ts), 2),
                      "join_scaling_bound": round(t1 / (N * max(ts)), 3)}), flush=True)
