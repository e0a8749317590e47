"""Latency / throughput of the f4 streaming path (stream_push) at the C4 train size: d = 10,000
random-walk streams, n_train = 200,000, k = 64, m = 256, FP32, inputs on the device.  Each push
of n_new points = Alg. 1 lines 4-5 for the new columns + the AB-join of the completed windows
against all 199,745 train windows of every group + their finalize.

    python tools/stream_bench.py [--d 10000] [--n 200000] [--k 64] [--m 256] [--reps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_03393_b200 as skmp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=10000)
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--sizes", default="1,16,256,4096")
a = ap.parse_args()
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
T = torch.randn(a.d, a.n, device=dev, generator=g).cumsum_(dim=1)
ids = np.arange(a.d, dtype=np.uint64)
sk = skmp.sketch_build(T, ids, a.k, seed=1)
del T
sizes = [int(x) for x in a.sizes.split(",")]
total = sum(s * (a.reps + 2) for s in sizes) + a.m
st = skmp.Stream(sk, a.m, capacity=total)
n_sub_tr = a.n - a.m + 1
# warm the stream with m - 1 points so that every later point completes one window
st.push(torch.randn(a.d, a.m - 1, device=dev, generator=g).cumsum_(dim=1))
for s in sizes:
    blocks = [torch.randn(a.d, s, device=dev, generator=g).cumsum_(dim=1) for _ in range(a.reps + 2)]
    for b in blocks[:2]:
        st.push(b)
    torch.cuda.synchronize()
    ts = []
    for b in blocks[2:]:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.push(b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    cells = s * n_sub_tr * a.k
    print(json.dumps({"n_new": s, "ms_per_push_median": round(ms, 4), "ms_min": round(min(ts), 4),
                      "windows_per_s": round(s / ms * 1e3, 1), "cells_per_s": cells / ms * 1e3,
                      "d": a.d, "n_train": a.n, "k": a.k, "m": a.m, "dtype": "f32"}), flush=True)
top = st.topk(3)
print(json.dumps({"top": [(x.t, x.g, round(x.score, 4)) for x in top]}))
