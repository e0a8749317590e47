"""Host vs device time of each call of one C4 bench step (diagnostic): every call is bracketed by
torch.cuda.synchronize(), so `host` is the call's wall time including its GPU work and `gpu` the
CUDA-event time of the same bracket.  usage: python tools/phase_probe.py [--config c4] [--iters 4]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_03393_b200 as skmp  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=4)
a = ap.parse_args()
cfg = synthgen.CONFIGS[a.config]
dev = torch.device("cuda", 0)
ids = synthgen.stream_ids(cfg)
add_ids, del_ids = synthgen.dynamic_ids(cfg)
Td = torch.from_numpy(synthgen.streams(cfg, ids)).to(dev)
Ta = torch.from_numpy(synthgen.streams(cfg, add_ids)).to(dev) if len(add_ids) else None
pos = {int(j): q for q, j in enumerate(ids)}
Tdl = Td[[pos[int(j)] for j in del_ids]].contiguous() if len(del_ids) else None
torch.cuda.synchronize()


def timed(name, f, rec):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    r = f()
    e1.record()
    torch.cuda.synchronize()
    rec.setdefault(name, []).append(((time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)))
    return r


rec = {}
for it in range(a.iters + 1):
    r = {} if it == 0 else rec
    sk = timed("sketch_build", lambda: skmp.sketch_build(Td, ids, cfg.k, seed=cfg.seed), r)
    if Ta is not None:
        timed("add_dim", lambda: skmp.sketch_add_dim(sk, Ta, add_ids), r)
    if Tdl is not None:
        timed("del_dim", lambda: skmp.sketch_del_dim(sk, Tdl, del_ids), r)
    w = timed("mp_create", lambda: skmp.mp_create(sk.R, cfg.m), r)
    timed("mp_join", lambda: skmp.mp_join(w), r)
    fin = timed("mp_finalize", lambda: skmp.mp_finalize(w), r)
    timed("discord_topk", lambda: skmp.discord_topk(*fin, m=cfg.m, top=2 * cfg.n_discords), r)
    timed("mp_free", lambda: w.free(), r)
    timed("sketch_free", lambda: sk.free(), r)
for k, v in rec.items():
    h = np.array(v)
    print(f"{k:14s} host {np.median(h[:, 0]):9.3f} ms   gpu {np.median(h[:, 1]):9.3f} ms")
