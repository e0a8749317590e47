"""GPU: bench.py's multi-rank branch (world > 1) for real on the one-GPU box — two ranks sharing
cuda:0 over a gloo process group (CUDA tensors staged through host memory around each
collective; no kernel of one rank waits on another's).  It runs exactly the code the driver's
torchrun N-GPU launch runs: streams sharded over the ranks + sum-all-reduce of the partial FP64
sketches (Alg. 1 is linear), each rank's equal-cost diagonal band (mp_band) + the
max-all-reduce of the profile keys, the sharded finalize, rank 0's discord_topk, and Alg. 3 over
every rank's own members of J_g* merged by discord_dims_merge.

Checks:
* the 2-rank keys / P / I / top-K / Alg. 3 result are bit-identical to ONE rank joining the same
  (all-reduced) sketch: the band split and the reductions change nothing;
* against the 1-rank bench run: the sketch agrees to FP64 rounding (the all-reduce only reorders
  the FP64 sum), and the top-K (t, g) list and Alg. 3's j* are the same.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(tmp, tag, config, shape, world):
    out = os.path.join(tmp, f"{tag}.npz")
    args = ["--config", config, "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
            "--dump", out]
    if shape:
        args += ["--shape", shape]
    if world == 1:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), *args]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), *args,
               "--backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return dict(np.load(out))


@pytest.mark.parametrize("config,shape", [("c2", ""), ("c3", "d=200,n=20000,k=8")])
def test_two_ranks_on_one_gpu_equal_one_rank(cuda, tmp_path, config, shape):
    import torch
    import paper_2311_03393_b200 as skmp
    two = _bench(str(tmp_path), "two", config, shape, 2)
    one = _bench(str(tmp_path), "one", config, shape, 1)
    # (1) one rank joining the 2-rank run's (all-reduced) sketch reproduces it bit for bit
    R = torch.from_numpy(two["R"]).to(cuda)
    m = {"c2": 100, "c3": 128}[config]
    w = skmp.mp_create(R, m)
    skmp.mp_join(w)
    keys, _ = skmp.mp_keys(w)
    keys = keys.cpu().numpy()
    P, I, inert = skmp.mp_finalize(w)
    w.free()
    assert np.array_equal(keys, two["keys"]), "band split + key all-reduce changed the keys"
    assert np.array_equal(P.cpu().numpy(), two["P"]) and np.array_equal(I.cpu().numpy(), two["I"])
    assert np.array_equal(inert, two["inert"])
    top = skmp.discord_topk(P, I, inert, m=m, top=len(two["top"]))
    assert np.array_equal(np.array([(d.t, d.g, d.nn) for d in top]), two["top"])
    assert np.array_equal(np.array([d.score for d in top]), two["top_score"])
    # (2) against the 1-rank bench: the sketch differs only by the FP64 summation order
    scale = np.abs(one["R64"]).max() + 1.0
    assert np.abs(two["R64"] - one["R64"]).max() <= 1e-12 * scale
    assert np.array_equal(two["top"][:, :2], one["top"][:, :2]), (two["top"][:5], one["top"][:5])
    assert np.array_equal(two["dim"], one["dim"]) and np.array_equal(two["dim_score"], one["dim_score"])
    print(f"{config}: 2 ranks on one GPU == 1 rank (keys, P, I, top-{len(top)}, Alg. 3 j* = {int(two['dim'][0])})")


def test_two_ranks_full_bench_line(cuda):
    """The whole default bench path at N = 2 (incl. the pipelined e2e leg through pinned host
    inputs and the max-over-ranks timing) runs and prints one complete JSON line."""
    import json
    args = ["--config", "c5", "--shape", "d=200,n=40000,k=8", "--steps", "2", "--warmup", "3", "--e2e-steps", "2",
            "--no-cpu-baseline", "--backend", "gloo"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["roofline"]["frac"] > 0 and d["gpu_launches"] > 0
