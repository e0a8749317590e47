"""dist.py's GPU paths in a one-rank NCCL group (the only multi-process shape one GPU allows):
mp_selfjoin_dist, finalize_dist and mp_abjoin_dist must reproduce the single-call results
exactly.  The band split and key reduce across 2 ranks are covered by test_dist_gloo.py (host
logic) and by the band-invariance tests (kernels)."""
from __future__ import annotations

import socket

import pytest

import synthgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg(cuda):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_one_rank_dist_paths(cuda, pg, dtype):
    import torch
    import paper_2311_03393_b200 as skmp
    from paper_2311_03393_b200 import dist as sdist
    tdt = torch.float32 if dtype == "f32" else torch.float64
    R = torch.from_numpy(synthgen.mp_series(3, 6000, seed=5, kind="mix")).to(cuda, tdt)
    P0, I0, in0 = skmp.mp_selfjoin(R, 64)
    P1, I1, in1 = sdist.mp_selfjoin_dist(R, 64)
    assert torch.equal(P0, P1) and torch.equal(I0, I1) and (in0 == in1).all()
    w = skmp.mp_create(R, 64)
    skmp.mp_join(w)
    P2, I2, _ = sdist.finalize_dist(w)
    assert torch.equal(P0, P2) and torch.equal(I0, I2)
    w.free()
    RB = torch.from_numpy(synthgen.mp_series(3, 4500, seed=6, kind="mix")).to(cuda, tdt)
    A0 = skmp.mp_abjoin(R, RB, 64, both=True)
    A1 = sdist.mp_abjoin_dist(R, RB, 64, both=True)
    for x, y in zip(A0[:4], A1[:4]):
        assert torch.equal(x, y)
    assert (A0[4] == A1[4]).all()


def test_one_rank_sketch_reduce_and_alg3(cuda, pg):
    """allreduce_sketch (NCCL sum of the FP64 master + refresh) and detect_dimension_dist (Alg. 3
    with the maxima all-gathered) in a one-rank group equal the single-process calls."""
    import numpy as np
    import torch
    import paper_2311_03393_b200 as skmp
    from paper_2311_03393_b200 import dist as sdist
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=30, n=3000, k=4)
    T = torch.from_numpy(synthgen.streams(cfg)).to(cuda)
    ids = synthgen.stream_ids(cfg)
    sk = skmp.sketch_build(T, ids, cfg.k, seed=cfg.seed)
    R0 = sk.R.clone()
    sdist.allreduce_sketch(sk)
    torch.cuda.synchronize()
    assert torch.equal(sk.R, R0)
    P, I, inert = skmp.mp_selfjoin(sk.R, cfg.m)
    top = skmp.discord_topk(P, I, inert, m=cfg.m, top=1)
    a = skmp.detect_dimension(sk, [(T, ids)], top[0].t, top[0].g, cfg.m)
    b = sdist.detect_dimension_dist(sk, [(T, ids)], top[0].t, top[0].g, cfg.m, cuda)
    assert a[0] == b[0] and abs(a[1] - b[1]) <= 1e-12 * abs(a[1]) and a[2] == b[2]
