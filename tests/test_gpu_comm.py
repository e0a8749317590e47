"""The native multi-GPU entry points (skmp_comm_*, sketch_allreduce, mp_selfjoin_dist) in a
one-rank NCCL communicator — the only shape one GPU allows: the band split and the collectives
must reproduce the single-GPU calls bit for bit.  (Multi-rank host logic: test_dist_gloo.py.)"""
from __future__ import annotations

import numpy as np
import pytest

import synthgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(cuda):
    import paper_2311_03393_b200 as skmp
    c = skmp.Comm(skmp.Comm.unique_id(), 1, 0)
    yield c
    c.free()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_native_dist_equals_single(cuda, comm, dtype):
    import torch
    import paper_2311_03393_b200 as skmp
    tdt = torch.float32 if dtype == "f32" else torch.float64
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=20, n=4000, k=4)
    T = torch.from_numpy(synthgen.streams(cfg)).to(cuda, tdt)
    ids = synthgen.stream_ids(cfg)
    sk = skmp.sketch_build(T, ids, cfg.k, seed=cfg.seed)
    R0 = sk.R.clone()
    skmp.sketch_allreduce(comm, sk)
    torch.cuda.synchronize()
    assert torch.equal(sk.R, R0)
    P0, I0, in0 = skmp.mp_selfjoin(sk.R, cfg.m)
    P1, I1, in1 = skmp.mp_selfjoin_dist(comm, sk.R, cfg.m)
    torch.cuda.synchronize()
    assert torch.equal(P0, P1) and torch.equal(I0, I1) and np.array_equal(in0, in1)
