"""Multi-rank host logic on CPU (gloo, world size 2): the diagonal-band partition (mp_band of the
C-ABI, host-only), the max-reduce of packed profile keys (dist.reduce_keys) and the sum-reduce of
partial sketches — checked against the oracle computed over the whole problem.  The GPU kernels
are not involved (they are covered by the -m gpu parity tests, incl. band invariance)."""
from __future__ import annotations

import math
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen
from oracle import reference as ref
from oracle.hashplan import plan_count_sketch


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ord32(f: float) -> int:
    b = struct.unpack("<i", struct.pack("<f", f))[0]
    return b if b >= 0 else b ^ 0x7FFFFFFF


def _ord64(f: float) -> int:
    b = struct.unpack("<q", struct.pack("<d", f))[0]
    return b if b >= 0 else b ^ 0x7FFFFFFFFFFFFFFF


def _band_keys(r, m, excl, lo, hi, words):
    """Oracle keys of one diagonal band: for every row i the best rho over j with |i-j| in
    [max(lo, excl+1), hi), packed like the library's keys (larger is better)."""
    Z, flat = ref.znorm_windows(r, m)
    n_sub = Z.shape[0]
    keys = np.full((n_sub, words), np.iinfo(np.int64).min, dtype=np.int64)
    a = max(lo, excl + 1)
    for i in range(n_sub):
        best = None
        for j in range(n_sub):
            dd = abs(i - j)
            if dd < a or dd >= hi:
                continue
            rho = 1.0 - float(((Z[i] - Z[j]) ** 2).sum()) / (2 * m)
            if best is None or rho > best[0] or (rho == best[0] and j < best[1]):
                best = (rho, j)
        if best is None:
            continue
        rho, j = best
        if words == 1:
            v = (_ord32(float(np.float32(rho))) << 32) | (0xFFFFFFFF - j)
            keys[i, 0] = v if v < (1 << 63) else v - (1 << 64)
        else:
            keys[i, 0] = _ord64(rho)
            keys[i, 1] = -1 - j
    return keys


def _pack(rho, j, words):
    if words == 1:
        v = (_ord32(float(np.float32(rho))) << 32) | (0xFFFFFFFF - int(j))
        return [v if v < (1 << 63) else v - (1 << 64)]
    return [_ord64(float(rho)), -1 - int(j)]


def _ab_band_keys(a, b, m, band1, band2, words):
    """Oracle keys of one AB band: pass 1 cells (i, j = i + delta), delta in band1 (test rows i,
    train columns j); pass 2 cells (j, i = j + delta), delta in band2.  Returns (keys of the test
    windows, keys of the train windows), each window's best over the cells of the band."""
    Za, _ = ref.znorm_windows(a, m)
    Zb, _ = ref.znorm_windows(b, m)
    nA, nB = Za.shape[0], Zb.shape[0]
    rho = np.empty((nA, nB))
    for i in range(nA):
        rho[i] = 1.0 - ((Za[i] - Zb) ** 2).sum(axis=1) / (2 * m)
    delta = np.arange(nB)[None, :] - np.arange(nA)[:, None]        # j - i
    cover = ((delta >= band1[0]) & (delta < band1[1])) | ((-delta >= band2[0]) & (-delta < band2[1]))
    out = []
    for M in (np.where(cover, rho, -np.inf), np.where(cover.T, rho.T, -np.inf)):
        keys = np.full((M.shape[0], words), np.iinfo(np.int64).min, dtype=np.int64)
        for i in range(M.shape[0]):
            if np.isfinite(M[i]).any():
                j = int(np.argmax(M[i]))            # first maximum = smallest index (reading 8)
                keys[i] = _pack(M[i, j], j, words)
        out.append(keys)
    return out


def _worker(rank, world, port, q):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import paper_2311_03393_b200 as skmp
        from paper_2311_03393_b200 import dist as sdist
        out = {}
        # ---- join: bands + key reduce ----------------------------------------------------
        r = synthgen.mp_series(1, 420, seed=11, kind="mix")[0]
        m = 16
        excl = 8
        n_sub = len(r) - m + 1
        for dtype, words in ((skmp.F32, 1), (skmp.F64, 2)):
            lo, hi = sdist.band_for_rank(n_sub, excl, dtype, world, rank)
            k = torch.from_numpy(_band_keys(r, m, excl, lo, hi, words).reshape(-1).copy())
            sdist.reduce_keys(k, words)
            out[f"keys{words}"] = k.numpy().reshape(n_sub, words)
            out[f"band{words}"] = (lo, hi)
        # ---- AB-join: bands over both passes + key reduce of both sides --------------------
        ra = synthgen.mp_series(1, 150, seed=12, kind="mix")[0]
        rb = synthgen.mp_series(1, 260, seed=13, kind="mix")[0]
        for dtype, words in ((skmp.F32, 1), (skmp.F64, 2)):
            b1, b2 = skmp.mp_abband(len(ra) - m + 1, len(rb) - m + 1, dtype, world, rank)
            ka, kb = _ab_band_keys(ra, rb, m, b1, b2, words)
            for nm, kk in (("A", ka), ("B", kb)):
                t = torch.from_numpy(kk.reshape(-1).copy())
                sdist.reduce_keys(t, words)
                out[f"ab{nm}{words}"] = t.numpy().reshape(-1, words)
            out[f"abband{words}"] = (b1, b2)
        # ---- sketch: shard streams, sum partial sketches ---------------------------------
        cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=9, n=600, k=3)
        ids = np.arange(cfg.d)
        mine = sdist.shard(ids, rank, world)
        T = synthgen.streams(cfg, mine)
        g, s = plan_count_sketch(mine, cfg.k, cfg.seed)
        Rp, _, _ = ref.sketch(T, cfg.k, g, s)
        Rt = torch.from_numpy(Rp.copy())
        dist.all_reduce(Rt, op=dist.ReduceOp.SUM)
        out["sketch"] = Rt.numpy()
        # ---- sharded finalize: zero-filled slices sum-reduce to the full profile -----------
        P, I, _ = ref.selfjoin_brute(r, m, excl)
        lo, hi = sdist.row_range(len(P), world, rank)
        Ps = torch.zeros(len(P), dtype=torch.float64)
        Is = torch.zeros(len(P), dtype=torch.int64)
        Ps[lo:hi] = torch.from_numpy(P[lo:hi])
        Is[lo:hi] = torch.from_numpy(I[lo:hi])
        dist.reduce(Ps, 0, op=dist.ReduceOp.SUM)
        dist.reduce(Is, 0, op=dist.ReduceOp.SUM)
        out["fin"] = (Ps.numpy(), Is.numpy(), (lo, hi))
        # ---- Alg. 3 across ranks: global first strict maximum in rank order --------------
        D = skmp.DimResult
        locs = [D(2.5, 11, 40, 3), D(2.5, 23, 7, 2)]          # a tie: rank 0 must win
        out["dim_tie"] = sdist.gather_dimension(locs[rank], "cpu")
        out["dim_none"] = sdist.gather_dimension(D(0.0, 0, 0, 0) if rank == 0 else D(1.0, 5, 3, 4), "cpu")
        # ids >= 2^53 (64-bit keyed names) must cross ranks exactly (no float64 rounding)
        big = [D(1.5, 2**64 - 3, 9, 1), D(2.0, 2**53 + 1, 8, 1)]
        out["dim_big"] = sdist.gather_dimension(big[rank], "cpu")
        out["dim_empty"] = sdist.gather_dimension(D(0.0, 0, 0, 0), "cpu")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_bands_and_reductions():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r = synthgen.mp_series(1, 420, seed=11, kind="mix")[0]
    m, excl = 16, 8
    P, I, _ = ref.selfjoin_brute(r, m, excl)
    for words in (1, 2):
        # the two bands tile [0, n_sub) on the tile grid
        b0, b1 = res[0][f"band{words}"], res[1][f"band{words}"]
        assert b0[0] == 0 and b0[1] == b1[0] and b1[1] == len(P)
        for rank in range(world):
            keys = res[rank][f"keys{words}"]
            if words == 1:
                j = 0xFFFFFFFF - (keys[:, 0] & 0xFFFFFFFF)
            else:
                j = -1 - keys[:, 1]
            Z, _ = ref.znorm_windows(r, m)
            for i in range(len(P)):
                if j[i] != I[i]:  # only a tie at the key's precision is acceptable
                    d = math.sqrt(((Z[i] - Z[j[i]]) ** 2).sum())
                    assert abs(d - P[i]) <= (1e-6 if words == 1 else 1e-12) * max(P[i], 1.0), (i, j[i], I[i])
    # AB-join: the ranks' bands cover both passes; reduced keys give Def. 6's AB profiles
    ra = synthgen.mp_series(1, 150, seed=12, kind="mix")[0]
    rb = synthgen.mp_series(1, 260, seed=13, kind="mix")[0]
    Za, _ = ref.znorm_windows(ra, m)
    Zb, _ = ref.znorm_windows(rb, m)
    for words in (1, 2):
        (a1, c1), (a2, c2) = res[0][f"abband{words}"]
        (b1_, d1), (b2_, d2) = res[1][f"abband{words}"]
        assert a1 == 0 and (c1 == b1_ or b1_ == d1) and max(c1, d1) == Zb.shape[0]
        assert max(c2, d2) == Za.shape[0] and min(x for x in (a2, b2_) if x > 0) == 1
        for nm, (x, y, Zx, Zy) in (("A", (ra, rb, Za, Zb)), ("B", (rb, ra, Zb, Za))):
            Pab, Iab = ref.abjoin_brute(x, y, m)
            for rank in range(world):
                keys = res[rank][f"ab{nm}{words}"]
                j = 0xFFFFFFFF - (keys[:, 0] & 0xFFFFFFFF) if words == 1 else -1 - keys[:, 1]
                assert np.all(keys[:, 0] > np.iinfo(np.int64).min)   # every window got a candidate
                for i in np.where(j != Iab)[0]:
                    d = math.sqrt(((Zx[i] - Zy[j[i]]) ** 2).sum())
                    assert abs(d - Pab[i]) <= (1e-6 if words == 1 else 1e-12) * max(Pab[i], 1.0), (nm, i, j[i])
    # sharded finalize reassembles the whole profile on rank 0; ranks' slices tile [0, n_sub)
    Pf, If, (lo0, hi0) = res[0]["fin"]
    assert np.array_equal(Pf, P) and np.array_equal(If, I)
    assert lo0 == 0 and res[0]["fin"][2][1] == res[1]["fin"][2][0] and res[1]["fin"][2][1] == len(P)
    for rank in range(world):
        assert res[rank]["dim_tie"] == (11, 2.5, 40)
        assert res[rank]["dim_none"] == (5, 1.0, 3)
        assert res[rank]["dim_big"] == (2**53 + 1, 2.0, 8)
        assert res[rank]["dim_empty"] is None
    cfg = synthgen.scaled(synthgen.CONFIGS["c2"], d=9, n=600, k=3)
    T = synthgen.streams(cfg)
    g, s = plan_count_sketch(np.arange(cfg.d), cfg.k, cfg.seed)
    R, _, _ = ref.sketch(T, cfg.k, g, s)
    for rank in range(world):
        np.testing.assert_allclose(res[rank]["sketch"], R, atol=1e-12)
