"""Multi-GPU orchestration of the hot path, one process per GPU.

Sketch: streams are sharded over ranks; each rank builds the partial sketch of its shard with
the shared (seeded, id-keyed) plan, and the FP64 master accumulators are sum-all-reduced
(linearity of Alg. 1), then re-rounded on every rank (sketch_refresh).
Join: the diagonals are split into equal-cost bands on the tile grid (mp_band, rank_diagonals);
each rank joins its band into its own profile keys, which are max-all-reduced (FP32: one signed
int64 MAX on {orderable rho, ~j}; FP64: MAX on the value word, then MAX on the index word among
the ranks holding that value), after which any rank can finalize.

AB-join: the same scheme over its two passes taken as one diagonal sequence (mp_abband); the
keys of both sides are max-all-reduced and each side's windows are finalized in row slices.

Only the collectives live here (torch.distributed: NCCL on GPUs, gloo in the CPU tests);
every computation step is a C-ABI call into libsketchmp.so.
"""
from __future__ import annotations

import numpy as np

import torch
import torch.distributed as dist

from . import (F32, F64, Sketch, detect_dimension, mp_abband, mp_band, mp_create, mp_create_ab, mp_finalize,
               mp_finalize_ab, mp_finalize_rows, mp_join, mp_join_ab, mp_keys, mp_tile_width, sketch_refresh,
               sketch_view64)

INT64_MIN = -(1 << 63)


def shard(ids, rank: int, world: int):
    """Contiguous id shard of `rank` (streams are independent, so any split is valid)."""
    return np.array_split(np.asarray(ids), world)[rank]


def band_for_rank(n_sub: int, excl: int, dtype: int, world: int, rank: int) -> tuple[int, int]:
    return mp_band(n_sub, excl, dtype, world, rank)


def rank_diagonals(n_sub: int, excl: int, dtype: int, world: int, rank: int) -> list[tuple[int, int]]:
    """Diagonal ranges rank `rank` joins: its equal-cost band of the whole join (mp_band; one
    rank: everything).  A variant that had every rank also join the first block (to fill all keys
    with good thresholds first) was measured slower: that block is the most expensive one
    (tools/band_balance.py)."""
    if world == 1:
        return [(0, n_sub)]
    return [mp_band(n_sub, excl, dtype, world, rank)]


def allreduce_sketch(sk: Sketch, group=None) -> None:
    """Sum the per-rank partial FP64 sketches in place and refresh the dtype copy."""
    R64 = sketch_view64(sk)
    dist.all_reduce(R64, op=dist.ReduceOp.SUM, group=group)
    sketch_refresh(sk)


def reduce_keys(keys: torch.Tensor, words: int, group=None) -> None:
    """In-place max-reduce of profile keys across ranks (the NCCL min-with-index reduce of
    SURVEY §8(e), expressed on the library's larger-is-better key words)."""
    if words == 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
        return
    kv = keys.view(-1, 2)
    v = kv[:, 0].clone()
    dist.all_reduce(v, op=dist.ReduceOp.MAX, group=group)
    idx = kv[:, 1].clone()
    idx.masked_fill_(kv[:, 0] != v, INT64_MIN)
    dist.all_reduce(idx, op=dist.ReduceOp.MAX, group=group)
    kv[:, 0].copy_(v)
    kv[:, 1].copy_(idx)


def mp_selfjoin_dist(R: torch.Tensor, m: int, *, excl: int = -1, reseed_rows: int = 0, group=None,
                     finalize_on_all: bool = False):
    """Self-join of R (k x n, replicated on every rank) split into diagonal bands over the ranks
    of `group`.  Returns (P, I, inert) on rank 0 (and on all ranks if finalize_on_all)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = R.shape[1]
    n_sub = n - m + 1
    e = (m + 1) // 2 if excl < 0 else excl
    dtype = F32 if R.dtype == torch.float32 else F64
    w = mp_create(R, m, excl=e, reseed_rows=reseed_rows)
    for lo, hi in rank_diagonals(n_sub, e, dtype, world, rank):
        if hi > lo:
            mp_join(w, lo, hi)
    keys, words = mp_keys(w)
    reduce_keys(keys, words, group)
    out = None
    if rank == 0 or finalize_on_all:
        out = mp_finalize(w)
    w.free()
    return out


def detect_dimension_dist(sk: Sketch, sources, t: int, g: int, m: int, device, group=None):
    """Alg. 3 with the streams sharded over ranks (each rank's sketch plan holds its own shard):
    every rank scores its members of J_g (discord_dims), then the (score, plan order) maxima are
    all-gathered and every rank returns the same (id*, score, nn).  Ranks hold contiguous id
    shards, so (rank, local order) is the global plan order of Alg. 3's scan."""
    return gather_dimension(detect_dimension(sk, sources, t, g, m), device, group)


def gather_dimension(loc, device, group=None):
    """All-gather every rank's local Alg. 3 winner (id, score, nn) or None and return the global
    one: the first strict maximum in rank order (ranks hold contiguous id shards)."""
    world = dist.get_world_size(group)
    row = torch.tensor([-1.0, 0.0, 0.0, 0.0], dtype=torch.float64, device=device) if loc is None else \
        torch.tensor([1.0, loc[1], float(loc[0]), float(loc[2])], dtype=torch.float64, device=device)
    allr = [torch.empty_like(row) for _ in range(world)]
    dist.all_gather(allr, row, group=group)
    best = None
    for r in range(world):
        ok, sc, j, nn = (float(x) for x in allr[r].tolist())
        if ok > 0 and (best is None or sc > best[1]):  # strict: the earliest rank wins ties
            best = (int(j), sc, int(nn))
    return best


def row_range(n_sub: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous window slice of `rank` for the sharded finalize."""
    b = np.linspace(0, n_sub, world + 1).astype(np.int64)
    return int(b[rank]), int(b[rank + 1])


def finalize_dist(w, group=None, dst: int = 0):
    """Sharded finalize after the key reduce (every rank holds all keys): each rank resolves its
    slice of windows into zero-filled full-size P / I, which are sum-reduced to rank `dst` (x + 0
    is exact).  Returns (P, I, inert) on `dst`, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = row_range(w.n_sub, world, rank)
    P, I, inert = mp_finalize_rows(w, lo, hi)
    dist.reduce(P, dst, op=dist.ReduceOp.SUM, group=group)
    dist.reduce(I, dst, op=dist.ReduceOp.SUM, group=group)
    return (P, I, inert) if rank == dst else None



def mp_abjoin_dist(RA: torch.Tensor, RB: torch.Tensor, m: int, *, reseed_rows: int = 0, both: bool = False,
                   group=None, dst: int = 0):
    """AB-join of RA (test) against RB (train), both replicated on every rank, its two passes split
    into equal-cell diagonal bands over the ranks of `group` (mp_abband).  Keys of both sides
    are max-reduced (a pass-2 band also feeds the test side's keys), then each rank finalizes a
    slice of the test windows (and of the train windows with both=True), sum-reduced to `dst`.
    Returns (PA, IA, inert) or (PA, IA, PB, IB, inert) on `dst`, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    a = mp_create_ab(RA, m, reseed_rows=reseed_rows)
    b = mp_create_ab(RB, m, reseed_rows=reseed_rows)
    (l1, h1), (l2, h2) = mp_abband(a.n_sub, b.n_sub, a.dtype, world, rank)
    if l1 < h1:
        mp_join_ab(a, b, l1, h1)   # pass 1: test rows, train columns
    if l2 < h2:
        mp_join_ab(b, a, l2, h2)   # pass 2: train rows, test columns
    for w in ((a, b) if both else (a,)):
        keys, words = mp_keys(w)
        reduce_keys(keys, words, group)
    out = []
    inert = None
    for w, o in ((a, b), (b, a)) if both else ((a, b),):
        lo, hi = row_range(w.n_sub, world, rank)
        if hi == 0:
            lo = hi = w.n_sub   # empty slice ((0, 0) would mean all windows)
        P, I, inert = mp_finalize_ab(w, o, lo, hi)
        dist.reduce(P, dst, op=dist.ReduceOp.SUM, group=group)
        dist.reduce(I, dst, op=dist.ReduceOp.SUM, group=group)
        out += [P, I]
    a.free()
    b.free()
    return (*out, inert) if rank == dst else None
