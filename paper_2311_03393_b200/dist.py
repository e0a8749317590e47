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

Only the collectives live here (torch.distributed: NCCL on GPUs, gloo in the CPU tests and in
the one-GPU multi-rank test, where CUDA tensors are staged through host memory around each
collective); every computation step is a C-ABI call into libsketchmp.so.
"""
from __future__ import annotations

import numpy as np

import torch
import torch.distributed as dist

from . import (F32, F64, DimResult, Sketch, discord_dims_group, discord_dims_merge, mp_abband, mp_band,
               mp_create, mp_create_ab, mp_finalize, mp_finalize_ab, mp_finalize_rows, mp_join, mp_join_ab, mp_keys, mp_tile_width, sketch_refresh,
               sketch_view64)

INT64_MIN = -(1 << 63)


def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_reduce(t: torch.Tensor, op=dist.ReduceOp.SUM, group=None) -> None:
    """dist.all_reduce in place; CUDA tensors go through host memory under gloo."""
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def reduce(t: torch.Tensor, dst: int, op=dist.ReduceOp.SUM, group=None) -> None:
    if _staged(t, group):
        h = t.cpu()
        dist.reduce(h, dst, op=op, group=group)
        t.copy_(h)
    else:
        dist.reduce(t, dst, op=op, group=group)


def broadcast(t: torch.Tensor, src: int, group=None) -> None:
    if _staged(t, group):
        h = t.cpu()
        dist.broadcast(h, src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src, group=group)


def all_gather(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    world = dist.get_world_size(group)
    src = t.cpu() if _staged(t, group) else t
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src, group=group)
    return out


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
    all_reduce(R64, op=dist.ReduceOp.SUM, group=group)
    sketch_refresh(sk)


def reduce_keys(keys: torch.Tensor, words: int, group=None) -> None:
    """In-place max-reduce of profile keys across ranks (the NCCL min-with-index reduce of
    SURVEY §8(e), expressed on the library's larger-is-better key words)."""
    if words == 1:
        all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
        return
    kv = keys.view(-1, 2)
    v = kv[:, 0].clone()
    all_reduce(v, op=dist.ReduceOp.MAX, group=group)
    idx = kv[:, 1].clone()
    idx.masked_fill_(kv[:, 0] != v, INT64_MIN)
    all_reduce(idx, op=dist.ReduceOp.MAX, group=group)
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
    every rank scores its members of J_g (discord_dims_group), then the ranks' winners are
    all-gathered and merged by the C-ABI (discord_dims_merge: first strict maximum in rank
    order; ranks hold contiguous id shards, so rank order is J_g's plan order).  Every rank
    returns the same (id*, score, nn), or None when no rank holds a member of J_g."""
    return gather_dimension(discord_dims_group(sk, g, sources, t, m), device, group)


def gather_dimension(loc: DimResult, device, group=None):
    """All-gather every rank's DimResult as four exact 64-bit words (score bits, id, nn,
    n_scored; the id travels as int64 bits, so ids >= 2^53 survive) and merge them in rank
    order through discord_dims_merge."""
    world = dist.get_world_size(group)
    words = np.array([loc.score], dtype=np.float64).view(np.int64).tolist() + \
        np.array([loc.id], dtype=np.uint64).view(np.int64).tolist() + [int(loc.nn), int(loc.n_scored)]
    row = torch.tensor(words, dtype=torch.int64, device=device)
    h = torch.stack([x.cpu() for x in all_gather(row, group)]).numpy()
    parts = [DimResult(float(h[r, 0:1].view(np.float64)[0]), int(h[r, 1:2].view(np.uint64)[0]), int(h[r, 2]),
                       int(h[r, 3])) for r in range(world)]
    best = discord_dims_merge(parts)
    return None if best.n_scored == 0 else (int(best.id), float(best.score), int(best.nn))


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
    reduce(P, dst, op=dist.ReduceOp.SUM, group=group)
    reduce(I, dst, op=dist.ReduceOp.SUM, group=group)
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
        reduce(P, dst, op=dist.ReduceOp.SUM, group=group)
        reduce(I, dst, op=dist.ReduceOp.SUM, group=group)
        out += [P, I]
    a.free()
    b.free()
    return (*out, inert) if rank == dst else None
