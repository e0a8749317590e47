"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module is INPUT PLUMBING ONLY.  It holds none of the method's arithmetic
(no z-normalisation, no sketch, no matrix profile); both `oracle/` and the CUDA
path consume the arrays it returns, byte-identical.  The recipes follow
SURVEY.md §8(d) ("Generators per config"), which stands in for the paper's
missing datasets:

* C2's d=51 mirrors SWaT's 51 sensors (§4.4),
* C3's d≈1,000 mirrors the payment network's ≈1,000 categories (§4.3),
* C4's d=10,000 is §4.1's largest d, random walks as in §4.1,
* C1 and C5 are BASELINE.json-only shapes.

Seeding: config seed s_c = 2311033930 + c; stream with id j is drawn from
numpy.random.default_rng([s_c, j]) so streams can be produced independently and
added/deleted by id; injections use default_rng([s_c, 0xD15C0]); the dense
projection matrix uses default_rng([s_c, 0x5EED]).  The population std used to
size an injection is the stream's std *before* injection (amplitude only).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 2311033930


@dataclass(frozen=True)
class Config:
    name: str
    index: int
    d: int
    n: int
    m: int
    k: int
    dtype: str            # "f64" | "f32"
    proj: str             # "dense" | "count"
    kind: str             # stream generator family
    n_discords: int
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    @property
    def n_sub(self) -> int:
        return self.n - self.m + 1

    @property
    def excl(self) -> int:
        return (self.m + 1) // 2

    def cells(self) -> int:
        """Exact evaluated pairs k*(n_sub-r-1)(n_sub-r)/2 (SURVEY §8(c) reading 17)."""
        a = self.n_sub - self.excl - 1
        return self.k * a * (a + 1) // 2


CONFIGS = {
    "c1": Config("c1", 1, d=8, n=2000, m=50, k=4, dtype="f64", proj="dense",
                 kind="randwalk", n_discords=1),
    "c2": Config("c2", 2, d=51, n=20000, m=100, k=16, dtype="f64", proj="count",
                 kind="periodic_mix", n_discords=3),
    "c3": Config("c3", 3, d=1000, n=100000, m=128, k=32, dtype="f32", proj="count",
                 kind="ar1_daily", n_discords=10),
    "c4": Config("c4", 4, d=10000, n=200000, m=256, k=64, dtype="f32", proj="count",
                 kind="randwalk", n_discords=20, extra={"n_add": 500, "n_del": 500}),
    "c5": Config("c5", 5, d=2000, n=2000000, m=256, k=32, dtype="f32", proj="count",
                 kind="seasonal_noise", n_discords=50),
}


def scaled(cfg: Config, *, d: int | None = None, n: int | None = None, k: int | None = None,
           m: int | None = None, name: str | None = None) -> Config:
    """Same recipe and seed, smaller shape (for oracle-sized parity cases)."""
    return Config(name or f"{cfg.name}s", cfg.index, d=d or cfg.d, n=n or cfg.n, m=m or cfg.m,
                  k=k or cfg.k, dtype=cfg.dtype, proj=cfg.proj, kind=cfg.kind,
                  n_discords=cfg.n_discords, extra=dict(cfg.extra))


# ----------------------------------------------------------------------------------------------
# per-stream base generators (before injection)
# ----------------------------------------------------------------------------------------------

def _stream_rng(cfg: Config, sid: int) -> np.random.Generator:
    return np.random.default_rng([cfg.seed, int(sid)])


def _base_stream(cfg: Config, sid: int, n: int) -> np.ndarray:
    rng = _stream_rng(cfg, sid)
    t = np.arange(n, dtype=np.float64)
    if cfg.kind == "randwalk":
        return np.cumsum(rng.standard_normal(n))
    if cfg.kind == "periodic_mix":
        c = int(rng.integers(1, 4))
        x = np.zeros(n)
        for _ in range(c):
            p = int(rng.integers(200, 2001))
            a = rng.uniform(0.5, 1.5)
            ph = rng.uniform(0.0, 2.0 * math.pi)
            x += a * np.sin(2.0 * math.pi * t / p + ph)
        return x + rng.normal(0.0, 0.1, n)
    if cfg.kind == "ar1_daily":
        from scipy.signal import lfilter
        phi = rng.uniform(0.8, 0.99)
        eps = rng.standard_normal(n)
        x0 = rng.normal(0.0, 1.0 / math.sqrt(1.0 - phi * phi))
        # x_t = phi x_{t-1} + eps_t with x_{-1} chosen so that x_0 ~ N(0, 1/(1-phi^2))
        eps[0] = x0
        x = lfilter([1.0], [1.0, -phi], eps)
        amp = 1.0 / math.sqrt(1.0 - phi * phi)
        th = rng.uniform(0.0, 2.0 * math.pi)
        return x + amp * np.sin(2.0 * math.pi * t / 1440.0 + th)
    if cfg.kind == "seasonal_noise":
        a = rng.uniform(0.5, 1.5)
        th = rng.uniform(0.0, 2.0 * math.pi)
        return a * np.sin(2.0 * math.pi * t / 10080.0 + th) + rng.normal(0.0, 0.2, n)
    raise ValueError(cfg.kind)


# ----------------------------------------------------------------------------------------------
# injected discords
# ----------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Injection:
    sid: int        # stream id
    t: int          # start sample
    kind: str       # "sine_burst" | "level_shift" | "spike"
    length: int
    period: float   # for sine bursts
    amp_sigmas: float


def _place(rng: np.random.Generator, count: int, n: int, m: int) -> list[int]:
    """Starts >= m from either end, pairwise >= 2m apart (SURVEY §8(d) 'Injection placement')."""
    starts: list[int] = []
    lo, hi = m, n - 2 * m
    tries = 0
    while len(starts) < count:
        tries += 1
        if tries > 100000:
            raise RuntimeError("cannot place injections")
        s = int(rng.integers(lo, hi))
        if all(abs(s - o) >= 2 * m for o in starts):
            starts.append(s)
    return starts


def injections(cfg: Config, d: int | None = None) -> list[Injection]:
    d = cfg.d if d is None else d
    n, m = cfg.n, cfg.m
    if cfg.name.startswith("c1"):
        return [Injection(0, min(1200, n - 2 * m), "sine_burst", 50, 10.0, 3.0)]
    rng = np.random.default_rng([cfg.seed, 0xD15C0])
    count = min(cfg.n_discords, max(1, (n - 3 * m) // (4 * m)))  # scaled-down configs: fewer fit
    starts = _place(rng, count, n, m)
    out: list[Injection] = []
    for q, s in enumerate(starts):
        if cfg.kind == "periodic_mix":
            nstreams = int(rng.integers(1, 4))
            sids = rng.choice(d, size=nstreams, replace=False)
            for sid in sids:
                out.append(Injection(int(sid), s, "sine_burst", m, m / 5.0, 3.0))
        elif cfg.kind == "ar1_daily":
            sid = int(rng.integers(0, d))
            if q % 2 == 0:
                out.append(Injection(sid, s, "level_shift", m, 0.0, 4.0))
            else:
                out.append(Injection(sid, s + m // 2, "spike", 1, 0.0, 10.0))
        elif cfg.kind == "randwalk":
            sid = int(rng.integers(0, d))
            out.append(Injection(sid, s, "sine_burst", m, 51.0, 3.0))
        elif cfg.kind == "seasonal_noise":
            sid = int(rng.integers(0, d))
            if q % 2 == 0:
                out.append(Injection(sid, s, "level_shift", m, 0.0, 4.0))
            else:
                out.append(Injection(sid, s, "sine_burst", m, m / 5.0, 3.0))
    return out


def _apply(x: np.ndarray, inj: Injection, sigma: float) -> None:
    a = inj.amp_sigmas * sigma
    if inj.kind == "sine_burst":
        u = np.arange(inj.length, dtype=np.float64)
        x[inj.t:inj.t + inj.length] += a * np.sin(2.0 * math.pi * u / inj.period)
    elif inj.kind == "level_shift":
        x[inj.t:inj.t + inj.length] += a
    elif inj.kind == "spike":
        x[inj.t] += a


def stream(cfg: Config, sid: int, injs: list[Injection] | None = None) -> np.ndarray:
    """One stream (FP64), with the config's injections for this id applied."""
    x = _base_stream(cfg, sid, cfg.n)
    mine = [q for q in (injs if injs is not None else injections(cfg)) if q.sid == sid]
    if mine:
        sigma = float(np.std(x))  # amplitude scale only (pre-injection population std)
        for q in mine:
            _apply(x, q, sigma)
    return x


def streams(cfg: Config, ids=None, *, out: np.ndarray | None = None, threads: int | None = None) -> np.ndarray:
    """d x n array (config dtype) of streams with the given ids (default 0..d-1)."""
    ids = np.arange(cfg.d) if ids is None else np.asarray(ids)
    injs = injections(cfg)
    if out is None:
        out = np.empty((len(ids), cfg.n), dtype=cfg.np_dtype)
    threads = threads or min(32, os.cpu_count() or 1)

    def work(r):
        out[r] = stream(cfg, int(ids[r]), injs)

    if len(ids) * cfg.n < 2_000_000 or threads == 1:
        for r in range(len(ids)):
            work(r)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(len(ids))))
    return out


def stream_ids(cfg: Config) -> np.ndarray:
    return np.arange(cfg.d, dtype=np.uint64)


def dense_S(cfg: Config) -> np.ndarray:
    """Dense Gaussian projection (BASELINE C1 'Gaussian projection matrix'), k x d, N(0,1), unscaled."""
    return np.random.default_rng([cfg.seed, 0x5EED]).standard_normal((cfg.k, cfg.d))


def dynamic_ids(cfg: Config) -> tuple[np.ndarray, np.ndarray]:
    """C4 dynamic test: ids to add (fresh random walks d..d+n_add-1) and ids to delete
    (drawn from the non-injected originals)."""
    n_add = cfg.extra.get("n_add", 0)
    n_del = cfg.extra.get("n_del", 0)
    add = np.arange(cfg.d, cfg.d + n_add, dtype=np.uint64)
    inj = {q.sid for q in injections(cfg)}
    pool = np.array([j for j in range(cfg.d) if j not in inj], dtype=np.uint64)
    rng = np.random.default_rng([cfg.seed, 0xDE1])
    dele = np.sort(rng.choice(pool, size=min(n_del, len(pool)), replace=False)).astype(np.uint64)
    return add, dele


# ----------------------------------------------------------------------------------------------
# sketch-like series for matrix-profile tests (inputs of mp_selfjoin directly)
# ----------------------------------------------------------------------------------------------

def mp_series(k: int, n: int, seed: int, kind: str = "mix", dtype=np.float64) -> np.ndarray:
    """k x n series with the statistics of a sketch of z-normalised streams: each row is a signed
    sum of a few independent random-walk / periodic / noise components (scaled), so windows are
    well conditioned yet structured.  `kind` in {"mix", "randwalk", "noise", "seasonal"}."""
    rng = np.random.default_rng([seed, 0x5E51E5])
    t = np.arange(n, dtype=np.float64)
    out = np.empty((k, n), dtype=np.float64)
    for g in range(k):
        if kind == "randwalk":
            x = np.cumsum(rng.standard_normal(n))
        elif kind == "noise":
            x = rng.standard_normal(n)
        elif kind == "seasonal":
            x = np.sin(2 * math.pi * t / rng.integers(50, 500) + rng.uniform(0, 6.3)) + 0.2 * rng.standard_normal(n)
        else:
            rw = np.cumsum(rng.standard_normal(n))
            rw = (rw - rw.mean()) / (rw.std() + 1e-30)
            per = np.sin(2 * math.pi * t / rng.integers(30, 400) + rng.uniform(0, 6.3))
            x = rw + per + 0.3 * rng.standard_normal(n)
        out[g] = x
    return out.astype(dtype)


def mp_series_torch(k: int, n: int, seed: int, device, dtype):
    """Large sketch-like series generated with torch (Philox on the device) for full-size GPU
    cases; same family as mp_series(kind='mix') but a different random stream.  Input plumbing."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    t = torch.arange(n, device=device, dtype=torch.float64)
    out = torch.empty((k, n), device=device, dtype=torch.float64)
    for r in range(k):
        rw = torch.cumsum(torch.randn(n, generator=g, device=device, dtype=torch.float64), 0)
        rw = (rw - rw.mean()) / rw.std(unbiased=False)
        per = torch.sin(2 * math.pi * t / (30 + 370 * torch.rand(1, generator=g, device=device, dtype=torch.float64))
                        + 6.3 * torch.rand(1, generator=g, device=device, dtype=torch.float64))
        out[r] = rw + per + 0.3 * torch.randn(n, generator=g, device=device, dtype=torch.float64)
    return out.to(dtype)


def streams_torch(cfg: Config, device, ids=None, dtype=None):
    """Large-config streams generated on `device` with torch (Philox), same recipe families as
    `streams` but a different random stream (documented in DESIGN.md).  Used by bench.py for C5
    where the numpy recipe would cost minutes of host time.  Input plumbing."""
    import torch
    ids = np.arange(cfg.d) if ids is None else np.asarray(ids)
    dtype = dtype or (torch.float64 if cfg.dtype == "f64" else torch.float32)
    n = cfg.n
    out = torch.empty((len(ids), n), device=device, dtype=dtype)
    t = torch.arange(n, device=device, dtype=torch.float32)
    injs = injections(cfg)
    by_sid: dict[int, list[Injection]] = {}
    for q in injs:
        by_sid.setdefault(q.sid, []).append(q)
    g = torch.Generator(device=device)
    for r, sid in enumerate(ids):
        g.manual_seed(cfg.seed * 1_000_003 + int(sid))
        if cfg.kind == "randwalk":
            x = torch.cumsum(torch.randn(n, generator=g, device=device, dtype=torch.float64), 0)
        elif cfg.kind == "seasonal_noise":
            a = 0.5 + torch.rand(1, generator=g, device=device)
            th = 2 * math.pi * torch.rand(1, generator=g, device=device)
            x = (a * torch.sin(2 * math.pi * t / 10080.0 + th)).double() \
                + 0.2 * torch.randn(n, generator=g, device=device, dtype=torch.float64)
        else:
            x = torch.from_numpy(_base_stream(cfg, int(sid), n)).to(device)
        mine = by_sid.get(int(sid), [])
        if mine:
            sigma = float(x.std(unbiased=False))
            for q in mine:
                a = q.amp_sigmas * sigma
                if q.kind == "sine_burst":
                    u = torch.arange(q.length, device=device, dtype=torch.float64)
                    x[q.t:q.t + q.length] += a * torch.sin(2 * math.pi * u / q.period)
                elif q.kind == "level_shift":
                    x[q.t:q.t + q.length] += a
                else:
                    x[q.t] += a
        out[r] = x.to(dtype)
    return out
