#!/usr/bin/env python
"""bench.py — the hot path of arXiv 2311.03393 on B200: sketch -> self-join -> discord top-K.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One STEP = one pass of every SURVEY §8(a) row over one batch of synthetic input.  Default
workload C5 (BASELINE.json configs[4], the configuration BASELINE's metric "MP cell updates/s at
1/2/4/8 B200" is quoted on: d=2,000 seasonal-plus-noise streams, n=2,000,000, m=256, k=32, FP32,
50 injected discords); `--config c4` runs configs[3] (d=10,000 random walks, n=200,000, m=256,
k=64, the dynamic add-500/delete-500 configuration):
  a2-a4  sketch_build over the d streams (count sketch, Alg. 1)
  a5     sketch_add_dim of 500 new streams + sketch_del_dim of 500 originals (§3.3)
  a6-a9  mp_create (window prep) + mp_join (the diagonal recurrence) + mp_finalize
  a10-11 discord_topk (Alg. 2 combine + ordered top-K)
  f2     discord_dims over the top discord's group (Alg. 3 dimension detection)
Multi-GPU (torchrun, N>1): streams are sharded over ranks, partial sketches are sum-all-reduced
(NCCL), each rank joins its diagonal band (mp_band) and the profile keys are max-all-reduced
(NCCL); every rank finalizes a slice of the windows (reduced to rank 0), rank 0 ranks the
discords, and Alg. 3 runs on every rank's own streams of the group (all-gathered maxima).
Strong scaling (fixed total work).  `--gpus N` without a torchrun environment re-launches this
script as N ranks (python -m torch.distributed.run --nproc-per-node N, 127.0.0.1); rank 0 prints
the one JSON line.

`value` = exact join cells per step (k (n_sub-r-1)(n_sub-r)/2) / device step time, inputs
resident in HBM.  `e2e` = the same with the inputs in pinned HOST memory handed to the C-ABI
(its H2D staging inside the timed region) and the top-K read back to the host, batches
pipelined with paper_2311_03393_b200.pipeline.Prefetcher (batch s+1 staged while batch s joins).
The reference arm (--impl reference) times the ORACLE (oracle/, plain C brute force) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MP cell updates/s (k·n²/2) at 1/2/4/8 B200; sketch HBM GB/s"
UNIT = "cell updates/s"
FP32_PIPE_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # B200: 148 SMs x 128 FP32 lanes x FMA x max clock
FLOPS_PER_CELL = 6                                    # 2 FFMA (4 flop) + 2 FMUL (2 flop), DESIGN.md §5
FP64_PIPE_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
FFMA_MEASURED = 0.971    # FFMA warp-instructions / clk / SMSP measured (profiles/r1b_pipe_mix.txt)
DFMA_MEASURED = 0.4865 / 0.5  # DFMA 0.4865 warp-instr / clk / SMSP of 0.5 (profiles/r1b_fp64_rate.txt)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "c5"))
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--top", type=int, default=0, help="discords per step (default 2 x injected)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="pipelined e2e batches (default 5; 3 for C5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reseed", type=int, default=0)
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process group backend (gloo: the one-GPU multi-rank test, ranks share cuda:0)")
    ap.add_argument("--shape", default="", help="test shapes: scale the config, e.g. d=200,n=20000,k=8")
    ap.add_argument("--dump", default="", help="rank 0 writes the last step's keys / P / I / top-K here (.npz)")
    return ap.parse_args()


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: run this script as N ranks, one per GPU (the driver's own
    launch line), and pass rank 0's JSON line through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("relaunch:", " ".join(cmd))
    return subprocess.call(cmd)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def join_kernel_name(dtype: str) -> str:
    if dtype == "f32" and os.environ.get("SKMP_JOIN_IMPL", "x2")[:1] != "s" and os.environ.get("SKMP_JOIN_D", "8") == "8":
        return "join_x2_kernel (mp_join_x2.cu, packed f32x2)"
    return "join_kernel (mp_join.cu)"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def workload_desc(cfg, top):
    return (f"{cfg.name}: d={cfg.d} streams, n={cfg.n}, m={cfg.m}, k={cfg.k}, {cfg.dtype}, "
            f"{'count sketch' if cfg.proj == 'count' else 'dense projection'}, {cfg.kind}; step = "
            f"sketch_build + add {cfg.extra.get('n_add', 0)} + delete {cfg.extra.get('n_del', 0)} + "
            f"self-join + top-{top} + Alg. 3 dimension of the top discord")


# ----------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampler unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
# reference arm: the oracle on the host cores
# ----------------------------------------------------------------------------------------------
def oracle_sample(cfg, seconds: float, threads: int):
    """Time the oracle's brute-force self-join (oracle/mp_brute.c) on whole rows of one
    sketch-length series; returns (cells/s, rows, seconds).  A row-wise brute force evaluates each
    unordered pair twice, so cells = rows * admissible pairs per row / 2."""
    import synthgen
    from oracle import reference as ref
    r = synthgen.mp_series(1, cfg.n, seed=cfg.seed, kind="randwalk")[0]
    n_sub, excl = cfg.n_sub, cfg.excl
    pairs_per_row = n_sub - 2 * excl - 1
    rng = np.random.default_rng(cfg.seed)
    # calibrate with one row per thread
    rows = rng.integers(0, n_sub, threads)
    t0 = time.perf_counter()
    ref.selfjoin_rows(r, cfg.m, excl, rows=rows, threads=threads)
    dt = time.perf_counter() - t0
    nrows = max(threads, int(threads * max(1.0, (seconds - dt) / max(dt, 1e-3))))
    rows = rng.integers(0, n_sub, nrows)
    t0 = time.perf_counter()
    ref.selfjoin_rows(r, cfg.m, excl, rows=rows, threads=threads)
    dt2 = time.perf_counter() - t0
    cells = nrows * pairs_per_row / 2
    return cells / dt2, nrows, dt2


def run_reference(args, cfg, top):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    budget = max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for s in range(args.warmup + args.steps):
        v, nrows, dt = oracle_sample(cfg, budget, threads)
        if s >= args.warmup:
            vals.append((v, nrows, dt))
    value = statistics.mean(v for v, _, _ in vals)
    ms = statistics.mean(dt for _, _, dt in vals) * 1e3
    sample = (f"oracle/mp_brute.c explicit-difference brute force, {vals[-1][1]} random whole rows of one "
              f"n={cfg.n}, m={cfg.m} sketch-length series per step (~{budget:.0f} s), {threads} OpenMP threads; "
              f"cells = rows x admissible pairs / 2")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_desc(cfg, top)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu": cpu_model(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return relaunch(args)
    import synthgen
    cfg = synthgen.CONFIGS[args.config]
    if args.shape:
        cfg = synthgen.scaled(cfg, **{kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.shape.split(",")})
    top = args.top or max(3, 2 * cfg.n_discords)
    if args.e2e_steps <= 0:
        args.e2e_steps = 3 if cfg.n * cfg.d >= 4_000_000_000 else 5
    if args.impl == "reference":
        return run_reference(args, cfg, top)

    import torch
    import torch.distributed as dist

    import paper_2311_03393_b200 as skmp
    from paper_2311_03393_b200 import dist as sdist
    from paper_2311_03393_b200.pipeline import Prefetcher

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.backend == "gloo":   # test mode: every rank on one GPU, collectives staged via host
        local = local % torch.cuda.device_count()
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPUs "
                         "(one process per GPU; --backend gloo shares one GPU for tests)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    skmp.lib()
    tdt = torch.float32 if cfg.dtype == "f32" else torch.float64
    dcode = skmp.F32 if cfg.dtype == "f32" else skmp.F64

    # ---------------- inputs (generated by synthgen, resident before timing) ----------------
    t_gen = time.perf_counter()
    ids_all = synthgen.stream_ids(cfg)
    add_ids, del_ids = synthgen.dynamic_ids(cfg)
    my_ids = sdist.shard(ids_all, rank, world)
    my_add = sdist.shard(add_ids, rank, world)
    my_del = np.array([j for j in del_ids if j in set(my_ids.tolist())], dtype=np.uint64)
    pos = {int(j): q for q, j in enumerate(my_ids)}
    big = cfg.d * cfg.n >= 2_000_000_000 // world and cfg.kind == "seasonal_noise"
    if big:
        # C5 (16 GB): numpy would cost minutes of host time; same recipe family on the device
        # (synthgen.streams_torch, Philox), host copy only for the e2e leg
        Td = synthgen.streams_torch(cfg, dev, my_ids)
        Tadd = synthgen.streams_torch(cfg, dev, my_add) if len(my_add) else None
        Tdel = Td[[pos[int(j)] for j in my_del]].contiguous() if len(my_del) else None
        host_T = host_add = host_del = None
    else:
        host_T = torch.from_numpy(synthgen.streams(cfg, my_ids)).pin_memory()
        host_add = torch.from_numpy(synthgen.streams(cfg, my_add)).pin_memory() if len(my_add) else None
        host_del = host_T[[pos[int(j)] for j in my_del]].contiguous().pin_memory() if len(my_del) else None
        Td = host_T.to(dev, non_blocking=False)
        Tadd = host_add.to(dev) if host_add is not None else None
        Tdel = host_del.to(dev) if host_del is not None else None
    torch.cuda.synchronize()
    log(f"[rank {rank}] inputs ready in {time.perf_counter() - t_gen:.1f}s: T {tuple(Td.shape)}, "
        f"add {0 if Tadd is None else Tadd.shape[0]}, del {0 if Tdel is None else Tdel.shape[0]}")

    n_sub, excl, m, k = cfg.n_sub, cfg.excl, cfg.m, cfg.k
    ranges = sdist.rank_diagonals(n_sub, excl, dcode, world, rank)
    cells_total = cfg.cells()
    cells_band = 0  # cells this rank's join launches compute (incl. the shared first block)
    for lo, hi in ranges:
        a0 = max(lo, excl + 1)
        b0 = min(max(hi, a0), n_sub)
        cells_band += k * ((b0 - a0) * n_sub - (b0 * (b0 - 1) - a0 * (a0 - 1)) // 2)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    S_dense = synthgen.dense_S(cfg)[:, [int(j) for j in my_ids]] if cfg.proj == "dense" else None
    dumpbox: dict = {}

    def build(T):
        if S_dense is not None:  # C1's Gaussian projection (reading 1)
            return skmp.sketch_build(T, my_ids, k, proj=skmp.PROJ_DENSE, S=S_dense)
        return skmp.sketch_build(T, my_ids, k, seed=cfg.seed)

    def stage(T, Ta, Tdl, e=None):
        """a1-a5 of one batch: sketch of the rank's streams + add / delete (no collective)."""
        sk = build(T)
        if e: e[1].record()
        if Ta is not None:
            skmp.sketch_add_dim(sk, Ta, my_add)
        if Tdl is not None:
            skmp.sketch_del_dim(sk, Tdl, my_del)
        return sk

    def step(T, Ta, Tdl, timers=None, sk=None, on_join=None):
        e = [ev() for _ in range(7)] if timers is not None else None
        if e: e[0].record()
        if sk is None:
            sk = stage(T, Ta, Tdl, e)
        elif e:
            e[1].record()
        if world > 1:
            sdist.allreduce_sketch(sk)
        if e: e[2].record()
        if args.dump:
            dumpbox["R"] = sk.R.cpu().numpy()
            dumpbox["R64"] = sk.R64.cpu().numpy()
        w = skmp.mp_create(sk.R, m, reseed_rows=args.reseed)
        if e: e[3].record()
        for lo, hi in ranges:
            if hi > lo:
                skmp.mp_join(w, lo, hi)
        if on_join is not None:  # e2e pipeline: stage the next batch while this join runs
            on_join()
        if e: e[4].record()
        if world > 1:
            keys, words = skmp.mp_keys(w)
            sdist.reduce_keys(keys, words)
        if args.dump:
            dumpbox["keys"] = skmp.mp_keys(w)[0].cpu().numpy()
        res = None
        if world > 1:  # every rank resolves a slice of the windows, P / I reduced to rank 0
            fin = sdist.finalize_dist(w)
        else:
            fin = skmp.mp_finalize(w)
        if rank == 0:
            P, I, inert = fin
            res = skmp.discord_topk(P, I, inert, m=m, top=top)
            if args.dump:
                dumpbox.update(P=P.cpu().numpy(), I=I.cpu().numpy(), inert=inert,
                               top=np.array([(d.t, d.g, d.nn) for d in res]),
                               top_score=np.array([d.score for d in res]))
        w.free()
        if e: e[5].record()
        # Alg. 3: the dimension j* of the top discord inside its group J_g*
        tg = torch.tensor([res[0].t, res[0].g] if rank == 0 else [0, 0], dtype=torch.int64, device=dev)
        if world > 1:
            sdist.broadcast(tg, 0)
        t_star, g_star = (int(x) for x in tg.tolist())
        sources = [(T, my_ids), (Ta, my_add)]
        if world > 1:
            dim = sdist.detect_dimension_dist(sk, sources, t_star, g_star, m, dev)
        else:
            dim = skmp.detect_dimension(sk, sources, t_star, g_star, m)
        sk.free()
        if args.dump:
            dumpbox["dim"] = np.array([] if dim is None else [dim[0], dim[2]], dtype=np.uint64)
            dumpbox["dim_score"] = np.array([] if dim is None else [dim[1]])
        if e:
            e[6].record()
            timers.append(e)
        return res, dim

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- warm-up + timed region (inputs in HBM) ----------------
    for _ in range(max(3, args.warmup)):
        step(Td, Tadd, Tdel)
    barrier()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    timers: list = []
    launches0 = skmp.skmp_launch_count()
    barrier()
    t_start, t_end = ev(), ev()
    t_start.record()
    res = None
    for _ in range(args.steps):
        res = step(Td, Tadd, Tdel, timers)
    t_end.record()
    barrier()
    launches = skmp.skmp_launch_count() - launches0
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    phase = {
        "sketch_build_ms": statistics.mean(e[0].elapsed_time(e[1]) for e in timers),
        "add_del_ms": statistics.mean(e[1].elapsed_time(e[2]) for e in timers),
        "mp_prep_ms": statistics.mean(e[2].elapsed_time(e[3]) for e in timers),
        "mp_join_ms": statistics.mean(e[3].elapsed_time(e[4]) for e in timers),
        "finalize_topk_ms": statistics.mean(e[4].elapsed_time(e[5]) for e in timers),
        "alg3_dims_ms": statistics.mean(e[5].elapsed_time(e[6]) for e in timers),
    }
    t = torch.tensor([elapsed_ms, phase["mp_join_ms"]], device=dev, dtype=torch.float64)
    if world > 1:
        sdist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, join_ms_max = float(t[0]), float(t[1])
    ms_per_step = elapsed_ms / args.steps
    value = cells_total / (ms_per_step / 1e3)

    # ---------------- e2e: host (pinned) inputs through the C-ABI ----------------
    e2e = None
    if not args.no_e2e and host_T is None:
        try:  # pinned host copies of the device-generated inputs (needs ~d*n*4 bytes of host RAM)
            def pinned(x):
                return torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x)
            host_T = pinned(Td)
            host_add = pinned(Tadd) if Tadd is not None else None
            host_del = pinned(Tdel) if Tdel is not None else None
        except RuntimeError as ex:
            log(f"[rank {rank}] e2e skipped: {ex}")
    dim_rows = None
    if not args.no_e2e and host_T is not None:
        step(host_T, host_add, host_del)  # warm the staging pool
        # members of the top discord's group (the streams Alg. 3 stages each step), all ranks
        gsk = build(Td)
        if Tadd is not None:
            skmp.sketch_add_dim(gsk, Tadd, my_add)
        if Tdel is not None:
            skmp.sketch_del_dim(gsk, Tdel, my_del)
        gt = torch.tensor([res[0][0].g if rank == 0 else 0], dtype=torch.int64, device=dev)
        if world > 1:
            sdist.broadcast(gt, 0)
        dim_rows = len(skmp.group_rows(gsk, int(gt.item())))
        gsk.free()
        pf = Prefetcher(dev)
        # warm the pipelined path once (prefetch stream, its pool blocks, the handoff)
        pending = [pf.run(stage, host_T, host_add, host_del)]
        pf.handoff()
        step(host_T, host_add, host_del, sk=pending.pop(0),
             on_join=lambda: pending.append(pf.run(stage, host_T, host_add, host_del)))
        pf.handoff()
        pending.pop(0).free()
        barrier()
        # batches pipelined: batch s+1's H2D staging + sketch (a1-a5, on the prefetch stream,
        # issued right after batch s's join launch) overlaps that join; every batch's inputs
        # still cross PCIe inside the timed region, which starts before batch 0's staging
        s0, s1 = ev(), ev()
        s0.record()
        dbg = os.environ.get("BENCH_DEBUG_E2E")
        tl, bl = [], []

        def staged(*a):
            if dbg:
                bl.append((ev(), ev()))
                bl[-1][0].record()
            out = stage(*a)
            if dbg:
                bl[-1][1].record()
            return out
        pending = [pf.run(staged, host_T, host_add, host_del, after=s0)]

        def prefetch():
            pending.append(pf.run(staged, host_T, host_add, host_del))
        for b in range(args.e2e_steps):
            pf.handoff()
            step(host_T, host_add, host_del, sk=pending.pop(0), timers=tl if dbg else None,
                 on_join=prefetch if b + 1 < args.e2e_steps else None)
        s1.record()
        barrier()
        if dbg:
            for b, e in enumerate(tl):
                log(f"  A step {b}: " + " ".join(f"{s0.elapsed_time(x):7.1f}" for x in e))
            for b, (x, y) in enumerate(bl):
                log(f"  B stage {b}: {s0.elapsed_time(x):7.1f} -> {s0.elapsed_time(y):7.1f}")
        et = torch.tensor([s0.elapsed_time(s1)], device=dev, dtype=torch.float64)
        if world > 1:
            sdist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms = float(et[0]) / args.e2e_steps
        esz = host_T.element_size()
        h2d = (host_T.numel() + (0 if host_add is None else host_add.numel())
               + (0 if host_del is None else host_del.numel())) * esz
        h2d += dim_rows * cfg.n * esz  # Alg. 3 stages its group's host rows
        if world > 1:
            hb = torch.tensor([h2d], device=dev, dtype=torch.float64)
            sdist.all_reduce(hb)
            h2d = int(hb.item())
        d2h = top * (8 + 4 + 8 + 8) + 4 + 16  # top-K tuples + count + Alg. 3 result
        e2e = {"value": cells_total / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "pipelined": "batch s+1's H2D + sketch (Prefetcher stream, issued after batch s's join launch) "
                            "overlaps that join; "
                            "timed from before batch 0's staging to batch K-1's results on the host"}

    if rank != 0:
        dist.destroy_process_group()
        return 0
    if args.dump:
        np.savez(args.dump, **dumpbox)

    # ---------------- roofline of the dominant kernel (the join) ----------------
    pk = peaks()
    join_flops = cells_band * FLOPS_PER_CELL
    achieved = join_flops / (phase["mp_join_ms"] / 1e3) / 1e12
    peak = FP32_PIPE_TFLOPS if cfg.dtype == "f32" else FP64_PIPE_TFLOPS
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "join_traffic.json")))
        for ent in (prof if isinstance(prof, list) else [prof]):   # one entry per config (ncu captures)
            if ent.get("config") == cfg.name and ent.get("world", 1) == world:
                traffic = ent["dram_bytes_per_launch"]
    except Exception:
        pass
    sk_bytes = 2 * cfg.d * cfg.n * (4 if cfg.dtype == "f32" else 8) // world + \
        cfg.k * cfg.n * (8 + (4 if cfg.dtype == "f32" else 0))
    sk_gbs = sk_bytes / (phase["sketch_build_ms"] / 1e3) / 1e9
    hbm_peak = pk.get("hbm_gbs", 6557.1)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": workload_desc(cfg, top), "cells_per_step": cells_total,
                   "nominal_cells_k_n2_over_2": cfg.k * cfg.n * cfg.n // 2,
                   "l2": "inputs larger than L2 (no flush needed)",
                   "parallelism": f"streams sharded x{world} + sum-allreduce; diagonal bands x{world} + max-allreduce"
                   if world > 1 else "single GPU"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": join_kernel_name(cfg.dtype),
                     "note": f"{FLOPS_PER_CELL} algorithmic FLOP per cell x cells of this rank's band / mean "
                             f"mp_join event time; peak = 148 SM x {128 if cfg.dtype == 'f32' else 64} lanes x 2 x "
                             f"1.965 GHz (derived, DESIGN.md §5)",
                     "pipe_frac": (cells_band / (phase['mp_join_ms'] / 1e3)) * 4 /
                                  (148 * (128 if cfg.dtype == 'f32' else 64) * 1.965e9),
                     "peak_measured": peak * (FFMA_MEASURED if cfg.dtype == "f32" else DFMA_MEASURED),
                     "peak_measured_note": "dependent-chain microbenchmark on one B200 (FFMA 0.971 warp-instr/clk/SMSP, "
                                           "profiles/r1b_pipe_mix.txt; DFMA profiles/r1b_fp64_rate.txt): the issue "
                                           "rate a plain FMA stream actually reaches; frac is against the derived peak"},
        "sketch": {"bound": "hbm", "achieved": sk_gbs, "peak": hbm_peak, "unit": "GB/s",
                   "frac": sk_gbs / hbm_peak, "bytes_per_build": sk_bytes,
                   "note": "algorithmic bytes 2 d n b + k n (8 + b) over sketch_build event time (includes its "
                           "flag D2H); peak = MEASURED_PEAKS.json hbm_gbs (of measured)"},
        "phases_ms": phase,
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
    }
    if res is not None:
        res, dim = res
        out["top"] = [(d.t, d.g, round(d.score, 4)) for d in res[:8]]
        if dim is not None:
            out["alg3"] = {"t": res[0].t, "g": res[0].g, "j_star_id": dim[0], "score": round(dim[1], 4),
                           "nn": dim[2]}
    if world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        v, nrows, dt = oracle_sample(cfg, 12.0, threads)
        out["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": threads, "cpu": cpu_model(), "kind": "oracle",
            "sample": f"oracle/mp_brute.c brute force on {nrows} random whole rows of one n={cfg.n}, m={cfg.m} "
                      f"series ({dt:.1f} s); cells = rows x admissible pairs / 2"}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
