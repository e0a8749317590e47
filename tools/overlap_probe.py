"""Probe (diagnostic): does a large pinned H2D copy on one stream overlap a join on another?
Events on both streams, no threads.   python tools/overlap_probe.py"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np, torch
import paper_2311_03393_b200 as skmp
dev = torch.device("cuda:0")
d, n, k, m = 10000, 200000, 64, 256
hostT = torch.randn(d, n).pin_memory()
buf = torch.empty(d, n, device=dev)
R = torch.randn(k, n, device=dev).cumsum_(1)
sA, sB = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ids = np.arange(d, dtype=np.uint64)
for mode in ("copy alone", "join alone", "join then copy", "join then sketch_build", "copy then join"):
    torch.cuda.synchronize()
    z, ja, jb, ca, cb = E(), E(), E(), E(), E()
    torch.cuda.current_stream().record_event(z)
    sA.wait_event(z); sB.wait_event(z)
    def do_join():
        with torch.cuda.stream(sA):
            ja.record(); w = skmp.mp_create(R, m); skmp.mp_join(w); jb.record()
        return w
    def do_copy():
        with torch.cuda.stream(sB):
            ca.record(); buf.copy_(hostT, non_blocking=True); cb.record()
    w = None
    if mode == "copy alone":
        do_copy()
    elif mode == "join alone":
        w = do_join()
    elif mode == "join then copy":
        w = do_join(); do_copy()
    elif mode == "copy then join":
        do_copy(); w = do_join()
    else:
        w = do_join()
        with torch.cuda.stream(sB):
            ca.record(); sk = skmp.sketch_build(hostT, ids, k, seed=1); cb.record()
    torch.cuda.synchronize()
    out = [mode]
    if w is not None:
        out.append(f"join {z.elapsed_time(ja):7.1f} -> {z.elapsed_time(jb):7.1f} ms")
        w.free()
    if mode != "join alone":
        out.append(f"copy {z.elapsed_time(ca):7.1f} -> {z.elapsed_time(cb):7.1f} ms")
    print(" | ".join(out), flush=True)
