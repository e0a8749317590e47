"""Time the join kernel alone on a C4/C5-shaped sketch (k x n FP32, synthetic, on device)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_03393_b200 as skmp
import synthgen

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--reseed", type=int, default=0)
ap.add_argument("--ab", type=int, default=0, help="AB-join: test length nA (train = --n)")
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
R = synthgen.mp_series_torch(a.k, a.n, 7, "cuda", dt)
if a.ab:
    RA = synthgen.mp_series_torch(a.k, a.ab, 8, "cuda", dt)
    cells = a.k * (a.ab - a.m + 1) * (a.n - a.m + 1)
    skmp.mp_abjoin(RA, R, a.m, reseed_rows=a.reseed, both=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); skmp.mp_abjoin(RA, R, a.m, reseed_rows=a.reseed, both=True); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    lanes = 128 if a.dtype == "f32" else 64
    print(f"AB-join k={a.k} nA={a.ab} nB={a.n} m={a.m} {a.dtype}: {t:.2f} ms (create + both passes + both finalizes), "
          f"{cells / t * 1e3:.3e} cells/s, pipe {cells / t * 1e3 * 4 / (148 * lanes * 1.965e9):.3f}")
    sys.exit(0)
n_sub = a.n - a.m + 1
excl = (a.m + 1) // 2
aa = n_sub - excl - 1
cells = a.k * aa * (aa + 1) // 2
w = skmp.mp_create(R, a.m, reseed_rows=a.reseed)
skmp.mp_join(w)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    w2 = skmp.mp_create(R, a.m, reseed_rows=a.reseed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); skmp.mp_join(w2); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)); w2.free()
t = min(ts)
print(f"D={os.environ.get('SKMP_JOIN_D','8')} k={a.k} n={a.n} m={a.m} {a.dtype}: join {t:.2f} ms, "
      f"{cells / t * 1e3:.3e} cells/s, pipe {cells / t * 1e3 * 4 / (148 * (128 if a.dtype=='f32' else 64) * 1.965e9):.3f}")
