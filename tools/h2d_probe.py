"""Probe (diagnostic): repeated 8 GB pinned H2D copies, to separate host/PCIe variance from the library."""
import torch, time
x = torch.empty(10000, 200000).pin_memory()
y = torch.empty(10000, 200000, device="cuda")
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"copy {i}: {dt*1e3:7.1f} ms  {x.numel()*4/dt/1e9:6.1f} GB/s", flush=True)
