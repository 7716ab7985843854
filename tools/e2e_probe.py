"""Where the host-buffer (e2e) time goes: pinned H2D / D2H bandwidth of the
c2 inputs and outputs, and Context.solve wall time vs chunk count."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06779_b200 as pd  # noqa: E402
from paper_1609_06779_b200 import workload as W  # noqa: E402

n, B = 32, 65536
x = torch.empty((3, B, n), dtype=torch.float64).pin_memory()
y = torch.empty((B, n), dtype=torch.float64).pin_memory()
d = torch.empty((3, B, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t0) / 10
t0 = time.perf_counter()
for _ in range(10):
    y.copy_(d[0], non_blocking=True)
torch.cuda.synchronize()
d2h = (time.perf_counter() - t0) / 10
print(f"H2D {x.numel() * 8 / h2d / 1e9:.1f} GB/s ({h2d * 1e3:.3f} ms for {x.numel() * 8 / 2**20:.0f} MiB); "
      f"D2H {y.numel() * 8 / d2h / 1e9:.1f} GB/s ({d2h * 1e3:.3f} ms)")
ctx = pd.Context(0)
cell = W.workload_seed(42, n, B)
links = W.workload_chains(cell, n, B)
q, qd, tau = W.workload_inputs(cell, n, B, 0)
ctx.set_models(links, None)
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (q, qd, tau)]
out = torch.empty((B, n), dtype=torch.float64).pin_memory().numpy()
for algo in ("abia", "jsiia"):
    for _ in range(3):
        ctx.solve(pd.FdAlgo[algo], *pin, out=out)
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.solve(pd.FdAlgo[algo], *pin, out=out)
    dt = (time.perf_counter() - t0) / 20
    print(f"solve {algo}: {dt * 1e3:.3f} ms/step, {B / dt / 1e6:.1f} M solves/s (chunks env {os.environ.get('PD_E2E_CHUNKS')})")

# raw PCIe duplex: H2D of the inputs and D2H of an output on separate streams at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty((B, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
both = (time.perf_counter() - t0) / 10
print(f"H2D + D2H concurrently: {both * 1e3:.3f} ms (serial would be {(h2d + d2h) * 1e3:.3f} ms)")
