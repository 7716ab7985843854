"""Timeline of one host-buffer solve (c2): per-chunk H2D / compute / D2H
completion times from the PD_E2E_TRACE events, and the call's wall time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06779_b200 as pd  # noqa: E402
from paper_1609_06779_b200 import workload as W  # noqa: E402

n, B = 32, 65536
ctx = pd.Context(0)
cell = W.workload_seed(42, n, B)
ctx.set_models(W.workload_chains(cell, n, B), None)
q, qd, tau = W.workload_inputs(cell, n, B, 0)
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (q, qd, tau)]
out = torch.empty((B, n), dtype=torch.float64).pin_memory().numpy()
sts = tuple(torch.zeros(B, dtype=torch.int32).pin_memory().numpy() for _ in range(3))
for _ in range(5):
    ctx.solve(pd.FdAlgo.abia, *pin, out=out, status_out=sts)
for mode in ("status",):
    t0 = time.perf_counter()
    for _ in range(20):
        if mode == "status":
            ctx.solve(pd.FdAlgo.abia, *pin, out=out, status_out=sts)
        else:
            ctx._check(ctx._L.pd_forward_dynamics(ctx._h, 0, B, pin[0].ctypes.data, pin[1].ctypes.data,
                                                  pin[2].ctypes.data, out.ctypes.data, None, None, None))
    print(f"{mode}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms/call", flush=True)
