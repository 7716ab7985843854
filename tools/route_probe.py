"""Time one workload's device solve under different kernel-selection batches
(pd_set_selection_batch), i.e. the alternative routes the dispatcher has for
the same problems. Usage: python tools/route_probe.py WORKLOAD SEL [SEL ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1609_06779_b200 import Context, FdAlgo  # noqa: E402

name = sys.argv[1]
wl = bench.WORKLOADS[name]
ctx = Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
links, inp, _ = bench.gen_workload(wl, 0)
if isinstance(links, bench.DeviceChains):
    ctx.set_models_workload(links.cell, wl["n"], links.count, g0=links.g0)
else:
    ctx.set_models(links, None)
B, n = inp[0].shape
dev = [tuple(torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in inp)]
base = None
for sel in map(int, sys.argv[2:]):
    ctx.set_selection_batch(sel)
    ms, _, qdd = bench.time_device(ctx, wl["algo"], B, n, dev, 20, 3, stream)
    out = qdd.cpu().numpy()
    if base is None:
        base = out
    gap = np.abs(out - base).max()
    print(f"{name} sel={sel}: {ms / 20:.4f} ms/step  variant {ctx.last_variant()}  max|diff| vs first {gap:.2e}",
          flush=True)
