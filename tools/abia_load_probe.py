"""ABIA ring kernel time vs how many SMs stream at once (c2 chains, n = 32,
224-chain tiles forced by the selection batch): B = k x 224 for k CTAs of one
tile each, then 2 tiles per CTA. Separates the per-tile latency of the
passes from the HBM contention when every SM runs pass A together.
Usage: python tools/abia_load_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1609_06779_b200 import Context  # noqa: E402
from paper_1609_06779_b200 import workload as W  # noqa: E402

n = 32
ctx = Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
ctx.set_selection_batch(65536)
for k in [1, 8, 37, 74, 111, 148, 222, 296]:
    B = 224 * k
    cell = W.workload_seed(42, n, B)
    ctx.set_models_workload(cell, n, B)
    q, qd, tau = W.workload_inputs(cell, n, B, 0)
    dev = [tuple(torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in (q, qd, tau))]
    ms, _, _ = bench.time_device(ctx, "abia", B, n, dev, 50, 5, stream)
    us = ms / 50 * 1e3
    print(f"ctas-worth {k:4d}  B {B:6d}  {us:8.1f} us/launch  {ctx.last_variant()}  "
          f"{B * 256 * n / us / 1e3:7.1f} GB/s algorithmic", flush=True)
