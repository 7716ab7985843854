"""Diagnostic: device-path solves (pd_forward_dynamics_device) vs host-path
solves for each algorithm; prints timings and max differences."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1609_06779_b200 as pd
from paper_1609_06779_b200 import workload as W

ctx = pd.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
for algo, n, B in (("abia", 32, 65536), ("jsiia", 32, 65536), ("cfa", 256, 4096), ("abia", 1024, 1)):
    cell = W.workload_seed(42, n, B)
    links = W.workload_chains(cell, n, B)
    q, qd, tau = W.workload_inputs(cell, n, B, 0)
    ctx.set_models(links, None)
    ref, st, _, _ = ctx.solve(pd.FdAlgo[algo], q, qd, tau)
    dq, dqd, dtau = (torch.from_numpy(np.ascontiguousarray(a.T)).cuda() for a in (q, qd, tau))
    dqdd = torch.zeros((n, B), dtype=torch.float64, device="cuda")
    dst = torch.full((3, B), -1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.solve_device(pd.FdAlgo[algo], B, dq.data_ptr(), dqd.data_ptr(), dtau.data_ptr(), dqdd.data_ptr(),
                     dst[0].data_ptr(), dst[1].data_ptr(), dst[2].data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    got = dqdd.cpu().numpy().T
    print(algo, n, B, "ms", e0.elapsed_time(e1), "launches", ctx.kernel_launches() - l0,
          "status", np.unique(dst[0].cpu().numpy()), "host status", np.unique(st),
          "max|dev-host|", np.abs(got - ref).max(), flush=True)
