"""The multi-GPU path with the real kernels: two processes (one pd_ctx each,
the way torchrun runs one rank per GPU; here both ranks share cuda:0, the only
device a test box has) each generate their contiguous shard of a c5-shaped
batch on the device (pd_set_models_workload with the shard's first chain),
solve it with kernels selected for the whole batch (pd_set_selection_batch),
and rank 0 gathers the rows over gloo. The gathered q̈ must be bit-identical to
one process solving the whole batch -- SURVEY.md §8e, the GPU analogue of
acceptance_main.cpp:495-580."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, B = 64, 40000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve(ctx, algo, cell, lo, hi):
    import torch
    from paper_1609_06779_b200 import workload as W
    ms, _ = ctx.set_models_workload(cell, N, hi - lo, g0=lo)
    assert (ms == 0).all()
    q, qd, tau = (np.ascontiguousarray(a[lo:hi]) for a in W.workload_inputs(cell, N, B, 0))
    dev = torch.device("cuda", 0)
    dq, dqd, dtau = (torch.from_numpy(np.ascontiguousarray(a.T)).to(dev) for a in (q, qd, tau))
    dqdd = torch.empty((N, hi - lo), dtype=torch.float64, device=dev)
    st = torch.empty((3, hi - lo), dtype=torch.int32, device=dev)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.solve_device(algo, hi - lo, dq.data_ptr(), dqd.data_ptr(), dtau.data_ptr(), dqdd.data_ptr(), st[0].data_ptr(),
                     st[1].data_ptr(), st[2].data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    assert (st[0] == 0).all()
    return dqdd.cpu().numpy().T.copy()


def _worker(rank, world, port, out_path, algo_name):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1609_06779_b200 as pd
    from paper_1609_06779_b200 import workload as W
    from paper_1609_06779_b200.sharding import gather_rows, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = pd.Context(0)
    ctx.set_selection_batch(B)
    lo, hi = shard_bounds(B, world, rank)
    qdd = _solve(ctx, pd.FdAlgo[algo_name], W.workload_seed(42, N, B), lo, hi)
    full = gather_rows(qdd, B, world, rank)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("algo", ["abia", "cfa"])
def test_two_process_shards_are_bit_identical(tmp_path, algo):
    import paper_1609_06779_b200 as pd
    from paper_1609_06779_b200 import workload as W
    out = str(tmp_path / "qdd.npy")
    mp.spawn(_worker, args=(2, _free_port(), out, algo), nprocs=2, join=True)
    got = np.load(out)
    ctx = pd.Context(0)
    whole = _solve(ctx, pd.FdAlgo[algo], W.workload_seed(42, N, B), 0, B)
    assert got.shape == whole.shape
    assert np.array_equal(got, whole)
