"""World-size-2 gloo run of the multi-GPU host path on CPU: each rank takes
its contiguous shard of one batch, solves it (the oracle stands in for the
device here -- this exercises partition and gather, not the kernels), and
rank 0 gathers; the result must be bit-identical to the unsharded solve
(acceptance_main.cpp:495-580's worker-count determinism, across ranks)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import pyoracle as po
    from paper_1609_06779_b200.sharding import gather_rows, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, B = 8, 37
    cell = po.workload_seed(42, n, B)
    b, e = shard_bounds(B, world, rank)
    links = po.workload_chains(cell, n, e - b, g0=b)
    q, qd, tau = (x[b:e] for x in po.workload_inputs(cell, n, B, 0))
    qdd, st = po.batch_forward_dynamics("abia", links, [0, 0, -9.81], q, qd, tau, nthreads=1)
    assert (st == 0).all()
    full = gather_rows(qdd, B, world, rank)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path, oracle):
    out = str(tmp_path / "qdd.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    n, B = 8, 37
    cell = oracle.workload_seed(42, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    ref, _ = oracle.batch_forward_dynamics("abia", links, [0, 0, -9.81], q, qd, tau, nthreads=1)
    assert np.array_equal(got, ref)
