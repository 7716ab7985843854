"""Small solves that launch every default kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck). Each line names the kernel
variant that ran; exit status 1 if any slot fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06779_b200 as pd  # noqa: E402
from paper_1609_06779_b200 import workload as W  # noqa: E402

ctx = pd.Context(0)
bad = 0


def run(algo, n, B, sel=0):
    global bad
    cell = W.workload_seed(7, n, B)
    ctx.set_models(W.workload_chains(cell, n, B), None)
    ctx.set_selection_batch(sel)
    q, qd, tau = W.workload_inputs(cell, n, B, 0)
    qdd, st, _, _ = ctx.solve(algo, q, qd, tau)
    ctx.set_selection_batch(0)
    ok = (st == 0).all() and np.isfinite(qdd).all()
    bad += not ok
    print(f"{algo.name:5s} n={n:4d} B={B:6d} sel={sel}: {ctx.last_variant()}  {'ok' if ok else 'FAILED'}", flush=True)


A, J, C = pd.FdAlgo.abia, pd.FdAlgo.jsiia, pd.FdAlgo.cfa
run(A, 16, 300)            # abia_ring_kernel (<64> tiles)
run(A, 32, 600, 65536)     # abia_ring_kernel<224>, 2 tiles per CTA when the grid is full
run(A, 8, 40)              # lane / ring, small
run(A, 8, 148 * 224 + 77)  # abia_ring_kernel<224>: 2 tiles through one CTA's ring, ragged last tile
run(A, 8, 600, 1 << 20)    # abia_ring8_kernel (256-chain tiles, setmaxnreg register split)
run(A, 70, 3)              # abia_cta_kernel
run(J, 32, 200)            # jsiia_dmma_kernel
run(J, 64, 100)            # jsiia_dmma_kernel, 8 blocks
run(J, 100, 6)             # jsiia_tiled_kernel
run(J, 300, 1)             # cooperative grid Cholesky + wavefront solves
run(J, 1050, 1)            # more tile rows (33) than solve warps (16)
run(C, 40, 100)            # cfa_row_kernel
run(C, 64, 300, 1 << 20)   # tau_surplus_lane_kernel + cfa_row_kernel
run(C, 300, 2)             # cfa_cta_kernel / coop OEE
run(C, 700, 1)             # cooperative OEE
# inverse dynamics, link states, M, the building blocks, operator builders, device workloads
n, B = 12, 64
cell = W.workload_seed(3, n, B)
links = W.workload_chains(cell, n, B)
q, qd, tau = W.workload_inputs(cell, n, B, 0)
ctx.set_models(links, None)
ctx.inverse_dynamics(q, qd, tau)
ctx.link_states(q, qd, tau)
ctx.joint_space_inertia(q)
rel, base, tr, sc = ctx.assemble_kinematics(q)
Jm = ctx.link_inertias()
ctx.articulated_body_inertias(tr, Jm, sc)
Wb = ctx.constraint_basis(sc.reshape(-1, 6)).reshape(B, n, 6, 5)
ops = ctx.cfa_operators(Jm, tr, sc, Wb)
ctx.cfa_apply(0, ops, q)
rng = np.random.default_rng(1)
ctx.block_bidiag_solve6(rng.standard_normal((4, 9, 6, 6)) * 0.3, rng.standard_normal((4, 10, 6)))
d = np.tile(np.eye(5) * 4.0, (4, 10, 1, 1))
ctx.block_tridiag_solve5(d, np.tile(np.eye(5) * 0.5, (4, 9, 1, 1)), rng.standard_normal((4, 10, 5)))
ctx.block_bidiag_solve(rng.standard_normal((3, 20, 3, 3)) * 0.3, rng.standard_normal((3, 21, 3)), True)
d2 = np.tile(np.eye(2) * 4.0, (3, 12, 1, 1))
ctx.block_tridiag_solve(d2, np.tile(np.eye(2) * 0.5, (3, 11, 1, 1)), rng.standard_normal((3, 12, 2, 3)))
st = pd.OeeState(d2[0].copy(), np.tile(np.eye(2) * 0.5, (11, 1, 1)), rng.standard_normal((12, 2)))
pd.oee_eliminate_round(st, ctx=ctx)
pd.oee_eliminate_round(st, ctx=ctx)
ms, _ = ctx.set_models_workload(W.workload_seed(42, 20, 500), 20, 500)
print("operators / ID / building blocks / device workload: done", flush=True)
sys.exit(1 if bad else 0)
