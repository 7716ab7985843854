"""GPU parity of the §8f row-1/row-2 entry points through the C-ABI against the
CPU oracle: inverse dynamics with the reference's IdOptions
(inverse_dynamics.hpp:23-28), bias_torque, link_states
(inverse_dynamics.cpp:166-196) and joint_space_inertia
(forward_dynamics.cpp:70-80).

Tolerances: 1e-12 relative for torques / link states (the reference's own
sequential-NE check, tests/test_invdyn.cpp:50-110) and M (closed-form CRBA vs
the reference's column probes)."""
import numpy as np
import pytest

import paper_1609_06779_b200 as pd

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_gap(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


def batch(oracle, n, B, seed):
    links = np.stack([oracle.random_chain(n, seed + c)[0] for c in range(B)])
    rng = np.random.default_rng(seed)
    q, qd, qdd = rng.uniform(-3, 3, (B, n)), rng.uniform(-2, 2, (B, n)), rng.uniform(-5, 5, (B, n))
    return links, q, qd, qdd


def options(seed, gravity=True):
    rng = np.random.default_rng(seed)
    return pd.IdOptions(rng.uniform(-1, 1, 6), rng.uniform(-2, 2, 6), rng.uniform(-3, 3, 6), gravity)


@pytest.mark.parametrize("n", [1, 2, 7, 32, 65])
@pytest.mark.parametrize("gravity", [True, False])
def test_inverse_dynamics_options(oracle, gpu_ctx, n, gravity):
    B = 24
    links, q, qd, qdd = batch(oracle, n, B, 500 + n)
    o = options(n, gravity)
    gpu_ctx.set_models(links, None)
    tau = gpu_ctx.inverse_dynamics_opts(q, qd, qdd, o)
    for b in range(B):
        want = oracle.inverse_dynamics(links[b], [0, 0, -9.81], q[b], qd[b], qdd[b], o.base_velocity,
                                       o.base_acceleration, o.tip_wrench, gravity)
        assert rel_gap(tau[b], want) <= TOL


@pytest.mark.parametrize("n", [1, 6, 33])
def test_default_options_match_plain_call(oracle, gpu_ctx, n):
    links, q, qd, qdd = batch(oracle, n, 16, 700 + n)
    gpu_ctx.set_models(links, None)
    a = gpu_ctx.inverse_dynamics(q, qd, qdd)
    b = gpu_ctx.inverse_dynamics_opts(q, qd, qdd, pd.IdOptions())
    c = gpu_ctx.inverse_dynamics_opts(q, qd, qdd, None)
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("n", [1, 9, 40])
def test_bias_torque(oracle, gpu_ctx, n):
    links, q, qd, _ = batch(oracle, n, 12, 900 + n)
    gpu_ctx.set_models(links, None)
    tau = gpu_ctx.bias_torque(q, qd)
    for b in range(len(links)):
        want = oracle.inverse_dynamics(links[b], [0, 0, -9.81], q[b], qd[b], np.zeros(n))
        assert rel_gap(tau[b], want) <= TOL
    chain = pd.RobotChain.from_records(links[0])
    assert rel_gap(pd.bias_torque(chain, q[0], qd[0]), tau[0]) <= 1e-15


@pytest.mark.parametrize("n", [1, 4, 31])
def test_link_states(oracle, gpu_ctx, n):
    links, q, qd, qdd = batch(oracle, n, 10, 1100 + n)
    o = options(1100 + n)
    gpu_ctx.set_models(links, None)
    v, a, f = gpu_ctx.link_states(q, qd, qdd, o)
    for b in range(len(links)):
        wv, wa, wf = oracle.link_states(links[b], [0, 0, -9.81], q[b], qd[b], qdd[b], o.base_velocity,
                                        o.base_acceleration, o.tip_wrench, True)
        assert rel_gap(v[b], wv) <= TOL
        assert rel_gap(a[b], wa) <= TOL
        assert rel_gap(f[b], wf) <= TOL
    chain = pd.RobotChain.from_records(links[0])
    st = pd.link_states(chain, q[0], qd[0], qdd[0], o)
    assert np.allclose(st.force, f[0], rtol=0, atol=1e-13 * max(1, np.abs(f[0]).max()))


@pytest.mark.parametrize("n", [1, 2, 8, 33, 64, 100])
def test_joint_space_inertia(oracle, gpu_ctx, n):
    B = 6
    links, q, _, _ = batch(oracle, n, B, 1300 + n)
    gpu_ctx.set_models(links, None)
    M = gpu_ctx.joint_space_inertia(q)
    for b in range(B):
        want = oracle.joint_space_inertia(links[b], q[b])
        assert rel_gap(M[b], want) <= TOL
        assert np.array_equal(M[b], M[b].T)  # exactly symmetric, like 0.5 (M + M^T)
    chain = pd.RobotChain.from_records(links[0])
    assert np.array_equal(pd.joint_space_inertia(chain, q[0]), M[0])


def test_shared_model_and_device_path(oracle, gpu_ctx):
    import torch
    n, B = 12, 300
    links, g = oracle.random_chain(n, 4242)
    rng = np.random.default_rng(3)
    q, qd, qdd = rng.uniform(-3, 3, (B, n)), rng.uniform(-2, 2, (B, n)), rng.uniform(-5, 5, (B, n))
    gpu_ctx.set_models(links[None], None)
    tau = gpu_ctx.inverse_dynamics(q, qd, qdd)
    for b in range(0, B, 37):
        assert rel_gap(tau[b], oracle.inverse_dynamics(links, g, q[b], qd[b], qdd[b])) <= TOL
    # device buffers, [link][problem]
    dq, dqd, dqdd = (torch.tensor(x.T.copy(), device="cuda") for x in (q, qd, qdd))
    dtau = torch.empty_like(dq)
    gpu_ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    gpu_ctx.inverse_dynamics_device(B, dq.data_ptr(), dqd.data_ptr(), dqdd.data_ptr(), dtau.data_ptr())
    gpu_ctx.synchronize()
    gpu_ctx.set_stream(None)
    assert np.array_equal(dtau.cpu().numpy().T, tau)


def test_errors(oracle):
    links, _ = oracle.random_chain(3, 1)
    chain = pd.RobotChain.from_records(links)
    with pytest.raises(pd.InvalidArgument, match="qdot has length 2 but the chain has 3 joints"):
        pd.inverse_dynamics(chain, np.zeros(3), np.zeros(2), np.zeros(3))
    with pytest.raises(pd.InvalidArgument, match="assemble_kinematics: q has length 4 but the chain has 3 joints"):
        pd.joint_space_inertia(chain, np.zeros(4))
    with pytest.raises(pd.InvalidArgument, match="assemble_kinematics: q has length 2 but the chain has 3 joints"):
        pd.inverse_dynamics(chain, np.zeros(2), np.zeros(2), np.zeros(2))
    bad = links.copy()
    bad[1, 0] = -1.0  # mass
    with pytest.raises(pd.InvalidArgument, match="mass must be positive"):
        pd.inverse_dynamics(pd.RobotChain.from_records(bad), np.zeros(3), np.zeros(3), np.zeros(3))
    with pytest.raises(pd.InvalidArgument, match="mass must be positive"):
        pd.joint_space_inertia(pd.RobotChain.from_records(bad), np.zeros(3))
    # the reference validates the link inertias before the rate lengths (model.cpp:148-155 first)
    with pytest.raises(pd.InvalidArgument, match="mass must be positive"):
        pd.inverse_dynamics(pd.RobotChain.from_records(bad), np.zeros(3), np.zeros(2), np.zeros(3))


@pytest.mark.parametrize("n,count,g0", [(8, 3000, 0), (64, 1500, 123456), (1, 5, 7)])
def test_device_workload_generator(oracle, gpu_ctx, n, count, g0):
    """§8f row 3: the device generator reproduces the host generator (and
    through it the reference's random_chain / workload_chains): the integer
    streams and every draw are bit exact (mass, com); fields through sin/cos
    are within a few ulp -- the device's sin/cos are correctly rounded, glibc's
    return the other neighbour in ~0.3% of evaluations (profiles/)."""
    import torch
    cell = oracle.workload_seed(42, n, 1 << 20)
    host = oracle.workload_chains(cell, n, count, g0)
    d = torch.empty((count, n, 31), dtype=torch.float64, device="cuda")
    gpu_ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    gpu_ctx.workload_chains_device(cell, n, count, d.data_ptr(), g0)
    gpu_ctx.synchronize()
    gpu_ctx.set_stream(None)
    dev = d.cpu().numpy()
    assert np.array_equal(dev[..., 0:4], host[..., 0:4])  # mass, com: pure draws
    assert np.array_equal(dev[..., 16:19], host[..., 16:19])  # linear screw part (zeros)
    # all fields are O(0.1..10): a last-bit difference in sin/cos moves them by ~1e-16
    assert np.abs(dev - host).max() <= 1e-14
    assert (dev != host).any(axis=2).mean() < 0.05


def test_set_models_workload_matches_host_models(oracle, gpu_ctx):
    n, B = 24, 2000
    cell = oracle.workload_seed(42, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    gpu_ctx.set_models(oracle.workload_chains(cell, n, B), None)
    a, st, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    ms, _ = gpu_ctx.set_models_workload(cell, n, B)
    assert (ms == 0).all()
    b, st2, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    assert (st == 0).all() and (st2 == 0).all()
    for k in range(0, B, 97):
        assert rel_gap(b[k], a[k]) <= 1e-12
