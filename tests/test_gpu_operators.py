"""The reference's chain operators on the device (SURVEY.md §8a rows a4, a5,
a11, a15-a17) through the C-ABI and the Python mirror, against the CPU oracle
and the properties tests/test_fwddyn.cpp:141-252 checks:
assemble_kinematics / link_inertias (model.cpp:117-155),
articulated_body_inertias (forward_dynamics.cpp:120-163),
build_constraint_basis (:245-259), build_cfa_operators (:261-357) and the
CfaOperators stencils (:359-416)."""
import numpy as np
import pytest

import paper_1609_06779_b200 as pd

pytestmark = pytest.mark.gpu


def sample(oracle, n, seed):
    links, g = oracle.random_chain(n, seed)
    rng = np.random.default_rng(seed ^ 0xF00D)
    return pd.RobotChain.from_records(links, g), links, rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), \
        rng.uniform(-10, 10, n)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


@pytest.mark.parametrize("n", [1, 2, 9, 64])
def test_kinematics_and_link_inertias_vs_oracle(oracle, n):
    chain, links, q, _, _ = sample(oracle, n, 4200 + n)
    kin = pd.assemble_kinematics(chain, q)
    orel, otr, obase = oracle.assemble_kinematics(links, q)
    assert np.abs(kin.rotation.reshape(n, 9) - orel[:, :9]).max() < 1e-14
    assert np.abs(kin.translation - orel[:, 9:]).max() < 1e-14
    assert np.abs(kin.base_transport - obase).max() < 1e-14
    if n > 1:
        assert np.abs(kin.transport - otr).max() < 1e-13
    assert np.array_equal(kin.screw, links[:, 13:19])
    J = pd.link_inertias(chain)
    for i in range(n):
        ref = oracle.spatial_inertia(links[i, 0], links[i, 1:4], links[i, 4:13].reshape(3, 3))
        assert rel(J[i], ref) < 1e-15


def test_link_inertias_reject_bad_links(oracle):
    chain, *_ = sample(oracle, 4, 17)
    chain.links[2].mass = -1.0
    with pytest.raises(pd.InvalidArgument, match="^spatial inertia: mass must be positive$"):
        pd.link_inertias(chain)


def test_articulated_inertias_properties_and_oracle(oracle):
    """test_fwddyn.cpp:141-161, plus the oracle's values at 1e-12."""
    chain, links, q, _, _ = sample(oracle, 7, 6100)
    kin = pd.assemble_kinematics(chain, q)
    J = pd.link_inertias(chain)
    tr = pd.ExecTrace()
    ab = pd.articulated_body_inertias(kin, J, trace=tr)
    assert tr.longest_sequential_link_chain == 7
    assert np.array_equal(ab.inertia[6], J[6])
    for i in range(7):
        s = kin.screw[i]
        assert np.array_equal(ab.inertia[i], ab.inertia[i].T)
        assert abs(ab.joint_inertia[i] - s @ ab.inertia[i] @ s) < 1e-12 * ab.joint_inertia[i]
        assert np.linalg.norm(ab.gain[i] * ab.joint_inertia[i] - ab.inertia[i] @ s) < 1e-10
        assert np.linalg.eigvalsh(ab.inertia[i]).min() > 0
    oI, olam, og = oracle.articulated_body_inertias(links, q)
    assert rel(ab.inertia, oI) < 1e-12 and rel(ab.joint_inertia, olam) < 1e-12 and rel(ab.gain, og) < 1e-12


def test_articulated_inertias_degenerate_joint(oracle, gpu_ctx):
    """A joint whose articulated inertia about its axis vanishes reports the
    reference's DynamicsError (forward_dynamics.cpp:140-144)."""
    n = 3
    tr = np.tile(np.eye(6), (1, n - 1, 1, 1))
    inertia = np.tile(np.eye(6), (n, 1, 1))
    inertia[2] = np.diag([1, 1, 0.0, 1, 1, 1])  # tip link: no inertia about z
    screw = np.tile([0, 0, 1.0, 0, 0, 0], (1, n, 1))
    _, _, _, st, ix = gpu_ctx.articulated_body_inertias(tr, inertia[None], screw)
    assert st[0] == pd.api._capi.SLOT_DEGENERATE_ARTICULATION and ix[0] == 2


def test_constraint_basis(oracle):
    """test_fwddyn.cpp:163-185 and bit-identity with the oracle's Householder."""
    chain, links, *_ = sample(oracle, 6, 321)
    b = pd.build_constraint_basis(chain).basis
    for i in range(6):
        w, s = b[i], links[i, 13:19]
        assert np.linalg.norm(w.T @ w - np.eye(5)) < 1e-14
        assert np.linalg.norm(w.T @ s) < 1e-14
        sq = np.concatenate([w, s[:, None]], axis=1)
        assert np.linalg.norm(sq.T @ sq - np.eye(6)) < 1e-13
    assert np.array_equal(pd.build_constraint_basis(chain).basis, b)
    assert np.abs(b - oracle.constraint_basis(links)).max() < 1e-15


def dense_ops(ops):
    n = len(ops.joint_diag)
    A, B, Cm = np.zeros((5 * n, 5 * n)), np.zeros((5 * n, n)), np.zeros((n, n))
    for i in range(n):
        A[5 * i:5 * i + 5, 5 * i:5 * i + 5] = ops.diag[i]
        B[5 * i:5 * i + 5, i] = ops.cross_diag[i]
        Cm[i, i] = ops.joint_diag[i]
        if i + 1 < n:
            A[5 * i:5 * i + 5, 5 * i + 5:5 * i + 10] = ops.upper[i]
            A[5 * i + 5:5 * i + 10, 5 * i:5 * i + 5] = ops.upper[i].T
            B[5 * i:5 * i + 5, i + 1] = ops.cross_super[i]
            B[5 * i + 5:5 * i + 10, i] = ops.cross_sub[i]
            Cm[i, i + 1] = Cm[i + 1, i] = ops.joint_off[i]
    return A, B, Cm


@pytest.mark.parametrize("n", [1, 2, 4, 9])
def test_cfa_operators_match_dense_projections(oracle, n):
    """test_fwddyn.cpp:187-206 (1e-12) and the oracle's operators."""
    chain, links, q, _, _ = sample(oracle, n, 5200 + n)
    kin = pd.assemble_kinematics(chain, q)
    basis = pd.build_constraint_basis(chain)
    ops = pd.build_cfa_operators(chain, kin, basis)
    J = pd.link_inertias(chain)
    jinv = np.zeros((6 * n, 6 * n))
    p = np.eye(6 * n)
    for i in range(n):
        jinv[6 * i:6 * i + 6, 6 * i:6 * i + 6] = np.linalg.inv(J[i])
        if i + 1 < n:
            p[6 * i:6 * i + 6, 6 * i + 6:6 * i + 12] = -kin.transport[i].T
    core = p.T @ jinv @ p
    W = np.zeros((6 * n, 5 * n))
    S = np.zeros((6 * n, n))
    for i in range(n):
        W[6 * i:6 * i + 6, 5 * i:5 * i + 5] = basis.basis[i]
        S[6 * i:6 * i + 6, i] = kin.screw[i]
    A, B, Cm = dense_ops(ops)
    assert rel(A, W.T @ core @ W) < 1e-12
    assert rel(B, W.T @ core @ S) < 1e-12
    assert rel(Cm, S.T @ core @ S) < 1e-12
    o = oracle.cfa_operators(links, q)
    assert rel(ops.diag, o["diag"]) < 1e-12 and rel(ops.cross_diag, o["cross_diag"]) < 1e-12
    assert rel(ops.joint_diag, o["joint_diag"]) < 1e-12
    if n > 1:
        assert rel(ops.upper, o["upper"]) < 1e-12 and rel(ops.joint_off, o["joint_off"]) < 1e-12


def test_operator_applications_match_dense(oracle):
    """test_fwddyn.cpp:208-232."""
    chain, links, q, _, _ = sample(oracle, 8, 5300)
    kin = pd.assemble_kinematics(chain, q)
    ops = pd.build_cfa_operators(chain, kin, pd.build_constraint_basis(chain))
    _, B, Cm = dense_ops(ops)
    rng = np.random.default_rng(64)
    v, f = rng.uniform(-2, 2, 8), rng.uniform(-2, 2, 40)
    assert np.linalg.norm(ops.apply_cross(v).ravel() - B @ v) < 1e-13
    assert np.linalg.norm(ops.apply_cross_transpose(f.reshape(8, 5)) - B.T @ f) < 1e-13
    assert np.linalg.norm(ops.apply_joint(v) - Cm @ v) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16])
def test_schur_complement_inverts_the_joint_space_inertia(oracle, n):
    """test_fwddyn.cpp:234-252: (C - B^T A^-1 B) M = I within 1e-7."""
    chain, links, q, _, _ = sample(oracle, n, 7300 + n)
    kin = pd.assemble_kinematics(chain, q)
    ops = pd.build_cfa_operators(chain, kin, pd.build_constraint_basis(chain))
    A, B, Cm = dense_ops(ops)
    M = pd.joint_space_inertia(chain, q)
    assert np.linalg.norm((Cm - B.T @ np.linalg.solve(A, B)) @ M - np.eye(n)) < 1e-7


def test_batched_operator_calls(oracle, gpu_ctx):
    """The C-ABI entries are batched: 300 chains of 12 links in one call each,
    against the oracle chain by chain."""
    n, B = 12, 300
    cell = oracle.workload_seed(5, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, _, _ = oracle.workload_inputs(cell, n, B, 0)
    gpu_ctx.set_models(links, None)
    rel_, base, tr, sc = gpu_ctx.assemble_kinematics(q)
    J = gpu_ctx.link_inertias()
    abi, lam, gain, st, _ = gpu_ctx.articulated_body_inertias(tr, J, sc)
    assert (st == 0).all()
    W = gpu_ctx.constraint_basis(sc.reshape(-1, 6)).reshape(B, n, 6, 5)
    ops = gpu_ctx.cfa_operators(J, tr, sc, W)
    assert (ops["status"] == 0).all()
    for b in (0, 151, B - 1):
        orel, otr, _ = oracle.assemble_kinematics(links[b], q[b])
        assert np.abs(rel_[b] - orel).max() < 1e-14 and np.abs(tr[b] - otr).max() < 1e-13
        oI, olam, _ = oracle.articulated_body_inertias(links[b], q[b])
        assert rel(abi[b], oI) < 1e-12 and rel(lam[b], olam) < 1e-12
        o = oracle.cfa_operators(links[b], q[b])
        assert rel(ops["diag"][b], o["diag"]) < 1e-12 and rel(ops["joint_off"][b], o["joint_off"]) < 1e-12


def test_batch_over_a_device_list_is_bit_identical(oracle):
    """batch_forward_dynamics(devices=[...]) splits each bucket into
    contiguous slices, one context per device (here three contexts on device
    0): bit-identical to the one-device call, which matches the oracle."""
    problems = []
    for k in range(400):
        n = 9 if k % 3 else 30
        chain, _, q, qd, tau = sample(oracle, n, 900 + k)
        problems.append(pd.FdProblem(chain, q, qd, tau))
    for algo in pd.FdAlgo:
        one = pd.batch_forward_dynamics(problems, algo)
        three = pd.batch_forward_dynamics(problems, algo, devices=[0, 0, 0])
        assert all(a.ok() and b.ok() and np.array_equal(a.qddot, b.qddot) for a, b in zip(one, three))
        p = problems[5]
        ref = oracle.forward_dynamics(algo.name, p.chain.to_records(), p.chain.gravity, p.q, p.qdot, p.tau)
        assert rel(one[5].qddot, ref) <= 1e-9


@pytest.mark.parametrize("n", [1, 2, 3, 7, 20])
def test_propagations_match_sequential_newton_euler(oracle, n):
    """test_invdyn.cpp:50-76: propagate_velocities / _accelerations / _forces
    (block bi-diagonal scans on the device) against the sequential
    Newton-Euler oracle at 1e-12, scan rounds ceil_log2(n); and
    inverse_dynamics_assembled == inverse_dynamics."""
    chain, links, q, qd, _ = sample(oracle, n, 100 + n)
    qdd = np.random.default_rng(1000 + n).uniform(-5, 5, n)
    kin = pd.assemble_kinematics(chain, q)
    J = pd.link_inertias(chain)
    ref_v, ref_a, ref_f = oracle.newton_euler(links, chain.gravity, q, qd, qdd, True)[:3]
    tv, ta, tf = pd.ScanTrace(), pd.ScanTrace(), pd.ScanTrace()
    v = pd.propagate_velocities(kin, qd, None, tv)
    a = pd.propagate_accelerations(kin, v, qd, qdd, np.concatenate([np.zeros(3), -chain.gravity]), ta)
    f = pd.propagate_forces(kin, v, a, J, None, tf)
    for got, want in ((v, ref_v), (a, ref_a), (f, ref_f)):
        gaps = np.linalg.norm(got - want, axis=1) / np.maximum(1.0, np.linalg.norm(want, axis=1))
        assert gaps.max() < 1e-12
    assert tv.rounds == ta.rounds == tf.rounds == pd.ceil_log2(n)
    tr = pd.ExecTrace()
    tau = pd.inverse_dynamics_assembled(kin, J, chain.gravity, qd, qdd, trace=tr)
    assert rel(tau, pd.inverse_dynamics(chain, q, qd, qdd)) < 1e-12
    assert tr.scan_rounds_max == pd.ceil_log2(n)
