"""The reference's unit and acceptance suites (proj/tests/*.cpp), ported to
run against the CPU oracle: independent routes (sequential recursions, dense
solves, matrix exponentials, closed forms) with the reference's tolerances.
This is what makes the oracle a trustworthy checker for the GPU path."""
import numpy as np
import pytest
from scipy.linalg import expm

RNG = np.random.default_rng


def rel_gap(a, b):
    """oracles.hpp:64-66"""
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1.0, np.linalg.norm(b))


def skew(a):
    return np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])


def rand_rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q * np.sign(np.linalg.det(q))


def sample(oracle, n, seed, q_rng=(-3, 3), qd_rng=(-2, 2), t_rng=(-10, 10)):
    links, g = oracle.random_chain(n, seed)
    r = RNG(seed ^ 0xF00D)
    return links, g, r.uniform(*q_rng, n), r.uniform(*qd_rng, n), r.uniform(*t_rng, n)


# ------------------------------------------------------------------ spatial (test_spatial.cpp)
def test_small_adjoint_layout_and_bracket(oracle):
    r = RNG(1)
    V, W = r.normal(size=6), r.normal(size=6)
    ad = oracle.small_adjoint(V)
    assert np.array_equal(ad[:3, :3], skew(V[:3])) and np.array_equal(ad[3:, 3:], skew(V[:3]))
    assert np.array_equal(ad[3:, :3], skew(V[3:])) and not ad[:3, 3:].any()
    assert np.allclose(ad @ W, -oracle.small_adjoint(W) @ V, atol=1e-14)  # antisymmetry
    assert np.allclose(ad @ V, 0, atol=1e-14)


def test_adjoint_homomorphism(oracle):
    """test_spatial.cpp:53-79: Ad(T1 T2) = Ad(T1) Ad(T2), Ad(T) Ad(T^-1) = I."""
    r = RNG(2)
    R1, R2, p1, p2 = rand_rot(r), rand_rot(r), r.normal(size=3), r.normal(size=3)
    A12 = oracle.adjoint_of(R1 @ R2, R1 @ p2 + p1)
    assert np.allclose(A12, oracle.adjoint_of(R1, p1) @ oracle.adjoint_of(R2, p2), atol=1e-12)
    assert np.allclose(oracle.adjoint_of(R1, p1) @ oracle.adjoint_of(R1.T, -R1.T @ p1), np.eye(6), atol=1e-12)


@pytest.mark.parametrize("screw", [[0, 0, 1, 0, 0, 0], [0.6, 0, 0.8, 0, 0, 0], [0, 0, 0, 1, 0, 0],
                                   [0.3, 0.4, 0.0, 0.5, 0.1, 0.7071]])
def test_screw_exp_vs_matrix_exponential(oracle, screw):
    """test_spatial.cpp:96-134 (exp_via_matrix, oracles.hpp:182-191)."""
    s = np.asarray(screw, float)
    for q in (0.0, 0.3, -1.7, 2.5):
        R, p = oracle.screw_exp(s, q)
        h = np.zeros((4, 4))
        h[:3, :3] = skew(s[:3])
        h[:3, 3] = s[3:]
        E = expm(q * h)
        assert np.allclose(R, E[:3, :3], atol=1e-12) and np.allclose(p, E[:3, 3], atol=1e-12)


def test_spatial_inertia_blocks_and_rejections(oracle):
    """test_spatial.cpp:156-212."""
    m, c, Ic = 2.0, np.array([0.1, -0.2, 0.3]), np.diag([0.3, 0.4, 0.5])
    J = oracle.spatial_inertia(m, c, Ic)
    cx = skew(c)
    assert np.allclose(J[:3, :3], Ic + m * cx @ cx.T) and np.allclose(J[:3, 3:], m * cx)
    assert np.allclose(J[3:, :3], m * cx.T) and np.allclose(J[3:, 3:], m * np.eye(3))
    assert np.array_equal(J, J.T) and np.linalg.eigvalsh(J).min() > 0
    for bad, msg in ((dict(mass=0.0), "mass must be positive"), (dict(mass=np.nan), "mass must be positive"),
                     (dict(Ic=np.diag([1, 1, -1.0])), "positive definite"),
                     (dict(Ic=np.array([[1, 0.5, 0], [0, 1, 0], [0, 0, 1.0]])), "symmetric"),
                     (dict(com=np.array([np.inf, 0, 0])), "finite")):
        kw = dict(mass=m, com=c, Ic=Ic)
        kw.update(bad)
        with pytest.raises(oracle.OracleError) as e:
            oracle.spatial_inertia(kw["mass"], kw["com"], kw["Ic"])
        assert e.value.kind == "invalid_argument" and msg in str(e.value)


# ------------------------------------------------------------------ model (test_model.cpp)
def test_validate_chain_messages(oracle):
    """test_model.cpp:37-68."""
    good, _ = oracle.random_chain(3, 7)
    oracle.validate_chain(good)
    cases = [(1, 0, -2.0, "link 1: mass must be positive"), (0, 13, 2.0, "unit norm")]
    for li, field, val, msg in cases:
        bad = good.copy()
        bad[li, field] = val
        with pytest.raises(oracle.OracleError) as e:
            oracle.validate_chain(bad)
        assert e.value.kind == "ModelError" and msg in str(e.value)
    bad = good.copy()
    bad[2, 4 + 1] += 1.0
    with pytest.raises(oracle.OracleError, match="link 2: rotational inertia must be symmetric"):
        oracle.validate_chain(bad)
    bad = good.copy()
    bad[1, 19:28] *= 1.5
    with pytest.raises(oracle.OracleError, match="orthonormal"):
        oracle.validate_chain(bad)
    with pytest.raises(oracle.OracleError, match="gravity"):
        oracle.validate_chain(good, [np.inf, 0, 0])


def test_kinematics_vs_matrix_exponential(oracle):
    """test_model.cpp:70-95."""
    links, _ = oracle.random_chain(6, 99)
    q = RNG(42).uniform(-2, 2, 6)
    rel, tr, base = oracle.assemble_kinematics(links, q)
    for i in range(6):
        s = links[i, 13:19]
        h = np.zeros((4, 4))
        h[:3, :3] = skew(s[:3])
        h[:3, 3] = s[3:]
        H = np.eye(4)
        H[:3, :3] = links[i, 19:28].reshape(3, 3)
        H[:3, 3] = links[i, 28:31]
        E = expm(-q[i] * h) @ H
        assert np.allclose(rel[i, :9].reshape(3, 3), E[:3, :3], atol=1e-12)
        assert np.allclose(rel[i, 9:], E[:3, 3], atol=1e-12)
    for i in range(5):
        assert np.array_equal(tr[i], oracle.adjoint_of(rel[i + 1, :9].reshape(3, 3), rel[i + 1, 9:]))


def test_random_chain_deterministic(oracle):
    a, _ = oracle.random_chain(12, 2024)
    b, _ = oracle.random_chain(12, 2024)
    c, _ = oracle.random_chain(12, 2025)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    with pytest.raises(oracle.OracleError):
        oracle.random_chain(0, 1)


# ------------------------------------------------------------------ scan (test_scan.cpp)
def test_integer_scan_and_depth(oracle):
    for n in (1, 2, 3, 5, 8, 13, 64, 100, 130):
        out, rounds = oracle.scan_int64(np.arange(1, n + 1))
        assert list(out) == list(np.cumsum(np.arange(1, n + 1)))
        assert rounds == int(np.ceil(np.log2(n))) if n > 1 else rounds == 0


@pytest.mark.parametrize("D", [1, 2, 6])
def test_bidiag_vs_recurrence_and_dense(oracle, D):
    """test_scan.cpp:92-120: 1e-12 vs the recurrence, 1e-10 vs dense LU."""
    r = RNG(31 + D)
    for n in list(range(1, 20)) + [33, 64]:
        for upper in (False, True):
            c = 0.5 * r.uniform(-1, 1, (max(n - 1, 1), D, D))[: n - 1] if n > 1 else np.zeros((0, D, D))
            rhs = r.uniform(-1, 1, (n, D))
            x, rounds = oracle.bidiag_solve(c, rhs, upper=upper)
            ref = np.zeros_like(rhs)
            if not upper:
                ref[0] = rhs[0]
                for k in range(1, n):
                    ref[k] = c[k - 1] @ ref[k - 1] + rhs[k]
            else:
                ref[n - 1] = rhs[n - 1]
                for k in range(n - 2, -1, -1):
                    ref[k] = c[k] @ ref[k + 1] + rhs[k]
            assert rel_gap(x, ref) < 1e-12
            Md = np.eye(n * D)
            for k in range(n - 1):
                if not upper:
                    Md[(k + 1) * D:(k + 2) * D, k * D:(k + 1) * D] = -c[k]
                else:
                    Md[k * D:(k + 1) * D, (k + 1) * D:(k + 2) * D] = -c[k]
            assert rel_gap(x.ravel(), np.linalg.solve(Md, rhs.ravel())) < 1e-10
            assert rounds == (0 if n == 1 else int(np.ceil(np.log2(n))))


# ------------------------------------------------------------------ OEE (test_oee.cpp)
def random_tridiag(B, n, r):
    """oracles.hpp:160-177."""
    upper = r.uniform(-1, 1, (max(n - 1, 0), B, B))
    diag = np.zeros((n, B, B))
    for k in range(n):
        a = r.uniform(-1, 1, (B, B))
        dom = 1.0 + (np.linalg.norm(upper[k - 1]) if k > 0 else 0) + (np.linalg.norm(upper[k]) if k + 1 < n else 0)
        diag[k] = a @ a.T + dom * np.eye(B)
    return diag, upper


def dense(diag, upper):
    n, B = diag.shape[0], diag.shape[1]
    A = np.zeros((n * B, n * B))
    for k in range(n):
        A[k * B:(k + 1) * B, k * B:(k + 1) * B] = diag[k]
        if k + 1 < n:
            A[k * B:(k + 1) * B, (k + 1) * B:(k + 2) * B] = upper[k]
            A[(k + 1) * B:(k + 2) * B, k * B:(k + 1) * B] = upper[k].T
    return A


@pytest.mark.parametrize("B", [1, 2, 5])
def test_oee_vs_thomas_and_dense(oracle, B):
    """test_oee.cpp:20-44 (1e-10), acceptance criterion 1 (1e-9 up to n=128)."""
    r = RNG(101 + B)
    for n in list(range(1, 49)) + [64, 100, 128]:
        diag, upper = random_tridiag(B, n, r)
        rhs = r.uniform(-1, 1, (n, B))
        x, rounds = oracle.tridiag_solve(diag, upper, rhs)
        xt, _ = oracle.tridiag_solve(diag, upper, rhs, thomas=True)
        xd = np.linalg.solve(dense(diag, upper), rhs.ravel())
        assert rel_gap(x.ravel(), xt.ravel()) < 1e-10
        assert rel_gap(x.ravel(), xd) < 1e-10
        assert rounds == (0 if n == 1 else int(np.ceil(np.log2(n))))


def test_oee_multi_rhs(oracle):
    """test_oee.cpp:46-58."""
    r = RNG(111)
    diag, upper = random_tridiag(5, 17, r)
    rhs = r.uniform(-1, 1, (17, 5, 3))
    x, _ = oracle.tridiag_solve(diag, upper, rhs)
    xd = np.linalg.solve(dense(diag, upper), rhs.reshape(85, 3))
    assert np.abs(x.reshape(85, 3) - xd).max() < 1e-10


def test_oee_rounds_symmetry_and_distance(oracle):
    """test_oee.cpp:60-94: every intermediate D stays symmetric; couplings
    shrink by the distance, which doubles each round."""
    r = RNG(121)
    for n in (5, 16, 33, 100):
        diag, upper = random_tridiag(5, n, r)
        rhs = r.uniform(-1, 1, (n, 5))
        d, c, h = diag, upper, 1
        for rd in range(1, int(np.ceil(np.log2(n))) + 1):
            d, c, rhs = oracle.oee_round(d, c, rhs, h, rd - 1)
            h *= 2
            assert max(np.abs(x - x.T).max() for x in d) < 1e-10
            assert len(c) == max(n - h, 0)
        assert len(c) == 0


def test_oee_singular_pivot_reports_round_and_block(oracle):
    """test_oee.cpp:106-126."""
    diag = np.stack([np.eye(2), np.zeros((2, 2)), np.eye(2)])
    upper = np.stack([0.1 * np.eye(2), 0.1 * np.eye(2)])
    with pytest.raises(oracle.OracleError) as e:
        oracle.tridiag_solve(diag, upper, np.ones((3, 2)))
    assert (e.value.round, e.value.index) == (1, 1) and "singular pivot" in str(e.value)
    diag = np.stack([np.zeros((2, 2)), np.eye(2), np.eye(2)])
    with pytest.raises(oracle.OracleError) as e:
        oracle.tridiag_solve(diag, upper, np.ones((3, 2)), thomas=True)
    assert e.value.kind == "DynamicsError"


def test_fullpivlu_rank_threshold(oracle):
    m = np.eye(5)
    assert oracle.fullpivlu_rank5(m) == 5
    m[4, 4] = 1e-17
    assert oracle.fullpivlu_rank5(m) == 4


# ------------------------------------------------------------------ inverse dynamics (test_invdyn.cpp)
@pytest.mark.parametrize("n", [1, 2, 3, 7, 20])
def test_scan_propagation_matches_sequential_ne(oracle, n):
    """test_invdyn.cpp:50-110 at 1e-12."""
    links, g = oracle.random_chain(n, 100 + n)
    r = RNG(n)
    q, qd, qdd = r.uniform(-3, 3, n), r.uniform(-2, 2, n), r.uniform(-5, 5, n)
    v, a, f = oracle.link_states(links, g, q, qd, qdd)
    sv, sa, sf, st = oracle.newton_euler(links, g, q, qd, qdd)
    for got, want in ((v, sv), (a, sa), (f, sf)):
        assert max(np.linalg.norm(got[i] - want[i]) / max(1, np.linalg.norm(want[i])) for i in range(n)) < 1e-12
    assert rel_gap(oracle.inverse_dynamics(links, g, q, qd, qdd), st) < 1e-12
    assert rel_gap(oracle.inverse_dynamics(links, g, q, qd, qdd, apply_gravity=False),
                   oracle.newton_euler(links, g, q, qd, qdd, apply_gravity=False)[3]) < 1e-12


def test_acceleration_is_velocity_derivative(oracle):
    """test_invdyn.cpp:144-170."""
    links, g = oracle.random_chain(5, 909)
    r = RNG(909)
    q, qd, qdd = r.uniform(-3, 3, 5), r.uniform(-2, 2, 5), r.uniform(-5, 5, 5)
    h = 1e-5
    vel = lambda t: oracle.link_states(links, g, q + t * qd + 0.5 * t * t * qdd, qd + t * qdd, qdd,
                                       apply_gravity=False)[0]
    _, acc, _ = oracle.link_states(links, g, q, qd, qdd, apply_gravity=False)
    num = (vel(h) - vel(-h)) / (2 * h)
    for i in range(5):
        assert np.linalg.norm(num[i] - acc[i]) / max(1, np.linalg.norm(acc[i])) < 1e-5


def test_tip_wrench_statics(oracle):
    """test_invdyn.cpp:180-204."""
    links, g = oracle.random_chain(3, 4242)
    q = RNG(777).uniform(-2, 2, 3)
    tip = np.array([0.4, -0.2, 0.9, -1.0, 2.5, 0.3])
    tau = oracle.inverse_dynamics(links, g, q, np.zeros(3), np.zeros(3), tip=tip, apply_gravity=False)
    _, tr, _ = oracle.assemble_kinematics(links, q)
    carried = tip.copy()
    exp = np.zeros(3)
    exp[2] = links[2, 13:19] @ carried
    for i in (1, 0):
        carried = tr[i].T @ carried
        exp[i] = links[i, 13:19] @ carried
    assert rel_gap(tau, exp) < 1e-13


# ------------------------------------------------------------------ forward dynamics (test_fwddyn.cpp)
@pytest.mark.parametrize("n", [1, 3, 8, 20])
def test_joint_space_inertia(oracle, n):
    """test_fwddyn.cpp:66-80."""
    links, g, q, _, _ = sample(oracle, n, 9000 + n)
    M = oracle.joint_space_inertia(links, q)
    assert rel_gap(M, oracle.mass_matrix_ne(links, q)) < 1e-10
    assert np.array_equal(M, M.T) and np.linalg.eigvalsh(M).min() > 0


@pytest.mark.parametrize("n", [1, 2, 5, 10, 30])
def test_all_algorithms_recover_dense_solve(oracle, n):
    """test_fwddyn.cpp:82-103: JSIIA vs dense 1e-9, ABIA and CFA vs JSIIA 1e-8."""
    for trial in range(3):
        links, g, q, qd, tau = sample(oracle, n, 400 + 10 * n + trial)
        ref = oracle.dense_forward_dynamics(links, g, q, qd, tau)
        j = oracle.forward_dynamics("jsiia", links, g, q, qd, tau)
        assert rel_gap(j, ref) < 1e-9
        assert rel_gap(oracle.forward_dynamics("abia", links, g, q, qd, tau), j) < 1e-8
        assert rel_gap(oracle.forward_dynamics("cfa", links, g, q, qd, tau), j) < 1e-8


def test_articulated_inertia_properties(oracle):
    """test_fwddyn.cpp:141-161."""
    links, g, q, _, _ = sample(oracle, 7, 6100)
    I, lam, gain = oracle.articulated_body_inertias(links, q)
    J6 = oracle.spatial_inertia(links[6, 0], links[6, 1:4], links[6, 4:13].reshape(3, 3))
    assert np.array_equal(I[6], J6)
    for i in range(7):
        s = links[i, 13:19]
        assert np.array_equal(I[i], I[i].T)
        assert abs(lam[i] - s @ I[i] @ s) < 1e-12 * lam[i]
        assert np.linalg.norm(gain[i] * lam[i] - I[i] @ s) < 1e-10
        assert np.linalg.eigvalsh(I[i]).min() > 0


def test_constraint_basis_orthonormal(oracle):
    """test_fwddyn.cpp:163-185."""
    links, _ = oracle.random_chain(6, 321)
    W = oracle.constraint_basis(links)
    for i in range(6):
        s = links[i, 13:19]
        assert np.linalg.norm(W[i].T @ W[i] - np.eye(5)) < 1e-14
        assert np.linalg.norm(W[i].T @ s) < 1e-14
        sq = np.column_stack([W[i], s])
        assert np.linalg.norm(sq.T @ sq - np.eye(6)) < 1e-13
    assert np.array_equal(W, oracle.constraint_basis(links))


def cfa_dense(oracle, links, q):
    n = len(links)
    ops = oracle.cfa_operators(links, q)
    A = dense(ops["diag"], ops["upper"])
    Bm = np.zeros((5 * n, n))
    C = np.diag(ops["joint_diag"])
    for i in range(n):
        Bm[5 * i:5 * i + 5, i] = ops["cross_diag"][i]
        if i + 1 < n:
            Bm[5 * i:5 * i + 5, i + 1] = ops["cross_super"][i]
            Bm[5 * (i + 1):5 * (i + 1) + 5, i] = ops["cross_sub"][i]
            C[i, i + 1] = C[i + 1, i] = ops["joint_off"][i]
    return A, Bm, C


@pytest.mark.parametrize("n", [1, 2, 4, 9])
def test_cfa_operators_match_dense_projections(oracle, n):
    """test_fwddyn.cpp:187-206 at 1e-12."""
    links, g, q, _, _ = sample(oracle, n, 5200 + n)
    _, tr, _ = oracle.assemble_kinematics(links, q)
    jinv = np.zeros((6 * n, 6 * n))
    P = np.eye(6 * n)
    for i in range(n):
        J = oracle.spatial_inertia(links[i, 0], links[i, 1:4], links[i, 4:13].reshape(3, 3))
        jinv[6 * i:6 * i + 6, 6 * i:6 * i + 6] = np.linalg.inv(J)
        if i + 1 < n:
            P[6 * i:6 * i + 6, 6 * (i + 1):6 * (i + 1) + 6] = -tr[i].T
    core = P.T @ jinv @ P
    W = oracle.constraint_basis(links)
    Wd = np.zeros((6 * n, 5 * n))
    Sd = np.zeros((6 * n, n))
    for i in range(n):
        Wd[6 * i:6 * i + 6, 5 * i:5 * i + 5] = W[i]
        Sd[6 * i:6 * i + 6, i] = links[i, 13:19]
    A, Bm, C = cfa_dense(oracle, links, q)
    assert rel_gap(A, Wd.T @ core @ Wd) < 1e-12
    assert rel_gap(Bm, Wd.T @ core @ Sd) < 1e-12
    assert rel_gap(C, Sd.T @ core @ Sd) < 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16])
def test_schur_identity_inverts_joint_space_inertia(oracle, n):
    """test_fwddyn.cpp:234-252: (C - B^T A^-1 B) M = I at 1e-7."""
    links, g, q, _, _ = sample(oracle, n, 7300 + n)
    A, Bm, C = cfa_dense(oracle, links, q)
    M = oracle.joint_space_inertia(links, q)
    assert np.linalg.norm((C - Bm.T @ np.linalg.solve(A, Bm)) @ M - np.eye(n)) < 1e-7


def test_execution_traces(oracle):
    """test_fwddyn.cpp:263-283."""
    links, g, q, qd, tau = sample(oracle, 13, 1300)
    depth = 4
    _, tj = oracle.forward_dynamics("jsiia", links, g, q, qd, tau, trace=True)
    _, ta = oracle.forward_dynamics("abia", links, g, q, qd, tau, trace=True)
    _, tc = oracle.forward_dynamics("cfa", links, g, q, qd, tau, trace=True)
    assert tj[1] == 0 and tj[2] == depth and tj[0] > 0
    assert ta[1] == 13 and ta[2] == depth
    assert tc[1] == 0 and tc[2] == depth and tc[3] == depth


def test_batch_slot_identity_and_isolation(oracle):
    """test_fwddyn.cpp:298-341: batch == single calls bitwise; per-slot errors."""
    for algo in ("jsiia", "abia", "cfa"):
        links, g, q, qd, tau = sample(oracle, 6, 600)
        B = 5
        Q, QD, T = np.tile(q, (B, 1)), np.tile(qd, (B, 1)), np.tile(tau, (B, 1))
        Q[2] += 0.1
        out, st = oracle.batch_forward_dynamics(algo, links[None], g, Q, QD, T)
        assert (st == 0).all()
        for b in range(B):
            assert np.array_equal(out[b], oracle.forward_dynamics(algo, links, g, Q[b], QD[b], T[b]))
    bad = links.copy()
    bad[2, 0] = -1.0
    out, st = oracle.batch_forward_dynamics("abia", np.stack([links, bad]), g, Q[:2], QD[:2], T[:2])
    assert list(st) == [0, 1]


def test_input_validation(oracle):
    """test_fwddyn.cpp:343-361."""
    links, g = oracle.random_chain(3, 77)
    for algo in ("jsiia", "abia", "cfa"):
        with pytest.raises(oracle.OracleError) as e:
            oracle.forward_dynamics(algo, links, g, np.zeros(2), np.zeros(3), np.zeros(3))
        assert e.value.kind == "invalid_argument" and "forward dynamics" in str(e.value)
    with pytest.raises(oracle.OracleError, match="no links"):
        oracle.forward_dynamics("jsiia", np.zeros((0, 31)), g, [], [], [])


# ------------------------------------------------------------------ acceptance (acceptance_main.cpp)
@pytest.mark.parametrize("n", [1, 2, 5, 10, 50, 200])
def test_acceptance_cross_algorithm_agreement(oracle, n):
    """Criterion 2: 1e-8 for n in {1,2,5,10,50,200}; 2 chains x a few states."""
    states = 6 if n >= 50 else 25
    for c in range(2):
        links, g = oracle.random_chain(n, 9100 + 10 * n + c)
        r = RNG(40 + 2 * n + c)
        Q, QD, T = r.uniform(-3, 3, (states, n)), r.uniform(-2, 2, (states, n)), r.uniform(-10, 10, (states, n))
        j, _ = oracle.batch_forward_dynamics("jsiia", links[None], g, Q, QD, T)
        a, _ = oracle.batch_forward_dynamics("abia", links[None], g, Q, QD, T)
        cf, _ = oracle.batch_forward_dynamics("cfa", links[None], g, Q, QD, T)
        for s in range(states):
            assert rel_gap(a[s], j[s]) <= 1e-8 and rel_gap(cf[s], j[s]) <= 1e-8


def test_acceptance_round_trips(oracle):
    """Criterion 4: ID(FD(tau)) = tau and FD(ID(qdd)) = qdd at 1e-8, n = 20."""
    links, g = oracle.random_chain(20, 777)
    r = RNG(778)
    for _ in range(5):
        q, qd, qdd, tau = r.uniform(-3, 3, 20), r.uniform(-2, 2, 20), r.uniform(-10, 10, 20), r.uniform(-10, 10, 20)
        t_of_qdd = oracle.inverse_dynamics(links, g, q, qd, qdd)
        for algo in ("jsiia", "abia", "cfa"):
            acc = oracle.forward_dynamics(algo, links, g, q, qd, tau)
            assert rel_gap(oracle.inverse_dynamics(links, g, q, qd, acc), tau) <= 1e-8
            assert rel_gap(oracle.forward_dynamics(algo, links, g, q, qd, t_of_qdd), qdd) <= 1e-8


def test_acceptance_determinism_across_thread_counts(oracle):
    """Criterion 8: bit-identical results for 1, 4 and 8 workers."""
    n, B = 16, 64
    cell = oracle.workload_seed(42, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 3)
    for algo in ("jsiia", "abia", "cfa"):
        ref, _ = oracle.batch_forward_dynamics(algo, links, [0, 0, -9.81], q, qd, tau, nthreads=1)
        for w in (4, 8):
            got, _ = oracle.batch_forward_dynamics(algo, links, [0, 0, -9.81], q, qd, tau, nthreads=w)
            assert np.array_equal(ref, got)
