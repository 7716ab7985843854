"""GPU parity of the paper's building block 2 on its own: batched symmetric
block tri-diagonal solves by odd-even elimination with 5x5 blocks
(pd_block_tridiag_solve5 <- oee_solve<5,1>, include/pardyn/oee.hpp:149-189)
against the oracle's restatement, including the reference's singular-pivot
report (tests/test_oee.cpp:106-126: round, block)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_system(rng, n):
    diag = np.empty((n, 5, 5))
    for k in range(n):
        a = rng.uniform(-1, 1, (5, 5))
        diag[k] = a @ a.T + 6.0 * np.eye(5)
    upper = rng.uniform(-1, 1, (max(n - 1, 0), 5, 5))
    rhs = rng.uniform(-5, 5, (n, 5))
    return diag, upper, rhs


@pytest.mark.parametrize("n", [1, 2, 3, 7, 33, 64, 200, 256])
def test_oee5_matches_oracle(oracle, gpu_ctx, n):
    rng = np.random.default_rng(n)
    B = 4
    systems = [random_system(rng, n) for _ in range(B)]
    diag = np.stack([s[0] for s in systems])
    upper = np.stack([s[1] for s in systems]) if n > 1 else np.zeros((B, 0, 5, 5))
    rhs = np.stack([s[2] for s in systems])
    x, st, rd, ix = gpu_ctx.block_tridiag_solve5(diag, upper, rhs)
    assert (st == 0).all()
    for b in range(B):
        want, rounds = oracle.tridiag_solve(diag[b], upper[b] if n > 1 else np.zeros((1, 5, 5)), rhs[b])
        want = want.reshape(n, 5)
        assert np.linalg.norm(x[b] - want) / max(1.0, np.linalg.norm(want)) <= 1e-12
        # and it solves the system
        full = np.zeros((5 * n, 5 * n))
        for k in range(n):
            full[5 * k:5 * k + 5, 5 * k:5 * k + 5] = diag[b, k]
            if k + 1 < n:
                full[5 * k:5 * k + 5, 5 * k + 5:5 * k + 10] = upper[b, k]
                full[5 * k + 5:5 * k + 10, 5 * k:5 * k + 5] = upper[b, k].T
        assert np.linalg.norm(full @ x[b].ravel() - rhs[b].ravel()) <= 1e-10 * np.linalg.norm(rhs[b])


@pytest.mark.parametrize("kind", ["negative_definite", "indefinite"])
@pytest.mark.parametrize("n", [1, 2, 9, 64])
def test_oee5_non_spd_pivots(oracle, gpu_ctx, kind, n):
    """Invertible but not positive definite pivots: the reference's
    coefficient_solve uses FullPivLU (oee.hpp:40-51), not a Cholesky, so
    these systems solve (oee.hpp notes intermediate pivots are symmetric but
    not guaranteed positive definite)."""
    rng = np.random.default_rng(100 + n)
    B = 3
    diag = np.empty((B, n, 5, 5))
    for b in range(B):
        for k in range(n):
            if kind == "negative_definite":
                a = rng.uniform(-1, 1, (5, 5))
                diag[b, k] = -(a @ a.T + 6.0 * np.eye(5))
            else:
                q, _ = np.linalg.qr(rng.uniform(-1, 1, (5, 5)))
                diag[b, k] = q @ np.diag([7.0, -6.5, 8.0, -7.5, 6.0]) @ q.T
    upper = rng.uniform(-1, 1, (B, max(n - 1, 0), 5, 5))
    rhs = rng.uniform(-5, 5, (B, n, 5))
    x, st, rd, ix = gpu_ctx.block_tridiag_solve5(diag, upper, rhs)
    assert (st == 0).all(), (st, rd, ix)
    for b in range(B):
        want, _ = oracle.tridiag_solve(diag[b], upper[b] if n > 1 else np.zeros((1, 5, 5)), rhs[b])
        want = want.reshape(n, 5)
        assert np.linalg.norm(x[b] - want) / max(1.0, np.linalg.norm(want)) <= 1e-11


def test_oee5_diag_minus_identity(oracle, gpu_ctx):
    """The advisor's case: diag = -I, upper = 0 (invertible, negative definite)."""
    n = 4
    diag = np.stack([-np.eye(5)] * n)[None]
    upper = np.zeros((1, n - 1, 5, 5))
    rhs = np.arange(n * 5, dtype=float).reshape(1, n, 5)
    x, st, _, _ = gpu_ctx.block_tridiag_solve5(diag, upper, rhs)
    assert st[0] == 0
    assert np.array_equal(x[0], -rhs[0])


@pytest.mark.parametrize("case", ["pivot_row1", "pivot_row0", "final"])
def test_oee5_singular_reports_like_the_reference(oracle, gpu_ctx, case):
    n = 3
    eye = np.eye(5)
    if case == "pivot_row1":     # test_oee.cpp:106-126 with 5x5 blocks
        diag = np.stack([eye, np.zeros((5, 5)), eye])
    elif case == "pivot_row0":
        diag = np.stack([np.zeros((5, 5)), eye, eye])
    else:                        # n = 1: no rounds, the final solve is singular
        n = 1
        diag = np.zeros((1, 5, 5))
    upper = np.stack([0.1 * eye] * (n - 1)) if n > 1 else np.zeros((0, 5, 5))
    rhs = np.ones((n, 5))
    x, st, rd, ix = gpu_ctx.block_tridiag_solve5(diag[None], upper[None], rhs[None])
    with pytest.raises(oracle.OracleError) as e:
        oracle.tridiag_solve(diag, upper if n > 1 else np.zeros((1, 5, 5)), rhs)
    assert st[0] != 0
    assert (rd[0], ix[0]) == (e.value.round, e.value.index)
    import paper_1609_06779_b200 as pd
    assert pd.api._capi.slot_message(st[0], rd[0], ix[0], n) == str(e.value)


# ---- building block 1: the block bi-diagonal scan (scan.hpp:100-168)
@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 100, 1024, 1500])
@pytest.mark.parametrize("upper", [False, True])
def test_bidiag6_matches_oracle(oracle, gpu_ctx, n, upper):
    rng = np.random.default_rng(n + 7 * upper)
    B = 3
    coupling = rng.uniform(-0.25, 0.25, (B, max(n - 1, 0), 6, 6))  # contractive: well-conditioned recursion
    rhs = rng.uniform(-1, 1, (B, n, 6))
    x = gpu_ctx.block_bidiag_solve6(coupling, rhs, upper)
    for b in range(B):
        want, _ = oracle.bidiag_solve(coupling[b] if n > 1 else np.zeros((1, 6, 6)), rhs[b], upper)
        assert np.linalg.norm(x[b] - want) / max(1.0, np.linalg.norm(want)) <= 1e-13


def test_bidiag6_spec_known_answer(gpu_ctx):
    """b = [2, 2], c = [1, 0, 0] -> [1, 2, 4] (scalar blocks
    embedded as 2 I and e), and the upper orientation -> [4, 2, 1]."""
    coupling = np.stack([2.0 * np.eye(6)] * 2)[None]
    rhs = np.zeros((1, 3, 6))
    rhs[0, 0] = 1.0
    x = gpu_ctx.block_bidiag_solve6(coupling, rhs, False)
    assert np.array_equal(x[0, :, 0], [1.0, 2.0, 4.0]) and np.array_equal(x[0, :, 5], [1.0, 2.0, 4.0])
    rhs_u = np.zeros((1, 3, 6))
    rhs_u[0, 2] = 1.0
    xu = gpu_ctx.block_bidiag_solve6(coupling, rhs_u, True)
    assert np.array_equal(xu[0, :, 0], [4.0, 2.0, 1.0])


def test_single_system_api(oracle, gpu_ctx):
    """Module-level mirrors of the reference's single-system calls
    (solve_lower/upper_bidiag, oee_solve) with their traces and errors."""
    import paper_1609_06779_b200 as pd
    st = pd.ScanTrace()
    x = pd.solve_lower_bidiag(np.stack([2.0 * np.eye(6)] * 2), np.vstack([np.ones(6), np.zeros((2, 6))]), st,
                              ctx=gpu_ctx)
    assert np.array_equal(x[:, 0], [1.0, 2.0, 4.0]) and st.rounds == 2
    xu = pd.solve_upper_bidiag(np.stack([2.0 * np.eye(6)] * 2), np.vstack([np.zeros((2, 6)), np.ones(6)]),
                               ctx=gpu_ctx)
    assert np.array_equal(xu[:, 0], [4.0, 2.0, 1.0])
    rng = np.random.default_rng(11)
    diag, upper, rhs = random_system(rng, 40)
    ot = pd.OeeTrace()
    x5 = pd.oee_solve(diag, upper, rhs, ot, ctx=gpu_ctx)
    want, _ = gpu_ctx.block_tridiag_solve5(diag[None], upper[None], rhs[None])[:2]
    assert np.array_equal(x5, want[0]) and ot.rounds == 6
    d3 = np.stack([np.eye(5), np.zeros((5, 5)), np.eye(5)])
    with pytest.raises(pd.SingularBlockError) as e:
        pd.oee_solve(d3, np.stack([0.1 * np.eye(5)] * 2), np.ones((3, 5)), ctx=gpu_ctx)
    assert (e.value.round(), e.value.index()) == (1, 1)
    assert "odd-even elimination: singular pivot block (round 1, block 1)" in str(e.value)
