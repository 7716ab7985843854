"""GPU parity of the two building blocks at every block size the reference's
templates take, not only the sizes the dynamics use: BlockBiDiagSystem<D>
with solve_lower_bidiag / solve_upper_bidiag (scan.hpp:100-168, D = 1..6,
pd_block_bidiag_solve) and oee_solve<B, M> (oee.hpp:149-189, B = 1..6,
M = 1..4, pd_block_tridiag_solve). Ported from the reference's
tests/test_oee.cpp (agreement with a dense solve for B = 1, 2, 5 and n up to
48, multi-column right-hand sides, the B = 2 singular-pivot report, the
one-row system, reproducibility) and tests/test_scan.cpp (the D = 2 affine
recursion); the dense / sequential references are numpy."""
import numpy as np
import pytest

import paper_1609_06779_b200 as pd

pytestmark = pytest.mark.gpu


def random_tridiag(rng, n, b):
    """oracles.hpp:161-177: random couplings, diagonal a a^T + (1 + norms of
    the adjacent couplings) I -- symmetric, block diagonally dominant."""
    upper = rng.uniform(-1, 1, (max(n - 1, 0), b, b))
    diag = np.empty((n, b, b))
    for k in range(n):
        a = rng.uniform(-1, 1, (b, b))
        dom = 1.0
        if k > 0:
            dom += np.linalg.norm(upper[k - 1])
        if k + 1 < n:
            dom += np.linalg.norm(upper[k])
        diag[k] = a @ a.T + dom * np.eye(b)
    return diag, upper


def dense(diag, upper):
    n, b = diag.shape[0], diag.shape[1]
    full = np.zeros((n * b, n * b))
    for k in range(n):
        full[b * k:b * k + b, b * k:b * k + b] = diag[k]
        if k + 1 < n:
            full[b * k:b * k + b, b * k + b:b * k + 2 * b] = upper[k]
            full[b * k + b:b * k + 2 * b, b * k:b * k + b] = upper[k].T
    return full


def rel_gap(x, want):
    return np.linalg.norm(x - want) / max(1.0, np.linalg.norm(want))


@pytest.mark.parametrize("b", [1, 2, 5])
def test_oee_agrees_with_dense_solve_all_sizes(gpu_ctx, b):
    """test_oee.cpp:22-43: n = 1..48, rel gap < 1e-10, ceil_log2(n) rounds."""
    rng = np.random.default_rng(101 + b)
    for n in range(1, 49):
        S = 2
        systems = [random_tridiag(rng, n, b) for _ in range(S)]
        diag = np.stack([s[0] for s in systems])
        upper = np.stack([s[1] for s in systems]) if n > 1 else np.zeros((S, 0, b, b))
        rhs = rng.uniform(-1, 1, (S, n, b))
        x, st, _, _ = gpu_ctx.block_tridiag_solve(diag, upper, rhs)
        assert (st == 0).all(), (b, n)
        for s in range(S):
            want = np.linalg.solve(dense(diag[s], upper[s]), rhs[s].ravel()).reshape(n, b)
            assert rel_gap(x[s], want) < 1e-10, (b, n, rel_gap(x[s], want))
        tr = pd.OeeTrace()
        one = pd.oee_solve(diag[0], upper[0], rhs[0], tr, ctx=gpu_ctx)
        assert np.array_equal(one, x[0]) and tr.rounds == pd.ceil_log2(n)


@pytest.mark.parametrize("b,m", [(3, 1), (4, 2), (6, 1), (6, 4), (5, 3), (2, 3), (1, 4)])
@pytest.mark.parametrize("n", [1, 7, 17, 64, 256])
def test_oee_block_and_column_counts(gpu_ctx, b, m, n):
    """Every (B, M) instantiation against a dense solve; (5, 3) at n = 17 is
    test_oee.cpp:45-58 (multi-column right-hand sides carried through the
    rounds)."""
    rng = np.random.default_rng(1000 * b + 10 * m + n)
    diag, upper = random_tridiag(rng, n, b)
    rhs = rng.uniform(-1, 1, (n, b, m))
    x = pd.oee_solve(diag, upper, rhs, ctx=gpu_ctx)
    assert x.shape == (n, b, m)
    A = dense(diag, upper)
    for c in range(m):
        want = np.linalg.solve(A, rhs[:, :, c].ravel()).reshape(n, b)
        assert rel_gap(x[:, :, c], want) < 1e-10


def test_oee_singular_pivot_block_size_2(gpu_ctx):
    """test_oee.cpp:106-126: a rank-deficient pivot in the first round is
    reported with round 1 and block 1."""
    diag = np.stack([np.eye(2), np.zeros((2, 2)), np.eye(2)])
    upper = np.stack([0.1 * np.eye(2)] * 2)
    with pytest.raises(pd.SingularBlockError) as e:
        pd.oee_solve(diag, upper, np.ones((3, 2)), ctx=gpu_ctx)
    assert (e.value.round(), e.value.index()) == (1, 1)
    assert "singular pivot" in str(e.value)


def test_oee_single_row_needs_no_rounds(gpu_ctx):
    """test_oee.cpp:96-104."""
    rng = np.random.default_rng(123)
    diag, upper = random_tridiag(rng, 1, 5)
    rhs = rng.uniform(-1, 1, (1, 5))
    tr = pd.OeeTrace()
    x = pd.oee_solve(diag, upper, rhs, tr, ctx=gpu_ctx)
    assert tr.rounds == 0
    assert np.linalg.norm(diag[0] @ x[0] - rhs[0]) < 1e-12


def test_oee_reproducible(gpu_ctx):
    """test_oee.cpp:128-140: the same system twice gives bit-identical x."""
    for b in (2, 5):
        diag, upper = random_tridiag(np.random.default_rng(131), 37, b)
        rhs = np.random.default_rng(132).uniform(-1, 1, (37, b))
        xa = pd.oee_solve(diag, upper, rhs, ctx=gpu_ctx)
        xb = pd.oee_solve(diag.copy(), upper.copy(), rhs.copy(), ctx=gpu_ctx)
        assert np.array_equal(xa, xb)


def recursion(coupling, rhs, upper):
    n = rhs.shape[0]
    x = np.empty_like(rhs)
    if upper:
        x[n - 1] = rhs[n - 1]
        for k in range(n - 2, -1, -1):
            x[k] = coupling[k] @ x[k + 1] + rhs[k]
    else:
        x[0] = rhs[0]
        for k in range(1, n):
            x[k] = coupling[k - 1] @ x[k - 1] + rhs[k]
    return x


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("n", [1, 2, 9, 31, 33, 100, 1000])
@pytest.mark.parametrize("upper", [False, True])
def test_bidiag_every_block_size(gpu_ctx, d, n, upper):
    """scan.hpp:100-168 for D = 1..6 against the sequential recursion."""
    rng = np.random.default_rng(10 * d + n + 1000 * upper)
    S = 3
    coupling = rng.uniform(-0.5, 0.5, (S, max(n - 1, 0), d, d)) / np.sqrt(d)  # contractive
    rhs = rng.uniform(-1, 1, (S, n, d))
    x = gpu_ctx.block_bidiag_solve(coupling, rhs, upper)
    for s in range(S):
        want = recursion(coupling[s], rhs[s], upper)
        assert rel_gap(x[s], want) <= 1e-13


def test_affine_composition_carries_the_recursion(gpu_ctx):
    """test_scan.cpp:48-71: nine D = 2 steps with random coefficients; the
    scan's prefixes hold x[k] = c[k] x[k-1] + o[k]."""
    rng = np.random.default_rng(21)
    coupling = rng.uniform(-1, 1, (8, 2, 2))
    rhs = rng.uniform(-1, 1, (9, 2))
    tr = pd.ScanTrace()
    x = pd.solve_lower_bidiag(coupling, rhs, tr, ctx=gpu_ctx)
    want = recursion(coupling, rhs, False)
    assert np.abs(x[0] - want[0]).max() < 1e-14
    assert np.abs(x - want).max() < 1e-12
    assert tr.rounds == 4


@pytest.mark.parametrize("b", [2, 5])
@pytest.mark.parametrize("n", [5, 16, 33, 100])
def test_elimination_rounds_on_a_state(gpu_ctx, b, n):
    """test_oee.cpp:60-94: pivots stay symmetric round to round, the
    couplings shrink by rows and the distance doubles; after the last round
    every row solves alone (coefficient_solve), bit for bit what oee_solve
    returns (same kernel arithmetic, state through memory)."""
    rng = np.random.default_rng(121 + n + b)
    diag, upper = random_tridiag(rng, n, b)
    rhs = rng.uniform(-1, 1, (n, b))
    st = pd.OeeState(diag.copy(), upper.copy(), rhs.copy())
    rounds = pd.ceil_log2(n)
    for j in range(rounds):
        pd.oee_eliminate_round(st, ctx=gpu_ctx)
        assert np.abs(st.diag - np.transpose(st.diag, (0, 2, 1))).max() < 1e-10
        assert st.distance == 2 << j and st.coupling.shape[0] == max(0, n - (2 << j))
    assert st.round == rounds and st.coupling.shape[0] == 0
    x = pd.oee_solve(diag, upper, rhs, ctx=gpu_ctx)
    xr = np.stack([pd.coefficient_solve(st.diag[k], st.rhs[k], st.round, k, ctx=gpu_ctx) for k in range(n)])
    assert np.array_equal(xr, x)


def test_elimination_round_singular_pivot_leaves_state(gpu_ctx):
    """oee.hpp:130-138: a singular pivot throws (round, block) and the state
    is not advanced."""
    diag = np.stack([np.eye(2), np.zeros((2, 2)), np.eye(2)])
    st = pd.OeeState(diag.copy(), np.stack([0.1 * np.eye(2)] * 2), np.ones((3, 2)))
    with pytest.raises(pd.SingularBlockError) as e:
        pd.oee_eliminate_round(st, ctx=gpu_ctx)
    assert (e.value.round(), e.value.index()) == (1, 1)
    assert st.round == 0 and st.distance == 1 and np.array_equal(st.diag, diag)
    with pytest.raises(pd.SingularBlockError) as e2:
        pd.coefficient_solve(np.zeros((3, 3)), np.ones((3, 6)), 4, 9, ctx=gpu_ctx)
    assert (e2.value.round(), e2.value.index()) == (4, 9)
    x = pd.coefficient_solve(2.0 * np.eye(3), np.ones((3, 6)), 1, 0, ctx=gpu_ctx)  # > 4 columns: two launches
    assert np.array_equal(x, 0.5 * np.ones((3, 6)))
