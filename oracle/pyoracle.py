"""TEST INFRASTRUCTURE — ctypes bindings of the CPU oracle (oracle/oracle.hpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module; the product path (paper_1609_06779_b200) never does.

Chains travel as float64 arrays of shape (n, 31) in LinkSpec field order
(mass, com[3], inertia_rot[9] row-major, joint_screw[6], home R[9], home p[3]),
see oracle.hpp kLinkFields.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

JSIIA, ABIA, CFA = 0, 1, 2
ALGOS = {"jsiia": JSIIA, "abia": ABIA, "cfa": CFA}

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_mt19937_64_nth.restype = C.c_uint64
        L.orc_mt19937_64_nth.argtypes = [C.c_uint64, C.c_int64]
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_workload_seed.restype = C.c_uint64
        L.orc_workload_seed.argtypes = [C.c_uint64, C.c_int, C.c_int]
        L.orc_random_chain.argtypes = [C.c_int, C.c_uint64, _D, _D, C.c_char_p, C.c_int]
        L.orc_workload_chains.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, _D]
        L.orc_workload_inputs.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, _D, _D, _D]
        L.orc_validate_chain.argtypes = [C.c_int, _D, _D, C.c_char_p, C.c_int]
        L.orc_spatial_inertia.argtypes = [C.c_double, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_screw_exp.argtypes = [_D, C.c_double, _D, _D]
        L.orc_small_adjoint.argtypes = [_D, _D]
        L.orc_adjoint_of.argtypes = [_D, _D, _D]
        L.orc_assemble_kinematics.argtypes = [C.c_int, _D, _D, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_inverse_dynamics.argtypes = [C.c_int, _D, _D, _D, _D, _D, _D, _D, _D, C.c_int, _D, _I,
                                           C.c_char_p, C.c_int]
        L.orc_link_states.argtypes = [C.c_int, _D, _D, _D, _D, _D, _D, _D, _D, C.c_int, _D, _D, _D,
                                      C.c_char_p, C.c_int]
        L.orc_newton_euler.argtypes = [C.c_int, _D, _D, _D, _D, _D, C.c_int, _D, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_joint_space_inertia.argtypes = [C.c_int, _D, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_forward_dynamics.argtypes = [C.c_int, C.c_int, _D, _D, _D, C.c_int, _D, C.c_int, _D, C.c_int, _D, _I,
                                           _I, _I, C.c_char_p, C.c_int]
        L.orc_batch_forward_dynamics.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int64, _D, _D, _D, _D, _D,
                                                 _D, _I, C.c_int]
        L.orc_articulated_body_inertias.argtypes = [C.c_int, _D, _D, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_constraint_basis.argtypes = [C.c_int, _D, _D]
        L.orc_cfa_operators.argtypes = [C.c_int, _D, _D, _D, _D, _D, _D, _D, _D, _D, C.c_char_p, C.c_int]
        L.orc_bidiag_solve.argtypes = [C.c_int, C.c_int, C.c_int, _D, _D, _D, _I]
        L.orc_scan_int64.argtypes = [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _I]
        L.orc_tridiag_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _D, _D, _D, _D, _I, _I, _I,
                                        C.c_char_p, C.c_int]
        L.orc_oee_round.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _D, _D, _D]
        L.orc_fullpivlu_rank5.argtypes = [_D]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(Exception):
    """Carries the reference exception class as `kind` and its message."""

    KINDS = {1: "invalid_argument", 2: "ModelError", 3: "DynamicsError", 4: "SingularBlockError", 7: "internal"}

    def __init__(self, status, msg, round_=-1, index=-1):
        super().__init__(msg)
        self.status = status
        self.kind = self.KINDS.get(status, "unknown")
        self.round = round_
        self.index = index


def _check(st, err, r=None, i=None):
    if st != 0:
        raise OracleError(st, err.value.decode(), r.value if r is not None else -1, i.value if i is not None else -1)


def _err():
    return C.create_string_buffer(512)


# ---------------------------------------------------------------- RNG / model
def mt19937_64_nth(seed, nth):
    return int(lib().orc_mt19937_64_nth(seed, nth))


def mix(x):
    return int(lib().orc_mix(x))


def workload_seed(seed, n_links, n_groups):
    return int(lib().orc_workload_seed(seed, n_links, n_groups))


def random_chain(n, seed):
    links = np.zeros((n, 31))
    g = np.zeros(3)
    e = _err()
    _check(lib().orc_random_chain(n, seed, _p(links), _p(g), e, 512), e)
    return links, g


def workload_chains(cell_seed, n_links, n_groups, g0=0):
    links = np.zeros((n_groups, n_links, 31))
    st = lib().orc_workload_chains(cell_seed, n_links, g0, n_groups, _p(links))
    assert st == 0
    return links


def workload_inputs(cell_seed, n_links, n_groups, repeat):
    q = np.zeros((n_groups, n_links))
    qd = np.zeros_like(q)
    dr = np.zeros_like(q)
    lib().orc_workload_inputs(cell_seed, n_links, n_groups, repeat, _p(q), _p(qd), _p(dr))
    return q, qd, dr


def validate_chain(links, gravity=None):
    links = _f(links)
    g = _f(gravity if gravity is not None else [0, 0, -9.81])
    e = _err()
    _check(lib().orc_validate_chain(links.shape[0], _p(links), _p(g), e, 512), e)


def spatial_inertia(mass, com, Ic):
    out = np.zeros(36)
    e = _err()
    _check(lib().orc_spatial_inertia(float(mass), _p(_f(com)), _p(_f(Ic)), _p(out), e, 512), e)
    return out.reshape(6, 6)


def screw_exp(s, q):
    R = np.zeros(9)
    p = np.zeros(3)
    lib().orc_screw_exp(_p(_f(s)), float(q), _p(R), _p(p))
    return R.reshape(3, 3), p


def small_adjoint(v):
    out = np.zeros(36)
    lib().orc_small_adjoint(_p(_f(v)), _p(out))
    return out.reshape(6, 6)


def adjoint_of(R, p):
    out = np.zeros(36)
    lib().orc_adjoint_of(_p(_f(R)), _p(_f(p)), _p(out))
    return out.reshape(6, 6)


def assemble_kinematics(links, q):
    links = _f(links)
    n = links.shape[0]
    rel = np.zeros((n, 12))
    tr = np.zeros((max(n - 1, 0), 36))
    base = np.zeros(36)
    e = _err()
    _check(lib().orc_assemble_kinematics(n, _p(links), _p(_f(q)), _p(rel), _p(tr) if n > 1 else None,
                                         _p(base), e, 512), e)
    return rel, tr.reshape(-1, 6, 6), base.reshape(6, 6)


# ---------------------------------------------------------------- dynamics
def _opt6(v):
    return None if v is None else _p(_f(v))


def inverse_dynamics(links, gravity, q, qd, qdd, base_v=None, base_a=None, tip=None, apply_gravity=True,
                     trace=False):
    links = _f(links)
    n = links.shape[0]
    tau = np.zeros(n)
    tr = (C.c_int * 4)()
    e = _err()
    _check(lib().orc_inverse_dynamics(n, _p(links), _p(_f(gravity)), _p(_f(q)), _p(_f(qd)), _p(_f(qdd)),
                                      _opt6(base_v), _opt6(base_a), _opt6(tip), int(apply_gravity), _p(tau),
                                      tr if trace else None, e, 512), e)
    return (tau, list(tr)) if trace else tau


def link_states(links, gravity, q, qd, qdd, base_v=None, base_a=None, tip=None, apply_gravity=True):
    links = _f(links)
    n = links.shape[0]
    v, a, f = np.zeros((n, 6)), np.zeros((n, 6)), np.zeros((n, 6))
    e = _err()
    _check(lib().orc_link_states(n, _p(links), _p(_f(gravity)), _p(_f(q)), _p(_f(qd)), _p(_f(qdd)),
                                 _opt6(base_v), _opt6(base_a), _opt6(tip), int(apply_gravity), _p(v), _p(a),
                                 _p(f), e, 512), e)
    return v, a, f


def newton_euler(links, gravity, q, qd, qdd, apply_gravity=True):
    links = _f(links)
    n = links.shape[0]
    v, a, f, t = np.zeros((n, 6)), np.zeros((n, 6)), np.zeros((n, 6)), np.zeros(n)
    e = _err()
    _check(lib().orc_newton_euler(n, _p(links), _p(_f(gravity)), _p(_f(q)), _p(_f(qd)), _p(_f(qdd)),
                                  int(apply_gravity), _p(v), _p(a), _p(f), _p(t), e, 512), e)
    return v, a, f, t


def joint_space_inertia(links, q, gravity=(0, 0, -9.81)):
    links = _f(links)
    n = links.shape[0]
    M = np.zeros((n, n))
    e = _err()
    _check(lib().orc_joint_space_inertia(n, _p(links), _p(_f(gravity)), _p(_f(q)), _p(M), e, 512), e)
    return M


def mass_matrix_ne(links, q):
    """oracles.hpp:267-278: columns of sequential NE with unit qdd, gravity off."""
    n = len(links)
    M = np.zeros((n, n))
    for j in range(n):
        u = np.zeros(n)
        u[j] = 1.0
        M[:, j] = newton_euler(links, [0, 0, 0], q, np.zeros(n), u, apply_gravity=False)[3]
    return M


def dense_forward_dynamics(links, gravity, q, qd, tau):
    """oracles.hpp:280-287: tau - NE bias solved against the NE mass matrix."""
    n = len(links)
    bias = newton_euler(links, gravity, q, qd, np.zeros(n))[3]
    return np.linalg.solve(mass_matrix_ne(links, q), np.asarray(tau) - bias)


def forward_dynamics(algo, links, gravity, q, qd, tau, trace=False):
    links = _f(links).reshape(-1, 31)
    n = links.shape[0]
    q, qd, tau = _f(q), _f(qd), _f(tau)
    qdd = np.zeros(max(n, 1))
    tr = (C.c_int * 4)()
    r, i = C.c_int(-1), C.c_int(-1)
    e = _err()
    algo = ALGOS.get(algo, algo)
    _check(lib().orc_forward_dynamics(algo, n, _p(links) if n else None, _p(_f(gravity)), _p(q), len(q), _p(qd),
                                      len(qd), _p(tau), len(tau), _p(qdd), tr if trace else None, C.byref(r),
                                      C.byref(i), e, 512), e, r, i)
    qdd = qdd[:n]
    return (qdd, list(tr)) if trace else qdd


def batch_forward_dynamics(algo, models, gravity, q, qd, tau, nthreads=0):
    """models: (M, n, 31) with M == 1 (shared) or M == batch; q: (batch, n)."""
    models = _f(models)
    q, qd, tau = _f(q), _f(qd), _f(tau)
    B, n = q.shape
    gravity = _f(np.broadcast_to(np.asarray(gravity, dtype=np.float64), (models.shape[0], 3)))
    qdd = np.zeros_like(q)
    st = np.zeros(B, dtype=np.int32)
    lib().orc_batch_forward_dynamics(ALGOS.get(algo, algo), B, n, models.shape[0], _p(models), _p(gravity),
                                     _p(q), _p(qd), _p(tau), _p(qdd), st.ctypes.data_as(_I), int(nthreads))
    return qdd, st


def articulated_body_inertias(links, q):
    links = _f(links)
    n = links.shape[0]
    I, lam, g = np.zeros((n, 36)), np.zeros(n), np.zeros((n, 6))
    e = _err()
    _check(lib().orc_articulated_body_inertias(n, _p(links), _p(_f(q)), _p(I), _p(lam), _p(g), e, 512), e)
    return I.reshape(n, 6, 6), lam, g


def constraint_basis(links):
    links = _f(links)
    n = links.shape[0]
    out = np.zeros((n, 30))
    lib().orc_constraint_basis(n, _p(links), _p(out))
    return out.reshape(n, 6, 5)


def cfa_operators(links, q):
    links = _f(links)
    n = links.shape[0]
    m = max(n - 1, 1)
    d, u = np.zeros((n, 25)), np.zeros((m, 25))
    cs, cd, cu = np.zeros((m, 5)), np.zeros((n, 5)), np.zeros((m, 5))
    jd, jo = np.zeros(n), np.zeros(m)
    e = _err()
    _check(lib().orc_cfa_operators(n, _p(links), _p(_f(q)), _p(d), _p(u), _p(cs), _p(cd), _p(cu), _p(jd), _p(jo),
                                   e, 512), e)
    k = n - 1
    return dict(diag=d.reshape(n, 5, 5), upper=u[:k].reshape(k, 5, 5), cross_sub=cs[:k], cross_diag=cd,
                cross_super=cu[:k], joint_diag=jd, joint_off=jo[:k])


# ---------------------------------------------------------------- primitives
def bidiag_solve(coupling, rhs, upper=False):
    rhs = _f(rhs)
    n, D = rhs.shape
    x = np.zeros_like(rhs)
    r = C.c_int(0)
    c = _f(coupling) if n > 1 else np.zeros((1, D, D))
    st = lib().orc_bidiag_solve(D, int(upper), n, _p(c), _p(rhs), _p(x), C.byref(r))
    assert st == 0
    return x, r.value


def scan_int64(items):
    a = np.ascontiguousarray(items, dtype=np.int64)
    out = np.zeros_like(a)
    r = C.c_int(0)
    lib().orc_scan_int64(len(a), a.ctypes.data_as(C.POINTER(C.c_int64)), out.ctypes.data_as(C.POINTER(C.c_int64)),
                         C.byref(r))
    return out, r.value


def tridiag_solve(diag, upper, rhs, thomas=False):
    diag = _f(diag)
    n, B = diag.shape[0], diag.shape[1]
    rhs = _f(rhs).reshape(n, B, -1)
    M = rhs.shape[2]
    x = np.zeros_like(rhs)
    up = _f(upper) if n > 1 else np.zeros((1, B, B))
    rr, ri, ro = C.c_int(0), C.c_int(-1), C.c_int(-1)
    e = _err()
    _check(lib().orc_tridiag_solve(B, M, int(thomas), n, _p(diag), _p(up), _p(rhs), _p(x), C.byref(ro),
                                   C.byref(rr), C.byref(ri), e, 512), e, rr, ri)
    return x, ro.value


def oee_round(diag, coupling, rhs, distance, round_):
    diag, rhs = _f(diag).copy(), _f(rhs).copy()
    n, B = diag.shape[0], diag.shape[1]
    c = np.zeros((max(n, 1), B, B))
    c[: len(coupling)] = coupling
    st = lib().orc_oee_round(B, n, distance, round_, _p(diag), _p(c), _p(rhs))
    assert st == 0, st
    return diag, c[: max(n - 2 * distance, 0)], rhs


def fullpivlu_rank5(m):
    return int(lib().orc_fullpivlu_rank5(_p(_f(m))))
