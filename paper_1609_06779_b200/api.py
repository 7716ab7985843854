"""Python mirror of the reference's forward-dynamics API over the C-ABI.

Same names, argument meaning and error behaviour as
proj/core/include/pardyn/forward_dynamics.hpp and inverse_dynamics.hpp:

  FdAlgo {jsiia, abia, cfa}                    forward_dynamics.hpp:29
  forward_dynamics(chain, q, qdot, tau, algo)  forward_dynamics.hpp:103-105
  jsiia_/abia_/cfa_forward_dynamics            forward_dynamics.hpp:38-42,58-62,98-101
  FdProblem / FdResult                         forward_dynamics.hpp:111-123
  batch_forward_dynamics(problems, algo)       forward_dynamics.hpp:125-126
  IdOptions / LinkStates                       inverse_dynamics.hpp:23-34
  inverse_dynamics / bias_torque / link_states inverse_dynamics.hpp:71-83
  joint_space_inertia(chain, q)                forward_dynamics.hpp:34-35
  validate_chain / load_chain / save_chain     model.hpp:56-82, model.cpp:75-115,244-337
  LinkSpec / RobotChain                        model.hpp:17-30
  ModelError / DynamicsError / SingularBlockError(round, index)   types.hpp:21-46
  std::invalid_argument -> InvalidArgument (a ValueError)

Every solve runs on the GPU through libpardyn_b200.so (no CPU fallback).
Batches are bucketed by link count, packed, solved with one C-ABI call per
bucket and scattered back; per-slot errors carry the reference's messages.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _capi


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class ModelError(RuntimeError):
    """pardyn::ModelError (types.hpp:21-24)."""


class DynamicsError(RuntimeError):
    """pardyn::DynamicsError (types.hpp:28-31)."""


class SingularBlockError(DynamicsError):
    """pardyn::SingularBlockError (types.hpp:35-46)."""

    def __init__(self, round_: int, index: int, what: str):
        super().__init__(what)
        self._round, self._index = round_, index

    def round(self) -> int:
        return self._round

    def index(self) -> int:
        return self._index


class CudaError(RuntimeError):
    pass


class FdAlgo(enum.IntEnum):
    jsiia = _capi.PD_JSIIA
    abia = _capi.PD_ABIA
    cfa = _capi.PD_CFA


@dataclass
class SE3Transform:
    """spatial.hpp:75-97: x_target = rotation @ x_source + translation."""
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class LinkSpec:
    """model.hpp:17-23 (defaults match the reference). joint_screw stacks
    (angular, linear) -- Twist::stacked() of the reference."""
    mass: float = 1.0
    com: np.ndarray = field(default_factory=lambda: np.zeros(3))
    inertia_rot: np.ndarray = field(default_factory=lambda: np.eye(3))
    joint_screw: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 1.0, 0.0, 0.0, 0.0]))
    home_transform: SE3Transform = field(default_factory=SE3Transform)

    def to_record(self) -> np.ndarray:
        h = self.home_transform
        return np.concatenate([[self.mass], np.ravel(self.com), np.ravel(self.inertia_rot), np.ravel(self.joint_screw),
                               np.ravel(h.rotation), np.ravel(h.translation)]).astype(np.float64)

    @staticmethod
    def from_record(r) -> "LinkSpec":
        r = np.asarray(r, dtype=np.float64)
        return LinkSpec(float(r[0]), r[1:4].copy(), r[4:13].reshape(3, 3).copy(), r[13:19].copy(),
                        SE3Transform(r[19:28].reshape(3, 3).copy(), r[28:31].copy()))


@dataclass
class RobotChain:
    """model.hpp:25-30."""
    links: List[LinkSpec] = field(default_factory=list)
    gravity: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -9.81]))

    def size(self) -> int:
        return len(self.links)

    def to_records(self) -> np.ndarray:
        if not self.links:
            return np.zeros((0, _capi.LINK_FIELDS))
        return np.stack([l.to_record() for l in self.links])

    @staticmethod
    def from_records(records, gravity=(0.0, 0.0, -9.81)) -> "RobotChain":
        return RobotChain([LinkSpec.from_record(r) for r in np.asarray(records)], np.asarray(gravity, np.float64))


@dataclass
class ExecTrace:
    """trace.hpp:24-39, filled with the designed dependency structure of the
    kernel variant that ran."""
    parallel_link_stages: int = 0
    longest_sequential_link_chain: int = 0
    scan_rounds_max: int = 0
    oee_rounds: int = 0


@dataclass
class FdProblem:
    chain: RobotChain
    q: np.ndarray
    qdot: np.ndarray
    tau: np.ndarray


@dataclass
class FdResult:
    qddot: np.ndarray = field(default_factory=lambda: np.zeros(0))
    error: str = ""

    def ok(self) -> bool:
        return self.error == ""


@dataclass
class IdOptions:
    """inverse_dynamics.hpp:23-28: base twist / acceleration (angular, linear),
    tip wrench (moment, force) in the last link's frame, gravity switch."""
    base_velocity: np.ndarray = field(default_factory=lambda: np.zeros(6))
    base_acceleration: np.ndarray = field(default_factory=lambda: np.zeros(6))
    tip_wrench: np.ndarray = field(default_factory=lambda: np.zeros(6))
    apply_gravity: bool = True

    def to_c(self) -> "_capi.IdOptions":
        o = _capi.IdOptions()
        for k in range(6):
            o.base_velocity[k] = float(np.ravel(self.base_velocity)[k])
            o.base_acceleration[k] = float(np.ravel(self.base_acceleration)[k])
            o.tip_wrench[k] = float(np.ravel(self.tip_wrench)[k])
        o.apply_gravity = 1 if self.apply_gravity else 0
        return o


@dataclass
class LinkStates:
    """inverse_dynamics.hpp:30-34: per-link twists, accelerations, wrenches,
    each (n, 6) stacked (angular|moment, linear|force)."""
    velocity: np.ndarray
    acceleration: np.ndarray
    force: np.ndarray


def ceil_log2(n: int) -> int:
    k, p = 0, 1
    while p < n:
        p <<= 1
        k += 1
    return k


# --------------------------------------------------------------------------- context
class Context:
    """A pd_ctx on one CUDA device (one per process per device)."""

    def __init__(self, device: int = 0):
        L = _capi.load()
        h = C.c_void_p()
        st = L.pd_create(C.byref(h), int(device))
        if st != _capi.PD_OK:
            raise CudaError(f"pd_create(device={device}) failed: {L.pd_status_string(st).decode()}")
        self._h = h
        self._L = L
        self.device = device
        self._models_key = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.pd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _check(self, st):
        if st == _capi.PD_OK:
            return
        msg = self._L.pd_last_error(self._h).decode()
        if st == _capi.PD_INVALID_ARGUMENT:
            raise InvalidArgument(msg)
        raise CudaError(f"{self._L.pd_status_string(st).decode()}: {msg}")

    def set_models(self, links: np.ndarray, gravity: Optional[np.ndarray] = None):
        """links: (M, n, 31) float64; gravity: (M, 3) or None. Returns
        (model_status, model_rule) int32 arrays."""
        links = np.ascontiguousarray(links, dtype=np.float64)
        M, n = links.shape[0], links.shape[1]
        g = None if gravity is None else np.ascontiguousarray(np.broadcast_to(gravity, (M, 3)), dtype=np.float64)
        ms = np.zeros(M, np.int32)
        mr = np.zeros(M, np.int32)
        self._check(self._L.pd_set_models(self._h, M, n, _capi.dptr(links), _capi.dptr(g), _capi.iptr(ms),
                                          _capi.iptr(mr)))
        self.n_links, self.n_models = n, M
        return ms, mr

    def set_models_workload(self, cell_seed: int, n_links: int, count: int, g0: int = 0, gravity=None):
        """Chains [g0, g0+count) of the reference benchmark cell generated,
        validated and packed on the device (no host model buffer). Returns
        (model_status, model_rule)."""
        g = None if gravity is None else np.ascontiguousarray(gravity, dtype=np.float64).reshape(3)
        ms = np.zeros(count, np.int32)
        mr = np.zeros(count, np.int32)
        self._check(self._L.pd_set_models_workload(self._h, int(cell_seed), int(n_links), int(g0), int(count),
                                                   _capi.dptr(g), _capi.iptr(ms), _capi.iptr(mr)))
        self.n_links, self.n_models = n_links, count
        return ms, mr

    def workload_chains_device(self, cell_seed: int, n_links: int, count: int, d_links, g0: int = 0):
        """Raw link records [count][n][31] into the device pointer d_links."""
        self._check(self._L.pd_workload_chains_device(self._h, int(cell_seed), int(n_links), int(g0), int(count),
                                                      d_links))

    def solve(self, algo, q, qdot, tau, out=None, status_out=None):
        """Host-buffer solve: q/qdot/tau (B, n) -> (qddot, status, round, index).
        `out` may be a preallocated (pinned) (B, n) float64 array and
        `status_out` a preallocated triple of (B,) int32 arrays (reused across
        calls, like C callers reuse their slot arrays)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        tau = np.ascontiguousarray(tau, dtype=np.float64)
        B = q.shape[0]
        qdd = np.empty_like(q) if out is None else out
        if status_out is None:
            st, rd, ix = np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32)
        else:
            st, rd, ix = status_out
        self._check(self._L.pd_forward_dynamics(self._h, int(algo), B, _capi.dptr(q), _capi.dptr(qd), _capi.dptr(tau),
                                                _capi.dptr(qdd), _capi.iptr(st), _capi.iptr(rd), _capi.iptr(ix)))
        return qdd, st, rd, ix

    def solve_traced(self, algo, q, qdot, tau):
        """Host-buffer solve through the log-depth (CTA-per-chain) variants,
        returning (qddot, status, round, index, ExecTrace of the variant)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        tau = np.ascontiguousarray(tau, dtype=np.float64)
        B = q.shape[0]
        qdd = np.empty_like(q)
        st, rd, ix = np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32)
        tr = _capi.ExecTraceC()
        self._check(self._L.pd_forward_dynamics_traced(self._h, int(algo), B, _capi.dptr(q), _capi.dptr(qd),
                                                       _capi.dptr(tau), _capi.dptr(qdd), _capi.iptr(st),
                                                       _capi.iptr(rd), _capi.iptr(ix), C.byref(tr)))
        return qdd, st, rd, ix, ExecTrace(tr.parallel_link_stages, tr.longest_sequential_link_chain,
                                          tr.scan_rounds_max, tr.oee_rounds)

    def last_variant(self) -> str:
        """Kernel variant(s) the last forward-dynamics call ran."""
        return self._L.pd_last_variant(self._h).decode()

    def last_trace(self) -> "ExecTrace":
        tr = _capi.ExecTraceC()
        self._check(self._L.pd_last_trace(self._h, C.byref(tr)))
        return ExecTrace(tr.parallel_link_stages, tr.longest_sequential_link_chain, tr.scan_rounds_max,
                         tr.oee_rounds)

    def set_selection_batch(self, batch: int):
        """Select kernels for `batch` problems (0 = each call's own batch):
        the parts of a split batch then run the whole batch's variants."""
        self._check(self._L.pd_set_selection_batch(self._h, int(batch)))

    def solve_device(self, algo, batch, d_q, d_qd, d_tau, d_qdd, d_st=None, d_rd=None, d_ix=None):
        """Device solve on raw device pointers ([link][problem] layout)."""
        self._check(self._L.pd_forward_dynamics_device(self._h, int(algo), int(batch), d_q, d_qd, d_tau, d_qdd, d_st,
                                                       d_rd, d_ix))

    def inverse_dynamics(self, q, qdot, qddot):
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        qdd = np.ascontiguousarray(qddot, dtype=np.float64)
        tau = np.empty_like(q)
        self._check(self._L.pd_inverse_dynamics(self._h, q.shape[0], _capi.dptr(q), _capi.dptr(qd), _capi.dptr(qdd),
                                                _capi.dptr(tau)))
        return tau

    def inverse_dynamics_opts(self, q, qdot, qddot, opts: Optional["IdOptions"] = None):
        """(B, n) host arrays -> tau (B, n); opts None = defaults."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        qdd = np.ascontiguousarray(qddot, dtype=np.float64)
        tau = np.empty_like(q)
        o = None if opts is None else C.byref(opts.to_c())
        self._check(self._L.pd_inverse_dynamics_opts(self._h, q.shape[0], _capi.dptr(q), _capi.dptr(qd),
                                                     _capi.dptr(qdd), o, _capi.dptr(tau)))
        return tau

    def inverse_dynamics_device(self, batch, d_q, d_qd, d_qdd, d_tau, opts: Optional["IdOptions"] = None):
        """Device inverse dynamics on raw device pointers ([link][problem])."""
        o = None if opts is None else C.byref(opts.to_c())
        self._check(self._L.pd_inverse_dynamics_device(self._h, int(batch), d_q, d_qd, d_qdd, o, d_tau))

    def bias_torque(self, q, qdot):
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        tau = np.empty_like(q)
        self._check(self._L.pd_bias_torque(self._h, q.shape[0], _capi.dptr(q), _capi.dptr(qd), _capi.dptr(tau)))
        return tau

    def link_states(self, q, qdot, qddot, opts: Optional["IdOptions"] = None):
        """(B, n) host arrays -> (velocity, acceleration, force), each (B, n, 6)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qdot, dtype=np.float64)
        qdd = np.ascontiguousarray(qddot, dtype=np.float64)
        B, n = q.shape
        v, a, f = (np.empty((B, n, 6)) for _ in range(3))
        o = None if opts is None else C.byref(opts.to_c())
        self._check(self._L.pd_link_states(self._h, B, _capi.dptr(q), _capi.dptr(qd), _capi.dptr(qdd), o,
                                           _capi.dptr(v), _capi.dptr(a), _capi.dptr(f)))
        return v, a, f

    def joint_space_inertia(self, q):
        """(B, n) host array -> M (B, n, n)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        B, n = q.shape
        M = np.empty((B, n, n))
        self._check(self._L.pd_joint_space_inertia(self._h, B, _capi.dptr(q), _capi.dptr(M)))
        return M

    # ---- the reference's operator builders, batched (pd_assemble_kinematics ... pd_cfa_apply)
    def assemble_kinematics(self, q):
        """q (B, n) against the current models -> rel (B, n, 12) [R row-major, p],
        base_transport (B, 6, 6), transport (B, n-1, 6, 6), screw (B, n, 6)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        B, n = q.shape
        rel, base = np.empty((B, n, 12)), np.empty((B, 6, 6))
        tr, sc = np.empty((B, max(n - 1, 0), 6, 6)), np.empty((B, n, 6))
        self._check(self._L.pd_assemble_kinematics(self._h, B, _capi.dptr(q), _capi.dptr(rel), _capi.dptr(base),
                                                   _capi.dptr(tr), _capi.dptr(sc)))
        return rel, base, tr, sc

    def link_inertias(self):
        """Spatial inertias of the current models -> (M, n, 6, 6)."""
        out = np.empty((max(self.n_models, 1), self.n_links, 6, 6))
        self._check(self._L.pd_link_inertias(self._h, _capi.dptr(out)))
        return out

    def articulated_body_inertias(self, transport, inertia, screw):
        """transport (B, n-1, 6, 6), inertia (B, n, 6, 6) or (n, 6, 6) shared,
        screw (B, n, 6) -> abi (B, n, 6, 6), joint_inertia (B, n), gain (B, n, 6),
        status (B,), index (B,)."""
        screw = np.ascontiguousarray(screw, dtype=np.float64)
        B, n = screw.shape[:2]
        inertia = np.ascontiguousarray(inertia, dtype=np.float64)
        shared = inertia.ndim == 3
        transport = np.ascontiguousarray(transport, dtype=np.float64).reshape(B, max(n - 1, 0), 6, 6)
        abi, lam, gain = np.empty((B, n, 6, 6)), np.empty((B, n)), np.empty((B, n, 6))
        st, ix = np.empty(B, np.int32), np.empty(B, np.int32)
        self._check(self._L.pd_articulated_body_inertias(
            self._h, B, n, _capi.dptr(transport), _capi.dptr(inertia), int(shared), _capi.dptr(screw),
            _capi.dptr(abi), _capi.dptr(lam), _capi.dptr(gain), _capi.iptr(st), _capi.iptr(ix)))
        return abi, lam, gain, st, ix

    def constraint_basis(self, screw):
        """screw (K, 6) -> basis (K, 6, 5)."""
        screw = np.ascontiguousarray(screw, dtype=np.float64).reshape(-1, 6)
        out = np.empty((screw.shape[0], 6, 5))
        self._check(self._L.pd_constraint_basis(self._h, screw.shape[0], _capi.dptr(screw), _capi.dptr(out)))
        return out

    def cfa_operators(self, inertia, transport, screw, basis):
        """-> dict of constraint diag (B, n, 5, 5) / upper (B, n-1, 5, 5),
        cross_sub / cross_super (B, n-1, 5), cross_diag (B, n, 5), joint_diag
        (B, n), joint_off (B, n-1), plus status / index (B,)."""
        screw = np.ascontiguousarray(screw, dtype=np.float64)
        B, n = screw.shape[:2]
        e = max(n - 1, 0)
        inertia = np.ascontiguousarray(inertia, dtype=np.float64)
        shared = inertia.ndim == 3
        transport = np.ascontiguousarray(transport, dtype=np.float64).reshape(B, e, 6, 6)
        basis = np.ascontiguousarray(basis, dtype=np.float64).reshape(B, n, 6, 5)
        o = {"diag": np.empty((B, n, 5, 5)), "upper": np.empty((B, e, 5, 5)), "cross_sub": np.empty((B, e, 5)),
             "cross_diag": np.empty((B, n, 5)), "cross_super": np.empty((B, e, 5)), "joint_diag": np.empty((B, n)),
             "joint_off": np.empty((B, e)), "status": np.empty(B, np.int32), "index": np.empty(B, np.int32)}
        self._check(self._L.pd_cfa_operators(
            self._h, B, n, _capi.dptr(inertia), int(shared), _capi.dptr(transport), _capi.dptr(screw),
            _capi.dptr(basis), *(_capi.dptr(o[k]) for k in ("diag", "upper", "cross_sub", "cross_diag",
                                                            "cross_super", "joint_diag", "joint_off")),
            _capi.iptr(o["status"]), _capi.iptr(o["index"])))
        return o

    def propagate(self, kind, base_transport, transport, screw, boundary, qdot=None, qddot=None, velocity=None,
                  acceleration=None, inertia=None):
        """One of the three propagations of inverse_dynamics.cpp:27-120 over
        dense kinematics (pd_propagate): kind PD_PROPAGATE_VELOCITIES /
        _ACCELERATIONS / _FORCES; arrays batched as in the C-ABI; -> (B, n, 6)."""
        screw = np.ascontiguousarray(screw, dtype=np.float64)
        B, n = screw.shape[:2]
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        inertia = f(inertia)
        shared = inertia is not None and inertia.ndim == 3
        out = np.empty((B, n, 6))
        args = [f(base_transport), f(np.reshape(transport, (B, max(n - 1, 0), 6, 6))), screw, inertia]
        self._check(self._L.pd_propagate(self._h, int(kind), B, n, *(_capi.dptr(a) for a in args), int(shared),
                                         *(_capi.dptr(f(a)) for a in (qdot, qddot, velocity, acceleration)),
                                         _capi.dptr(f(np.ravel(boundary))), _capi.dptr(out)))
        return out

    def cfa_apply(self, op, ops, x):
        """CfaOperators::apply_* on the device: op PD_APPLY_CROSS (x (B, n) ->
        (B, n, 5)), PD_APPLY_CROSS_TRANSPOSE ((B, n, 5) -> (B, n)),
        PD_APPLY_JOINT ((B, n) -> (B, n))."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        B, n = x.shape[:2]
        out = np.empty((B, n, 5) if op == _capi.PD_APPLY_CROSS else (B, n))
        f = {k: np.ascontiguousarray(ops[k], dtype=np.float64)
             for k in ("cross_sub", "cross_diag", "cross_super", "joint_diag", "joint_off")}
        self._check(self._L.pd_cfa_apply(self._h, int(op), B, n, *(_capi.dptr(f[k]) for k in (
            "cross_sub", "cross_diag", "cross_super", "joint_diag", "joint_off")), _capi.dptr(x), _capi.dptr(out)))
        return out

    def block_bidiag_solve(self, coupling, rhs, upper=False):
        """Batched scan solve of BlockBiDiagSystem<D> (D = 1..6): coupling
        (B, n-1, D, D), rhs (B, n, D) -> x (B, n, D) (scan.hpp:100-168)."""
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        B, n, d = rhs.shape
        coupling = np.ascontiguousarray(coupling, dtype=np.float64) if n > 1 else np.zeros((B, 0, d, d))
        x = np.empty_like(rhs)
        self._check(self._L.pd_block_bidiag_solve(self._h, d, B, n, 1 if upper else 0, _capi.dptr(coupling),
                                                  _capi.dptr(rhs), _capi.dptr(x)))
        return x

    def block_bidiag_solve6(self, coupling, rhs, upper=False):
        """block_bidiag_solve for the dynamics' 6x6 blocks."""
        return self.block_bidiag_solve(coupling, rhs, upper)

    def block_tridiag_solve(self, diag, upper, rhs):
        """Batched OEE (oee_solve<B, M>, B = 1..6, M = 1..4): diag (S, n, B, B),
        upper (S, n-1, B, B), rhs (S, n, B) or (S, n, B, M) -> (x shaped like
        rhs, status, round, index) per system."""
        diag = np.ascontiguousarray(diag, dtype=np.float64)
        S, n, b = diag.shape[0], diag.shape[1], diag.shape[2]
        upper = np.ascontiguousarray(upper, dtype=np.float64) if n > 1 else np.zeros((S, 0, b, b))
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        m = 1 if rhs.ndim == 3 else rhs.shape[3]
        x = np.empty_like(rhs)
        st, rd, ix = (np.zeros(S, np.int32) for _ in range(3))
        self._check(self._L.pd_block_tridiag_solve(self._h, b, m, S, n, _capi.dptr(diag), _capi.dptr(upper),
                                                   _capi.dptr(rhs), _capi.dptr(x), _capi.iptr(st), _capi.iptr(rd),
                                                   _capi.iptr(ix)))
        return x, st, rd, ix

    def block_tridiag_solve5(self, diag, upper, rhs):
        """block_tridiag_solve for the constraint operator's 5x5 blocks."""
        return self.block_tridiag_solve(diag, upper, rhs)

    def set_stream(self, stream_ptr):
        """Run on a CUDA stream (cudaStream_t as int). 0 = the legacy default
        stream (what torch.cuda.current_stream() is unless a stream is set);
        None restores the context's own stream."""
        if stream_ptr is None:
            self._check(self._L.pd_set_stream(self._h, None))
        else:
            self._check(self._L.pd_set_stream(self._h, C.c_void_p(stream_ptr if stream_ptr else 1)))

    def synchronize(self):
        self._check(self._L.pd_synchronize(self._h))

    def probe_fp64_peak(self):
        """Measured dense FP64 FMA throughput (TFLOP/s) of this device."""
        tf, ms = C.c_double(0), C.c_double(0)
        self._check(self._L.pd_probe_fp64_peak(self._h, C.byref(tf), C.byref(ms)))
        return tf.value

    def kernel_launches(self) -> int:
        return int(self._L.pd_kernel_launches(self._h))

    def kernel_variant(self, algo, n) -> str:
        return self._L.pd_kernel_variant(self._h, int(algo), int(n)).decode()


_tls = threading.local()
_default_device = 0


def set_device(device: int) -> None:
    """CUDA device the calling thread's free-function solves run on
    (pardyn::gpu::set_device in the C++ drop-in)."""
    global _default_device
    _default_device = int(device)
    ctx = getattr(_tls, "ctx", None)
    if ctx is not None and ctx.device != _default_device:
        _tls.ctx = None


def default_context() -> Context:
    """The calling thread's context. A pd_ctx is used from one host thread at
    a time and the free functions are set_models + solve pairs, so every
    thread gets its own (the reference's free functions are reentrant,
    SPEC.md:97-98)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context(_default_device)
    return ctx


# --------------------------------------------------------------------------- errors
def _raise_slot(code, round_, index, n):
    msg = _capi.slot_message(code, round_, index, n)
    if code in (_capi.SLOT_BAD_MODEL, _capi.SLOT_BAD_SIZE):
        raise InvalidArgument(msg)
    if code in (_capi.SLOT_OEE_SINGULAR_PIVOT, _capi.SLOT_OEE_SINGULAR_FINAL):
        raise SingularBlockError(int(round_), int(index), msg)
    raise DynamicsError(msg)


def _check_sizes(chain: RobotChain, q, qdot, tau):
    """forward_dynamics.cpp:19-31."""
    n = chain.size()
    if n == 0:
        raise InvalidArgument("forward dynamics: chain has no links")
    if len(q) != n or len(qdot) != n or len(tau) != n:
        raise InvalidArgument("forward dynamics: q, qdot and tau must each have one entry per joint "
                              f"(chain has {n})")


# --------------------------------------------------------------------------- API
def forward_dynamics(chain: RobotChain, q, qdot, tau, algo: FdAlgo, trace: Optional[ExecTrace] = None,
                     ctx: Optional[Context] = None) -> np.ndarray:
    try:
        algo = FdAlgo(int(algo))
    except ValueError:
        raise InvalidArgument("forward_dynamics: unknown algorithm") from None
    _check_sizes(chain, q, qdot, tau)
    ctx = ctx or default_context()
    ctx.set_models(chain.to_records()[None], np.asarray(chain.gravity, np.float64)[None])
    args = (np.asarray(q, np.float64)[None], np.asarray(qdot, np.float64)[None], np.asarray(tau, np.float64)[None])
    if trace is None:
        qdd, st, rd, ix = ctx.solve(algo, *args)
    else:  # the log-depth variants, counters from the variant that ran
        qdd, st, rd, ix, tr = ctx.solve_traced(algo, *args)
    if st[0] != _capi.SLOT_OK:
        _raise_slot(st[0], rd[0], ix[0], chain.size())
    if trace is not None:
        trace.parallel_link_stages += tr.parallel_link_stages
        trace.longest_sequential_link_chain = max(trace.longest_sequential_link_chain,
                                                  tr.longest_sequential_link_chain)
        trace.scan_rounds_max = max(trace.scan_rounds_max, tr.scan_rounds_max)
        trace.oee_rounds = tr.oee_rounds if algo == FdAlgo.cfa else trace.oee_rounds
    return qdd[0]


def jsiia_forward_dynamics(chain, q, qdot, tau, trace=None, ctx=None):
    return forward_dynamics(chain, q, qdot, tau, FdAlgo.jsiia, trace, ctx)


def abia_forward_dynamics(chain, q, qdot, tau, trace=None, ctx=None):
    return forward_dynamics(chain, q, qdot, tau, FdAlgo.abia, trace, ctx)


def cfa_forward_dynamics(chain, q, qdot, tau, trace=None, ctx=None):
    return forward_dynamics(chain, q, qdot, tau, FdAlgo.cfa, trace, ctx)


def batch_forward_dynamics(problems: Sequence[FdProblem], algo: FdAlgo, ctx: Optional[Context] = None,
                           devices: Optional[Sequence[int]] = None) -> List[FdResult]:
    """forward_dynamics.cpp:466-481: independent problems, per-slot errors,
    never raises per problem. Problems are bucketed by link count; with a
    device list each bucket is split into contiguous slices, one thread and
    one context per device, every slice selecting kernels for the whole
    bucket -- the result is bit-identical to the one-device call."""
    algo = FdAlgo(int(algo))
    out = [FdResult() for _ in problems]
    buckets = {}
    for k, p in enumerate(problems):
        try:
            _check_sizes(p.chain, p.q, p.qdot, p.tau)
        except InvalidArgument as e:
            out[k].error = str(e)
            continue
        buckets.setdefault(p.chain.size(), []).append(k)
    if not buckets:
        return out
    devices = list(devices) if devices else None
    for n, idx in buckets.items():
        links = np.stack([problems[k].chain.to_records() for k in idx])
        grav = np.stack([np.asarray(problems[k].chain.gravity, np.float64) for k in idx])
        q = np.stack([np.asarray(problems[k].q, np.float64) for k in idx])
        qd = np.stack([np.asarray(problems[k].qdot, np.float64) for k in idx])
        tau = np.stack([np.asarray(problems[k].tau, np.float64) for k in idx])
        B = len(idx)
        qdd, st = np.empty((B, n)), np.empty(B, np.int32)
        rd, ix = np.empty(B, np.int32), np.empty(B, np.int32)

        def run(c, lo, hi):
            c.set_selection_batch(B)
            try:
                c.set_models(links[lo:hi], grav[lo:hi])
                qdd[lo:hi], st[lo:hi], rd[lo:hi], ix[lo:hi] = c.solve(algo, q[lo:hi], qd[lo:hi], tau[lo:hi])
            finally:
                c.set_selection_batch(0)

        G = min(len(devices), B) if devices else 1
        if G <= 1:
            run(ctx or (default_context() if not devices else _device_context(devices[0])), 0, B)
        else:
            errors = []

            def worker(g):
                try:
                    run(_device_context(devices[g]), B * g // G, B * (g + 1) // G)
                except Exception as e:  # re-raised on the calling thread
                    errors.append(e)
            threads = [threading.Thread(target=worker, args=(g,)) for g in range(G)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            if errors:
                raise errors[0]
        for j, k in enumerate(idx):
            if st[j] == _capi.SLOT_OK:
                out[k].qddot = qdd[j].copy()
            else:
                out[k].error = _capi.slot_message(st[j], rd[j], ix[j], n)
    return out


def _device_context(device: int) -> Context:
    """The calling thread's context on `device` (sharded batch calls)."""
    ctxs = getattr(_tls, "by_device", None)
    if ctxs is None:
        ctxs = _tls.by_device = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _id_sizes(chain: RobotChain, **vecs):
    """inverse_dynamics.cpp:10-17 (check_joint_size)."""
    n = chain.size()
    for name, v in vecs.items():
        if len(v) != n:
            raise InvalidArgument(f"{name} has length {len(v)} but the chain has {n} joints")


def _one_model(chain: RobotChain, q, ctx: Optional[Context]) -> Context:
    """The reference's order: assemble_kinematics checks q (model.cpp:117-124),
    then link_inertias validates every link (model.cpp:148-155,
    spatial.cpp:72-87); the rate checks come after (inverse_dynamics.cpp:10-17)."""
    n = chain.size()
    if len(q) != n:
        raise InvalidArgument(f"assemble_kinematics: q has length {len(q)} but the chain has {n} joints")
    ctx = ctx or default_context()
    ms, mr = ctx.set_models(chain.to_records()[None], np.asarray(chain.gravity, np.float64)[None])
    if ms[0] != _capi.SLOT_OK:
        raise InvalidArgument(_capi.slot_message(ms[0], 0, mr[0], chain.size()))
    return ctx


def inverse_dynamics(chain: RobotChain, q, qdot, qddot, opts: Optional[IdOptions] = None,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:166-173 (IdOptions defaults when opts is None)."""
    if chain.size() == 0:
        _id_sizes(chain, q=q, qdot=qdot, qddot=qddot)
        return np.zeros(0)
    ctx = _one_model(chain, q, ctx)
    _id_sizes(chain, qdot=qdot, qddot=qddot)
    return ctx.inverse_dynamics_opts(np.asarray(q, np.float64)[None], np.asarray(qdot, np.float64)[None],
                                     np.asarray(qddot, np.float64)[None], opts)[0]


def bias_torque(chain: RobotChain, q, qdot, ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:175-179."""
    if chain.size() == 0:
        _id_sizes(chain, q=q, qdot=qdot)
        return np.zeros(0)
    ctx = _one_model(chain, q, ctx)
    _id_sizes(chain, qdot=qdot)
    return ctx.bias_torque(np.asarray(q, np.float64)[None], np.asarray(qdot, np.float64)[None])[0]


def link_states(chain: RobotChain, q, qdot, qddot, opts: Optional[IdOptions] = None,
                ctx: Optional[Context] = None) -> LinkStates:
    """inverse_dynamics.cpp:181-196."""
    if chain.size() == 0:
        _id_sizes(chain, q=q, qdot=qdot, qddot=qddot)
        z = np.zeros((0, 6))
        return LinkStates(z, z.copy(), z.copy())
    ctx = _one_model(chain, q, ctx)
    _id_sizes(chain, qdot=qdot, qddot=qddot)
    v, a, f = ctx.link_states(np.asarray(q, np.float64)[None], np.asarray(qdot, np.float64)[None],
                              np.asarray(qddot, np.float64)[None], opts)
    return LinkStates(v[0], a[0], f[0])


def joint_space_inertia(chain: RobotChain, q, ctx: Optional[Context] = None) -> np.ndarray:
    """forward_dynamics.cpp:70-80: M(q), symmetric."""
    if chain.size() == 0 and len(q) == 0:
        return np.zeros((0, 0))
    ctx = _one_model(chain, q, ctx)
    return ctx.joint_space_inertia(np.asarray(q, np.float64)[None])[0]


# --------------------------------------------------------------------------- chain operators
@dataclass
class ChainKinematics:
    """model.hpp:37-49: rel[i] maps link-(i-1) into link-i coordinates
    (rotation (n, 3, 3), translation (n, 3)); transport[i] = Ad(rel[i+1])."""
    rotation: np.ndarray
    translation: np.ndarray
    base_transport: np.ndarray
    transport: np.ndarray
    screw: np.ndarray

    def size(self) -> int:
        return self.screw.shape[0]


@dataclass
class ArticulatedBodyInertias:
    """forward_dynamics.hpp:44-52."""
    inertia: np.ndarray        # (n, 6, 6)
    joint_inertia: np.ndarray  # (n,)
    gain: np.ndarray           # (n, 6)


@dataclass
class ConstraintBasis:
    """forward_dynamics.hpp:64-69: basis (n, 6, 5)."""
    basis: np.ndarray


@dataclass
class CfaOperators:
    """forward_dynamics.hpp:73-91; apply_* run on the device."""
    diag: np.ndarray
    upper: np.ndarray
    cross_sub: np.ndarray
    cross_diag: np.ndarray
    cross_super: np.ndarray
    joint_diag: np.ndarray
    joint_off: np.ndarray

    def _blocks(self):
        return {k: getattr(self, k)[None] for k in ("cross_sub", "cross_diag", "cross_super", "joint_diag",
                                                    "joint_off")}

    def apply_cross(self, v, ctx: Optional[Context] = None):
        """forward_dynamics.cpp:359-376: v (n,) -> (n, 5)."""
        v = np.asarray(v, np.float64)
        if len(v) != len(self.cross_diag):
            raise InvalidArgument("apply_cross: one entry per link expected")
        return (ctx or default_context()).cfa_apply(_capi.PD_APPLY_CROSS, self._blocks(), v[None])[0]

    def apply_cross_transpose(self, f, ctx: Optional[Context] = None):
        """forward_dynamics.cpp:378-399: f (n, 5) -> (n,)."""
        f = np.asarray(f, np.float64).reshape(-1, 5)
        if f.shape[0] != len(self.cross_diag):
            raise InvalidArgument("apply_cross_transpose: one constraint block per link expected")
        return (ctx or default_context()).cfa_apply(_capi.PD_APPLY_CROSS_TRANSPOSE, self._blocks(), f[None])[0]

    def apply_joint(self, v, ctx: Optional[Context] = None):
        """forward_dynamics.cpp:401-416: v (n,) -> (n,)."""
        v = np.asarray(v, np.float64)
        if len(v) != len(self.joint_diag):
            raise InvalidArgument("apply_joint: one entry per link expected")
        return (ctx or default_context()).cfa_apply(_capi.PD_APPLY_JOINT, self._blocks(), v[None])[0]


def assemble_kinematics(chain: RobotChain, q, ctx: Optional[Context] = None) -> ChainKinematics:
    """model.cpp:117-146 on the device."""
    ctx = _one_model(chain, q, ctx)
    rel, base, tr, sc = ctx.assemble_kinematics(np.asarray(q, np.float64)[None])
    return ChainKinematics(rel[0, :, :9].reshape(-1, 3, 3), rel[0, :, 9:], base[0], tr[0], sc[0])


def link_inertias(chain: RobotChain, ctx: Optional[Context] = None) -> np.ndarray:
    """model.cpp:148-155 on the device: (n, 6, 6); a bad link raises the
    spatial_inertia_from message."""
    ctx = _one_model(chain, np.zeros(chain.size()), ctx)
    return ctx.link_inertias()[0]


def articulated_body_inertias(kin: ChainKinematics, inertia, trace: Optional[ExecTrace] = None,
                              ctx: Optional[Context] = None) -> ArticulatedBodyInertias:
    """forward_dynamics.cpp:120-163 on the device (the n-link tip-to-base walk)."""
    n = kin.size()
    inertia = np.asarray(inertia, np.float64).reshape(n, 6, 6)
    abi, lam, gain, st, ix = (ctx or default_context()).articulated_body_inertias(
        kin.transport[None], inertia[None], kin.screw[None])
    if st[0] != _capi.SLOT_OK:
        _raise_slot(st[0], 0, ix[0], n)
    if trace is not None:
        trace.longest_sequential_link_chain = max(trace.longest_sequential_link_chain, n)
    return ArticulatedBodyInertias(abi[0], lam[0], gain[0])


def build_constraint_basis(chain: RobotChain, ctx: Optional[Context] = None) -> ConstraintBasis:
    """forward_dynamics.cpp:245-259 on the device (Householder complement)."""
    screws = np.stack([np.asarray(l.joint_screw, np.float64) for l in chain.links]) if chain.links else \
        np.zeros((0, 6))
    if not chain.links:
        return ConstraintBasis(np.zeros((0, 6, 5)))
    return ConstraintBasis((ctx or default_context()).constraint_basis(screws))


def build_cfa_operators(chain: RobotChain, kin: ChainKinematics, basis: ConstraintBasis,
                        trace: Optional[ExecTrace] = None, ctx: Optional[Context] = None) -> CfaOperators:
    """forward_dynamics.cpp:261-357 on the device."""
    n = chain.size()
    if n == 0:
        raise InvalidArgument("build_cfa_operators: chain has no links")
    if basis.basis.shape[0] != n or kin.size() != n:
        raise InvalidArgument("build_cfa_operators: kinematics and basis must match the chain")
    ctx = ctx or default_context()
    J = link_inertias(chain, ctx)
    o = ctx.cfa_operators(J[None], kin.transport[None], kin.screw[None], basis.basis[None])
    if o["status"][0] != _capi.SLOT_OK:
        _raise_slot(o["status"][0], 0, o["index"][0], n)
    if trace is not None:
        trace.parallel_link_stages += 2
    return CfaOperators(*(o[k][0] for k in ("diag", "upper", "cross_sub", "cross_diag", "cross_super",
                                            "joint_diag", "joint_off")))


def _check_joint_size(kin: ChainKinematics, v, name):
    """inverse_dynamics.cpp:10-17."""
    if len(v) != kin.size():
        raise InvalidArgument(f"{name} has length {len(v)} but the chain has {kin.size()} joints")


def propagate_velocities(kin: ChainKinematics, qdot, base_velocity=None, trace: Optional[ScanTrace] = None,
                         ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:27-51 on the device (block bi-diagonal scan): (n, 6) twists."""
    _check_joint_size(kin, qdot, "qdot")
    n = kin.size()
    if trace is not None:
        trace.rounds = ceil_log2(n)
    if n == 0:
        return np.zeros((0, 6))
    bv = np.zeros(6) if base_velocity is None else np.asarray(base_velocity, np.float64)
    return (ctx or default_context()).propagate(_capi.PD_PROPAGATE_VELOCITIES, kin.base_transport[None],
                                                kin.transport[None], kin.screw[None], bv,
                                                qdot=np.asarray(qdot, np.float64)[None])[0]


def propagate_accelerations(kin: ChainKinematics, velocity, qdot, qddot, base_acceleration=None,
                            trace: Optional[ScanTrace] = None, ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:53-84 on the device: (n, 6) accelerations."""
    _check_joint_size(kin, qdot, "qdot")
    _check_joint_size(kin, qddot, "qddot")
    n = kin.size()
    if trace is not None:
        trace.rounds = ceil_log2(n)
    if n == 0:
        return np.zeros((0, 6))
    ba = np.zeros(6) if base_acceleration is None else np.asarray(base_acceleration, np.float64)
    return (ctx or default_context()).propagate(
        _capi.PD_PROPAGATE_ACCELERATIONS, kin.base_transport[None], kin.transport[None], kin.screw[None], ba,
        qdot=np.asarray(qdot, np.float64)[None], qddot=np.asarray(qddot, np.float64)[None],
        velocity=np.asarray(velocity, np.float64).reshape(1, n, 6))[0]


def propagate_forces(kin: ChainKinematics, velocity, acceleration, inertia, tip_wrench=None,
                     trace: Optional[ScanTrace] = None, ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:86-120 on the device: (n, 6) wrenches."""
    n = kin.size()
    if trace is not None:
        trace.rounds = ceil_log2(n)
    if n == 0:
        return np.zeros((0, 6))
    tw = np.zeros(6) if tip_wrench is None else np.asarray(tip_wrench, np.float64)
    return (ctx or default_context()).propagate(
        _capi.PD_PROPAGATE_FORCES, None, kin.transport[None], kin.screw[None], tw,
        velocity=np.asarray(velocity, np.float64).reshape(1, n, 6),
        acceleration=np.asarray(acceleration, np.float64).reshape(1, n, 6),
        inertia=np.asarray(inertia, np.float64).reshape(1, n, 6, 6))[0]


def inverse_dynamics_assembled(kin: ChainKinematics, inertia, gravity, qdot, qddot, opts: Optional[IdOptions] = None,
                               trace: Optional[ExecTrace] = None, ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_dynamics.cpp:122-164: the three propagations, tau_i = S_i . F_i."""
    opts = opts or IdOptions()
    sv, sa, sf = ScanTrace(), ScanTrace(), ScanTrace()
    vel = propagate_velocities(kin, qdot, opts.base_velocity, sv, ctx)
    ba = np.array(opts.base_acceleration, np.float64).copy()
    if opts.apply_gravity:
        ba[3:] -= np.asarray(gravity, np.float64)
    acc = propagate_accelerations(kin, vel, qdot, qddot, ba, sa, ctx)
    frc = propagate_forces(kin, vel, acc, inertia, opts.tip_wrench, sf, ctx)
    if trace is not None:
        trace.scan_rounds_max = max(trace.scan_rounds_max, sv.rounds, sa.rounds, sf.rounds)
        trace.parallel_link_stages += 5
    return np.einsum("ij,ij->i", kin.screw, frc)


# --------------------------------------------------------------------------- model files
# --------------------------------------------------------------------------- building blocks
@dataclass
class ScanTrace:
    """trace.hpp ScanTrace: rounds of the Hillis-Steele scan (ceil_log2(n))."""
    rounds: int = 0


@dataclass
class OeeTrace:
    """trace.hpp OeeTrace: odd-even elimination rounds (ceil_log2(n))."""
    rounds: int = 0


def _bidiag(coupling, rhs, upper, trace, ctx):
    rhs = np.asarray(rhs, dtype=np.float64)
    if rhs.ndim != 2 or not 1 <= rhs.shape[1] <= 6:
        raise InvalidArgument("block bi-diagonal solve: rhs must be (n, D) with 1 <= D <= 6")
    n, d = rhs.shape
    coupling = np.asarray(coupling, dtype=np.float64)
    if coupling.size and coupling.shape[-2:] != (d, d):
        raise InvalidArgument("block bi-diagonal solve: coupling blocks must be D x D")
    coupling = coupling.reshape(-1, d, d)
    if n > 0 and coupling.shape[0] != n - 1:
        raise InvalidArgument("block bi-diagonal solve: need n - 1 coupling blocks for n right-hand sides")
    if trace is not None:
        trace.rounds = ceil_log2(n)
    if n == 0:
        return np.zeros((0, d))
    return (ctx or default_context()).block_bidiag_solve(coupling[None], rhs[None], upper=upper)[0]


def solve_lower_bidiag(coupling, rhs, trace: Optional[ScanTrace] = None, ctx: Optional[Context] = None):
    """solve_lower_bidiag<D> (scan.hpp:115-140) of one BlockBiDiagSystem<D>:
    x_0 = r_0, x_i = C_i x_{i-1} + r_i; coupling (n-1, D, D), rhs (n, D)."""
    return _bidiag(coupling, rhs, False, trace, ctx)


def solve_upper_bidiag(coupling, rhs, trace: Optional[ScanTrace] = None, ctx: Optional[Context] = None):
    """solve_upper_bidiag<D> (scan.hpp:143-168): the reversed index order."""
    return _bidiag(coupling, rhs, True, trace, ctx)


def oee_solve(diag, upper, rhs, trace: Optional[OeeTrace] = None, ctx: Optional[Context] = None):
    """oee_solve<B, M> (oee.hpp:149-189) of one SymBlockTriDiagSystem<B>:
    diag (n, B, B), upper (n-1, B, B), rhs (n, B) or (n, B, M) -> x shaped
    like rhs (B <= 6, M <= 4). Raises SingularBlockError(round, index) with
    the reference's message."""
    diag = np.asarray(diag, dtype=np.float64)
    if diag.ndim != 3 or diag.shape[1] != diag.shape[2] or not 1 <= diag.shape[1] <= 6:
        raise InvalidArgument("odd-even elimination: diag must be (n, B, B) with 1 <= B <= 6")
    n, b = diag.shape[0], diag.shape[1]
    rhs = np.asarray(rhs, dtype=np.float64)
    upper = np.asarray(upper, dtype=np.float64).reshape(-1, b, b)
    if rhs.ndim not in (2, 3) or rhs.shape[0] != n or rhs.shape[1] != b or (n > 0 and upper.shape[0] != n - 1):
        raise InvalidArgument("odd-even elimination: inconsistent block counts")
    if rhs.ndim == 3 and not 1 <= rhs.shape[2] <= 4:
        raise InvalidArgument("odd-even elimination: 1 to 4 right-hand-side columns")
    if trace is not None:
        trace.rounds = ceil_log2(n)
    if n == 0:
        return np.zeros(rhs.shape)
    x, st, rd, ix = (ctx or default_context()).block_tridiag_solve(diag[None], upper[None], rhs[None])
    if st[0] != 0:
        _raise_slot(int(st[0]), int(rd[0]), int(ix[0]), n)
    return x[0]


@dataclass
class OeeState:
    """OeeState<B, M> (oee.hpp:57-67): diag (n, B, B), coupling (n - distance,
    B, B) linking row i to row i + distance, rhs (n, B) or (n, B, M)."""
    diag: np.ndarray
    coupling: np.ndarray
    rhs: np.ndarray
    distance: int = 1
    round: int = 0


def oee_eliminate_round(state: OeeState, ctx: Optional[Context] = None) -> None:
    """oee_eliminate_round (oee.hpp:69-145) on the GPU: advances `state` by
    one round in place (distance doubles, couplings shrink to n - 2h); a
    singular pivot raises SingularBlockError(round, block) and leaves the
    state as it was."""
    diag = np.ascontiguousarray(state.diag, dtype=np.float64)
    n, b = diag.shape[0], diag.shape[1]
    rhs = np.ascontiguousarray(state.rhs, dtype=np.float64)
    m = 1 if rhs.ndim == 2 else rhs.shape[2]
    h = int(state.distance)
    coupling = np.ascontiguousarray(np.asarray(state.coupling, dtype=np.float64).reshape(-1, b, b))
    if rhs.shape[0] != n or coupling.shape[0] != max(n - h, 0):
        raise InvalidArgument("odd-even elimination: inconsistent block counts")
    nu = max(n - 2 * h, 0)
    if n > 0:
        c = ctx or default_context()
        d1, c1, r1 = np.empty_like(diag), np.empty((nu, b, b)), np.empty_like(rhs)
        st, rd, ix = (np.zeros(1, np.int32) for _ in range(3))
        c._check(c._L.pd_oee_eliminate_rounds(c._h, b, m, 1, n, h, int(state.round), 1, _capi.dptr(diag),
                                              _capi.dptr(coupling), _capi.dptr(rhs), _capi.dptr(d1), _capi.dptr(c1),
                                              _capi.dptr(r1), _capi.iptr(st), _capi.iptr(rd), _capi.iptr(ix)))
        if st[0] != 0:
            _raise_slot(int(st[0]), int(rd[0]), int(ix[0]), n)
        state.diag, state.coupling, state.rhs = d1, c1, r1
    state.distance = 2 * h
    state.round = int(state.round) + 1


def coefficient_solve(pivot, rhs, round_: int, index: int, ctx: Optional[Context] = None):
    """coefficient_solve<B> (oee.hpp:34-51): pivot x = rhs by full-pivot LU on
    the GPU (a one-row elimination); SingularBlockError(round_, index) when
    the pivot is rank deficient."""
    pivot = np.asarray(pivot, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    b = pivot.shape[0]
    cols = rhs.reshape(b, -1)
    out = np.empty_like(cols)
    c = ctx or default_context()
    for c0 in range(0, cols.shape[1], 4):
        part = np.ascontiguousarray(cols[:, c0:c0 + 4])
        x, st, _, _ = c.block_tridiag_solve(pivot[None, None], np.zeros((1, 0, b, b)), part[None, None])
        if st[0] != 0:
            raise SingularBlockError(round_, index, f"odd-even elimination: singular pivot block (round {round_}, "
                                                    f"block {index})")
        out[:, c0:c0 + 4] = x[0, 0]
    return out.reshape(rhs.shape)


def _link_prefix(k: int) -> str:
    return f"link {k}"


def validate_chain(chain: RobotChain) -> None:
    """model.cpp:75-115 (ModelError with the reference's messages)."""
    if not chain.links:
        raise ModelError("chain must have at least one link")
    if not np.all(np.isfinite(chain.gravity)):
        raise ModelError("gravity must be finite")
    for k, l in enumerate(chain.links):
        if not (l.mass > 0.0) or not np.isfinite(l.mass):
            raise ModelError(f"{_link_prefix(k)}: mass must be positive")
        if not np.all(np.isfinite(l.com)):
            raise ModelError(f"{_link_prefix(k)}: com must be finite")
        I = np.asarray(l.inertia_rot, np.float64).reshape(3, 3)
        if not np.all(np.isfinite(I)) or np.abs(I - I.T).max() > 1e-9 * max(1.0, np.abs(I).max()):
            raise ModelError(f"{_link_prefix(k)}: rotational inertia must be symmetric")
        if not (np.linalg.eigvalsh(0.5 * (I + I.T)).min() > 0.0):
            raise ModelError(f"{_link_prefix(k)}: rotational inertia must be positive definite")
        s = np.asarray(l.joint_screw, np.float64)
        if not np.all(np.isfinite(s)):
            raise ModelError(f"{_link_prefix(k)}: joint_screw must be finite")
        nrm = float(np.linalg.norm(s))
        if abs(nrm - 1.0) > 1e-9:
            raise ModelError(f"{_link_prefix(k)}: joint_screw must have unit norm (got {nrm:.6f})")
        R = np.asarray(l.home_transform.rotation, np.float64).reshape(3, 3)
        ok = np.all(np.isfinite(R)) and np.all(np.isfinite(l.home_transform.translation))
        ok = ok and np.abs(R.T @ R - np.eye(3)).max() <= 1e-9 and np.linalg.det(R) > 0.0
        if not ok:
            raise ModelError(f"{_link_prefix(k)}: home_transform rotation must be orthonormal with determinant +1")


def load_chain(path: str) -> RobotChain:
    """model.cpp:254-310: the reference's JSON layout, validated."""
    import json
    import numbers
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ModelError(f"cannot open model file '{path}'") from None
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ModelError(f"model file '{path}': {e}") from None
    where = f"model file '{path}'"

    def need(j, field, w):
        if not isinstance(j, dict) or field not in j:
            raise ModelError(f"{w}: missing field '{field}'")
        return j[field]

    def number(j, field, w):
        v = need(j, field, w)
        if isinstance(v, bool) or not isinstance(v, numbers.Real):
            raise ModelError(f"{w}: field '{field}' must be a number")
        return float(v)

    def array(j, field, n, w):
        v = need(j, field, w)
        if not isinstance(v, list) or len(v) != n:
            raise ModelError(f"{w}: field '{field}' must be an array of {n} numbers")
        if any(isinstance(e, bool) or not isinstance(e, numbers.Real) for e in v):
            raise ModelError(f"{w}: field '{field}' must contain only numbers")
        return np.asarray(v, np.float64)

    n = need(doc, "n", where)
    if isinstance(n, bool) or not isinstance(n, int):
        raise ModelError(f"{where}: field 'n' must be an integer")
    gravity = array(doc, "gravity", 3, where)
    links = need(doc, "links", where)
    if not isinstance(links, list):
        raise ModelError(f"{where}: field 'links' must be an array")
    if len(links) != n:
        raise ModelError(f"{where}: field 'n' (= {n}) does not match the length of 'links' (= {len(links)})")
    out = []
    for k, j in enumerate(links):
        w = _link_prefix(k)
        if not isinstance(j, dict):
            raise ModelError(f"{w}: must be an object")
        home = need(j, "home_transform", w)
        mass = number(j, "mass", w)
        com = array(j, "com", 3, w)
        Ir = array(j, "inertia_rot", 9, w)
        screw = array(j, "joint_screw", 6, w)
        if not isinstance(home, dict):
            raise ModelError(f"{w}: field 'home_transform' must be an object")
        out.append(LinkSpec(mass, com, Ir.reshape(3, 3), screw,
                            SE3Transform(array(home, "rotation", 9, w).reshape(3, 3), array(home, "translation", 3, w))))
    chain = RobotChain(out, gravity)
    validate_chain(chain)
    return chain


def save_chain(chain: RobotChain, path: str) -> None:
    """model.cpp:312-337: indented JSON in the reference's field order; repr
    floats so that loading back reproduces the chain exactly."""
    import json
    doc = {"n": chain.size(), "gravity": [float(x) for x in chain.gravity], "links": [
        {"mass": float(l.mass), "com": [float(x) for x in np.ravel(l.com)],
         "inertia_rot": [float(x) for x in np.ravel(l.inertia_rot)],
         "joint_screw": [float(x) for x in np.ravel(l.joint_screw)],
         "home_transform": {"rotation": [float(x) for x in np.ravel(l.home_transform.rotation)],
                            "translation": [float(x) for x in np.ravel(l.home_transform.translation)]}}
        for l in chain.links]}
    try:
        with open(path, "w") as f:
            f.write(json.dumps(doc, indent=2) + "\n")
    except OSError:
        raise ModelError(f"cannot open model file '{path}' for writing") from None
