"""ctypes binding of the C-ABI (include/pardyn_c.h) of libpardyn_b200.so.

The shared library is built in-tree (paper_1609_06779_b200/lib/) by
``make -C paper_1609_06779_b200/csrc`` (or ``__graft_entry__.build()``).
There is no CPU fallback: if the library or a CUDA device is missing, calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libpardyn_b200.so")

PD_JSIIA, PD_ABIA, PD_CFA = 0, 1, 2
PD_OK, PD_INVALID_ARGUMENT, PD_MODEL_ERROR, PD_DYNAMICS_ERROR, PD_SINGULAR_BLOCK, PD_CUDA_ERROR, PD_NO_DEVICE, \
    PD_INTERNAL = range(8)
SLOT_OK, SLOT_DEGENERATE_ARTICULATION, SLOT_JSI_NOT_SPD, SLOT_JSI_REFINE_FAILED, SLOT_LINK_INERTIA_NOT_PD, \
    SLOT_OEE_SINGULAR_PIVOT, SLOT_OEE_SINGULAR_FINAL, SLOT_BAD_MODEL, SLOT_BAD_SIZE = range(9)
LINK_FIELDS = 31

# every symbol include/pardyn_c.h declares
EXPORTS = (
    "pd_create", "pd_destroy", "pd_abi_version", "pd_status_string", "pd_last_error", "pd_set_stream",
    "pd_synchronize", "pd_set_models", "pd_forward_dynamics", "pd_forward_dynamics_device", "pd_inverse_dynamics",
    "pd_slot_message", "pd_kernel_launches", "pd_kernel_variant", "pd_mix", "pd_workload_seed", "pd_random_chain",
    "pd_workload_chains", "pd_workload_inputs", "pd_probe_fp64_peak", "pd_inverse_dynamics_opts",
    "pd_inverse_dynamics_device", "pd_bias_torque", "pd_link_states", "pd_joint_space_inertia",
    "pd_workload_chains_device", "pd_set_models_workload", "pd_block_tridiag_solve5", "pd_block_bidiag_solve6", "pd_block_tridiag_solve", "pd_block_bidiag_solve", "pd_oee_eliminate_rounds",
    "pd_forward_dynamics_traced", "pd_last_variant", "pd_last_trace", "pd_set_selection_batch",
    "pd_assemble_kinematics", "pd_link_inertias", "pd_articulated_body_inertias", "pd_constraint_basis",
    "pd_cfa_operators", "pd_cfa_apply", "pd_host_alloc", "pd_host_free",
    "pd_propagate",
)
PD_PROPAGATE_VELOCITIES, PD_PROPAGATE_ACCELERATIONS, PD_PROPAGATE_FORCES = range(3)
PD_APPLY_CROSS, PD_APPLY_CROSS_TRANSPOSE, PD_APPLY_JOINT = range(3)


class IdOptions(C.Structure):
    """pd_id_options (include/pardyn_c.h) <- IdOptions (inverse_dynamics.hpp:23-28)."""
    _fields_ = [("base_velocity", C.c_double * 6), ("base_acceleration", C.c_double * 6),
                ("tip_wrench", C.c_double * 6), ("apply_gravity", C.c_int32)]

class ExecTraceC(C.Structure):
    """pd_exec_trace (include/pardyn_c.h) <- ExecTrace (trace.hpp:24-39)."""
    _fields_ = [("parallel_link_stages", C.c_int32), ("longest_sequential_link_chain", C.c_int32),
                ("scan_rounds_max", C.c_int32), ("oee_rounds", C.c_int32)]


_lib = None
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load libpardyn_b200.so (raises LibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(f"{LIB_PATH} not built; run `make -C paper_1609_06779_b200/csrc` "
                             "(or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    L.pd_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.pd_create.restype = C.c_int
    L.pd_destroy.argtypes = [C.c_void_p]
    L.pd_destroy.restype = None
    L.pd_abi_version.restype = C.c_int
    L.pd_status_string.argtypes = [C.c_int]
    L.pd_status_string.restype = C.c_char_p
    L.pd_last_error.argtypes = [C.c_void_p]
    L.pd_last_error.restype = C.c_char_p
    L.pd_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.pd_set_stream.restype = C.c_int
    L.pd_synchronize.argtypes = [C.c_void_p]
    L.pd_synchronize.restype = C.c_int
    L.pd_set_models.argtypes = [C.c_void_p, C.c_int64, C.c_int32, _D, _D, _I32, _I32]
    L.pd_set_models.restype = C.c_int
    L.pd_forward_dynamics.argtypes = [C.c_void_p, C.c_int, C.c_int64, _D, _D, _D, _D, _I32, _I32, _I32]
    L.pd_forward_dynamics.restype = C.c_int
    L.pd_forward_dynamics_device.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.pd_forward_dynamics_device.restype = C.c_int
    L.pd_inverse_dynamics.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D, _D]
    L.pd_inverse_dynamics.restype = C.c_int
    _OPT = C.POINTER(IdOptions)
    L.pd_inverse_dynamics_opts.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D, _OPT, _D]
    L.pd_inverse_dynamics_opts.restype = C.c_int
    L.pd_inverse_dynamics_device.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, _OPT,
                                             C.c_void_p]
    L.pd_inverse_dynamics_device.restype = C.c_int
    L.pd_bias_torque.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D]
    L.pd_bias_torque.restype = C.c_int
    L.pd_link_states.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D, _OPT, _D, _D, _D]
    L.pd_link_states.restype = C.c_int
    L.pd_joint_space_inertia.argtypes = [C.c_void_p, C.c_int64, _D, _D]
    L.pd_joint_space_inertia.restype = C.c_int
    L.pd_workload_chains_device.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
    L.pd_workload_chains_device.restype = C.c_int
    L.pd_set_models_workload.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int64, C.c_int64, _D, _I32, _I32]
    L.pd_set_models_workload.restype = C.c_int
    L.pd_block_bidiag_solve6.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, _D, _D, _D]
    L.pd_block_bidiag_solve6.restype = C.c_int
    L.pd_block_tridiag_solve5.argtypes = [C.c_void_p, C.c_int64, C.c_int32, _D, _D, _D, _D, _I32, _I32, _I32]
    L.pd_block_tridiag_solve5.restype = C.c_int
    L.pd_block_bidiag_solve.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32, _D, _D, _D]
    L.pd_block_bidiag_solve.restype = C.c_int
    L.pd_block_tridiag_solve.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _D, _D, _D, _D,
                                         _I32, _I32, _I32]
    L.pd_block_tridiag_solve.restype = C.c_int
    L.pd_oee_eliminate_rounds.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_int32, _D, _D, _D, _D, _D, _D, _I32, _I32, _I32]
    L.pd_oee_eliminate_rounds.restype = C.c_int
    L.pd_slot_message.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_int32]
    L.pd_slot_message.restype = None
    L.pd_kernel_launches.argtypes = [C.c_void_p]
    L.pd_kernel_launches.restype = C.c_int64
    L.pd_kernel_variant.argtypes = [C.c_void_p, C.c_int, C.c_int32]
    L.pd_kernel_variant.restype = C.c_char_p
    L.pd_mix.argtypes = [C.c_uint64]
    L.pd_mix.restype = C.c_uint64
    L.pd_workload_seed.argtypes = [C.c_uint64, C.c_int32, C.c_int64]
    L.pd_workload_seed.restype = C.c_uint64
    L.pd_random_chain.argtypes = [C.c_int32, C.c_uint64, _D]
    L.pd_random_chain.restype = None
    L.pd_workload_chains.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_int64, _D]
    L.pd_workload_chains.restype = None
    L.pd_workload_inputs.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_int64, _D, _D, _D]
    L.pd_workload_inputs.restype = None
    L.pd_probe_fp64_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.pd_probe_fp64_peak.restype = C.c_int
    _TR = C.POINTER(ExecTraceC)
    L.pd_forward_dynamics_traced.argtypes = [C.c_void_p, C.c_int, C.c_int64, _D, _D, _D, _D, _I32, _I32, _I32, _TR]
    L.pd_forward_dynamics_traced.restype = C.c_int
    L.pd_last_variant.argtypes = [C.c_void_p]
    L.pd_last_variant.restype = C.c_char_p
    L.pd_last_trace.argtypes = [C.c_void_p, _TR]
    L.pd_last_trace.restype = C.c_int
    L.pd_set_selection_batch.argtypes = [C.c_void_p, C.c_int64]
    L.pd_set_selection_batch.restype = C.c_int
    L.pd_assemble_kinematics.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D, _D, _D]
    L.pd_assemble_kinematics.restype = C.c_int
    L.pd_link_inertias.argtypes = [C.c_void_p, _D]
    L.pd_link_inertias.restype = C.c_int
    L.pd_articulated_body_inertias.argtypes = [C.c_void_p, C.c_int64, C.c_int32, _D, _D, C.c_int32, _D, _D, _D, _D,
                                               _I32, _I32]
    L.pd_articulated_body_inertias.restype = C.c_int
    L.pd_constraint_basis.argtypes = [C.c_void_p, C.c_int64, _D, _D]
    L.pd_constraint_basis.restype = C.c_int
    L.pd_cfa_operators.argtypes = [C.c_void_p, C.c_int64, C.c_int32, _D, C.c_int32, _D, _D, _D, _D, _D, _D, _D, _D,
                                   _D, _D, _I32, _I32]
    L.pd_cfa_operators.restype = C.c_int
    L.pd_cfa_apply.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, _D, _D, _D, _D, _D, _D, _D]
    L.pd_cfa_apply.restype = C.c_int
    L.pd_host_alloc.argtypes = [C.c_uint64, C.POINTER(C.c_void_p)]
    L.pd_host_alloc.restype = C.c_int
    L.pd_host_free.argtypes = [C.c_void_p]
    L.pd_host_free.restype = None
    L.pd_propagate.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, _D, _D, _D, _D, C.c_int32, _D, _D, _D, _D,
                               _D, _D]
    L.pd_propagate.restype = C.c_int
    _lib = L
    return L


def slot_message(code, round_, index, n_links):
    buf = C.create_string_buffer(512)
    load().pd_slot_message(int(code), int(round_), int(index), int(n_links), buf, 512)
    return buf.value.decode()


def dptr(a):
    return None if a is None else a.ctypes.data_as(_D)


def iptr(a):
    return None if a is None else a.ctypes.data_as(_I32)
