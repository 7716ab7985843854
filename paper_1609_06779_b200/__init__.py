"""B200-native batched forward dynamics of serial chains (arxiv 1609.06779).

Hot path: FP64 ABIA / JSIIA / CFA forward dynamics on sm_100a, behind the
C-ABI of libpardyn_b200.so (include/pardyn_c.h). This package is the Python
mirror of the reference's C++ API (proj/core/include/pardyn/*.hpp); the C++
drop-in lives in include/pardyn/ + paper_1609_06779_b200/cpp/.
"""
from .api import (  # noqa: F401
    ArticulatedBodyInertias,
    CfaOperators,
    ChainKinematics,
    ConstraintBasis,
    Context,
    SE3Transform,
    articulated_body_inertias,
    assemble_kinematics,
    build_cfa_operators,
    build_constraint_basis,
    link_inertias,
    CudaError,
    DynamicsError,
    ExecTrace,
    FdAlgo,
    FdProblem,
    FdResult,
    IdOptions,
    InvalidArgument,
    LinkSpec,
    LinkStates,
    ModelError,
    OeeTrace,
    RobotChain,
    ScanTrace,
    SingularBlockError,
    abia_forward_dynamics,
    batch_forward_dynamics,
    bias_torque,
    cfa_forward_dynamics,
    ceil_log2,
    default_context,
    set_device,
    forward_dynamics,
    inverse_dynamics,
    joint_space_inertia,
    jsiia_forward_dynamics,
    link_states,
    oee_solve,
    load_chain,
    save_chain,
    solve_lower_bidiag,
    solve_upper_bidiag,
    validate_chain,
)
from ._capi import LIB_PATH, LibraryMissing  # noqa: F401
