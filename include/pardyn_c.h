/*
 * pardyn_c.h — C-ABI of the B200-native batched forward-dynamics library
 * (libpardyn_b200.so). Plain pointers and sizes only; no C++ or torch types.
 *
 * This is the drop-in boundary for the reference library "pardyn"
 * (arxiv 1609.06779, /root/reference/proj/core). Each entry point names the
 * reference interface it replaces:
 *
 *   pd_algo                  <- enum class FdAlgo { jsiia, abia, cfa }
 *                               (include/pardyn/forward_dynamics.hpp:29)
 *   pd_set_models            <- the RobotChain / LinkSpec values carried by
 *                               FdProblem (model.hpp:17-30,
 *                               forward_dynamics.hpp:111-116) plus the
 *                               per-call spatial_inertia_from validation
 *                               (src/spatial.cpp:70-100)
 *   pd_forward_dynamics      <- batch_forward_dynamics(span<const FdProblem>,
 *                               FdAlgo) (forward_dynamics.hpp:125-126,
 *                               src/forward_dynamics.cpp:466-481) and, at
 *                               batch 1, forward_dynamics(...)
 *                               (forward_dynamics.hpp:103-105)
 *   pd_forward_dynamics_device  same, on device-resident buffers
 *   pd_slot_message          <- FdResult::error strings (e.what() of the
 *                               reference exceptions, types.hpp:21-46)
 *   pd_inverse_dynamics      <- inverse_dynamics(chain, q, qdot, qddot)
 *                               (inverse_dynamics.hpp:71-74), default
 *                               IdOptions
 *   pd_inverse_dynamics_opts <- inverse_dynamics(..., const IdOptions&)
 *                               (inverse_dynamics.hpp:23-28,71-74;
 *                               src/inverse_dynamics.cpp:122-173)
 *   pd_inverse_dynamics_device  same, device buffers [link][problem]
 *   pd_bias_torque           <- bias_torque (inverse_dynamics.hpp:77-78,
 *                               src/inverse_dynamics.cpp:175-179)
 *   pd_link_states           <- link_states (inverse_dynamics.hpp:81-83,
 *                               src/inverse_dynamics.cpp:181-196)
 *   pd_block_bidiag_solve    <- solve_lower_bidiag<D> / solve_upper_bidiag<D> (D <= 6)
 *   pd_block_bidiag_solve6   <- the D = 6 case
 *                               (include/pardyn/scan.hpp:100-168)
 *   pd_block_tridiag_solve   <- oee_solve<B,M> / SymBlockTriDiagSystem<B> (B <= 6, M <= 4)
 *   pd_block_tridiag_solve5  <- the oee_solve<5,1> case
 *   pd_oee_eliminate_rounds  <- oee_eliminate_round / OeeState<B,M> (oee.hpp:57-145)
 *                               (include/pardyn/oee.hpp:28-32,149-189)
 *   pd_workload_chains_device, pd_set_models_workload
 *                            <- workload_chains / random_chain on the device
 *                               (bench.cpp:357-366, model.cpp:157-185)
 *   pd_joint_space_inertia   <- joint_space_inertia(chain, q)
 *                               (forward_dynamics.hpp:34-35,
 *                               src/forward_dynamics.cpp:70-80)
 *   pd_forward_dynamics_traced, pd_exec_trace
 *                            <- forward_dynamics(..., ExecTrace* trace) and
 *                               the per-algorithm entry points with a trace
 *                               (forward_dynamics.hpp:38-42,58-62,98-105;
 *                               trace.hpp:24-39)
 *
 * Layouts
 *   LinkSpec record: 31 doubles, the field order of LinkSpec (model.hpp:17-23)
 *     [0] mass, [1..3] com, [4..12] inertia_rot row-major,
 *     [13..18] joint_screw (angular, linear), [19..27] home rotation
 *     row-major, [28..30] home translation.
 *   Host models:  links[model][link][31], gravity[model][3].
 *   Host states:  q/qdot/tau/qddot[problem][link] (one JointVector per row).
 *   Device states (pd_*_device): [link][problem] (problem fastest).
 *   Problem p uses model (n_models == 1 ? 0 : p).
 *
 * Errors never abort a batch: each slot gets a pd_slot_code plus
 * (round, index); pd_slot_message() rebuilds the reference's message.
 * A pd_ctx is used from one host thread at a time; contexts are independent.
 */
#ifndef PARDYN_C_H_
#define PARDYN_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_LINK_FIELDS 31
#define PD_ABI_VERSION 1

typedef enum pd_algo { PD_JSIIA = 0, PD_ABIA = 1, PD_CFA = 2 } pd_algo;

/* Call-level status. Classes mirror the reference's exceptions. */
typedef enum pd_status {
  PD_OK = 0,
  PD_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  PD_MODEL_ERROR = 2,      /* pardyn::ModelError */
  PD_DYNAMICS_ERROR = 3,   /* pardyn::DynamicsError */
  PD_SINGULAR_BLOCK = 4,   /* pardyn::SingularBlockError */
  PD_CUDA_ERROR = 5,
  PD_NO_DEVICE = 6,
  PD_INTERNAL = 7
} pd_status;

/* Per-slot outcome written by the kernels (or by host validation). */
typedef enum pd_slot_code {
  PD_SLOT_OK = 0,
  PD_SLOT_DEGENERATE_ARTICULATION = 1, /* index = joint    forward_dynamics.cpp:140-144 */
  PD_SLOT_JSI_NOT_SPD = 2,             /*                  forward_dynamics.cpp:93-98   */
  PD_SLOT_JSI_REFINE_FAILED = 3,       /*                  forward_dynamics.cpp:108-116 */
  PD_SLOT_LINK_INERTIA_NOT_PD = 4,     /*                  forward_dynamics.cpp:317-320 */
  PD_SLOT_OEE_SINGULAR_PIVOT = 5,      /* (round, block)   oee.hpp:132-137             */
  PD_SLOT_OEE_SINGULAR_FINAL = 6,      /* (round, block)   oee.hpp:182-187             */
  PD_SLOT_BAD_MODEL = 7,               /* index = spatial-inertia rule, spatial.cpp:72-87 */
  PD_SLOT_BAD_SIZE = 8                 /* check_sizes, forward_dynamics.cpp:19-31      */
} pd_slot_code;

/* Detail for PD_SLOT_BAD_MODEL (slot index field). */
typedef enum pd_model_rule {
  PD_RULE_MASS = 1,      /* "spatial inertia: mass must be positive" */
  PD_RULE_FINITE = 2,    /* "spatial inertia: parameters must be finite" */
  PD_RULE_SYMMETRIC = 3, /* "...rotational inertia must be symmetric" */
  PD_RULE_PD = 4         /* "...rotational inertia must be positive definite" */
} pd_model_rule;

typedef struct pd_ctx pd_ctx;

/* ExecTrace (trace.hpp:24-39): the dependency profile of the kernel variant
 * that ran. parallel_link_stages = per-link stages whose iterations ran
 * independently (a thread per link); longest_sequential_link_chain = the
 * longest link walk one thread carried a dependency through;
 * scan_rounds_max = Hillis-Steele combine rounds of the deepest link scan;
 * oee_rounds = odd-even elimination rounds. */
typedef struct pd_exec_trace {
  int32_t parallel_link_stages;
  int32_t longest_sequential_link_chain;
  int32_t scan_rounds_max;
  int32_t oee_rounds;
} pd_exec_trace;

/* Context on one CUDA device (ordinal). Owns device buffers and a stream. */
pd_status pd_create(pd_ctx** out, int device);
void pd_destroy(pd_ctx* ctx);
int pd_abi_version(void);
const char* pd_status_string(pd_status s);
/* Last call-level error text of this context ("" if none). */
const char* pd_last_error(const pd_ctx* ctx);

/* Use an external CUDA stream (cudaStream_t as void*; cudaStreamLegacy
 * ((void*)1) selects the legacy default stream); NULL restores the context's
 * own non-blocking stream. */
pd_status pd_set_stream(pd_ctx* ctx, void* stream);
pd_status pd_synchronize(pd_ctx* ctx);

/* Upload and pack a model set: n_models chains of n_links links each.
 * Validates every link with the spatial_inertia_from rules; a model whose
 * link fails gets model_status[m] = PD_SLOT_BAD_MODEL and model_rule[m] = the
 * rule (pd_model_rule) of the first failing link (nullable outputs). Problems
 * bound to a bad model report that code instead of being solved.
 * gravity may be NULL (default (0,0,-9.81) for every model). */
pd_status pd_set_models(pd_ctx* ctx, int64_t n_models, int32_t n_links, const double* links,
                        const double* gravity, int32_t* model_status, int32_t* model_rule);

/* Solve `batch` problems against the current models, host buffers in and out
 * ([problem][link]); blocks until results are on the host. slot_* outputs are
 * nullable. Returns PD_OK if the call ran (slots may still carry errors). */
pd_status pd_forward_dynamics(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* q, const double* qdot,
                              const double* tau, double* qddot, int32_t* slot_status, int32_t* slot_round,
                              int32_t* slot_index);

/* Same on device buffers in [link][problem] layout, asynchronous on the
 * context's stream. d_slot_* must be device int32 arrays of length batch;
 * each is nullable on its own (internal scratch then takes that output). */
pd_status pd_forward_dynamics_device(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* d_q,
                                     const double* d_qdot, const double* d_tau, double* d_qddot,
                                     int32_t* d_slot_status, int32_t* d_slot_round, int32_t* d_slot_index);

/* A traced solve (host buffers, as pd_forward_dynamics): runs the
 * CTA-per-chain variants whose link recursions are log-depth scans and OEE
 * rounds -- the parallel structure the reference's counters describe -- and
 * fills *trace (nullable) from that variant. The reference's expectations
 * (tests/test_fwddyn.cpp:263-283): JSIIA and CFA longest chain 0, ABIA n,
 * scan rounds ceil(log2 n), CFA OEE rounds ceil(log2 n). */
pd_status pd_forward_dynamics_traced(pd_ctx* ctx, pd_algo algo, int64_t batch, const double* q,
                                     const double* qdot, const double* tau, double* qddot, int32_t* slot_status,
                                     int32_t* slot_round, int32_t* slot_index, pd_exec_trace* trace);

/* The kernel variant(s) the last forward-dynamics call on this context ran
 * (e.g. "abia_ring_kernel<224> grid 148 tiles 293") and their ExecTrace. */
const char* pd_last_variant(const pd_ctx* ctx);
pd_status pd_last_trace(const pd_ctx* ctx, pd_exec_trace* trace);

/* Kernel choice depends on (algorithm, n, batch). A caller that splits one
 * batch over several calls or devices sets the whole batch here (0 = each
 * call's own batch): every part then runs the same variants and the results
 * are bit-identical to the unsplit call's (acceptance_main.cpp:495-580). */
pd_status pd_set_selection_batch(pd_ctx* ctx, int64_t batch);

/* Joint torques of inverse dynamics with default IdOptions (gravity on, no
 * base motion, no tip wrench), host buffers [problem][link]. */
pd_status pd_inverse_dynamics(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot,
                              const double* qddot, double* tau);

/* IdOptions (inverse_dynamics.hpp:23-28). Twists stack (angular, linear) in
 * base coordinates; the tip wrench stacks (moment, force) in the last link's
 * frame. A NULL options pointer means the defaults (zeros, gravity on). */
typedef struct pd_id_options {
  double base_velocity[6];
  double base_acceleration[6];
  double tip_wrench[6];
  int32_t apply_gravity;
} pd_id_options;

/* Inverse dynamics with options, host buffers [problem][link]. A model that
 * failed upload validation makes the call fail with PD_INVALID_ARGUMENT and
 * the reference's spatial-inertia message (pd_last_error), as the
 * reference's link_inertias throws. */
pd_status pd_inverse_dynamics_opts(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot,
                                   const double* qddot, const pd_id_options* opts, double* tau);

/* Same on device buffers in [link][problem] layout, asynchronous. */
pd_status pd_inverse_dynamics_device(pd_ctx* ctx, int64_t batch, const double* d_q, const double* d_qdot,
                                     const double* d_qddot, const pd_id_options* opts, double* d_tau);

/* Gravity, centrifugal and Coriolis torques (qddot = 0, default options). */
pd_status pd_bias_torque(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, double* tau);

/* Link twists, accelerations and wrenches of one inverse-dynamics evaluation,
 * each [problem][link][6] in the reference's link frames. */
pd_status pd_link_states(pd_ctx* ctx, int64_t batch, const double* q, const double* qdot, const double* qddot,
                         const pd_id_options* opts, double* velocity, double* acceleration, double* force);

/* Joint-space inertia matrices M(q), [problem][n][n] row-major (exactly
 * symmetric, as the reference's 0.5 (M + M^T)). */
pd_status pd_joint_space_inertia(pd_ctx* ctx, int64_t batch, const double* q, double* M);

/* Reference error message of a slot outcome into buf (always terminated). */
void pd_slot_message(int32_t code, int32_t round, int32_t index, int32_t n_links, char* buf, int32_t buflen);

/* Seeded synthetic workloads of the reference benchmark (product side,
 * host threads):
 *   pd_mix             <- mix (bench.cpp:42-47, splitmix64 finalizer)
 *   pd_workload_seed   <- workload_seed (bench.cpp:350-355)
 *   pd_random_chain    <- random_chain(n, seed) (model.cpp:157-185)
 *   pd_workload_chains <- workload_chains (bench.cpp:357-366), chains
 *                         [g0, g0+count) of the cell, links[chain][link][31]
 *   pd_workload_inputs <- workload_inputs (bench.cpp:368-383), [group][link] */
uint64_t pd_mix(uint64_t x);
uint64_t pd_workload_seed(uint64_t seed, int32_t n_links, int64_t n_groups);
void pd_random_chain(int32_t n_links, uint64_t seed, double* links);
void pd_workload_chains(uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count, double* links);
void pd_workload_inputs(uint64_t cell_seed, int32_t n_links, int64_t n_groups, int64_t repeat, double* q,
                        double* qdot, double* drive);

/* The paper's building block 1 on its own: `batch` block bi-diagonal
 * systems with dim x dim blocks (1 <= dim <= 6) and implicit identity diagonal
 * (BlockBiDiagSystem<D>, include/pardyn/scan.hpp:100-168), solved by an
 * all-prefix scan of affine elements: lower (upper = 0): x[0] = rhs[0],
 * x[k] = coupling[k-1] x[k-1] + rhs[k]; upper: x[n-1] = rhs[n-1],
 * x[k] = coupling[k] x[k+1] + rhs[k]. coupling [batch][n-1][dim*dim]
 * row-major, rhs / x [batch][n][dim], host buffers.
 *   pd_block_bidiag_solve   <- solve_lower_bidiag<D> / solve_upper_bidiag<D>
 *   pd_block_bidiag_solve6  the dim = 6 case (the dynamics' recurrences) */
pd_status pd_block_bidiag_solve(pd_ctx* ctx, int32_t dim, int64_t batch, int32_t n, int32_t upper,
                                const double* coupling, const double* rhs, double* x);
pd_status pd_block_bidiag_solve6(pd_ctx* ctx, int64_t batch, int32_t n, int32_t upper, const double* coupling,
                                 const double* rhs, double* x);

/* The paper's building block 2 on its own: `batch` symmetric block
 * tri-diagonal systems of n <= 256 block rows with 5x5 blocks solved by
 * odd-even elimination (oee_solve<5,1>, include/pardyn/oee.hpp:149-189):
 * diag [batch][n][25] (row-major, symmetric), upper [batch][n-1][25] (block
 * row k to k+1; the sub-diagonal blocks are their transposes), rhs
 * [batch][n][5] -> x [batch][n][5], host buffers. Per system: PD_SLOT_OK,
 * PD_SLOT_OEE_SINGULAR_PIVOT (round, block) or PD_SLOT_OEE_SINGULAR_FINAL
 * (rounds, block), the reference's smallest-failing-row rule. */
pd_status pd_block_tridiag_solve5(pd_ctx* ctx, int64_t batch, int32_t n, const double* diag, const double* upper,
                                  const double* rhs, double* x, int32_t* slot_status, int32_t* slot_round,
                                  int32_t* slot_index);
/* The same for block size `block` (1..6) and `cols` (1..4) right-hand-side
 * columns, oee_solve<B, M> (oee.hpp:149-189): diag / upper [..][block*block],
 * rhs / x [batch][n][block*cols] with each block row-major (element (r, c) at
 * r * cols + c). The singularity test is FullPivLU::isInvertible's with
 * threshold block * eps (oee.hpp:40-51). */
pd_status pd_block_tridiag_solve(pd_ctx* ctx, int32_t block, int32_t cols, int64_t batch, int32_t n,
                                 const double* diag, const double* upper, const double* rhs, double* x,
                                 int32_t* slot_status, int32_t* slot_round, int32_t* slot_index);
/* Odd-even elimination rounds on a state (OeeState<B, M> + oee_eliminate_round,
 * oee.hpp:57-145) for `batch` systems: diag [batch][n][block*block], coupling
 * [batch][max(n - distance, 0)][block*block] (coupling[i] links row i to row
 * i + distance), rhs [batch][n][block*cols], after `state_round` rounds. Runs
 * `rounds` more rounds (numbered state_round + 1, ...) and writes the advanced
 * state to diag_out / rhs_out (same shapes) and coupling_out
 * [batch][max(n - distance * 2^rounds, 0)][block*block]. A singular pivot
 * reports PD_SLOT_OEE_SINGULAR_PIVOT (round, block) for that system, whose
 * outputs are then unspecified. 1 <= n <= 256, block 1..6, cols 1..4. */
pd_status pd_oee_eliminate_rounds(pd_ctx* ctx, int32_t block, int32_t cols, int64_t batch, int32_t n,
                                  int32_t distance, int32_t state_round, int32_t rounds, const double* diag,
                                  const double* coupling, const double* rhs, double* diag_out,
                                  double* coupling_out, double* rhs_out, int32_t* slot_status, int32_t* slot_round,
                                  int32_t* slot_index);

/* The same chains generated on the device (§8f row 3), one thread per chain:
 *   pd_workload_chains_device  chains [g0, g0+count) into device memory,
 *                              d_links[chain][link][31], asynchronous
 *   pd_set_models_workload     generate, validate (spatial_inertia_from rules,
 *                              on the device) and pack them as the model set
 *                              without a host copy; gravity: 3 doubles for
 *                              every model or NULL (default)
 * Same mt19937_64 streams and arithmetic as pd_workload_chains (no FMA
 * contraction, IEEE sqrt): draws are bit exact; fields through sin/cos may
 * differ in the last bit, since the device's sin/cos are correctly rounded
 * (double-double evaluation) and glibc's are not always (~0.3% of
 * evaluations). */
pd_status pd_workload_chains_device(pd_ctx* ctx, uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count,
                                    double* d_links);
pd_status pd_set_models_workload(pd_ctx* ctx, uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count,
                                 const double* gravity, int32_t* model_status, int32_t* model_rule);

/* The reference's per-chain operator builders on the device, in its dense
 * representation. Host buffers,
 * blocks row-major, arrays problem-major; each call blocks until done.
 *
 *   pd_assemble_kinematics   <- assemble_kinematics(chain, q) (model.hpp:51-58,
 *                               src/model.cpp:117-146) against the current
 *                               models: rel [b][n][12] (R 9, p 3),
 *                               base_transport [b][36], transport [b][n-1][36]
 *                               (Ad of rel[i+1]), screw [b][n][6]
 *   pd_link_inertias         <- link_inertias(chain) (model.hpp:60-61,
 *                               src/model.cpp:148-155): [models][n][36]; a
 *                               model that failed validation fails the call
 *                               with the spatial_inertia_from message
 *   pd_articulated_body_inertias
 *                            <- articulated_body_inertias(kin, inertia)
 *                               (forward_dynamics.hpp:48-56,
 *                               src/forward_dynamics.cpp:120-163): inputs
 *                               transport [b][n-1][36], inertia [b][n][36]
 *                               ([n][36] for all if shared_inertia), screw
 *                               [b][n][6]; outputs abi [b][n][36],
 *                               joint_inertia [b][n], gain [b][n][6]; per
 *                               problem PD_SLOT_OK or
 *                               PD_SLOT_DEGENERATE_ARTICULATION (index = joint)
 *   pd_constraint_basis      <- build_constraint_basis(chain)
 *                               (forward_dynamics.hpp:64-71,
 *                               src/forward_dynamics.cpp:245-259): screw
 *                               [k][6] -> basis [k][30] (6x5)
 *   pd_cfa_operators         <- build_cfa_operators(chain, kin, basis)
 *                               (forward_dynamics.hpp:73-96,
 *                               src/forward_dynamics.cpp:261-357): inputs as
 *                               above plus basis [b][n][30]; outputs
 *                               constraint diag [b][n][25] / upper
 *                               [b][n-1][25], cross_sub / cross_super
 *                               [b][n-1][5], cross_diag [b][n][5],
 *                               joint_diag [b][n], joint_off [b][n-1]; per
 *                               problem PD_SLOT_OK or
 *                               PD_SLOT_LINK_INERTIA_NOT_PD (index = link)
 *   pd_cfa_apply             <- CfaOperators::apply_cross / apply_cross_transpose
 *                               / apply_joint (forward_dynamics.cpp:359-416):
 *                               in [b][n] -> out [b][n][5] (PD_APPLY_CROSS),
 *                               in [b][n][5] -> out [b][n] (PD_APPLY_CROSS_TRANSPOSE),
 *                               in [b][n] -> out [b][n] (PD_APPLY_JOINT) */
typedef enum pd_apply_op { PD_APPLY_CROSS = 0, PD_APPLY_CROSS_TRANSPOSE = 1, PD_APPLY_JOINT = 2 } pd_apply_op;

pd_status pd_assemble_kinematics(pd_ctx* ctx, int64_t batch, const double* q, double* rel, double* base_transport,
                                 double* transport, double* screw);
pd_status pd_link_inertias(pd_ctx* ctx, double* inertia);
pd_status pd_articulated_body_inertias(pd_ctx* ctx, int64_t batch, int32_t n, const double* transport,
                                       const double* inertia, int32_t shared_inertia, const double* screw,
                                       double* abi, double* joint_inertia, double* gain, int32_t* slot_status,
                                       int32_t* slot_index);
pd_status pd_constraint_basis(pd_ctx* ctx, int64_t count, const double* screw, double* basis);
pd_status pd_cfa_operators(pd_ctx* ctx, int64_t batch, int32_t n, const double* inertia, int32_t shared_inertia,
                           const double* transport, const double* screw, const double* basis, double* constraint_diag,
                           double* constraint_upper, double* cross_sub, double* cross_diag, double* cross_super,
                           double* joint_diag, double* joint_off, int32_t* slot_status, int32_t* slot_index);
pd_status pd_cfa_apply(pd_ctx* ctx, int32_t op, int64_t batch, int32_t n, const double* cross_sub,
                       const double* cross_diag, const double* cross_super, const double* joint_diag,
                       const double* joint_off, const double* in, double* out);

/* The three propagations of inverse dynamics over caller-supplied dense
 * kinematics (inverse_dynamics.hpp:36-66, src/inverse_dynamics.cpp:27-120),
 * each a block bi-diagonal system solved by the building-block scan
 * (pd_block_bidiag_solve6's kernel) after a device-side setup of its
 * couplings and right-hand sides:
 *   PD_PROPAGATE_VELOCITIES     V_0 = Ad_base V_b + S_0 qd_0, V_i = T_{i-1} V_{i-1} + S_i qd_i
 *                               (boundary = base twist; needs base_transport, qdot)
 *   PD_PROPAGATE_ACCELERATIONS  A_i = T_{i-1} A_{i-1} + S_i qdd_i + ad_{V_i}(S_i qd_i)
 *                               (boundary = base acceleration; needs velocity)
 *   PD_PROPAGATE_FORCES         F_i = T_i^T F_{i+1} + J_i A_i - ad_{V_i}^T (J_i V_i), F_{n-1} += tip
 *                               (boundary = tip wrench; needs inertia, velocity, acceleration)
 * Arrays: base_transport [b][36], transport [b][n-1][36], screw / velocity /
 * acceleration / out [b][n][6], inertia [b][n][36] ([n][36] if
 * shared_inertia), qdot / qddot [b][n], boundary [6]. */
typedef enum pd_propagate_kind {
  PD_PROPAGATE_VELOCITIES = 0,
  PD_PROPAGATE_ACCELERATIONS = 1,
  PD_PROPAGATE_FORCES = 2
} pd_propagate_kind;
pd_status pd_propagate(pd_ctx* ctx, int32_t kind, int64_t batch, int32_t n, const double* base_transport,
                       const double* transport, const double* screw, const double* inertia, int32_t shared_inertia,
                       const double* qdot, const double* qddot, const double* velocity, const double* acceleration,
                       const double* boundary, double* out);

/* Page-locked host memory for staging host-buffer calls (copies from it run
 * at PCIe DMA speed instead of through the driver's pageable bounce buffer).
 * The C++ drop-in packs its batch calls into such a buffer. */
pd_status pd_host_alloc(uint64_t bytes, void** out);
void pd_host_free(void* p);

/* Diagnostic: measured dense FP64 FMA throughput of this device (TFLOP/s),
 * the FP64 roofline denominator (no FP64 figure in MEASURED_PEAKS.json). */
pd_status pd_probe_fp64_peak(pd_ctx* ctx, double* tflops, double* elapsed_ms);

/* Number of kernels this context has launched since creation. */
int64_t pd_kernel_launches(const pd_ctx* ctx);

/* Name of the kernel variant pd_forward_dynamics would run for (algo, n). */
const char* pd_kernel_variant(const pd_ctx* ctx, pd_algo algo, int32_t n_links);

#ifdef __cplusplus
}
#endif

#endif /* PARDYN_C_H_ */
