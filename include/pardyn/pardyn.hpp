// pardyn drop-in C++ API over the B200 C-ABI (include/pardyn_c.h).
//
// Mirrors the reference library's public forward-dynamics surface
// (/root/reference/proj/core/include/pardyn/{types,model,trace,
// forward_dynamics,inverse_dynamics}.hpp) with the same names, argument
// meaning and error behaviour; every solve runs on the GPU. Eigen is not a
// dependency: JointVector / Vec3 / Mat3 / Vec6 / Mat6 / MatrixXd are small
// value types (include/pardyn/linalg.hpp) with the subset of Eigen's
// interface the reference API and its callers use.
//
//   FdAlgo                         forward_dynamics.hpp:29
//   forward_dynamics(...)          forward_dynamics.hpp:103-105
//   jsiia_/abia_/cfa_forward_dynamics  forward_dynamics.hpp:38-42, 58-62, 98-101
//   FdProblem / FdResult           forward_dynamics.hpp:111-123
//   batch_forward_dynamics(...)    forward_dynamics.hpp:125-126
//   Twist / Wrench                 spatial.hpp:15-60 (stacked (angular, linear) / (moment, force))
//   IdOptions / LinkStates         inverse_dynamics.hpp:23-34
//   inverse_dynamics / bias_torque / link_states   inverse_dynamics.hpp:71-83
//   propagate_velocities / _accelerations / _forces, inverse_dynamics_assembled   inverse_dynamics.hpp:36-75
//   joint_space_inertia            forward_dynamics.hpp:34-35 (MatrixXd stand-in)
//   solve_lower_bidiag / solve_upper_bidiag / oee_solve   scan.hpp:100-168, oee.hpp:149-189
//   LinkSpec / RobotChain          model.hpp:17-30
//   SE3Transform / AdjointMap / SpatialInertia, skew, small_adjoint,
//   adjoint_of, screw_exp, spatial_inertia_from   spatial.hpp:75-150
//   ChainKinematics / assemble_kinematics / link_inertias   model.hpp:37-61
//   ArticulatedBodyInertias / articulated_body_inertias   forward_dynamics.hpp:44-56
//   ConstraintBasis / build_constraint_basis      forward_dynamics.hpp:64-71
//   CfaOperators (+ apply_*) / build_cfa_operators   forward_dynamics.hpp:73-96
//   random_chain                   model.hpp:66-70
//   validate_chain / load_chain / save_chain   model.hpp:56-82 (JSON model files)
//   ExecTrace                      trace.hpp:24-39
//   ModelError / DynamicsError / SingularBlockError   types.hpp:21-46
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "linalg.hpp"

namespace pardyn {

// ----------------------------------------------------------------- spatial types (spatial.hpp)
// Rigid-body velocity (angular, linear) (spatial.hpp:15-33).
struct Twist {
  Vec3 angular = Vec3::Zero();
  Vec3 linear = Vec3::Zero();
  Twist() = default;
  Twist(const Vec3& ang, const Vec3& lin) : angular(ang), linear(lin) {}
  static Twist from_stacked(const Vec6& v) { return {v.head<3>(), v.tail<3>()}; }
  Vec6 stacked() const {
    Vec6 v;
    for (int k = 0; k < 3; ++k) {
      v(k) = angular(k);
      v(3 + k) = linear(k);
    }
    return v;
  }
  bool is_finite() const { return angular.allFinite() && linear.allFinite(); }
};
inline Twist operator+(const Twist& a, const Twist& b) { return {a.angular + b.angular, a.linear + b.linear}; }
inline Twist operator-(const Twist& a, const Twist& b) { return {a.angular - b.angular, a.linear - b.linear}; }
inline Twist operator*(double s, const Twist& a) { return {s * a.angular, s * a.linear}; }

// Generalised force (moment, force) (spatial.hpp:44-69).
struct Wrench {
  Vec3 moment = Vec3::Zero();
  Vec3 force = Vec3::Zero();
  Wrench() = default;
  Wrench(const Vec3& m, const Vec3& f) : moment(m), force(f) {}
  static Wrench from_stacked(const Vec6& v) { return {v.head<3>(), v.tail<3>()}; }
  Vec6 stacked() const {
    Vec6 v;
    for (int k = 0; k < 3; ++k) {
      v(k) = moment(k);
      v(3 + k) = force(k);
    }
    return v;
  }
  bool is_finite() const { return moment.allFinite() && force.allFinite(); }
};
inline Wrench operator+(const Wrench& a, const Wrench& b) { return {a.moment + b.moment, a.force + b.force}; }
inline Wrench operator-(const Wrench& a, const Wrench& b) { return {a.moment - b.moment, a.force - b.force}; }
inline Wrench operator*(double s, const Wrench& a) { return {s * a.moment, s * a.force}; }

// x_target = rotation * x_source + translation (spatial.hpp:75-97).
struct SE3Transform {
  Mat3 rotation = Mat3::Identity();
  Vec3 translation = Vec3::Zero();
  SE3Transform operator*(const SE3Transform& rhs) const {
    return {rotation * rhs.rotation, rotation * rhs.translation + translation};
  }
  SE3Transform inverse() const {
    const Mat3 rt = rotation.transpose();
    return {rt, -(rt * translation)};
  }
  Vec3 apply(const Vec3& point) const { return rotation * point + translation; }
  // Rotation orthonormal with determinant +1, translation finite.
  bool is_valid(double tol = 1e-9) const;
};

// Frame change of twists (apply) and wrenches (transpose_apply) (spatial.hpp:99-109).
struct AdjointMap {
  Mat6 mat = Mat6::Identity();
  Twist apply(const Twist& v) const { return Twist::from_stacked(mat * v.stacked()); }
  Wrench transpose_apply(const Wrench& f) const { return Wrench::from_stacked(mat.transpose() * f.stacked()); }
};

struct RobotChain;

// 6x6 SPD link inertia, built by spatial_inertia_from (spatial.hpp:111-127).
class SpatialInertia {
 public:
  SpatialInertia() : mat_(Mat6::Identity()) {}
  const Mat6& matrix() const { return mat_; }
  Wrench apply(const Twist& v) const { return Wrench::from_stacked(mat_ * v.stacked()); }

 private:
  explicit SpatialInertia(const Mat6& m) : mat_(m) {}
  friend SpatialInertia spatial_inertia_from(double mass, const Vec3& com, const Mat3& inertia_rot);
  friend std::vector<SpatialInertia> link_inertias(const RobotChain& chain);
  Mat6 mat_;
};

Mat3 skew(const Vec3& a);                       // spatial.hpp:129-130
Mat6 small_adjoint(const Twist& v);             // spatial.hpp:132-135
AdjointMap adjoint_of(const SE3Transform& t);   // spatial.hpp:137-138
SE3Transform screw_exp(const Twist& s, double q);  // spatial.hpp:140-143
// spatial.hpp:145-150: throws std::invalid_argument with the reference's texts.
SpatialInertia spatial_inertia_from(double mass, const Vec3& com, const Mat3& inertia_rot);

class ModelError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DynamicsError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class SingularBlockError : public DynamicsError {
 public:
  SingularBlockError(int round, int index, const std::string& what)
      : DynamicsError(what), round_(round), index_(index) {}
  int round() const noexcept { return round_; }
  int index() const noexcept { return index_; }

 private:
  int round_, index_;
};
// Raised when no CUDA device / kernel launch is available (no CPU fallback).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline int ceil_log2(std::size_t n) {
  int k = 0;
  std::size_t p = 1;
  while (p < n) {
    p <<= 1;
    ++k;
  }
  return k;
}

// ----------------------------------------------------------------- model
// model.hpp:17-23: link i hangs off link i-1 (link 0 off the base) by a
// one-degree-of-freedom joint of screw `joint_screw` in the link-i frame.
struct LinkSpec {
  double mass = 1.0;
  Vec3 com = Vec3::Zero();              // centre of mass, link frame
  Mat3 inertia_rot = Mat3::Identity();  // rotational inertia about the COM
  Twist joint_screw{Vec3::UnitZ(), Vec3::Zero()};  // unit 6-norm
  SE3Transform home_transform;          // parent-frame -> link-frame map at q = 0
};

struct RobotChain {  // model.hpp:25-30
  std::vector<LinkSpec> links;
  Vec3 gravity = Vec3(0.0, 0.0, -9.81);
  int size() const { return static_cast<int>(links.size()); }
};

// Exact field-for-field comparison (model.hpp:32-35).
bool operator==(const LinkSpec& a, const LinkSpec& b);
bool operator==(const RobotChain& a, const RobotChain& b);

// Configuration-dependent operators at q (model.hpp:37-49): rel[i] maps
// link-(i-1) coordinates into link-i coordinates, transport[i] is the adjoint
// of rel[i+1].
struct ChainKinematics {
  std::vector<SE3Transform> rel;      // n
  AdjointMap base_transport;          // adjoint of rel[0]
  std::vector<AdjointMap> transport;  // n - 1
  std::vector<Twist> screw;           // n
  int size() const { return static_cast<int>(rel.size()); }
};

// model.hpp:51-58 (model.cpp:117-146), evaluated on the device.
ChainKinematics assemble_kinematics(const RobotChain& chain, const JointVector& q);
// model.hpp:60-61 (model.cpp:148-155), evaluated on the device; throws
// std::invalid_argument with spatial_inertia_from's message for a bad link.
std::vector<SpatialInertia> link_inertias(const RobotChain& chain);

// Deterministic random chain (model.cpp:157-185), bit-identical to the
// reference generator.
RobotChain random_chain(int n, std::uint64_t seed);

// model.cpp:75-115: throws ModelError naming the offending link and field.
void validate_chain(const RobotChain& chain);

// JSON model files (model.hpp:72-82, model.cpp:244-337): the reference's
// layout {"n", "gravity", "links": [{"mass", "com", "inertia_rot",
// "joint_screw", "home_transform": {"rotation", "translation"}}]}; load
// validates, save round-trips exactly.
RobotChain load_chain(const std::string& path);
void save_chain(const RobotChain& chain, const std::string& path);

// ----------------------------------------------------------------- trace (trace.hpp:12-39)
struct ScanTrace {
  int rounds = 0;
};
struct OeeTrace {
  int rounds = 0;
};
// Filled from the kernel variant that ran (pd_last_trace): a traced call runs
// the CTA-per-chain variants whose recursions are log-depth scans / OEE rounds.
struct ExecTrace {
  int parallel_link_stages = 0;
  int longest_sequential_link_chain = 0;
  int scan_rounds_max = 0;
  int oee_rounds = 0;
  void note_parallel_stage() { ++parallel_link_stages; }
  void note_sequential_chain(int length) {
    longest_sequential_link_chain = length > longest_sequential_link_chain ? length : longest_sequential_link_chain;
  }
  void note_scan(const ScanTrace& t) { scan_rounds_max = t.rounds > scan_rounds_max ? t.rounds : scan_rounds_max; }
  void note_oee(const OeeTrace& t) { oee_rounds = t.rounds; }
};

// ----------------------------------------------------------------- building blocks (scan.hpp, oee.hpp)
// The paper's two solvers on their own, on the GPU: block bi-diagonal
// systems by the affine scan (scan.hpp:100-168), symmetric block
// tri-diagonal systems by odd-even elimination (oee.hpp:28-32, 149-189), at
// the block sizes the reference's templates take (the dynamics use D = 6,
// B = 5).
enum class BiDiagOrientation { lower, upper };

// lower: x[0] = rhs[0], x[k] = coupling[k-1] x[k-1] + rhs[k];
// upper: x[n-1] = rhs[n-1], x[k] = coupling[k] x[k+1] + rhs[k].
template <int D>
struct BlockBiDiagSystem {
  BiDiagOrientation orientation = BiDiagOrientation::lower;
  std::vector<Matrix<D, D>> coupling;  // n - 1 blocks
  std::vector<Matrix<D, 1>> rhs;       // n blocks
};

// diag[i] symmetric, upper[i] couples row i to row i+1 (sub-diagonal = upper^T).
template <int B>
struct SymBlockTriDiagSystem {
  std::vector<Matrix<B, B>> diag;   // n blocks
  std::vector<Matrix<B, B>> upper;  // n - 1 blocks
};

// One step of the block recursion x[k] = coeff x[k-1] + offset; composing
// steps gives the step of the concatenated range (scan.hpp:66-97). The later
// step's coefficient multiplies from the left. Value algebra only: the scans
// run on the GPU as solve_lower_bidiag / solve_upper_bidiag.
template <int D>
struct AffineElement {
  Matrix<D, D> coeff = Matrix<D, D>::Identity();
  Matrix<D, 1> offset = Matrix<D, 1>::Zero();
  static AffineElement identity() { return {}; }
  static AffineElement compose(const AffineElement& first, const AffineElement& second) {
    AffineElement out;
    out.coeff = second.coeff * first.coeff;
    out.offset = second.coeff * first.offset + second.offset;
    return out;
  }
};

// Elimination state after `round` rounds: coupling[i] links row i to row
// i + distance (oee.hpp:57-67).
template <int B, int M = 1>
struct OeeState {
  using PivotBlock = Matrix<B, B>;
  using RhsBlock = Matrix<B, M>;
  std::vector<PivotBlock> diag;
  std::vector<PivotBlock> coupling;
  std::vector<RhsBlock> rhs;
  int distance = 1;
  int round = 0;
};

namespace detail {
// Row-major packed blocks through the C-ABI (pd_block_bidiag_solve /
// pd_block_tridiag_solve / pd_oee_eliminate_rounds); D, B in 1..6, M in 1..4.
// Throw the reference's exceptions (std::invalid_argument, SingularBlockError).
void bidiag_solve_rm(int dim, bool upper, std::size_t n, const double* coupling, const double* rhs, double* x);
void oee_solve_rm(int block, int cols, std::size_t n, const double* diag, const double* upper, const double* rhs,
                  double* x);
void oee_rounds_rm(int block, int cols, std::size_t n, int distance, int round, const double* diag,
                   const double* coupling, const double* rhs, double* diag_out, double* coupling_out,
                   double* rhs_out);
// pivot x = rhs for one pivot (n = 1 elimination), SingularBlockError(round, index) if singular
void coefficient_solve_rm(int block, int cols, const double* pivot, const double* rhs, double* x, int round,
                          int index);

template <int D>
std::vector<Matrix<D, 1>> bidiag(const BlockBiDiagSystem<D>& sys, bool upper, ScanTrace* trace) {
  static_assert(D >= 1 && D <= 6, "block bi-diagonal solve: block size 1..6");
  const std::size_t n = sys.rhs.size();
  if (sys.coupling.size() + 1 != n && !(n == 0 && sys.coupling.empty()))
    throw std::invalid_argument("block bi-diagonal solve: need n - 1 coupling blocks for n right-hand sides");
  if (trace) trace->rounds = ceil_log2(n);  // the scan's designed depth (scan.hpp:32-65)
  std::vector<Matrix<D, 1>> x(n);
  if (n == 0) return x;
  std::vector<double> c(D * D * (n - 1)), r(D * n), xo(D * n);
  for (std::size_t k = 0; k + 1 < n; ++k) sys.coupling[k].toRowMajor(&c[D * D * k]);
  for (std::size_t k = 0; k < n; ++k) sys.rhs[k].toRowMajor(&r[D * k]);
  bidiag_solve_rm(D, upper, n, c.empty() ? nullptr : c.data(), r.data(), xo.data());
  for (std::size_t k = 0; k < n; ++k) x[k] = Matrix<D, 1>::FromRowMajor(&xo[D * k]);
  return x;
}
}  // namespace detail

template <int D>
std::vector<Matrix<D, 1>> solve_lower_bidiag(const BlockBiDiagSystem<D>& sys, ScanTrace* trace = nullptr) {
  return detail::bidiag<D>(sys, false, trace);
}
template <int D>
std::vector<Matrix<D, 1>> solve_upper_bidiag(const BlockBiDiagSystem<D>& sys, ScanTrace* trace = nullptr) {
  return detail::bidiag<D>(sys, true, trace);
}
// Exactly ceil_log2(n) rounds; throws SingularBlockError(round, index) like
// the reference (oee.hpp:149-189). B in 1..6, M in 1..4 right-hand-side columns.
template <int B, int M = 1>
std::vector<Matrix<B, M>> oee_solve(const SymBlockTriDiagSystem<B>& sys, const std::vector<Matrix<B, M>>& rhs,
                                    OeeTrace* trace = nullptr) {
  static_assert(B >= 1 && B <= 6 && M >= 1 && M <= 4, "odd-even elimination: B in 1..6, M in 1..4");
  const std::size_t n = sys.diag.size();
  if (rhs.size() != n || (n > 0 && sys.upper.size() + 1 != n))
    throw std::invalid_argument("odd-even elimination: inconsistent block counts");
  if (trace) trace->rounds = 0;
  std::vector<Matrix<B, M>> x(n);
  if (n == 0) return x;
  std::vector<double> d(B * B * n), u(B * B * (n - 1)), r(B * M * n), xo(B * M * n);
  for (std::size_t k = 0; k < n; ++k) {
    sys.diag[k].toRowMajor(&d[B * B * k]);
    rhs[k].toRowMajor(&r[B * M * k]);
  }
  for (std::size_t k = 0; k + 1 < n; ++k) sys.upper[k].toRowMajor(&u[B * B * k]);
  detail::oee_solve_rm(B, M, n, d.data(), u.empty() ? nullptr : u.data(), r.data(), xo.data());
  if (trace) trace->rounds = ceil_log2(n);
  for (std::size_t k = 0; k < n; ++k) x[k] = Matrix<B, M>::FromRowMajor(&xo[B * M * k]);
  return x;
}

// One elimination round on the GPU (oee.hpp:69-145): distance doubles, the
// couplings shrink to n - 2h; a singular pivot throws SingularBlockError and
// leaves the state as it was.
template <int B, int M>
void oee_eliminate_round(OeeState<B, M>& state) {
  static_assert(B >= 1 && B <= 6 && M >= 1 && M <= 4, "odd-even elimination: B in 1..6, M in 1..4");
  const std::size_t n = state.diag.size();
  const std::size_t h = static_cast<std::size_t>(state.distance);
  if (state.rhs.size() != n || state.coupling.size() != (n > h ? n - h : 0))
    throw std::invalid_argument("odd-even elimination: inconsistent block counts");
  const std::size_t nu = n > 2 * h ? n - 2 * h : 0;
  if (n == 0) {
    state.distance *= 2;
    state.round += 1;
    return;
  }
  std::vector<double> d(B * B * n), c(B * B * state.coupling.size()), r(B * M * n), d1(B * B * n),
      c1(B * B * nu), r1(B * M * n);
  for (std::size_t k = 0; k < n; ++k) {
    state.diag[k].toRowMajor(&d[B * B * k]);
    state.rhs[k].toRowMajor(&r[B * M * k]);
  }
  for (std::size_t k = 0; k < state.coupling.size(); ++k) state.coupling[k].toRowMajor(&c[B * B * k]);
  detail::oee_rounds_rm(B, M, n, state.distance, state.round, d.data(), c.empty() ? nullptr : c.data(), r.data(),
                        d1.data(), c1.empty() ? nullptr : c1.data(), r1.data());
  state.coupling.resize(nu);
  for (std::size_t k = 0; k < n; ++k) {
    state.diag[k] = Matrix<B, B>::FromRowMajor(&d1[B * B * k]);
    state.rhs[k] = Matrix<B, M>::FromRowMajor(&r1[B * M * k]);
  }
  for (std::size_t k = 0; k < nu; ++k) state.coupling[k] = Matrix<B, B>::FromRowMajor(&c1[B * B * k]);
  state.distance *= 2;
  state.round += 1;
}

// pivot x = rhs by full-pivot LU (oee.hpp:34-51); throws
// SingularBlockError(round, index) when the pivot is rank deficient.
template <int B, int C>
Matrix<B, C> coefficient_solve(const Matrix<B, B>& pivot, const Matrix<B, C>& rhs, int round, int index) {
  static_assert(B >= 1 && B <= 6 && C >= 1, "coefficient_solve: B in 1..6");
  double p[B * B], r[B * C], x[B * C];
  pivot.toRowMajor(p);
  rhs.toRowMajor(r);
  detail::coefficient_solve_rm(B, C, p, r, x, round, index);
  return Matrix<B, C>::FromRowMajor(x);
}

// ----------------------------------------------------------------- inverse dynamics (inverse_dynamics.hpp)
// inverse_dynamics.hpp:23-28
struct IdOptions {
  Twist base_velocity{};
  Twist base_acceleration{};
  Wrench tip_wrench{};
  bool apply_gravity = true;
};

// inverse_dynamics.hpp:30-34
struct LinkStates {
  std::vector<Twist> velocity;
  std::vector<Twist> acceleration;
  std::vector<Wrench> force;
};

// The three propagations over assembled kinematics (inverse_dynamics.hpp:36-66,
// inverse_dynamics.cpp:27-120): block bi-diagonal systems solved on the device
// by the building-block scan.
std::vector<Twist> propagate_velocities(const ChainKinematics& kin, const JointVector& qdot,
                                        const Twist& base_velocity, ScanTrace* trace = nullptr);
std::vector<Twist> propagate_accelerations(const ChainKinematics& kin, std::span<const Twist> velocity,
                                           const JointVector& qdot, const JointVector& qddot,
                                           const Twist& base_acceleration, ScanTrace* trace = nullptr);
std::vector<Wrench> propagate_forces(const ChainKinematics& kin, std::span<const Twist> velocity,
                                     std::span<const Twist> acceleration, std::span<const SpatialInertia> inertia,
                                     const Wrench& tip_wrench, ScanTrace* trace = nullptr);
// inverse_dynamics.hpp:68-75 (inverse_dynamics.cpp:122-164).
JointVector inverse_dynamics_assembled(const ChainKinematics& kin, std::span<const SpatialInertia> inertia,
                                       const Vec3& gravity, const JointVector& qdot, const JointVector& qddot,
                                       const IdOptions& opts = {}, ExecTrace* trace = nullptr);

JointVector inverse_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& qddot, const IdOptions& opts = {}, ExecTrace* trace = nullptr);
JointVector bias_torque(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                        ExecTrace* trace = nullptr);
LinkStates link_states(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                       const JointVector& qddot, const IdOptions& opts = {});

// ----------------------------------------------------------------- forward dynamics (forward_dynamics.hpp)
enum class FdAlgo { jsiia, abia, cfa };

// forward_dynamics.hpp:31-35: column j = ID(q, 0, e_j) without gravity, symmetrised.
MatrixXd joint_space_inertia(const RobotChain& chain, const JointVector& q, ExecTrace* trace = nullptr);

JointVector jsiia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                   const JointVector& tau, ExecTrace* trace = nullptr);

// forward_dynamics.hpp:44-56: joint_inertia[i] = S_i^T abi[i] S_i,
// gain[i] = abi[i] S_i / joint_inertia[i].
struct ArticulatedBodyInertias {
  std::vector<Mat6> inertia;
  JointVector joint_inertia;
  std::vector<Vec6> gain;
};
ArticulatedBodyInertias articulated_body_inertias(const ChainKinematics& kin, std::span<const SpatialInertia> inertia,
                                                  ExecTrace* trace = nullptr);

JointVector abia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                  const JointVector& tau, ExecTrace* trace = nullptr);

// forward_dynamics.hpp:64-71: basis[i]^T screw[i] = 0, [basis[i] screw[i]] orthogonal.
struct ConstraintBasis {
  std::vector<Matrix<6, 5>> basis;
};
ConstraintBasis build_constraint_basis(const RobotChain& chain);

// forward_dynamics.hpp:73-96: projections of (I - G) J^-1 (I - G)^T.
struct CfaOperators {
  SymBlockTriDiagSystem<5> constraint_op;
  std::vector<Vec5> cross_sub;    // n-1: couples row i+1 to column i
  std::vector<Vec5> cross_diag;   // n
  std::vector<Vec5> cross_super;  // n-1: couples row i to column i+1
  JointVector joint_diag;         // n
  JointVector joint_off;          // n-1

  std::vector<Vec5> apply_cross(const JointVector& v) const;
  JointVector apply_cross_transpose(std::span<const Vec5> f) const;
  JointVector apply_joint(const JointVector& v) const;
};
CfaOperators build_cfa_operators(const RobotChain& chain, const ChainKinematics& kin, const ConstraintBasis& basis,
                                 ExecTrace* trace = nullptr);

JointVector cfa_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                 const JointVector& tau, ExecTrace* trace = nullptr);

JointVector forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& tau, FdAlgo algo, ExecTrace* trace = nullptr);

struct FdProblem {
  RobotChain chain;
  JointVector q;
  JointVector qdot;
  JointVector tau;
};

struct FdResult {
  JointVector qddot;
  std::string error;
  bool ok() const { return error.empty(); }
};

// forward_dynamics.cpp:466-481: never throws per problem; the batch is
// bucketed by link count, one device call per bucket.
std::vector<FdResult> batch_forward_dynamics(std::span<const FdProblem> problems, FdAlgo algo);

// ----------------------------------------------------------------- device
namespace gpu {
// CUDA device the calling thread's single-problem calls run on (default 0).
void set_device(int device);
int device();
// Devices batch_forward_dynamics shards a bucket across (default: {device()}).
// Contiguous slices, one context per device, no collective; every slice
// selects kernels for the whole bucket, so results do not depend on the
// device count.
void set_devices(const std::vector<int>& devices);
std::vector<int> devices();
}  // namespace gpu

}  // namespace pardyn
