// pardyn drop-in C++ API over the B200 C-ABI (include/pardyn_c.h).
//
// Mirrors the reference library's public forward-dynamics surface
// (/root/reference/proj/core/include/pardyn/{types,model,trace,
// forward_dynamics,inverse_dynamics}.hpp) with the same names, argument
// meaning and error behaviour; every solve runs on the GPU. Eigen is not a
// dependency: JointVector / Vec3 / Mat3 / Vec6 are small value types with the
// subset of Eigen's interface the reference API and its callers use
// (size(), operator[], operator(), data(), Zero(), norm()).
//
//   FdAlgo                         forward_dynamics.hpp:29
//   forward_dynamics(...)          forward_dynamics.hpp:103-105
//   jsiia_/abia_/cfa_forward_dynamics  forward_dynamics.hpp:38-42, 58-62, 98-101
//   FdProblem / FdResult           forward_dynamics.hpp:111-123
//   batch_forward_dynamics(...)    forward_dynamics.hpp:125-126
//   Twist / Wrench                 spatial.hpp:15-60 (stacked (angular, linear) / (moment, force))
//   IdOptions / LinkStates         inverse_dynamics.hpp:23-34
//   inverse_dynamics / bias_torque / link_states   inverse_dynamics.hpp:71-83
//   joint_space_inertia            forward_dynamics.hpp:34-35 (MatrixXd stand-in)
//   solve_lower_bidiag / solve_upper_bidiag / oee_solve   scan.hpp:100-168, oee.hpp:149-189
//   LinkSpec / RobotChain          model.hpp:17-30
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

namespace pardyn {

// ----------------------------------------------------------------- types
class JointVector {
 public:
  JointVector() = default;
  explicit JointVector(std::size_t n) : v_(n, 0.0) {}
  JointVector(std::initializer_list<double> l) : v_(l) {}
  static JointVector Zero(std::size_t n) { return JointVector(n); }
  std::size_t size() const { return v_.size(); }
  double& operator[](std::size_t i) { return v_[i]; }
  double operator[](std::size_t i) const { return v_[i]; }
  double& operator()(std::size_t i) { return v_[i]; }
  double operator()(std::size_t i) const { return v_[i]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double norm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return std::sqrt(s);
  }
  JointVector operator-(const JointVector& o) const {
    JointVector r(size());
    for (std::size_t i = 0; i < size(); ++i) r[i] = v_[i] - o[i];
    return r;
  }
  bool operator==(const JointVector& o) const { return v_ == o.v_; }

 private:
  std::vector<double> v_;
};

using Vec3 = std::array<double, 3>;
using Vec6 = std::array<double, 6>;
using Mat3 = std::array<double, 9>;  // row-major

// Spatial vectors (spatial.hpp:15-60).
struct Twist {
  Vec3 angular{0.0, 0.0, 0.0};
  Vec3 linear{0.0, 0.0, 0.0};
  Vec6 stacked() const { return {angular[0], angular[1], angular[2], linear[0], linear[1], linear[2]}; }
  static Twist from_stacked(const Vec6& v) { return {{v[0], v[1], v[2]}, {v[3], v[4], v[5]}}; }
};
struct Wrench {
  Vec3 moment{0.0, 0.0, 0.0};
  Vec3 force{0.0, 0.0, 0.0};
  Vec6 stacked() const { return {moment[0], moment[1], moment[2], force[0], force[1], force[2]}; }
  static Wrench from_stacked(const Vec6& v) { return {{v[0], v[1], v[2]}, {v[3], v[4], v[5]}}; }
};

// Dense row-major matrix (the Eigen::MatrixXd that joint_space_inertia returns).
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(std::size_t r, std::size_t c) : r_(r), c_(c), v_(r * c, 0.0) {}
  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  double& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

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
struct LinkSpec {
  double mass = 1.0;
  Vec3 com{0.0, 0.0, 0.0};
  Mat3 inertia_rot{1, 0, 0, 0, 1, 0, 0, 0, 1};
  Vec6 joint_screw{0, 0, 1, 0, 0, 0};  // (angular, linear), unit 6-norm
  Mat3 home_rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};
  Vec3 home_translation{0.0, 0.0, 0.0};
};

struct RobotChain {
  std::vector<LinkSpec> links;
  Vec3 gravity{0.0, 0.0, -9.81};
  int size() const { return static_cast<int>(links.size()); }
};

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

// ----------------------------------------------------------------- trace
struct ExecTrace {
  int parallel_link_stages = 0;
  int longest_sequential_link_chain = 0;
  int scan_rounds_max = 0;
  int oee_rounds = 0;
};

// ----------------------------------------------------------------- dynamics
enum class FdAlgo { jsiia, abia, cfa };

JointVector forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& tau, FdAlgo algo, ExecTrace* trace = nullptr);
JointVector jsiia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                   const JointVector& tau, ExecTrace* trace = nullptr);
JointVector abia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                  const JointVector& tau, ExecTrace* trace = nullptr);
JointVector cfa_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                 const JointVector& tau, ExecTrace* trace = nullptr);

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

std::vector<FdResult> batch_forward_dynamics(std::span<const FdProblem> problems, FdAlgo algo);

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

JointVector inverse_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& qddot, const IdOptions& opts = {});
JointVector bias_torque(const RobotChain& chain, const JointVector& q, const JointVector& qdot);
LinkStates link_states(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                       const JointVector& qddot, const IdOptions& opts = {});
MatrixXd joint_space_inertia(const RobotChain& chain, const JointVector& q);

// ----------------------------------------------------------------- building blocks
// The paper's two solvers on their own (scan.hpp:100-168, oee.hpp:28-32,
// 149-189), on the GPU: 6x6 block bi-diagonal systems by the affine scan,
// symmetric 5x5 block tri-diagonal systems by odd-even elimination (the
// block sizes the dynamics use). Blocks are row-major.
enum class BiDiagOrientation { lower, upper };

template <int D>
struct BlockBiDiagSystem {
  BiDiagOrientation orientation = BiDiagOrientation::lower;
  std::vector<std::array<double, D * D>> coupling;  // n - 1 blocks
  std::vector<std::array<double, D>> rhs;           // n blocks
};

template <int B>
struct SymBlockTriDiagSystem {
  std::vector<std::array<double, B * B>> diag;   // n blocks
  std::vector<std::array<double, B * B>> upper;  // n - 1 blocks
};

struct ScanTrace {
  int rounds = 0;
};
struct OeeTrace {
  int rounds = 0;
};

std::vector<std::array<double, 6>> solve_lower_bidiag(const BlockBiDiagSystem<6>& sys, ScanTrace* trace = nullptr);
std::vector<std::array<double, 6>> solve_upper_bidiag(const BlockBiDiagSystem<6>& sys, ScanTrace* trace = nullptr);
// Throws SingularBlockError(round, index) like the reference.
std::vector<std::array<double, 5>> oee_solve(const SymBlockTriDiagSystem<5>& sys,
                                             const std::vector<std::array<double, 5>>& rhs,
                                             OeeTrace* trace = nullptr);

// ----------------------------------------------------------------- device
namespace gpu {
// CUDA device the calling thread's solves run on (default 0).
void set_device(int device);
int device();
}  // namespace gpu

}  // namespace pardyn
