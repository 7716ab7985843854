// The reference's operator suites (tests/test_fwddyn.cpp:141-283) written
// against the drop-in C++ API, whose assemble_kinematics, link_inertias,
// articulated_body_inertias, build_constraint_basis, build_cfa_operators,
// CfaOperators::apply_* and traced solves run on the device. Dense checks use
// small host matrices built here (test infrastructure); the column-probe
// joint-space inertia comes from the CPU oracle. One PASS/FAIL line per case;
// exit status = number of failures.
#include <pardyn/pardyn.hpp>

#include <algorithm>
#include <cmath>
#include <limits>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../oracle/oracle.hpp"

using namespace pardyn;

namespace {

int failures = 0;
void check(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

struct Sample {  // test_fwddyn.cpp:19-27
  RobotChain chain;
  JointVector q, qdot, tau;
};
JointVector uniform(std::mt19937_64& e, int n, double lo, double hi) {
  JointVector v(n);
  for (int i = 0; i < n; ++i) v[i] = lo + (hi - lo) * (static_cast<double>(e() >> 11) * 0x1.0p-53);
  return v;
}
Sample make_sample(int n, std::uint64_t seed) {
  Sample s;
  s.chain = random_chain(n, seed);
  std::mt19937_64 e(seed ^ 0xF00D);
  s.q = uniform(e, n, -3.0, 3.0);
  s.qdot = uniform(e, n, -2.0, 2.0);
  s.tau = uniform(e, n, -10.0, 10.0);
  return s;
}

template <int R, int C>
void put(MatrixXd& m, std::size_t r0, std::size_t c0, const Matrix<R, C>& b) {
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) m(r0 + r, c0 + c) = b(r, c);
}

// Dense lower Cholesky of an SPD matrix; false if a pivot is not positive.
bool cholesky(MatrixXd a, MatrixXd& L) {
  const std::size_t n = a.rows();
  L = MatrixXd(n, n);
  for (std::size_t k = 0; k < n; ++k) {
    double d = a(k, k);
    for (std::size_t j = 0; j < k; ++j) d -= L(k, j) * L(k, j);
    if (!(d > 0.0)) return false;
    L(k, k) = std::sqrt(d);
    for (std::size_t i = k + 1; i < n; ++i) {
      double v = a(i, k);
      for (std::size_t j = 0; j < k; ++j) v -= L(i, j) * L(k, j);
      L(i, k) = v / L(k, k);
    }
  }
  return true;
}
// X = A^-1 B for SPD A.
MatrixXd spd_solve(const MatrixXd& A, const MatrixXd& B) {
  MatrixXd L;
  cholesky(A, L);
  const std::size_t n = A.rows();
  MatrixXd X = B;
  for (std::size_t c = 0; c < B.cols(); ++c) {
    for (std::size_t i = 0; i < n; ++i) {
      double v = X(i, c);
      for (std::size_t j = 0; j < i; ++j) v -= L(i, j) * X(j, c);
      X(i, c) = v / L(i, i);
    }
    for (std::size_t i = n; i-- > 0;) {
      double v = X(i, c);
      for (std::size_t j = i + 1; j < n; ++j) v -= L(j, i) * X(j, c);
      X(i, c) = v / L(i, i);
    }
  }
  return X;
}
double rel_gap(const MatrixXd& a, const MatrixXd& b) { return (a - b).norm() / std::max(1.0, b.norm()); }

// (I - G)^T diag(J^-1) (I - G) (test_fwddyn.cpp:29-44)
MatrixXd dense_compliance_core(const RobotChain& chain, const ChainKinematics& kin) {
  const std::size_t n = chain.links.size();
  const auto inertia = link_inertias(chain);
  MatrixXd jinv(6 * n, 6 * n), p = MatrixXd::Identity(6 * n, 6 * n);
  for (std::size_t i = 0; i < n; ++i) {
    MatrixXd J(6, 6);
    put(J, 0, 0, inertia[i].matrix());
    const MatrixXd Ji = spd_solve(J, MatrixXd::Identity(6, 6));
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) jinv(6 * i + r, 6 * i + c) = Ji(r, c);
    if (i + 1 < n) put(p, 6 * i, 6 * (i + 1), -1.0 * kin.transport[i].mat.transpose());
  }
  return p.transpose() * jinv * p;
}
MatrixXd dense_basis(const ConstraintBasis& b) {
  const std::size_t n = b.basis.size();
  MatrixXd w(6 * n, 5 * n);
  for (std::size_t i = 0; i < n; ++i) put(w, 6 * i, 5 * i, b.basis[i]);
  return w;
}
MatrixXd dense_screws(const ChainKinematics& kin) {
  const std::size_t n = kin.screw.size();
  MatrixXd s(6 * n, n);
  for (std::size_t i = 0; i < n; ++i) put(s, 6 * i, i, kin.screw[i].stacked());
  return s;
}
MatrixXd dense_constraint_op(const CfaOperators& ops) {  // oracles.hpp:387-398
  const std::size_t n = ops.constraint_op.diag.size();
  MatrixXd a(5 * n, 5 * n);
  for (std::size_t i = 0; i < n; ++i) {
    put(a, 5 * i, 5 * i, ops.constraint_op.diag[i]);
    if (i + 1 < n) {
      put(a, 5 * i, 5 * (i + 1), ops.constraint_op.upper[i]);
      put(a, 5 * (i + 1), 5 * i, ops.constraint_op.upper[i].transpose());
    }
  }
  return a;
}
MatrixXd dense_cross_op(const CfaOperators& ops) {  // oracles.hpp:400-411
  const std::size_t n = ops.cross_diag.size();
  MatrixXd b(5 * n, n);
  for (std::size_t i = 0; i < n; ++i) {
    put(b, 5 * i, i, ops.cross_diag[i]);
    if (i + 1 < n) {
      put(b, 5 * i, i + 1, ops.cross_super[i]);
      put(b, 5 * (i + 1), i, ops.cross_sub[i]);
    }
  }
  return b;
}
MatrixXd dense_joint_op(const CfaOperators& ops) {  // oracles.hpp:413-424
  const std::size_t n = ops.joint_diag.size();
  MatrixXd c(n, n);
  for (std::size_t i = 0; i < n; ++i) {
    c(i, i) = ops.joint_diag[i];
    if (i + 1 < n) c(i, i + 1) = c(i + 1, i) = ops.joint_off[i];
  }
  return c;
}
MatrixXd as_col(const JointVector& v) {
  MatrixXd m(v.size(), 1);
  for (std::size_t i = 0; i < v.size(); ++i) m(i, 0) = v[i];
  return m;
}

oracle::RobotChain to_oracle(const RobotChain& c) {
  oracle::RobotChain o;
  o.gravity = oracle::v3(c.gravity(0), c.gravity(1), c.gravity(2));
  for (const auto& l : c.links) {
    double f[31];
    f[0] = l.mass;
    for (int k = 0; k < 3; ++k) f[1 + k] = l.com(k);
    l.inertia_rot.toRowMajor(f + 4);
    const Vec6 s = l.joint_screw.stacked();
    for (int k = 0; k < 6; ++k) f[13 + k] = s(k);
    l.home_transform.rotation.toRowMajor(f + 19);
    for (int k = 0; k < 3; ++k) f[28 + k] = l.home_transform.translation(k);
    o.links.push_back(oracle::link_from_flat(f));
  }
  return o;
}

}  // namespace

int main() {
  // kinematics and link inertias vs the oracle's restatement (model.cpp:117-155)
  {
    const Sample s = make_sample(9, 4242);
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const auto oc = to_oracle(s.chain);
    const auto ok = oracle::assemble_kinematics(oc, std::vector<double>(s.q.begin(), s.q.end()));
    const auto inertia = link_inertias(s.chain);
    const auto oin = oracle::link_inertias(oc);
    double worst = 0.0;
    for (int i = 0; i < 9; ++i) {
      for (int r = 0; r < 3; ++r) {
        worst = std::max(worst, std::fabs(kin.rel[i].translation(r) - ok.rel[i].p[r]));
        for (int c = 0; c < 3; ++c) worst = std::max(worst, std::fabs(kin.rel[i].rotation(r, c) - ok.rel[i].R(r, c)));
      }
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          if (i + 1 < 9) worst = std::max(worst, std::fabs(kin.transport[i].mat(r, c) - ok.transport[i](r, c)));
          worst = std::max(worst, std::fabs(inertia[i].matrix()(r, c) - oin[i](r, c)));
        }
    }
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) worst = std::max(worst, std::fabs(kin.base_transport.mat(r, c) - ok.base_transport(r, c)));
    check(worst < 1e-13, "assemble_kinematics / link_inertias match the oracle (" + std::to_string(worst) + ")");
    bool threw = false;
    try {
      assemble_kinematics(s.chain, JointVector::Zero(4));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "assemble_kinematics: q has length 4 but the chain has 9 joints";
    }
    check(threw, "assemble_kinematics size message");
  }

  // test_fwddyn.cpp:141-161
  {
    const Sample s = make_sample(7, 6100);
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const auto inertia = link_inertias(s.chain);
    ExecTrace tr;
    const ArticulatedBodyInertias ab = articulated_body_inertias(kin, inertia, &tr);
    bool ok = ab.inertia.size() == 7 && (ab.inertia[6] - inertia[6].matrix()).norm() == 0.0 &&
              tr.longest_sequential_link_chain == 7;
    for (int i = 0; i < 7; ++i) {
      const Vec6 screw = kin.screw[i].stacked();
      MatrixXd A(6, 6), L;
      put(A, 0, 0, ab.inertia[i]);
      ok = ok && (ab.inertia[i] - ab.inertia[i].transpose()).norm() == 0.0;
      ok = ok && std::abs(ab.joint_inertia[i] - screw.dot(ab.inertia[i] * screw)) < 1e-12 * ab.joint_inertia[i];
      ok = ok && (ab.gain[i] * ab.joint_inertia[i] - ab.inertia[i] * screw).norm() < 1e-10;
      ok = ok && cholesky(A, L);  // SPD
    }
    check(ok, "articulated inertias: tip equals the link, projections are SPD");
    const auto oab = oracle::articulated_body_inertias(oracle::assemble_kinematics(to_oracle(s.chain),
                                                                                   std::vector<double>(s.q.begin(), s.q.end())),
                                                       oracle::link_inertias(to_oracle(s.chain)));
    double worst = 0.0;
    for (int i = 0; i < 7; ++i)
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c)
          worst = std::max(worst, std::fabs(ab.inertia[i](r, c) - oab.inertia[i](r, c)) /
                                      std::max(1.0, std::fabs(oab.inertia[i](r, c))));
    check(worst < 1e-12, "articulated inertias match the oracle");
  }

  // test_fwddyn.cpp:163-185
  {
    const RobotChain chain = random_chain(6, 321);
    const ConstraintBasis basis = build_constraint_basis(chain);
    bool ok = basis.basis.size() == 6;
    for (int i = 0; i < 6; ++i) {
      const Matrix<6, 5>& w = basis.basis[i];
      const Vec6 screw = chain.links[i].joint_screw.stacked();
      ok = ok && (w.transpose() * w - Mat5::Identity()).norm() < 1e-14;
      ok = ok && (w.transpose() * screw).norm() < 1e-14;
      Mat6 square;
      for (int r = 0; r < 6; ++r) {
        for (int c = 0; c < 5; ++c) square(r, c) = w(r, c);
        square(r, 5) = screw(r);
      }
      ok = ok && (square.transpose() * square - Mat6::Identity()).norm() < 1e-13;
    }
    const ConstraintBasis again = build_constraint_basis(chain);
    for (int i = 0; i < 6; ++i) ok = ok && (basis.basis[i] - again.basis[i]).norm() == 0.0;
    check(ok, "constraint basis is the orthonormal complement of each screw, deterministically");
  }

  // test_fwddyn.cpp:187-206
  for (int n : {1, 2, 4, 9}) {
    const Sample s = make_sample(n, 5200 + static_cast<std::uint64_t>(n));
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const ConstraintBasis basis = build_constraint_basis(s.chain);
    ExecTrace tr;
    const CfaOperators ops = build_cfa_operators(s.chain, kin, basis, &tr);
    const MatrixXd core = dense_compliance_core(s.chain, kin);
    const MatrixXd w = dense_basis(basis), sc = dense_screws(kin);
    const double ga = rel_gap(dense_constraint_op(ops), w.transpose() * core * w);
    const double gb = rel_gap(dense_cross_op(ops), w.transpose() * core * sc);
    const double gc = rel_gap(dense_joint_op(ops), sc.transpose() * core * sc);
    check(ga < 1e-12 && gb < 1e-12 && gc < 1e-12 && tr.parallel_link_stages == 2,
          "CFA operators match their dense projections, n=" + std::to_string(n));
  }

  // test_fwddyn.cpp:208-232
  {
    const Sample s = make_sample(8, 5300);
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const CfaOperators ops = build_cfa_operators(s.chain, kin, build_constraint_basis(s.chain));
    const MatrixXd b = dense_cross_op(ops), c = dense_joint_op(ops);
    std::mt19937_64 e(64);
    const JointVector v = uniform(e, 8, -2.0, 2.0), f = uniform(e, 40, -2.0, 2.0);
    const std::vector<Vec5> bv = ops.apply_cross(v);
    MatrixXd bv_flat(40, 1);
    std::vector<Vec5> f_blocks(8);
    for (int i = 0; i < 8; ++i)
      for (int k = 0; k < 5; ++k) {
        bv_flat(5 * i + k, 0) = bv[i](k);
        f_blocks[i](k) = f[5 * i + k];
      }
    const bool ok = (bv_flat - b * as_col(v)).norm() < 1e-13 &&
                    (as_col(ops.apply_cross_transpose(f_blocks)) - b.transpose() * as_col(f)).norm() < 1e-13 &&
                    (as_col(ops.apply_joint(v)) - c * as_col(v)).norm() < 1e-13;
    check(ok, "tri-diagonal operator applications match the dense matrices");
  }

  // test_fwddyn.cpp:234-252
  for (int n : {1, 2, 3, 8, 16}) {
    const Sample s = make_sample(n, 7300 + static_cast<std::uint64_t>(n));
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const CfaOperators ops = build_cfa_operators(s.chain, kin, build_constraint_basis(s.chain));
    const MatrixXd a = dense_constraint_op(ops), b = dense_cross_op(ops), c = dense_joint_op(ops);
    const MatrixXd m = joint_space_inertia(s.chain, s.q);
    const MatrixXd inverse_via_schur = c - b.transpose() * spd_solve(a, b);
    check((inverse_via_schur * m - MatrixXd::Identity(n, n)).norm() < 1e-7,
          "eliminating the constraint forces inverts the joint-space inertia, n=" + std::to_string(n));
  }

  // test_fwddyn.cpp:254-261
  {
    const Sample s = make_sample(24, 8800);
    const JointVector qddot = jsiia_forward_dynamics(s.chain, s.q, s.qdot, s.tau);
    const JointVector surplus = s.tau - bias_torque(s.chain, s.q, s.qdot);
    const MatrixXd m = joint_space_inertia(s.chain, s.q);
    check((m * qddot - surplus).norm() <= 1e-9 * surplus.norm(), "the dense-inertia path meets its residual contract");
  }

  // test_fwddyn.cpp:263-283: the trace of the variant that ran
  {
    const Sample s = make_sample(13, 1300);
    const int depth = ceil_log2(13);
    ExecTrace dense, articulated, constraint;
    jsiia_forward_dynamics(s.chain, s.q, s.qdot, s.tau, &dense);
    abia_forward_dynamics(s.chain, s.q, s.qdot, s.tau, &articulated);
    cfa_forward_dynamics(s.chain, s.q, s.qdot, s.tau, &constraint);
    check(dense.longest_sequential_link_chain == 0 && dense.scan_rounds_max == depth &&
              dense.parallel_link_stages > 0,
          "JSIIA trace: no sequential walk, log-depth scans");
    check(articulated.longest_sequential_link_chain == 13 && articulated.scan_rounds_max == depth,
          "ABIA trace: the n-link articulated recursion, log-depth scans");
    check(constraint.longest_sequential_link_chain == 0 && constraint.scan_rounds_max == depth &&
              constraint.oee_rounds == depth,
          "CFA trace: no sequential walk, log-depth scans and OEE rounds");
    const JointVector plain = cfa_forward_dynamics(s.chain, s.q, s.qdot, s.tau);
    const JointVector traced = cfa_forward_dynamics(s.chain, s.q, s.qdot, s.tau, &constraint);
    check((plain - traced).norm() <= 1e-12 * std::max(1.0, plain.norm()), "traced and untraced solves agree");
  }

  // test_invdyn.cpp:50-76: the scan-backed propagations vs the sequential Newton-Euler oracle
  for (int n : {1, 2, 3, 7, 20}) {
    Sample s = make_sample(n, 100 + static_cast<std::uint64_t>(n));
    std::mt19937_64 e(1000 + n);
    const JointVector qddot = uniform(e, n, -5.0, 5.0);
    const ChainKinematics kin = assemble_kinematics(s.chain, s.q);
    const auto inertia = link_inertias(s.chain);
    std::vector<double> q(s.q.begin(), s.q.end()), qd(s.qdot.begin(), s.qdot.end()), qdd(qddot.begin(), qddot.end());
    const auto ref = oracle::newton_euler(to_oracle(s.chain), q, qd, qdd, true, nullptr);
    ScanTrace tv, ta, tf;
    const auto vel = propagate_velocities(kin, s.qdot, Twist{}, &tv);
    Twist base_acc;
    base_acc.linear = -1.0 * s.chain.gravity;
    const auto acc = propagate_accelerations(kin, vel, s.qdot, qddot, base_acc, &ta);
    const auto frc = propagate_forces(kin, vel, acc, inertia, Wrench{}, &tf);
    double worst = 0.0;
    for (int i = 0; i < n; ++i) {
      const Vec6 v = vel[i].stacked(), a = acc[i].stacked(), f = frc[i].stacked();
      double nv = 0, na = 0, nf = 0, dv = 0, da = 0, df = 0;
      for (int k = 0; k < 6; ++k) {
        nv += ref.velocity[i][k] * ref.velocity[i][k];
        na += ref.acceleration[i][k] * ref.acceleration[i][k];
        nf += ref.force[i][k] * ref.force[i][k];
        dv += (v(k) - ref.velocity[i][k]) * (v(k) - ref.velocity[i][k]);
        da += (a(k) - ref.acceleration[i][k]) * (a(k) - ref.acceleration[i][k]);
        df += (f(k) - ref.force[i][k]) * (f(k) - ref.force[i][k]);
      }
      worst = std::max(worst, std::max(std::sqrt(dv) / std::max(1.0, std::sqrt(nv)),
                                       std::max(std::sqrt(da) / std::max(1.0, std::sqrt(na)),
                                                std::sqrt(df) / std::max(1.0, std::sqrt(nf)))));
    }
    const int depth = ceil_log2(static_cast<std::size_t>(n));
    check(worst < 1e-12 && tv.rounds == depth && ta.rounds == depth && tf.rounds == depth,
          "propagate_velocities / _accelerations / _forces match sequential Newton-Euler, n=" + std::to_string(n));
    ExecTrace tr;
    const JointVector tau = inverse_dynamics_assembled(kin, inertia, s.chain.gravity, s.qdot, qddot, {}, &tr);
    const JointVector tau2 = inverse_dynamics(s.chain, s.q, s.qdot, qddot);
    check((tau - tau2).norm() <= 1e-12 * std::max(1.0, tau2.norm()) && tr.scan_rounds_max == depth,
          "inverse_dynamics_assembled == inverse_dynamics, n=" + std::to_string(n));
  }
  // test_invdyn.cpp:212-232: a moving base feeds into the link states
  {
    const Sample s = make_sample(4, 5115);
    std::mt19937_64 e(5115);
    const JointVector qddot = uniform(e, 4, -5.0, 5.0);
    std::vector<double> q(s.q.begin(), s.q.end()), qd(s.qdot.begin(), s.qdot.end()), qdd(qddot.begin(), qddot.end());
    const auto ref = oracle::newton_euler(to_oracle(s.chain), q, qd, qdd, false, nullptr);
    RobotChain tail;
    tail.gravity = s.chain.gravity;
    tail.links.assign(s.chain.links.begin() + 1, s.chain.links.end());
    const JointVector q3(s.q.begin() + 1, s.q.end()), qd3(s.qdot.begin() + 1, s.qdot.end()),
        qdd3(qddot.begin() + 1, qddot.end());
    const ChainKinematics kin = assemble_kinematics(tail, q3);
    auto tw = [](const auto& a) { return Twist(Vec3(a[0], a[1], a[2]), Vec3(a[3], a[4], a[5])); };
    const auto vel = propagate_velocities(kin, qd3, tw(ref.velocity[0]));
    const auto acc = propagate_accelerations(kin, vel, qd3, qdd3, tw(ref.acceleration[0]));
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 6; ++k)
        worst = std::max(worst, std::max(std::fabs(vel[i].stacked()(k) - ref.velocity[i + 1][k]),
                                         std::fabs(acc[i].stacked()(k) - ref.acceleration[i + 1][k])));
    check(worst < 1e-12, "a moving base feeds into the link states");
    ChainKinematics empty;
    ScanTrace et;
    check(propagate_velocities(empty, JointVector(0), Twist{}, &et).empty() && et.rounds == 0,
          "empty kinematics short-circuit cleanly");
  }

  // a device list shards the batch call; results equal the single-device call bit for bit
  {
    std::vector<FdProblem> probs;
    for (int k = 0; k < 300; ++k) {
      Sample s = make_sample(11, 900 + k);
      probs.push_back({s.chain, s.q, s.qdot, s.tau});
    }
    const auto one = batch_forward_dynamics(probs, FdAlgo::abia);
    gpu::set_devices({gpu::device(), gpu::device(), gpu::device()});  // three contexts, three slices
    const auto three = batch_forward_dynamics(probs, FdAlgo::abia);
    gpu::set_devices({});
    bool same = one.size() == three.size();
    for (std::size_t k = 0; same && k < one.size(); ++k) same = one[k].ok() && one[k].qddot == three[k].qddot;
    check(same, "batch sharded over a device list is bit-identical to one device");
  }

  // a large bucket over one device and over a device list (two slices on two
  // contexts): the same bits, per-slot errors in their slots, slots matching
  // the single-problem call
  {
    std::vector<FdProblem> probs;
    for (int k = 0; k < 40000; ++k) {
      Sample s = make_sample(4, 5000 + k);
      probs.push_back({s.chain, s.q, s.qdot, s.tau});
    }
    probs[3].tau = JointVector::Zero(3);                        // rejected on the host (sizes)
    probs[17001].q[1] = std::numeric_limits<double>::quiet_NaN();  // rejected by the kernel, second slice
    const auto one = batch_forward_dynamics(probs, FdAlgo::abia);
    gpu::set_devices({gpu::device(), gpu::device()});
    const auto two = batch_forward_dynamics(probs, FdAlgo::abia);
    gpu::set_devices({});
    bool same = one.size() == probs.size() && two.size() == probs.size();
    for (std::size_t k = 0; same && k < one.size(); ++k)
      same = one[k].ok() == two[k].ok() && one[k].qddot == two[k].qddot && one[k].error == two[k].error;
    check(same, "large batch: a device list gives the same bits");
    check(!one[3].ok() && one[3].error.find("forward dynamics") != std::string::npos && !one[17001].ok() &&
              !one[17001].error.empty() && one[17000].ok() && one[17002].ok(),
          "large batch: per-slot errors stay in their slots");
    double worst = 0.0;
    for (std::size_t k = 0; k < probs.size(); k += 997) {
      if (k == 3 || k == 17001) continue;
      const JointVector ref = forward_dynamics(probs[k].chain, probs[k].q, probs[k].qdot, probs[k].tau, FdAlgo::abia);
      worst = std::max(worst, (one[k].qddot - ref).norm() / std::max(1.0, ref.norm()));
    }
    check(worst < 1e-12, "large batch: slots match the single-problem call");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
