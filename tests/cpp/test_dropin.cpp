// The reference's test_fwddyn.cpp cases, written against the pardyn drop-in
// C++ API (include/pardyn/pardyn.hpp -> C-ABI -> sm_100a kernels), checked
// against the CPU oracle (oracle/oracle.hpp, test infrastructure only).
// Prints one PASS/FAIL line per case; exit status = number of failures.
#include <pardyn/pardyn.hpp>

#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "../../oracle/oracle.hpp"

using pardyn::FdAlgo;
using pardyn::JointVector;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

double rel_gap(const JointVector& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num) / std::max(1.0, std::sqrt(den));
}

oracle::RobotChain to_oracle(const pardyn::RobotChain& c) {
  oracle::RobotChain o;
  o.gravity = oracle::v3(c.gravity[0], c.gravity[1], c.gravity[2]);
  for (const auto& l : c.links) {
    double f[31];
    f[0] = l.mass;
    for (int k = 0; k < 3; ++k) f[1 + k] = l.com(k);
    l.inertia_rot.toRowMajor(f + 4);
    const pardyn::Vec6 s = l.joint_screw.stacked();
    for (int k = 0; k < 6; ++k) f[13 + k] = s(k);
    l.home_transform.rotation.toRowMajor(f + 19);
    for (int k = 0; k < 3; ++k) f[28 + k] = l.home_transform.translation(k);
    o.links.push_back(oracle::link_from_flat(f));
  }
  return o;
}

JointVector uniform(std::mt19937_64& e, int n, double lo, double hi) {
  JointVector v(n);
  for (int i = 0; i < n; ++i) v[i] = lo + (hi - lo) * (static_cast<double>(e() >> 11) * 0x1.0p-53);
  return v;
}

std::vector<double> as_vec(const JointVector& v) { return std::vector<double>(v.data(), v.data() + v.size()); }

}  // namespace

int main() {
  // all three algorithms vs the same algorithm's oracle (north star: 1e-9)
  for (int n : {1, 2, 5, 10, 30}) {
    for (std::uint64_t trial = 0; trial < 3; ++trial) {
      const pardyn::RobotChain chain = pardyn::random_chain(n, 400 + 10 * n + trial);
      std::mt19937_64 e((400 + 10 * n + trial) ^ 0xF00D);
      const JointVector q = uniform(e, n, -3, 3), qd = uniform(e, n, -2, 2), tau = uniform(e, n, -10, 10);
      const oracle::RobotChain oc = to_oracle(chain);
      for (FdAlgo a : {FdAlgo::jsiia, FdAlgo::abia, FdAlgo::cfa}) {
        const JointVector got = pardyn::forward_dynamics(chain, q, qd, tau, a);
        const auto want = oracle::forward_dynamics(oc, as_vec(q), as_vec(qd), as_vec(tau),
                                                   static_cast<oracle::FdAlgo>(static_cast<int>(a)));
        check(rel_gap(got, want) < 1e-9, "algo " + std::to_string(static_cast<int>(a)) + " n=" + std::to_string(n) +
                                             " trial " + std::to_string(trial) + " vs oracle");
      }
    }
  }

  // closed-form pendulum (test_fwddyn.cpp:105-122)
  {
    pardyn::RobotChain c;
    c.gravity = pardyn::Vec3(0.0, -9.81, 0.0);
    pardyn::LinkSpec l;
    l.mass = 1.3;
    l.com = pardyn::Vec3(0.45, 0, 0);
    l.inertia_rot = pardyn::Mat3::FromRowMajor({0.11, 0, 0, 0, 0.13, 0, 0, 0, 0.07});
    c.links.push_back(l);
    std::mt19937_64 e(111);
    bool ok = true;
    for (int t = 0; t < 20; ++t) {
      const JointVector q = uniform(e, 1, -6, 6), qd = uniform(e, 1, -4, 4), tau = uniform(e, 1, -8, 8);
      const double want = (tau[0] - 1.3 * 9.81 * 0.45 * std::cos(q[0])) / (0.07 + 1.3 * 0.45 * 0.45);
      for (FdAlgo a : {FdAlgo::jsiia, FdAlgo::abia, FdAlgo::cfa}) {
        const double got = pardyn::forward_dynamics(c, q, qd, tau, a)[0];
        ok = ok && std::abs(got - want) < 1e-8 * std::max(1.0, std::abs(want));
      }
    }
    check(ok, "closed-form pendulum, every algorithm");
  }

  // dispatcher reaches the algorithm it names (test_fwddyn.cpp:285-296)
  {
    const pardyn::RobotChain chain = pardyn::random_chain(4, 9100);
    const JointVector q{0.1, -0.2, 0.3, 0.4}, qd{0.5, 0.1, -0.3, 0.2}, tau{1, -1, 2, 0.5};
    check(pardyn::forward_dynamics(chain, q, qd, tau, FdAlgo::cfa) ==
              pardyn::cfa_forward_dynamics(chain, q, qd, tau),
          "dispatcher == cfa_forward_dynamics");
  }

  // batch: slot identity, per-slot errors, empty batch (test_fwddyn.cpp:298-341)
  {
    std::vector<pardyn::FdProblem> probs;
    for (int n = 1; n <= 8; ++n) {
      std::mt19937_64 e(600 + n);
      probs.push_back({pardyn::random_chain(n, 600 + n), uniform(e, n, -3, 3), uniform(e, n, -2, 2),
                       uniform(e, n, -10, 10)});
    }
    probs[2].tau = JointVector::Zero(1);
    const auto res = pardyn::batch_forward_dynamics(probs, FdAlgo::abia);
    bool ok = !res[2].ok() && res[2].error.find("forward dynamics") != std::string::npos;
    for (std::size_t i = 0; i < probs.size(); ++i) {
      if (i == 2) continue;
      const auto& p = probs[i];
      ok = ok && res[i].ok() && res[i].qddot == pardyn::forward_dynamics(p.chain, p.q, p.qdot, p.tau, FdAlgo::abia);
    }
    check(ok, "batch slot identity and error isolation");
    check(pardyn::batch_forward_dynamics({}, FdAlgo::cfa).empty(), "empty batch");
  }

  // validation and error classes (test_fwddyn.cpp:343-361, spatial.cpp:72-87)
  {
    const pardyn::RobotChain chain = pardyn::random_chain(3, 77);
    const JointVector good = JointVector::Zero(3), bad = JointVector::Zero(2);
    bool threw = false;
    try {
      pardyn::forward_dynamics(chain, bad, good, good, FdAlgo::jsiia);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "size mismatch -> std::invalid_argument");
    pardyn::RobotChain neg = chain;
    neg.links[1].mass = -2.0;
    std::string msg;
    try {
      pardyn::forward_dynamics(neg, good, good, good, FdAlgo::abia);
    } catch (const std::invalid_argument& e) {
      msg = e.what();
    }
    check(msg == "spatial inertia: mass must be positive", "negative mass -> spatial inertia message");
  }

  // inverse dynamics and bias torque vs the oracle
  {
    const pardyn::RobotChain chain = pardyn::random_chain(9, 2222);
    std::mt19937_64 e(2222);
    const JointVector q = uniform(e, 9, -3, 3), qd = uniform(e, 9, -2, 2), qdd = uniform(e, 9, -5, 5);
    const auto want = oracle::inverse_dynamics(to_oracle(chain), as_vec(q), as_vec(qd), as_vec(qdd));
    check(rel_gap(pardyn::inverse_dynamics(chain, q, qd, qdd), want) < 1e-12, "inverse dynamics vs oracle");
    check(pardyn::bias_torque(chain, q, qd) == pardyn::inverse_dynamics(chain, q, qd, JointVector::Zero(9)),
          "bias torque = ID(qdd = 0)");
  }
  // IdOptions, link states, joint-space inertia vs the oracle
  {
    const pardyn::RobotChain chain = pardyn::random_chain(11, 3333);
    std::mt19937_64 e(3333);
    const JointVector q = uniform(e, 11, -3, 3), qd = uniform(e, 11, -2, 2), qdd = uniform(e, 11, -5, 5);
    const JointVector a = uniform(e, 6, -1, 1), b = uniform(e, 6, -2, 2), w = uniform(e, 6, -3, 3);
    pardyn::IdOptions opts;
    opts.base_velocity = pardyn::Twist::from_stacked(pardyn::Vec6::FromRowMajor(a.data()));
    opts.base_acceleration = pardyn::Twist::from_stacked(pardyn::Vec6::FromRowMajor(b.data()));
    opts.tip_wrench = pardyn::Wrench::from_stacked(pardyn::Vec6::FromRowMajor(w.data()));
    opts.apply_gravity = false;
    oracle::IdOptions oo;
    for (int k = 0; k < 6; ++k) {
      oo.base_velocity[k] = a[k];
      oo.base_acceleration[k] = b[k];
      oo.tip_wrench[k] = w[k];
    }
    oo.apply_gravity = false;
    const oracle::RobotChain oc = to_oracle(chain);
    const auto want = oracle::inverse_dynamics(oc, as_vec(q), as_vec(qd), as_vec(qdd), oo);
    check(rel_gap(pardyn::inverse_dynamics(chain, q, qd, qdd, opts), want) < 1e-12, "ID with IdOptions vs oracle");
    const pardyn::LinkStates st = pardyn::link_states(chain, q, qd, qdd, opts);
    const oracle::LinkStates ost = oracle::link_states(oc, as_vec(q), as_vec(qd), as_vec(qdd), oo);
    double worst = 0.0;
    for (int i = 0; i < 11; ++i) {
      const pardyn::Vec6 v = st.velocity[i].stacked(), ac = st.acceleration[i].stacked(), f = st.force[i].stacked();
      for (int k = 0; k < 6; ++k) {
        worst = std::max(worst, std::fabs(v[k] - ost.velocity[i][k]) / std::max(1.0, std::fabs(ost.velocity[i][k])));
        worst = std::max(worst,
                         std::fabs(ac[k] - ost.acceleration[i][k]) / std::max(1.0, std::fabs(ost.acceleration[i][k])));
        worst = std::max(worst, std::fabs(f[k] - ost.force[i][k]) / std::max(1.0, std::fabs(ost.force[i][k])));
      }
    }
    check(worst < 1e-11, "link states vs oracle");
    const pardyn::MatrixXd M = pardyn::joint_space_inertia(chain, q);
    const oracle::MatX OM = oracle::joint_space_inertia(oc, as_vec(q));
    double mg = 0.0, sym = 0.0;
    for (int r = 0; r < 11; ++r)
      for (int c = 0; c < 11; ++c) {
        mg = std::max(mg, std::fabs(M(r, c) - OM(r, c)) / std::max(1.0, std::fabs(OM(r, c))));
        sym = std::max(sym, std::fabs(M(r, c) - M(c, r)));
      }
    check(mg < 1e-12 && sym == 0.0, "joint-space inertia vs oracle, exactly symmetric");
  }
  // the building blocks: scan and OEE (test_oee.cpp:106-126)
  {
    pardyn::BlockBiDiagSystem<6> sys;
    const pardyn::Mat6 two = 2.0 * pardyn::Mat6::Identity();
    sys.coupling = {two, two};
    sys.rhs = {pardyn::Vec6::Constant(1.0), pardyn::Vec6(), pardyn::Vec6()};
    pardyn::ScanTrace tr;
    const auto x = pardyn::solve_lower_bidiag(sys, &tr);
    check(x[0](0) == 1.0 && x[1](0) == 2.0 && x[2](5) == 4.0 && tr.rounds == 2, "scan known answer [1, 2, 4]");
    sys.orientation = pardyn::BiDiagOrientation::upper;
    sys.rhs = {pardyn::Vec6(), pardyn::Vec6(), pardyn::Vec6::Constant(1.0)};
    const auto xu = pardyn::solve_upper_bidiag(sys);
    check(xu[0](0) == 4.0 && xu[2](0) == 1.0, "upper scan known answer [4, 2, 1]");
    pardyn::SymBlockTriDiagSystem<5> t3;
    const pardyn::Mat5 eye = pardyn::Mat5::Identity(), tenth = 0.1 * eye;
    t3.diag = {eye, pardyn::Mat5(), eye};
    t3.upper = {tenth, tenth};
    const std::vector<pardyn::Vec5> ones(3, pardyn::Vec5::Constant(1.0));
    int rd = -1, ix = -1;
    try {
      pardyn::oee_solve(t3, ones);
    } catch (const pardyn::SingularBlockError& e) {
      rd = e.round();
      ix = e.index();
    }
    check(rd == 1 && ix == 1, "OEE singular pivot reports (round 1, block 1)");
    t3.diag = {eye, eye, eye};
    pardyn::OeeTrace ot;
    const auto xs = pardyn::oee_solve(t3, ones, &ot);
    double res = 0.0;  // (I + 0.1 (shift + shift^T)) x = 1
    for (int k = 0; k < 3; ++k)
      for (int e = 0; e < 5; ++e) {
        double v = xs[k](e);
        if (k > 0) v += 0.1 * xs[k - 1](e);
        if (k < 2) v += 0.1 * xs[k + 1](e);
        res = std::max(res, std::fabs(v - 1.0));
      }
    check(res < 1e-14 && ot.rounds == 2, "OEE solves a 3-block system");
    // other block sizes, as the reference's templates take them (test_oee.cpp:106-126, :45-58)
    pardyn::SymBlockTriDiagSystem<2> t2;
    t2.diag = {pardyn::Matrix<2, 2>::Identity(), pardyn::Matrix<2, 2>(), pardyn::Matrix<2, 2>::Identity()};
    t2.upper = {0.1 * pardyn::Matrix<2, 2>::Identity(), 0.1 * pardyn::Matrix<2, 2>::Identity()};
    rd = ix = -1;
    try {
      pardyn::oee_solve<2, 1>(t2, std::vector<pardyn::Matrix<2, 1>>(3, pardyn::Matrix<2, 1>::Constant(1.0)));
    } catch (const pardyn::SingularBlockError& e) {
      rd = e.round();
      ix = e.index();
    }
    check(rd == 1 && ix == 1, "OEE<2,1> singular pivot reports (round 1, block 1)");
    t3.diag = {eye, eye, eye};
    std::vector<pardyn::Matrix<5, 3>> rhs3(3, pardyn::Matrix<5, 3>::Constant(1.0));
    rhs3[1](2, 1) = -2.0;
    const auto x3 = pardyn::oee_solve<5, 3>(t3, rhs3);
    double res3 = 0.0;
    for (int k = 0; k < 3; ++k)
      for (int e = 0; e < 5; ++e)
        for (int c = 0; c < 3; ++c) {
          double v = x3[k](e, c);
          if (k > 0) v += 0.1 * x3[k - 1](e, c);
          if (k < 2) v += 0.1 * x3[k + 1](e, c);
          res3 = std::max(res3, std::fabs(v - rhs3[k](e, c)));
        }
    check(res3 < 1e-14, "OEE<5,3> carries three right-hand-side columns");
    pardyn::BlockBiDiagSystem<2> s2;
    s2.coupling = {pardyn::Matrix<2, 2>::FromRowMajor({0.0, 1.0, -1.0, 0.0})};
    s2.rhs = {pardyn::Matrix<2, 1>::FromRowMajor({1.0, 2.0}), pardyn::Matrix<2, 1>::FromRowMajor({0.5, 0.5})};
    const auto x2 = pardyn::solve_lower_bidiag(s2);
    check(x2[1](0) == 2.5 && x2[1](1) == -0.5, "scan<2>: x1 = C x0 + r1");
    // AffineElement composition order (scan.hpp:66-97)
    pardyn::AffineElement<2> e1, e2;
    e1.offset = s2.rhs[0];
    e2.coeff = s2.coupling[0];
    e2.offset = s2.rhs[1];
    const auto e12 = pardyn::AffineElement<2>::compose(e1, e2);
    check(e12.offset(0) == 2.5 && e12.offset(1) == -0.5, "AffineElement::compose(first, second)");
    // elimination rounds on a state (test_oee.cpp:60-94): pivots stay
    // symmetric round to round, couplings shrink by rows, distance doubles
    for (int n : {5, 16, 33, 100}) {
      pardyn::OeeState<5, 1> st;
      for (int k = 0; k < n; ++k) {
        pardyn::Mat5 a;
        for (int r = 0; r < 5; ++r)
          for (int c = 0; c < 5; ++c) a(r, c) = std::sin(1.3 * (k + 1) * (r + 1) + 0.7 * c);
        st.diag.push_back(a * a.transpose() + 4.0 * pardyn::Mat5::Identity());
        st.rhs.push_back(pardyn::Vec5::Constant(1.0 + 0.01 * k));
        if (k + 1 < n) st.coupling.push_back(0.2 * a);
      }
      const int rounds = pardyn::ceil_log2(static_cast<std::size_t>(n));
      double asym = 0.0;
      for (int j = 0; j < rounds; ++j) {
        pardyn::oee_eliminate_round(st);
        for (const auto& d : st.diag)
          for (int r = 0; r < 5; ++r)
            for (int c = 0; c < 5; ++c) asym = std::max(asym, std::fabs(d(r, c) - d(c, r)));
        check(st.distance == (2 << j) && st.coupling.size() == static_cast<std::size_t>(std::max(0, n - (2 << j))),
              "elimination round: distance doubles, couplings shrink by rows");
      }
      check(asym < 1e-10 && st.round == rounds && st.coupling.empty(), "pivots stay symmetric; all couplings gone");
      // the eliminated system decouples: each row solves alone, and agrees with oee_solve
      pardyn::SymBlockTriDiagSystem<5> sys;
      pardyn::OeeState<5, 1> st0;
      for (int k = 0; k < n; ++k) {
        pardyn::Mat5 a;
        for (int r = 0; r < 5; ++r)
          for (int c = 0; c < 5; ++c) a(r, c) = std::sin(1.3 * (k + 1) * (r + 1) + 0.7 * c);
        sys.diag.push_back(a * a.transpose() + 4.0 * pardyn::Mat5::Identity());
        st0.rhs.push_back(pardyn::Vec5::Constant(1.0 + 0.01 * k));
        if (k + 1 < n) sys.upper.push_back(0.2 * a);
      }
      const auto xs = pardyn::oee_solve(sys, st0.rhs);
      double gap = 0.0;
      for (int k = 0; k < n; ++k) {
        const pardyn::Vec5 xk = pardyn::coefficient_solve<5, 1>(st.diag[k], st.rhs[k], st.round, k);
        for (int e = 0; e < 5; ++e) gap = std::max(gap, std::fabs(xk(e) - xs[k](e)));
      }
      check(gap < 1e-12, "rounds + coefficient_solve reproduce oee_solve");
    }
    int cs_round = -1, cs_index = -1;
    try {
      pardyn::coefficient_solve<2, 1>(pardyn::Matrix<2, 2>(), pardyn::Matrix<2, 1>::Constant(1.0), 3, 7);
    } catch (const pardyn::SingularBlockError& e) {
      cs_round = e.round();
      cs_index = e.index();
    }
    check(cs_round == 3 && cs_index == 7, "coefficient_solve: singular pivot names (round, block)");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
