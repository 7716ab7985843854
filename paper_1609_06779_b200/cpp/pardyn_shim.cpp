// Implementation of the pardyn drop-in C++ API (include/pardyn/pardyn.hpp)
// over the C-ABI. Host side only: size checks, packing into the C-ABI
// layouts, bucketing batches by link count, and rebuilding the reference's
// exceptions / error strings from per-slot codes. No arithmetic of the
// dynamics happens here -- every solve is a pd_forward_dynamics call.
#include "../../include/pardyn/pardyn.hpp"

#include <map>
#include <memory>
#include <mutex>

#include "../../include/pardyn_c.h"

namespace pardyn {

namespace {

thread_local int t_device = 0;

// One pd_ctx per (thread, device): contexts are single-threaded objects.
struct CtxHolder {
  std::map<int, pd_ctx*> by_dev;
  ~CtxHolder() {
    for (auto& kv : by_dev) pd_destroy(kv.second);
  }
};
thread_local CtxHolder t_ctx;

pd_ctx* ctx() {
  auto it = t_ctx.by_dev.find(t_device);
  if (it != t_ctx.by_dev.end()) return it->second;
  pd_ctx* c = nullptr;
  const pd_status st = pd_create(&c, t_device);
  if (st != PD_OK)
    throw DeviceError(std::string("pardyn: cannot open CUDA device ") + std::to_string(t_device) + ": " +
                      pd_status_string(st));
  t_ctx.by_dev[t_device] = c;
  return c;
}

void check_call(pd_ctx* c, pd_status st) {
  if (st == PD_OK) return;
  const std::string msg = pd_last_error(c);
  if (st == PD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw DeviceError(std::string(pd_status_string(st)) + ": " + msg);
}

void append_link(const LinkSpec& l, std::vector<double>& out) {
  out.push_back(l.mass);
  out.insert(out.end(), l.com.begin(), l.com.end());
  out.insert(out.end(), l.inertia_rot.begin(), l.inertia_rot.end());
  out.insert(out.end(), l.joint_screw.begin(), l.joint_screw.end());
  out.insert(out.end(), l.home_rotation.begin(), l.home_rotation.end());
  out.insert(out.end(), l.home_translation.begin(), l.home_translation.end());
}

// forward_dynamics.cpp:19-31
void check_sizes(const RobotChain& chain, const JointVector& q, const JointVector& qdot, const JointVector& tau) {
  const std::size_t n = chain.links.size();
  if (n == 0) throw std::invalid_argument("forward dynamics: chain has no links");
  if (q.size() != n || qdot.size() != n || tau.size() != n)
    throw std::invalid_argument("forward dynamics: q, qdot and tau must each have one entry per joint (chain has " +
                                std::to_string(n) + ")");
}

std::string slot_message(int code, int round, int index, int n) {
  char buf[512];
  pd_slot_message(code, round, index, n, buf, sizeof(buf));
  return buf;
}

[[noreturn]] void throw_slot(int code, int round, int index, int n) {
  const std::string m = slot_message(code, round, index, n);
  if (code == PD_SLOT_BAD_MODEL || code == PD_SLOT_BAD_SIZE) throw std::invalid_argument(m);
  if (code == PD_SLOT_OEE_SINGULAR_PIVOT || code == PD_SLOT_OEE_SINGULAR_FINAL) throw SingularBlockError(round, index, m);
  throw DynamicsError(m);
}

void fill_trace(ExecTrace* t, FdAlgo algo, int n) {
  if (!t) return;
  const int L = ceil_log2(static_cast<std::size_t>(n));
  t->scan_rounds_max = std::max(t->scan_rounds_max, L);
  switch (algo) {
    case FdAlgo::jsiia:
      t->parallel_link_stages += 6;
      break;
    case FdAlgo::abia:
      t->parallel_link_stages += 6;
      t->longest_sequential_link_chain = std::max(t->longest_sequential_link_chain, n);
      break;
    case FdAlgo::cfa:
      t->parallel_link_stages += 9;
      t->oee_rounds = L;
      break;
  }
}

pd_algo to_c(FdAlgo a) {
  switch (a) {
    case FdAlgo::jsiia: return PD_JSIIA;
    case FdAlgo::abia: return PD_ABIA;
    case FdAlgo::cfa: return PD_CFA;
  }
  throw std::invalid_argument("forward_dynamics: unknown algorithm");
}

}  // namespace

namespace gpu {
void set_device(int device) { t_device = device; }
int device() { return t_device; }
}  // namespace gpu

RobotChain random_chain(int n, std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("random_chain: n must be at least 1");
  std::vector<double> rec(static_cast<std::size_t>(n) * PD_LINK_FIELDS);
  pd_random_chain(n, seed, rec.data());
  RobotChain c;
  c.links.resize(n);
  for (int i = 0; i < n; ++i) {
    const double* f = rec.data() + static_cast<std::size_t>(i) * PD_LINK_FIELDS;
    LinkSpec& l = c.links[i];
    l.mass = f[0];
    for (int k = 0; k < 3; ++k) l.com[k] = f[1 + k];
    for (int k = 0; k < 9; ++k) l.inertia_rot[k] = f[4 + k];
    for (int k = 0; k < 6; ++k) l.joint_screw[k] = f[13 + k];
    for (int k = 0; k < 9; ++k) l.home_rotation[k] = f[19 + k];
    for (int k = 0; k < 3; ++k) l.home_translation[k] = f[28 + k];
  }
  return c;
}

JointVector forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& tau, FdAlgo algo, ExecTrace* trace) {
  const pd_algo a = to_c(algo);
  check_sizes(chain, q, qdot, tau);
  const int n = chain.size();
  std::vector<double> links;
  links.reserve(static_cast<std::size_t>(n) * PD_LINK_FIELDS);
  for (const LinkSpec& l : chain.links) append_link(l, links);
  pd_ctx* c = ctx();
  check_call(c, pd_set_models(c, 1, n, links.data(), chain.gravity.data(), nullptr, nullptr));
  JointVector out(n);
  int32_t st = 0, rd = 0, ix = 0;
  check_call(c, pd_forward_dynamics(c, a, 1, q.data(), qdot.data(), tau.data(), out.data(), &st, &rd, &ix));
  if (st != PD_SLOT_OK) throw_slot(st, rd, ix, n);
  fill_trace(trace, algo, n);
  return out;
}

JointVector jsiia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                   const JointVector& tau, ExecTrace* trace) {
  return forward_dynamics(chain, q, qdot, tau, FdAlgo::jsiia, trace);
}
JointVector abia_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                  const JointVector& tau, ExecTrace* trace) {
  return forward_dynamics(chain, q, qdot, tau, FdAlgo::abia, trace);
}
JointVector cfa_forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                                 const JointVector& tau, ExecTrace* trace) {
  return forward_dynamics(chain, q, qdot, tau, FdAlgo::cfa, trace);
}

// forward_dynamics.cpp:466-481: never throws per problem. Problems are
// bucketed by link count; each bucket is one pd_forward_dynamics call.
std::vector<FdResult> batch_forward_dynamics(std::span<const FdProblem> problems, FdAlgo algo) {
  const pd_algo a = to_c(algo);
  std::vector<FdResult> out(problems.size());
  std::map<int, std::vector<std::size_t>> buckets;
  for (std::size_t k = 0; k < problems.size(); ++k) {
    const FdProblem& p = problems[k];
    try {
      check_sizes(p.chain, p.q, p.qdot, p.tau);
      buckets[p.chain.size()].push_back(k);
    } catch (const std::exception& e) {
      out[k].error = e.what();
    }
  }
  if (buckets.empty()) return out;
  pd_ctx* c = ctx();
  for (const auto& [n, idx] : buckets) {
    const std::size_t B = idx.size();
    std::vector<double> links, grav, q, qd, tau;
    links.reserve(B * n * PD_LINK_FIELDS);
    q.reserve(B * n);
    qd.reserve(B * n);
    tau.reserve(B * n);
    for (std::size_t k : idx) {
      const FdProblem& p = problems[k];
      for (const LinkSpec& l : p.chain.links) append_link(l, links);
      grav.insert(grav.end(), p.chain.gravity.begin(), p.chain.gravity.end());
      q.insert(q.end(), p.q.data(), p.q.data() + n);
      qd.insert(qd.end(), p.qdot.data(), p.qdot.data() + n);
      tau.insert(tau.end(), p.tau.data(), p.tau.data() + n);
    }
    check_call(c, pd_set_models(c, static_cast<int64_t>(B), n, links.data(), grav.data(), nullptr, nullptr));
    std::vector<double> qdd(B * n);
    std::vector<int32_t> st(B), rd(B), ix(B);
    check_call(c, pd_forward_dynamics(c, a, static_cast<int64_t>(B), q.data(), qd.data(), tau.data(), qdd.data(),
                                      st.data(), rd.data(), ix.data()));
    for (std::size_t j = 0; j < B; ++j) {
      FdResult& r = out[idx[j]];
      if (st[j] == PD_SLOT_OK) {
        r.qddot = JointVector(n);
        for (int i = 0; i < n; ++i) r.qddot[i] = qdd[j * n + i];
      } else {
        r.error = slot_message(st[j], rd[j], ix[j], n);
      }
    }
  }
  return out;
}

namespace {

void id_sizes(const RobotChain& chain, std::initializer_list<std::pair<const char*, const JointVector*>> args) {
  const std::size_t n = chain.links.size();
  for (const auto& a : args)  // inverse_dynamics.cpp:10-17
    if (a.second->size() != n)
      throw std::invalid_argument(std::string(a.first) + " has length " + std::to_string(a.second->size()) +
                                  " but the chain has " + std::to_string(n) + " joints");
}

// One shared model on this thread's context; a bad link throws as
// link_inertias -> spatial_inertia_from does (spatial.cpp:72-87).
pd_ctx* one_model(const RobotChain& chain) {
  const std::size_t n = chain.links.size();
  std::vector<double> links;
  for (const LinkSpec& l : chain.links) append_link(l, links);
  pd_ctx* c = ctx();
  int32_t ms = 0, mr = 0;
  check_call(c, pd_set_models(c, 1, static_cast<int32_t>(n), links.data(), chain.gravity.data(), &ms, &mr));
  if (ms != PD_SLOT_OK) throw std::invalid_argument(slot_message(ms, 0, mr, static_cast<int>(n)));
  return c;
}

pd_id_options to_c(const IdOptions& o) {
  pd_id_options r{};
  const Vec6 bv = o.base_velocity.stacked(), ba = o.base_acceleration.stacked(), tw = o.tip_wrench.stacked();
  for (int k = 0; k < 6; ++k) {
    r.base_velocity[k] = bv[k];
    r.base_acceleration[k] = ba[k];
    r.tip_wrench[k] = tw[k];
  }
  r.apply_gravity = o.apply_gravity ? 1 : 0;
  return r;
}

}  // namespace

JointVector inverse_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& qddot, const IdOptions& opts) {
  id_sizes(chain, {{"q", &q}, {"qdot", &qdot}, {"qddot", &qddot}});
  const std::size_t n = chain.links.size();
  if (n == 0) return JointVector();
  pd_ctx* c = one_model(chain);
  JointVector tau(n);
  const pd_id_options o = to_c(opts);
  check_call(c, pd_inverse_dynamics_opts(c, 1, q.data(), qdot.data(), qddot.data(), &o, tau.data()));
  return tau;
}

JointVector bias_torque(const RobotChain& chain, const JointVector& q, const JointVector& qdot) {
  id_sizes(chain, {{"q", &q}, {"qdot", &qdot}});
  const std::size_t n = chain.links.size();
  if (n == 0) return JointVector();
  pd_ctx* c = one_model(chain);
  JointVector tau(n);
  check_call(c, pd_bias_torque(c, 1, q.data(), qdot.data(), tau.data()));
  return tau;
}

LinkStates link_states(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                       const JointVector& qddot, const IdOptions& opts) {
  id_sizes(chain, {{"q", &q}, {"qdot", &qdot}, {"qddot", &qddot}});
  const std::size_t n = chain.links.size();
  LinkStates out;
  if (n == 0) return out;
  pd_ctx* c = one_model(chain);
  std::vector<double> v(6 * n), a(6 * n), f(6 * n);
  const pd_id_options o = to_c(opts);
  check_call(c, pd_link_states(c, 1, q.data(), qdot.data(), qddot.data(), &o, v.data(), a.data(), f.data()));
  auto six = [](const std::vector<double>& x, std::size_t i) {
    Vec6 r;
    for (int k = 0; k < 6; ++k) r[k] = x[6 * i + k];
    return r;
  };
  for (std::size_t i = 0; i < n; ++i) {
    out.velocity.push_back(Twist::from_stacked(six(v, i)));
    out.acceleration.push_back(Twist::from_stacked(six(a, i)));
    out.force.push_back(Wrench::from_stacked(six(f, i)));
  }
  return out;
}

MatrixXd joint_space_inertia(const RobotChain& chain, const JointVector& q) {
  const std::size_t n = chain.links.size();
  if (q.size() != n) throw std::invalid_argument("joint_space_inertia: q must have one entry per joint");
  MatrixXd M(n, n);
  if (n == 0) return M;
  pd_ctx* c = one_model(chain);
  check_call(c, pd_joint_space_inertia(c, 1, q.data(), M.data()));
  return M;
}

namespace {

std::vector<std::array<double, 6>> bidiag(const BlockBiDiagSystem<6>& sys, bool upper, ScanTrace* trace) {
  const std::size_t n = sys.rhs.size();
  if (sys.coupling.size() + 1 != n && !(n == 0 && sys.coupling.empty()))
    throw std::invalid_argument("block bi-diagonal solve: need n - 1 coupling blocks for n right-hand sides");
  if (trace) trace->rounds = ceil_log2(n);  // the scan's designed depth (scan.hpp:32-65)
  std::vector<std::array<double, 6>> x(n);
  if (n == 0) return x;
  std::vector<double> c, r, xo(6 * n);
  for (const auto& b : sys.coupling) c.insert(c.end(), b.begin(), b.end());
  for (const auto& b : sys.rhs) r.insert(r.end(), b.begin(), b.end());
  pd_ctx* cx = ctx();
  check_call(cx, pd_block_bidiag_solve6(cx, 1, static_cast<int32_t>(n), upper ? 1 : 0, c.empty() ? nullptr : c.data(),
                                       r.data(), xo.data()));
  for (std::size_t k = 0; k < n; ++k)
    for (int e = 0; e < 6; ++e) x[k][e] = xo[6 * k + e];
  return x;
}

}  // namespace

std::vector<std::array<double, 6>> solve_lower_bidiag(const BlockBiDiagSystem<6>& sys, ScanTrace* trace) {
  return bidiag(sys, false, trace);
}

std::vector<std::array<double, 6>> solve_upper_bidiag(const BlockBiDiagSystem<6>& sys, ScanTrace* trace) {
  return bidiag(sys, true, trace);
}

std::vector<std::array<double, 5>> oee_solve(const SymBlockTriDiagSystem<5>& sys,
                                             const std::vector<std::array<double, 5>>& rhs, OeeTrace* trace) {
  const std::size_t n = sys.diag.size();
  if (rhs.size() != n || (n > 0 && sys.upper.size() + 1 != n))
    throw std::invalid_argument("odd-even elimination: inconsistent block counts");
  if (trace) trace->rounds = ceil_log2(n);
  std::vector<std::array<double, 5>> x(n);
  if (n == 0) return x;
  std::vector<double> d, u, r, xo(5 * n);
  for (const auto& b : sys.diag) d.insert(d.end(), b.begin(), b.end());
  for (const auto& b : sys.upper) u.insert(u.end(), b.begin(), b.end());
  for (const auto& b : rhs) r.insert(r.end(), b.begin(), b.end());
  pd_ctx* cx = ctx();
  int32_t st = 0, rd = 0, ix = 0;
  check_call(cx, pd_block_tridiag_solve5(cx, 1, static_cast<int32_t>(n), d.data(), u.empty() ? nullptr : u.data(),
                                         r.data(), xo.data(), &st, &rd, &ix));
  if (st != PD_SLOT_OK) throw SingularBlockError(rd, ix, slot_message(st, rd, ix, static_cast<int>(n)));
  for (std::size_t k = 0; k < n; ++k)
    for (int e = 0; e < 5; ++e) x[k][e] = xo[5 * k + e];
  return x;
}

}  // namespace pardyn
