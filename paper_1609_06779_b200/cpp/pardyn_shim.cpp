// Implementation of the pardyn drop-in C++ API (include/pardyn/pardyn.hpp)
// over the C-ABI. Host side: size checks, packing into the C-ABI layouts,
// bucketing batches by link count, sharding buckets across devices, and
// rebuilding the reference's exceptions / error strings from per-slot codes.
// The dynamics, the chain operators and the building-block solves all run on
// the device; the only host arithmetic is the 3x3 / 6x6 value algebra of
// spatial.hpp (skew, adjoint_of, screw_exp, spatial_inertia_from).
#include "../../include/pardyn/pardyn.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/pardyn_c.h"
#include "records.hpp"

namespace pardyn {

namespace {

thread_local int t_device = 0;
thread_local std::vector<int> t_devices;  // empty: {t_device}

// pd_ctx objects of the calling thread, per (device, slot) -- contexts are
// single-threaded objects. Slot 0 serves the thread's own calls; a batch call
// lends slots 0.. to its worker threads (one each), so the contexts and their
// device buffers outlive the workers and are reused call to call.
struct CtxHolder {
  std::map<std::pair<int, int>, pd_ctx*> by_dev;
  ~CtxHolder() {
    for (auto& kv : by_dev) pd_destroy(kv.second);
  }
};
thread_local CtxHolder t_ctx;

pd_ctx* ctx_on(int device, int slot = 0) {
  auto it = t_ctx.by_dev.find({device, slot});
  if (it != t_ctx.by_dev.end()) return it->second;
  pd_ctx* c = nullptr;
  const pd_status st = pd_create(&c, device);
  if (st != PD_OK)
    throw DeviceError(std::string("pardyn: cannot open CUDA device ") + std::to_string(device) + ": " +
                      pd_status_string(st));
  t_ctx.by_dev[{device, slot}] = c;
  return c;
}
pd_ctx* ctx() { return ctx_on(t_device); }

void check_call(pd_ctx* c, pd_status st) {
  if (st == PD_OK) return;
  const std::string msg = pd_last_error(c);
  if (st == PD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw DeviceError(std::string(pd_status_string(st)) + ": " + msg);
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

pd_algo to_c(FdAlgo a) {
  switch (a) {
    case FdAlgo::jsiia: return PD_JSIIA;
    case FdAlgo::abia: return PD_ABIA;
    case FdAlgo::cfa: return PD_CFA;
  }
  throw std::invalid_argument("forward_dynamics: unknown algorithm");
}

// Merge the trace of the variant that ran into *t (trace.hpp:24-39 semantics:
// stages add up, the longest chain and deepest scan are maxima).
void merge_trace(ExecTrace* t, const pd_exec_trace& r) {
  if (!t) return;
  t->parallel_link_stages += r.parallel_link_stages;
  t->note_sequential_chain(r.longest_sequential_link_chain);
  t->note_scan(ScanTrace{r.scan_rounds_max});
  if (r.oee_rounds) t->note_oee(OeeTrace{r.oee_rounds});
}

void merge_last_trace(ExecTrace* t, pd_ctx* c) {
  if (!t) return;
  pd_exec_trace r{};
  check_call(c, pd_last_trace(c, &r));
  merge_trace(t, r);
}

// Upload one chain as the context's shared model; a bad link throws the way
// link_inertias -> spatial_inertia_from does (spatial.cpp:72-87).
pd_ctx* one_model(const RobotChain& chain) {
  std::vector<double> rec;
  detail::append_records(chain, rec);
  pd_ctx* c = ctx();
  int32_t ms = 0, mr = 0;
  const int n = chain.size();
  check_call(c, pd_set_models(c, 1, n, rec.data(), chain.gravity.data(), &ms, &mr));
  if (ms != PD_SLOT_OK) throw std::invalid_argument(slot_message(ms, 0, mr, n));
  return c;
}

template <int R, int C>
void put_block(const Matrix<R, C>& m, double* out) {
  m.toRowMajor(out);
}
template <int R, int C>
Matrix<R, C> get_block(const double* in) {
  return Matrix<R, C>::FromRowMajor(in);
}

}  // namespace

namespace gpu {
void set_device(int device) { t_device = device; }
int device() { return t_device; }
void set_devices(const std::vector<int>& devices) { t_devices = devices; }
std::vector<int> devices() { return t_devices.empty() ? std::vector<int>{t_device} : t_devices; }
}  // namespace gpu

// ----------------------------------------------------------------- spatial algebra (spatial.cpp:10-100)
Mat3 skew(const Vec3& a) { return Mat3::FromRowMajor({0.0, -a(2), a(1), a(2), 0.0, -a(0), -a(1), a(0), 0.0}); }

namespace {
void set3(Mat6& m, int r0, int c0, const Mat3& b) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m(r0 + r, c0 + c) = b(r, c);
}
}  // namespace

Mat6 small_adjoint(const Twist& v) {
  Mat6 ad;
  const Mat3 wx = skew(v.angular);
  set3(ad, 0, 0, wx);
  set3(ad, 3, 3, wx);
  set3(ad, 3, 0, skew(v.linear));
  return ad;
}

AdjointMap adjoint_of(const SE3Transform& t) {
  AdjointMap a;
  a.mat.setZero();
  set3(a.mat, 0, 0, t.rotation);
  set3(a.mat, 3, 3, t.rotation);
  set3(a.mat, 3, 0, skew(t.translation) * t.rotation);
  return a;
}

SE3Transform screw_exp(const Twist& s, double q) {
  const Vec3& w = s.angular;
  const Vec3& v = s.linear;
  const double wn = w.norm();
  SE3Transform t;
  if (wn < 1e-12) {  // pure translation along the linear part
    t.translation = q * v;
    return t;
  }
  const Mat3 wx = skew(w), wx2 = wx * wx;
  const double st = std::sin(wn * q), ct = std::cos(wn * q);
  t.rotation = Mat3::Identity() + (st / wn) * wx + ((1.0 - ct) / (wn * wn)) * wx2;
  t.translation = (q * Mat3::Identity() + ((1.0 - ct) / (wn * wn)) * wx + ((q - st / wn) / (wn * wn)) * wx2) * v;
  return t;
}

SpatialInertia spatial_inertia_from(double mass, const Vec3& com, const Mat3& inertia_rot) {
  if (!(mass > 0.0) || !std::isfinite(mass)) throw std::invalid_argument("spatial inertia: mass must be positive");
  if (!com.allFinite() || !inertia_rot.allFinite())
    throw std::invalid_argument("spatial inertia: parameters must be finite");
  double scale = 0.0, asym = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      scale = std::max(scale, std::fabs(inertia_rot(r, c)));
      asym = std::max(asym, std::fabs(inertia_rot(r, c) - inertia_rot(c, r)));
    }
  if (asym > 1e-9 * std::max(scale, 1.0))
    throw std::invalid_argument("spatial inertia: rotational inertia must be symmetric");
  if (!(detail::sym3_min_eig(inertia_rot) > 0.0))
    throw std::invalid_argument("spatial inertia: rotational inertia must be positive definite");
  const Mat3 cx = skew(com);
  Mat6 m;
  set3(m, 0, 0, inertia_rot + mass * (cx * cx.transpose()));
  set3(m, 0, 3, mass * cx);
  set3(m, 3, 0, mass * cx.transpose());
  set3(m, 3, 3, mass * Mat3::Identity());
  return SpatialInertia(m);
}

bool operator==(const LinkSpec& a, const LinkSpec& b) {
  return a.mass == b.mass && a.com == b.com && a.inertia_rot == b.inertia_rot &&
         a.joint_screw.angular == b.joint_screw.angular && a.joint_screw.linear == b.joint_screw.linear &&
         a.home_transform.rotation == b.home_transform.rotation &&
         a.home_transform.translation == b.home_transform.translation;
}
bool operator==(const RobotChain& a, const RobotChain& b) { return a.gravity == b.gravity && a.links == b.links; }

// ----------------------------------------------------------------- model (device)
RobotChain random_chain(int n, std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("random_chain: n must be at least 1");
  std::vector<double> rec(static_cast<std::size_t>(n) * PD_LINK_FIELDS);
  pd_random_chain(n, seed, rec.data());
  return detail::chain_from_records(rec.data(), n);
}

ChainKinematics assemble_kinematics(const RobotChain& chain, const JointVector& q) {
  const int n = chain.size();
  if (static_cast<int>(q.size()) != n)  // model.cpp:120-124
    throw std::invalid_argument("assemble_kinematics: q has length " + std::to_string(q.size()) +
                                " but the chain has " + std::to_string(n) + " joints");
  ChainKinematics kin;
  if (n == 0) return kin;
  pd_ctx* c = one_model(chain);
  std::vector<double> rel(12 * n), base(36), tr(36 * (n - 1)), sc(6 * n);
  check_call(c, pd_assemble_kinematics(c, 1, q.data(), rel.data(), base.data(), tr.data(), sc.data()));
  kin.rel.resize(n);
  kin.screw.resize(n);
  kin.transport.resize(n - 1);
  for (int i = 0; i < n; ++i) {
    kin.rel[i].rotation = get_block<3, 3>(&rel[12 * i]);
    kin.rel[i].translation = Vec3(rel[12 * i + 9], rel[12 * i + 10], rel[12 * i + 11]);
    kin.screw[i] = Twist::from_stacked(get_block<6, 1>(&sc[6 * i]));
  }
  kin.base_transport.mat = get_block<6, 6>(base.data());
  for (int i = 0; i + 1 < n; ++i) kin.transport[i].mat = get_block<6, 6>(&tr[36 * i]);
  return kin;
}

std::vector<SpatialInertia> link_inertias(const RobotChain& chain) {
  const int n = chain.size();
  std::vector<SpatialInertia> out(static_cast<std::size_t>(n));
  if (n == 0) return out;
  pd_ctx* c = one_model(chain);
  std::vector<double> J(36 * static_cast<std::size_t>(n));
  check_call(c, pd_link_inertias(c, J.data()));
  for (int i = 0; i < n; ++i) out[i] = SpatialInertia(get_block<6, 6>(&J[36 * i]));
  return out;
}

// ----------------------------------------------------------------- operators (device)
namespace {
void kin_arrays(const ChainKinematics& kin, std::vector<double>& tr, std::vector<double>& sc) {
  const int n = kin.size();
  tr.assign(36 * static_cast<std::size_t>(std::max(n - 1, 0)), 0.0);
  sc.assign(6 * static_cast<std::size_t>(n), 0.0);
  for (int i = 0; i + 1 < n; ++i) put_block(kin.transport[i].mat, &tr[36 * i]);
  for (int i = 0; i < n; ++i) put_block(kin.screw[i].stacked(), &sc[6 * i]);
}
}  // namespace

ArticulatedBodyInertias articulated_body_inertias(const ChainKinematics& kin, std::span<const SpatialInertia> inertia,
                                                  ExecTrace* trace) {
  const int n = kin.size();
  ArticulatedBodyInertias out;
  if (n == 0) return out;
  if (static_cast<int>(inertia.size()) != n || static_cast<int>(kin.transport.size()) != n - 1 ||
      static_cast<int>(kin.screw.size()) != n)
    throw std::invalid_argument("articulated_body_inertias: kinematics and inertias must match");
  std::vector<double> tr, sc, J(36 * static_cast<std::size_t>(n)), abi(36 * n), lam(n), gain(6 * n);
  kin_arrays(kin, tr, sc);
  for (int i = 0; i < n; ++i) put_block(inertia[i].matrix(), &J[36 * i]);
  pd_ctx* c = ctx();
  int32_t st = 0, ix = 0;
  check_call(c, pd_articulated_body_inertias(c, 1, n, tr.data(), J.data(), 0, sc.data(), abi.data(), lam.data(),
                                             gain.data(), &st, &ix));
  if (st != PD_SLOT_OK) throw_slot(st, 0, ix, n);
  out.inertia.resize(n);
  out.gain.resize(n);
  out.joint_inertia = JointVector(n);
  for (int i = 0; i < n; ++i) {
    out.inertia[i] = get_block<6, 6>(&abi[36 * i]);
    out.gain[i] = get_block<6, 1>(&gain[6 * i]);
    out.joint_inertia[i] = lam[i];
  }
  if (trace) trace->note_sequential_chain(n);  // the tip-to-base walk (forward_dynamics.cpp:160)
  return out;
}

ConstraintBasis build_constraint_basis(const RobotChain& chain) {
  const int n = chain.size();
  ConstraintBasis out;
  out.basis.resize(n);
  if (n == 0) return out;
  std::vector<double> sc(6 * static_cast<std::size_t>(n)), W(30 * static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) put_block(chain.links[i].joint_screw.stacked(), &sc[6 * i]);
  pd_ctx* c = ctx();
  check_call(c, pd_constraint_basis(c, n, sc.data(), W.data()));
  for (int i = 0; i < n; ++i) out.basis[i] = get_block<6, 5>(&W[30 * i]);
  return out;
}

CfaOperators build_cfa_operators(const RobotChain& chain, const ChainKinematics& kin, const ConstraintBasis& basis,
                                 ExecTrace* trace) {
  const int n = chain.size();
  if (n == 0) throw std::invalid_argument("build_cfa_operators: chain has no links");
  if (static_cast<int>(basis.basis.size()) != n || kin.size() != n)
    throw std::invalid_argument("build_cfa_operators: kinematics and basis must match the chain");
  const std::vector<SpatialInertia> inertia = link_inertias(chain);  // validates like the reference (:273)
  std::vector<double> tr, sc, J(36 * static_cast<std::size_t>(n)), W(30 * static_cast<std::size_t>(n));
  kin_arrays(kin, tr, sc);
  for (int i = 0; i < n; ++i) {
    put_block(inertia[i].matrix(), &J[36 * i]);
    put_block(basis.basis[i], &W[30 * i]);
  }
  const std::size_t e = static_cast<std::size_t>(n - 1);
  std::vector<double> D(25 * n), U(25 * e), bs(5 * e), bd(5 * n), bp(5 * e), cd(n), co(e);
  pd_ctx* c = ctx();
  int32_t st = 0, ix = 0;
  check_call(c, pd_cfa_operators(c, 1, n, J.data(), 0, tr.data(), sc.data(), W.data(), D.data(), U.data(), bs.data(),
                                 bd.data(), bp.data(), cd.data(), co.data(), &st, &ix));
  if (st != PD_SLOT_OK) throw_slot(st, 0, ix, n);
  CfaOperators ops;
  ops.constraint_op.diag.resize(n);
  ops.constraint_op.upper.resize(e);
  ops.cross_diag.resize(n);
  ops.cross_sub.resize(e);
  ops.cross_super.resize(e);
  ops.joint_diag = JointVector(n);
  ops.joint_off = JointVector(e);
  for (int i = 0; i < n; ++i) {
    ops.constraint_op.diag[i] = get_block<5, 5>(&D[25 * i]);
    ops.cross_diag[i] = get_block<5, 1>(&bd[5 * i]);
    ops.joint_diag[i] = cd[i];
  }
  for (std::size_t i = 0; i < e; ++i) {
    ops.constraint_op.upper[i] = get_block<5, 5>(&U[25 * i]);
    ops.cross_sub[i] = get_block<5, 1>(&bs[5 * i]);
    ops.cross_super[i] = get_block<5, 1>(&bp[5 * i]);
    ops.joint_off[i] = co[i];
  }
  if (trace) {  // per-link factor-solves, then per-row projections (forward_dynamics.cpp:322,354)
    trace->note_parallel_stage();
    trace->note_parallel_stage();
  }
  return ops;
}

namespace {
std::vector<double> flat5(const std::vector<Vec5>& v) {
  std::vector<double> out(5 * v.size());
  for (std::size_t i = 0; i < v.size(); ++i) put_block(v[i], &out[5 * i]);
  return out;
}
}  // namespace

std::vector<Vec5> CfaOperators::apply_cross(const JointVector& v) const {
  const std::size_t n = cross_diag.size();
  if (v.size() != n) throw std::invalid_argument("apply_cross: one entry per link expected");
  std::vector<Vec5> out(n);
  if (n == 0) return out;
  const std::vector<double> bs = flat5(cross_sub), bd = flat5(cross_diag), bp = flat5(cross_super);
  std::vector<double> r(5 * n);
  pd_ctx* c = ctx();
  check_call(c, pd_cfa_apply(c, PD_APPLY_CROSS, 1, static_cast<int32_t>(n), bs.data(), bd.data(), bp.data(), nullptr,
                             nullptr, v.data(), r.data()));
  for (std::size_t i = 0; i < n; ++i) out[i] = get_block<5, 1>(&r[5 * i]);
  return out;
}

JointVector CfaOperators::apply_cross_transpose(std::span<const Vec5> f) const {
  const std::size_t n = cross_diag.size();
  if (f.size() != n) throw std::invalid_argument("apply_cross_transpose: one constraint block per link expected");
  JointVector out(n);
  if (n == 0) return out;
  const std::vector<double> bs = flat5(cross_sub), bd = flat5(cross_diag), bp = flat5(cross_super),
                            ff = flat5(std::vector<Vec5>(f.begin(), f.end()));
  pd_ctx* c = ctx();
  check_call(c, pd_cfa_apply(c, PD_APPLY_CROSS_TRANSPOSE, 1, static_cast<int32_t>(n), bs.data(), bd.data(), bp.data(),
                             nullptr, nullptr, ff.data(), out.data()));
  return out;
}

JointVector CfaOperators::apply_joint(const JointVector& v) const {
  const std::size_t n = joint_diag.size();
  if (v.size() != n) throw std::invalid_argument("apply_joint: one entry per link expected");
  JointVector out(n);
  if (n == 0) return out;
  pd_ctx* c = ctx();
  check_call(c, pd_cfa_apply(c, PD_APPLY_JOINT, 1, static_cast<int32_t>(n), nullptr, nullptr, nullptr,
                             joint_diag.data(), joint_off.data(), v.data(), out.data()));
  return out;
}

// ----------------------------------------------------------------- forward dynamics (device)
JointVector forward_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& tau, FdAlgo algo, ExecTrace* trace) {
  const pd_algo a = to_c(algo);
  check_sizes(chain, q, qdot, tau);
  const int n = chain.size();
  pd_ctx* c = one_model(chain);
  JointVector out(n);
  int32_t st = 0, rd = 0, ix = 0;
  if (trace) {
    // log-depth (CTA) variants; the trace describes the variant that ran
    pd_exec_trace r{};
    check_call(c, pd_forward_dynamics_traced(c, a, 1, q.data(), qdot.data(), tau.data(), out.data(), &st, &rd, &ix,
                                             &r));
    if (st != PD_SLOT_OK) throw_slot(st, rd, ix, n);
    merge_trace(trace, r);
    return out;
  }
  check_call(c, pd_forward_dynamics(c, a, 1, q.data(), qdot.data(), tau.data(), out.data(), &st, &rd, &ix));
  if (st != PD_SLOT_OK) throw_slot(st, rd, ix, n);
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

namespace {

// Page-locked staging for the batch calls, one per thread, grown on demand:
// copies from it run at DMA speed (pageable host memory goes through the
// driver's bounce buffer at ~10 GB/s).
struct PinnedStage {
  void* p = nullptr;
  std::size_t cap = 0;
  ~PinnedStage() { pd_host_free(p); }
  double* get(std::size_t doubles) {
    const std::size_t want = doubles * sizeof(double);
    if (want > cap) {
      pd_host_free(p);
      p = nullptr;
      cap = 0;
      if (pd_host_alloc(want + (want >> 3), &p) != PD_OK || !p)
        throw DeviceError("pardyn: cannot allocate page-locked staging memory");
      cap = want + (want >> 3);
    }
    return static_cast<double*>(p);
  }
};
thread_local PinnedStage t_stage;

// Runs f(lo, hi) over [0, count) on up to hardware_concurrency threads
// (inline below `grain` items per thread).
template <class F>
void parallel_ranges(std::size_t count, std::size_t grain, F&& f) {
  const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t T = std::min<std::size_t>(hw, std::max<std::size_t>(1, count / std::max<std::size_t>(grain, 1)));
  if (T <= 1) {
    f(std::size_t{0}, count);
    return;
  }
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < T; ++t) pool.emplace_back([&, t] { f(count * t / T, count * (t + 1) / T); });
  f(std::size_t{0}, count / T);
  for (std::thread& th : pool) th.join();
}

// One bucket (equal n) packed for the C-ABI into page-locked staging:
// links [B][n][31], gravity [B][3], q / qd / tau / qdd [B][n], then the slot arrays.
struct Bucket {
  int n = 0;
  std::vector<std::size_t> idx;
  double *links = nullptr, *grav = nullptr, *q = nullptr, *qd = nullptr, *tau = nullptr, *qdd = nullptr;
  int32_t *st = nullptr, *rd = nullptr, *ix = nullptr;

  void layout(double* base) {
    const std::size_t B = idx.size(), nn = static_cast<std::size_t>(n);
    links = base;
    grav = links + B * nn * PD_LINK_FIELDS;
    q = grav + 3 * B;
    qd = q + B * nn;
    tau = qd + B * nn;
    qdd = tau + B * nn;
    st = reinterpret_cast<int32_t*>(qdd + B * nn);
    rd = st + B;
    ix = rd + B;
  }
  // problems [lo, hi) of the bucket into the staging (host threads). The
  // staging is only read back by the upload DMA, so the stores stream past the
  // caches (no read-for-ownership of ~0.5 GB of staging lines for a c2 batch).
  static void put(double* dst, double v) {
#if defined(__x86_64__)
    long long bits;
    std::memcpy(&bits, &v, sizeof bits);
    _mm_stream_si64(reinterpret_cast<long long*>(dst), bits);
#else
    *dst = v;
#endif
  }
  void pack(std::span<const FdProblem> problems, std::size_t lo, std::size_t hi) {
    const std::size_t nn = static_cast<std::size_t>(n);
    parallel_ranges(hi - lo, 1024, [&](std::size_t a, std::size_t b) {
      double r[PD_LINK_FIELDS];
      for (std::size_t j = lo + a; j < lo + b; ++j) {
        const FdProblem& p = problems[idx[j]];
        double* rec = links + j * nn * PD_LINK_FIELDS;
        for (std::size_t i = 0; i < nn; ++i) {
          detail::to_record(p.chain.links[i], r);
          for (int k = 0; k < PD_LINK_FIELDS; ++k) put(rec + i * PD_LINK_FIELDS + k, r[k]);
        }
        for (int k = 0; k < 3; ++k) put(grav + 3 * j + k, p.chain.gravity(k));
        for (std::size_t i = 0; i < nn; ++i) {
          put(q + j * nn + i, p.q[i]);
          put(qd + j * nn + i, p.qdot[i]);
          put(tau + j * nn + i, p.tau[i]);
        }
      }
#if defined(__x86_64__)
      _mm_sfence();
#endif
    });
  }
  static std::size_t doubles(std::size_t B, int n) {
    return B * n * PD_LINK_FIELDS + 3 * B + 4 * B * n + (3 * B + 1) / 2;
  }
};

// Solve slots [lo, hi) of a packed bucket on one device; every slice selects
// kernels for the whole bucket (pd_set_selection_batch), so the result does
// not depend on how the bucket was split.
void solve_slice(pd_ctx* c, pd_algo a, Bucket& b, std::size_t lo, std::size_t hi) {
  const std::size_t cnt = hi - lo, n = static_cast<std::size_t>(b.n);
  if (cnt == 0) return;
  check_call(c, pd_set_selection_batch(c, static_cast<int64_t>(b.idx.size())));
  check_call(c, pd_set_models(c, static_cast<int64_t>(cnt), b.n, b.links + lo * n * PD_LINK_FIELDS, b.grav + 3 * lo,
                              nullptr, nullptr));
  const pd_status s = pd_forward_dynamics(c, a, static_cast<int64_t>(cnt), b.q + lo * n, b.qd + lo * n,
                                          b.tau + lo * n, b.qdd + lo * n, b.st + lo, b.rd + lo, b.ix + lo);
  pd_set_selection_batch(c, 0);
  check_call(c, s);
}

}  // namespace

// forward_dynamics.cpp:466-481: never throws per problem. Problems are
// bucketed by link count; a bucket is packed (in parallel host threads) into
// page-locked staging and split into contiguous slices over gpu::devices(),
// one worker thread per device on a context the calling thread lends it (so
// the contexts and their device buffers are reused call to call). Packing the
// whole bucket before the first upload is deliberate: both are bound by host
// memory bandwidth, and overlapping them per slice measured slower
// (profiles/dropin_batch_r2.txt).
std::vector<FdResult> batch_forward_dynamics(std::span<const FdProblem> problems, FdAlgo algo) {
  const pd_algo a = to_c(algo);
  std::vector<FdResult> out(problems.size());
  std::map<int, Bucket> buckets;
  for (std::size_t k = 0; k < problems.size(); ++k) {
    const FdProblem& p = problems[k];
    try {
      check_sizes(p.chain, p.q, p.qdot, p.tau);
      buckets[p.chain.size()].idx.push_back(k);
    } catch (const std::exception& e) {
      out[k].error = e.what();
    }
  }
  const std::vector<int> devs = gpu::devices();
  for (auto& [n, b] : buckets) {
    b.n = n;
    const std::size_t B = b.idx.size();
    b.layout(t_stage.get(Bucket::doubles(B, n)));
    b.pack(problems, 0, B);
    const std::size_t G = std::min<std::size_t>(devs.size(), B);
    std::vector<pd_ctx*> ctxs;
    std::map<int, int> slots;  // a device listed twice gets distinct contexts
    for (std::size_t g = 0; g < G; ++g) ctxs.push_back(ctx_on(devs[g], slots[devs[g]]++));
    if (G <= 1) {
      solve_slice(ctxs[0], a, b, 0, B);
    } else {
      std::vector<std::thread> workers;
      std::vector<std::string> errors(G);
      std::vector<int> kinds(G, 0);
      for (std::size_t g = 0; g < G; ++g)
        workers.emplace_back([&, g] {
          try {
            solve_slice(ctxs[g], a, b, B * g / G, B * (g + 1) / G);
          } catch (const std::invalid_argument& e) {
            errors[g] = e.what();
            kinds[g] = 1;
          } catch (const std::exception& e) {
            errors[g] = e.what();
            kinds[g] = 2;
          }
        });
      for (std::thread& w : workers) w.join();
      for (std::size_t g = 0; g < G; ++g) {
        if (kinds[g] == 1) throw std::invalid_argument(errors[g]);
        if (kinds[g] == 2) throw DeviceError(errors[g]);
      }
    }
    parallel_ranges(B, 4096, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t j = lo; j < hi; ++j) {
        FdResult& r = out[b.idx[j]];
        if (b.st[j] == PD_SLOT_OK)
          r.qddot = JointVector(b.qdd + j * n, b.qdd + (j + 1) * n);
        else
          r.error = slot_message(b.st[j], b.rd[j], b.ix[j], n);
      }
    });
  }
  return out;
}

// ----------------------------------------------------------------- inverse dynamics (device)
namespace {

void id_sizes(const RobotChain& chain, std::initializer_list<std::pair<const char*, const JointVector*>> args) {
  const std::size_t n = chain.links.size();
  for (const auto& a : args)  // inverse_dynamics.cpp:10-17
    if (a.second->size() != n)
      throw std::invalid_argument(std::string(a.first) + " has length " + std::to_string(a.second->size()) +
                                  " but the chain has " + std::to_string(n) + " joints");
}

// model.cpp:120-124 (assemble_kinematics runs first in the reference)
void q_size(const RobotChain& chain, const JointVector& q) {
  if (q.size() != chain.links.size())
    throw std::invalid_argument("assemble_kinematics: q has length " + std::to_string(q.size()) +
                                " but the chain has " + std::to_string(chain.links.size()) + " joints");
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

namespace {

// inverse_dynamics.cpp:10-17
void check_joint_size(const ChainKinematics& kin, const JointVector& v, const char* name) {
  if (static_cast<int>(v.size()) != kin.size())
    throw std::invalid_argument(std::string(name) + " has length " + std::to_string(v.size()) + " but the chain has " +
                                std::to_string(kin.size()) + " joints");
}

std::vector<double> flat6(std::span<const Twist> v) {
  std::vector<double> out(6 * v.size());
  for (std::size_t i = 0; i < v.size(); ++i) put_block(v[i].stacked(), &out[6 * i]);
  return out;
}

// One propagation on the device (pd_propagate): kinematics and the per-kind inputs flattened.
std::vector<Vec6> propagate(int kind, const ChainKinematics& kin, const JointVector* qdot, const JointVector* qddot,
                            std::span<const Twist> velocity, std::span<const Twist> acceleration,
                            std::span<const SpatialInertia> inertia, const Vec6& boundary, ScanTrace* trace) {
  const int n = kin.size();
  if (trace) trace->rounds = ceil_log2(static_cast<std::size_t>(n));  // the scan's designed depth (scan.hpp:32-65)
  std::vector<Vec6> out(static_cast<std::size_t>(n));
  if (n == 0) return out;
  std::vector<double> tr, sc, base(36), J, vv, aa, bd(6), x(6 * static_cast<std::size_t>(n));
  kin_arrays(kin, tr, sc);
  put_block(kin.base_transport.mat, base.data());
  put_block(boundary, bd.data());
  if (!velocity.empty()) vv = flat6(velocity);
  if (!acceleration.empty()) aa = flat6(acceleration);
  if (!inertia.empty()) {
    J.resize(36 * static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) put_block(inertia[i].matrix(), &J[36 * i]);
  }
  pd_ctx* c = ctx();
  check_call(c, pd_propagate(c, kind, 1, n, base.data(), tr.empty() ? nullptr : tr.data(), sc.data(),
                             J.empty() ? nullptr : J.data(), 0, qdot ? qdot->data() : nullptr,
                             qddot ? qddot->data() : nullptr, vv.empty() ? nullptr : vv.data(),
                             aa.empty() ? nullptr : aa.data(), bd.data(), x.data()));
  for (int i = 0; i < n; ++i) out[i] = get_block<6, 1>(&x[6 * i]);
  return out;
}

template <class T>
std::vector<T> as_spatial(const std::vector<Vec6>& v) {
  std::vector<T> out;
  out.reserve(v.size());
  for (const Vec6& x : v) out.push_back(T::from_stacked(x));
  return out;
}

}  // namespace

std::vector<Twist> propagate_velocities(const ChainKinematics& kin, const JointVector& qdot,
                                        const Twist& base_velocity, ScanTrace* trace) {
  check_joint_size(kin, qdot, "qdot");
  return as_spatial<Twist>(propagate(PD_PROPAGATE_VELOCITIES, kin, &qdot, nullptr, {}, {}, {},
                                     base_velocity.stacked(), trace));
}

std::vector<Twist> propagate_accelerations(const ChainKinematics& kin, std::span<const Twist> velocity,
                                           const JointVector& qdot, const JointVector& qddot,
                                           const Twist& base_acceleration, ScanTrace* trace) {
  check_joint_size(kin, qdot, "qdot");
  check_joint_size(kin, qddot, "qddot");
  if (static_cast<int>(velocity.size()) != kin.size())
    throw std::invalid_argument("propagate_accelerations: one velocity per link expected");
  return as_spatial<Twist>(propagate(PD_PROPAGATE_ACCELERATIONS, kin, &qdot, &qddot, velocity, {}, {},
                                     base_acceleration.stacked(), trace));
}

std::vector<Wrench> propagate_forces(const ChainKinematics& kin, std::span<const Twist> velocity,
                                     std::span<const Twist> acceleration, std::span<const SpatialInertia> inertia,
                                     const Wrench& tip_wrench, ScanTrace* trace) {
  const int n = kin.size();
  if (static_cast<int>(velocity.size()) != n || static_cast<int>(acceleration.size()) != n ||
      static_cast<int>(inertia.size()) != n)
    throw std::invalid_argument("propagate_forces: one velocity, acceleration and inertia per link expected");
  return as_spatial<Wrench>(
      propagate(PD_PROPAGATE_FORCES, kin, nullptr, nullptr, velocity, acceleration, inertia, tip_wrench.stacked(), trace));
}

JointVector inverse_dynamics_assembled(const ChainKinematics& kin, std::span<const SpatialInertia> inertia,
                                       const Vec3& gravity, const JointVector& qdot, const JointVector& qddot,
                                       const IdOptions& opts, ExecTrace* trace) {
  const int n = kin.size();
  ScanTrace sv, sa, sf;
  const std::vector<Twist> vel = propagate_velocities(kin, qdot, opts.base_velocity, &sv);
  Twist base_acc = opts.base_acceleration;
  if (opts.apply_gravity) base_acc.linear -= gravity;  // inverse_dynamics.cpp:135-140
  const std::vector<Twist> acc = propagate_accelerations(kin, vel, qdot, qddot, base_acc, &sa);
  const std::vector<Wrench> frc = propagate_forces(kin, vel, acc, inertia, opts.tip_wrench, &sf);
  JointVector tau(n);
  for (int i = 0; i < n; ++i) tau[i] = kin.screw[i].stacked().dot(frc[i].stacked());  // :146-150
  if (trace) {
    trace->note_scan(sv);
    trace->note_scan(sa);
    trace->note_scan(sf);
    for (int k = 0; k < 5; ++k) trace->note_parallel_stage();  // kinematics, three source builds, extraction
  }
  return tau;
}

JointVector inverse_dynamics(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                             const JointVector& qddot, const IdOptions& opts, ExecTrace* trace) {
  q_size(chain, q);
  const std::size_t n = chain.links.size();
  if (n == 0) return JointVector();
  pd_ctx* c = one_model(chain);  // link_inertias validates before the rates are checked
  id_sizes(chain, {{"qdot", &qdot}, {"qddot", &qddot}});
  JointVector tau(n);
  const pd_id_options o = to_c(opts);
  check_call(c, pd_inverse_dynamics_opts(c, 1, q.data(), qdot.data(), qddot.data(), &o, tau.data()));
  merge_last_trace(trace, c);
  return tau;
}

JointVector bias_torque(const RobotChain& chain, const JointVector& q, const JointVector& qdot, ExecTrace* trace) {
  return inverse_dynamics(chain, q, qdot, JointVector::Zero(chain.links.size()), {}, trace);
}

LinkStates link_states(const RobotChain& chain, const JointVector& q, const JointVector& qdot,
                       const JointVector& qddot, const IdOptions& opts) {
  q_size(chain, q);
  const std::size_t n = chain.links.size();
  LinkStates out;
  if (n == 0) return out;
  pd_ctx* c = one_model(chain);
  id_sizes(chain, {{"qdot", &qdot}, {"qddot", &qddot}});
  std::vector<double> v(6 * n), a(6 * n), f(6 * n);
  const pd_id_options o = to_c(opts);
  check_call(c, pd_link_states(c, 1, q.data(), qdot.data(), qddot.data(), &o, v.data(), a.data(), f.data()));
  for (std::size_t i = 0; i < n; ++i) {
    out.velocity.push_back(Twist::from_stacked(get_block<6, 1>(&v[6 * i])));
    out.acceleration.push_back(Twist::from_stacked(get_block<6, 1>(&a[6 * i])));
    out.force.push_back(Wrench::from_stacked(get_block<6, 1>(&f[6 * i])));
  }
  return out;
}

MatrixXd joint_space_inertia(const RobotChain& chain, const JointVector& q, ExecTrace* trace) {
  const std::size_t n = chain.links.size();
  if (q.size() != n) throw std::invalid_argument("joint_space_inertia: q must have one entry per joint");
  MatrixXd M(n, n);
  if (n == 0) return M;
  pd_ctx* c = one_model(chain);
  check_call(c, pd_joint_space_inertia(c, 1, q.data(), M.data()));
  merge_last_trace(trace, c);
  return M;
}

// ----------------------------------------------------------------- building blocks (device)
namespace detail {

void bidiag_solve_rm(int dim, bool upper, std::size_t n, const double* coupling, const double* rhs, double* x) {
  pd_ctx* cx = ctx();
  check_call(cx, pd_block_bidiag_solve(cx, dim, 1, static_cast<int32_t>(n), upper ? 1 : 0, coupling, rhs, x));
}

void oee_solve_rm(int block, int cols, std::size_t n, const double* diag, const double* upper, const double* rhs,
                  double* x) {
  pd_ctx* cx = ctx();
  int32_t st = 0, rd = 0, ix = 0;
  check_call(cx, pd_block_tridiag_solve(cx, block, cols, 1, static_cast<int32_t>(n), diag, upper, rhs, x, &st, &rd,
                                        &ix));
  if (st != PD_SLOT_OK) throw SingularBlockError(rd, ix, slot_message(st, rd, ix, static_cast<int>(n)));
}

void oee_rounds_rm(int block, int cols, std::size_t n, int distance, int round, const double* diag,
                   const double* coupling, const double* rhs, double* diag_out, double* coupling_out,
                   double* rhs_out) {
  pd_ctx* cx = ctx();
  int32_t st = 0, rd = 0, ix = 0;
  check_call(cx, pd_oee_eliminate_rounds(cx, block, cols, 1, static_cast<int32_t>(n), distance, round, 1, diag,
                                         coupling, rhs, diag_out, coupling_out, rhs_out, &st, &rd, &ix));
  if (st != PD_SLOT_OK) throw SingularBlockError(rd, ix, slot_message(st, rd, ix, static_cast<int>(n)));
}

void coefficient_solve_rm(int block, int cols, const double* pivot, const double* rhs, double* x, int round,
                          int index) {
  // a one-row system is exactly a pivot solve: no rounds, the final block solve
  pd_ctx* cx = ctx();
  std::vector<double> rc(static_cast<std::size_t>(block) * std::min(cols, 4)), xc(rc.size());
  for (int c0 = 0; c0 < cols; c0 += 4) {  // the kernel carries up to 4 columns at a time
    const int w = std::min(4, cols - c0);
    for (int r = 0; r < block; ++r)
      for (int c = 0; c < w; ++c) rc[r * w + c] = rhs[r * cols + c0 + c];
    int32_t st = 0, rd = 0, ix = 0;
    check_call(cx, pd_block_tridiag_solve(cx, block, w, 1, 1, pivot, nullptr, rc.data(), xc.data(), &st, &rd, &ix));
    if (st != PD_SLOT_OK)
      throw SingularBlockError(round, index,
                               "odd-even elimination: singular pivot block (round " + std::to_string(round) +
                                   ", block " + std::to_string(index) + ")");
    for (int r = 0; r < block; ++r)
      for (int c = 0; c < w; ++c) x[r * cols + c0 + c] = xc[r * w + c];
  }
}

}  // namespace detail

}  // namespace pardyn
