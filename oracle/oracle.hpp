// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU restatement ("oracle") of the reference library pardyn's forward-
// dynamics path (arxiv 1609.06779), written without Eigen because Eigen3 is
// absent from this image, so the reference itself cannot be compiled here
// (SURVEY.md §0, §8c). Only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline leg may load this code, and only as the checker / the timed CPU
// reference arm -- never as the product path.
//
// Every function cites the reference file:line it restates (paths relative
// to /root/reference/proj/core). The restatement keeps the reference's
// algorithmic structure on purpose -- Hillis-Steele 6x6 affine scans,
// row-centric odd-even elimination with full-pivot LU, per-call kinematics /
// inertia / basis stages -- so that it is also the CPU baseline the GPU is
// compared against.
//
// Parity pinning: the reference ships no golden vectors and no test pins
// Eigen's bits. This oracle is pinned against the reference's
// own known-answer tests: the closed-form pendulum and planar 2-link arm
// (tests/support/oracles.hpp:293-382), the SPEC known-answer examples, the
// sequential Newton-Euler oracle, dense solves and the structural identities
// of tests/test_*.cpp, all re-run in tests/test_oracle_*.py. Bit-level parity
// with an Eigen build is unpinned.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------------------
// Fixed-size dense matrices (row-major).  Replaces Eigen's fixed-size types
// (include/pardyn/types.hpp:11-17).

template <int R, int C>
struct Mat {
  double a[R * C];
  double& operator()(int r, int c) { return a[r * C + c]; }
  double operator()(int r, int c) const { return a[r * C + c]; }
  double& operator[](int i) { return a[i]; }
  double operator[](int i) const { return a[i]; }
  static Mat Zero() {
    Mat m;
    for (int i = 0; i < R * C; ++i) m.a[i] = 0.0;
    return m;
  }
  static Mat Identity() {
    Mat m = Zero();
    for (int i = 0; i < (R < C ? R : C); ++i) m(i, i) = 1.0;
    return m;
  }
  Mat<C, R> T() const {
    Mat<C, R> t;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < C; ++c) t(c, r) = (*this)(r, c);
    return t;
  }
  double squaredNorm() const {
    double s = 0.0;
    for (int i = 0; i < R * C; ++i) s += a[i] * a[i];
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const {
    for (int i = 0; i < R * C; ++i)
      if (!std::isfinite(a[i])) return false;
    return true;
  }
};

template <int R, int C>
inline Mat<R, C> operator+(const Mat<R, C>& x, const Mat<R, C>& y) {
  Mat<R, C> o;
  for (int i = 0; i < R * C; ++i) o.a[i] = x.a[i] + y.a[i];
  return o;
}
template <int R, int C>
inline Mat<R, C> operator-(const Mat<R, C>& x, const Mat<R, C>& y) {
  Mat<R, C> o;
  for (int i = 0; i < R * C; ++i) o.a[i] = x.a[i] - y.a[i];
  return o;
}
template <int R, int C>
inline Mat<R, C> operator-(const Mat<R, C>& x) {
  Mat<R, C> o;
  for (int i = 0; i < R * C; ++i) o.a[i] = -x.a[i];
  return o;
}
template <int R, int C>
inline Mat<R, C> operator*(double s, const Mat<R, C>& x) {
  Mat<R, C> o;
  for (int i = 0; i < R * C; ++i) o.a[i] = s * x.a[i];
  return o;
}
template <int R, int K, int C>
inline Mat<R, C> operator*(const Mat<R, K>& x, const Mat<K, C>& y) {
  Mat<R, C> o;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) {
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += x(r, k) * y(k, c);
      o(r, c) = s;
    }
  return o;
}
template <int R, int C>
inline Mat<R, C>& operator+=(Mat<R, C>& x, const Mat<R, C>& y) {
  for (int i = 0; i < R * C; ++i) x.a[i] += y.a[i];
  return x;
}
template <int R, int C>
inline Mat<R, C>& operator-=(Mat<R, C>& x, const Mat<R, C>& y) {
  for (int i = 0; i < R * C; ++i) x.a[i] -= y.a[i];
  return x;
}
template <int N>
inline double dot(const Mat<N, 1>& x, const Mat<N, 1>& y) {
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += x.a[i] * y.a[i];
  return s;
}
template <int N>
inline double mtrace(const Mat<N, N>& x) {
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += x(i, i);
  return s;
}

using Vec3 = Mat<3, 1>;
using Mat3 = Mat<3, 3>;
using Vec5 = Mat<5, 1>;
using Mat5 = Mat<5, 5>;
using Vec6 = Mat<6, 1>;
using Mat6 = Mat<6, 6>;
using Mat65 = Mat<6, 5>;
using VecX = std::vector<double>;

inline Vec3 v3(double x, double y, double z) {
  Vec3 v;
  v[0] = x;
  v[1] = y;
  v[2] = z;
  return v;
}

// Dense n x n row-major matrix (Eigen::MatrixXd stand-in for JSIIA).
struct MatX {
  int n = 0;
  std::vector<double> a;
  MatX() = default;
  explicit MatX(int n_) : n(n_), a(static_cast<size_t>(n_) * n_, 0.0) {}
  double& operator()(int r, int c) { return a[static_cast<size_t>(r) * n + c]; }
  double operator()(int r, int c) const { return a[static_cast<size_t>(r) * n + c]; }
};

inline double vnorm(const VecX& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

// ---------------------------------------------------------------------------
// Errors (include/pardyn/types.hpp:21-46) and ceil_log2 (:49-57).

struct ModelError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DynamicsError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularBlockError : DynamicsError {
  SingularBlockError(int round, int index, const std::string& what)
      : DynamicsError(what), round_(round), index_(index) {}
  int round() const noexcept { return round_; }
  int index() const noexcept { return index_; }
  int round_, index_;
};

inline int ceil_log2(size_t n) {
  int k = 0;
  size_t p = 1;
  while (p < n) {
    p <<= 1;
    ++k;
  }
  return k;
}

// Trace counters (include/pardyn/trace.hpp:12-39).
struct ScanTrace {
  int rounds = 0;
};
struct OeeTrace {
  int rounds = 0;
};
struct ExecTrace {
  int parallel_link_stages = 0;
  int longest_sequential_link_chain = 0;
  int scan_rounds_max = 0;
  int oee_rounds = 0;
  void note_parallel_stage() { ++parallel_link_stages; }
  void note_sequential_chain(int l) {
    longest_sequential_link_chain = std::max(longest_sequential_link_chain, l);
  }
  void note_scan(const ScanTrace& t) { scan_rounds_max = std::max(scan_rounds_max, t.rounds); }
  void note_oee(const OeeTrace& t) { oee_rounds = t.rounds; }
};

// ---------------------------------------------------------------------------
// Spatial algebra (include/pardyn/spatial.hpp, src/spatial.cpp).
// Twists stack (angular, linear); wrenches (moment, force)  (spatial.hpp:7-10).

struct SE3 {
  Mat3 R = Mat3::Identity();
  Vec3 p = Vec3::Zero();
  // (a * b)(x) = a(b(x))   spatial.hpp:80-82
  SE3 operator*(const SE3& rhs) const {
    SE3 o;
    o.R = R * rhs.R;
    o.p = R * rhs.p + p;
    return o;
  }
  SE3 inverse() const {
    SE3 o;
    o.R = R.T();
    o.p = -(o.R * p);
    return o;
  }
  bool is_valid(double tol = 1e-9) const {  // spatial.cpp:36-41
    if (!R.allFinite() || !p.allFinite()) return false;
    const Mat3 g = R.T() * R - Mat3::Identity();
    double mx = 0.0;
    for (int i = 0; i < 9; ++i) mx = std::max(mx, std::fabs(g[i]));
    if (mx > tol) return false;
    const double det = R(0, 0) * (R(1, 1) * R(2, 2) - R(1, 2) * R(2, 1)) -
                       R(0, 1) * (R(1, 0) * R(2, 2) - R(1, 2) * R(2, 0)) +
                       R(0, 2) * (R(1, 0) * R(2, 1) - R(1, 1) * R(2, 0));
    return det > 0.0;
  }
};

// spatial.cpp:10-16
inline Mat3 skew(const Vec3& a) {
  Mat3 m;
  m(0, 0) = 0.0;   m(0, 1) = -a[2]; m(0, 2) = a[1];
  m(1, 0) = a[2];  m(1, 1) = 0.0;   m(1, 2) = -a[0];
  m(2, 0) = -a[1]; m(2, 1) = a[0];  m(2, 2) = 0.0;
  return m;
}

template <int R0, int C0, int R, int C>
inline void set_block(Mat<R, C>& m, const Mat3& b) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m(R0 + r, C0 + c) = b(r, c);
}
inline Vec6 stack(const Vec3& top, const Vec3& bot) {
  Vec6 v;
  for (int i = 0; i < 3; ++i) {
    v[i] = top[i];
    v[i + 3] = bot[i];
  }
  return v;
}
inline Vec3 head3(const Vec6& v) { return v3(v[0], v[1], v[2]); }
inline Vec3 tail3(const Vec6& v) { return v3(v[3], v[4], v[5]); }

// spatial.cpp:18-25: ad_V = [[w^, 0], [v^, w^]]
inline Mat6 small_adjoint(const Vec6& V) {
  Mat6 ad = Mat6::Zero();
  const Mat3 wx = skew(head3(V));
  set_block<0, 0>(ad, wx);
  set_block<3, 3>(ad, wx);
  set_block<3, 0>(ad, skew(tail3(V)));
  return ad;
}

// spatial.cpp:27-34: Ad(T) = [[R, 0], [p^ R, R]]
inline Mat6 adjoint_of(const SE3& t) {
  Mat6 a = Mat6::Zero();
  set_block<0, 0>(a, t.R);
  set_block<3, 3>(a, t.R);
  set_block<3, 0>(a, skew(t.p) * t.R);
  return a;
}

// spatial.cpp:43-68 (Rodrigues for a not-necessarily-unit angular part).
inline SE3 screw_exp(const Vec6& s, double q) {
  const Vec3 w = head3(s), v = tail3(s);
  const double wn = w.norm();
  SE3 t;
  if (wn < 1e-12) {
    t.p = q * v;
    return t;
  }
  const Mat3 wx = skew(w);
  const Mat3 wx2 = wx * wx;
  const double theta = wn * q;
  const double st = std::sin(theta), ct = std::cos(theta);
  t.R = Mat3::Identity() + (st / wn) * wx + ((1.0 - ct) / (wn * wn)) * wx2;
  t.p = (q * Mat3::Identity() + ((1.0 - ct) / (wn * wn)) * wx +
         ((q - st / wn) / (wn * wn)) * wx2) * v;
  return t;
}

// Smallest eigenvalue of a symmetric 3x3 by cyclic Jacobi (stands in for
// Eigen::SelfAdjointEigenSolver's minCoeff at spatial.cpp:83, model.cpp:96).
inline double sym3_min_eig(Mat3 m) {
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = m(0, 1) * m(0, 1) + m(0, 2) * m(0, 2) + m(1, 2) * m(1, 2);
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (m(p, q) == 0.0) continue;
        const double theta = (m(q, q) - m(p, p)) / (2.0 * m(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // rotate columns p,q
          const double mkp = m(k, p), mkq = m(k, q);
          m(k, p) = c * mkp - s * mkq;
          m(k, q) = s * mkp + c * mkq;
        }
        for (int k = 0; k < 3; ++k) {  // rotate rows p,q
          const double mpk = m(p, k), mqk = m(q, k);
          m(p, k) = c * mpk - s * mqk;
          m(q, k) = s * mpk + c * mqk;
        }
      }
  }
  return std::min(m(0, 0), std::min(m(1, 1), m(2, 2)));
}

inline double max_abs_asym(const Mat3& m) {
  double mx = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) mx = std::max(mx, std::fabs(m(r, c) - m(c, r)));
  return mx;
}
inline double max_abs(const Mat3& m) {
  double mx = 0.0;
  for (int i = 0; i < 9; ++i) mx = std::max(mx, std::fabs(m[i]));
  return mx;
}

// spatial.cpp:70-100. Throws std::invalid_argument with the reference's
// messages; assembles J = [[Ic + m cx cx^T, m cx], [m cx^T, m I]].
inline Mat6 spatial_inertia_from(double mass, const Vec3& com, const Mat3& Ic) {
  if (!(mass > 0.0) || !std::isfinite(mass))
    throw std::invalid_argument("spatial inertia: mass must be positive");
  if (!com.allFinite() || !Ic.allFinite())
    throw std::invalid_argument("spatial inertia: parameters must be finite");
  const double scale = max_abs(Ic);
  if (max_abs_asym(Ic) > 1e-9 * std::max(scale, 1.0))
    throw std::invalid_argument("spatial inertia: rotational inertia must be symmetric");
  if (!(sym3_min_eig(Ic) > 0.0))
    throw std::invalid_argument("spatial inertia: rotational inertia must be positive definite");
  const Mat3 cx = skew(com);
  const Mat3 cx_sq = cx * cx.T();
  Mat6 m;
  set_block<0, 0>(m, Ic + mass * cx_sq);
  set_block<0, 3>(m, mass * cx);
  set_block<3, 0>(m, mass * cx.T());
  set_block<3, 3>(m, mass * Mat3::Identity());
  return m;
}

// ---------------------------------------------------------------------------
// Model (include/pardyn/model.hpp, src/model.cpp).

struct LinkSpec {  // model.hpp:17-23
  double mass = 1.0;
  Vec3 com = Vec3::Zero();
  Mat3 inertia_rot = Mat3::Identity();
  Vec6 joint_screw = stack(v3(0, 0, 1), Vec3::Zero());
  SE3 home;
};

struct RobotChain {  // model.hpp:25-30
  std::vector<LinkSpec> links;
  Vec3 gravity = v3(0.0, 0.0, -9.81);
  int size() const { return static_cast<int>(links.size()); }
};

// Flat 31-double LinkSpec record used at every boundary of this repo:
//   [0] mass, [1..3] com, [4..12] inertia_rot row-major, [13..18] screw
//   (angular, linear), [19..27] home rotation row-major, [28..30] home
//   translation -- the field order of LinkSpec (model.hpp:17-23) and of the
//   JSON model format (model.hpp:72-77).
constexpr int kLinkFields = 31;

inline LinkSpec link_from_flat(const double* f) {
  LinkSpec l;
  l.mass = f[0];
  for (int i = 0; i < 3; ++i) l.com[i] = f[1 + i];
  for (int i = 0; i < 9; ++i) l.inertia_rot[i] = f[4 + i];
  for (int i = 0; i < 6; ++i) l.joint_screw[i] = f[13 + i];
  for (int i = 0; i < 9; ++i) l.home.R[i] = f[19 + i];
  for (int i = 0; i < 3; ++i) l.home.p[i] = f[28 + i];
  return l;
}
inline void link_to_flat(const LinkSpec& l, double* f) {
  f[0] = l.mass;
  for (int i = 0; i < 3; ++i) f[1 + i] = l.com[i];
  for (int i = 0; i < 9; ++i) f[4 + i] = l.inertia_rot[i];
  for (int i = 0; i < 6; ++i) f[13 + i] = l.joint_screw[i];
  for (int i = 0; i < 9; ++i) f[19 + i] = l.home.R[i];
  for (int i = 0; i < 3; ++i) f[28 + i] = l.home.p[i];
}
inline RobotChain chain_from_flat(int n, const double* links, const double* gravity) {
  RobotChain c;
  c.links.resize(n);
  for (int i = 0; i < n; ++i) c.links[i] = link_from_flat(links + static_cast<size_t>(i) * kLinkFields);
  if (gravity) c.gravity = v3(gravity[0], gravity[1], gravity[2]);
  return c;
}

struct ChainKinematics {  // model.hpp:42-49
  std::vector<SE3> rel;
  Mat6 base_transport;
  std::vector<Mat6> transport;  // n-1
  std::vector<Vec6> screw;
  int size() const { return static_cast<int>(rel.size()); }
};

// model.cpp:117-146
inline ChainKinematics assemble_kinematics(const RobotChain& chain, const VecX& q) {
  const int n = chain.size();
  if (static_cast<int>(q.size()) != n)
    throw std::invalid_argument("assemble_kinematics: q has length " + std::to_string(q.size()) +
                                " but the chain has " + std::to_string(n) + " joints");
  ChainKinematics kin;
  kin.rel.resize(n);
  kin.screw.resize(n);
  kin.transport.resize(n > 0 ? n - 1 : 0);
  for (int i = 0; i < n; ++i) {
    kin.screw[i] = chain.links[i].joint_screw;
    kin.rel[i] = screw_exp(chain.links[i].joint_screw, -q[i]) * chain.links[i].home;
  }
  if (n > 0) kin.base_transport = adjoint_of(kin.rel[0]);
  for (int i = 0; i + 1 < n; ++i) kin.transport[i] = adjoint_of(kin.rel[i + 1]);
  return kin;
}

// model.cpp:148-155
inline std::vector<Mat6> link_inertias(const RobotChain& chain) {
  std::vector<Mat6> out(chain.links.size());
  for (size_t i = 0; i < chain.links.size(); ++i)
    out[i] = spatial_inertia_from(chain.links[i].mass, chain.links[i].com, chain.links[i].inertia_rot);
  return out;
}

// model.cpp:75-115
inline void validate_chain(const RobotChain& chain) {
  if (chain.links.empty()) throw ModelError("chain must have at least one link");
  if (!chain.gravity.allFinite()) throw ModelError("gravity must be finite");
  for (int k = 0; k < chain.size(); ++k) {
    const LinkSpec& l = chain.links[k];
    const std::string pre = "link " + std::to_string(k);
    if (!(l.mass > 0.0) || !std::isfinite(l.mass)) throw ModelError(pre + ": mass must be positive");
    if (!l.com.allFinite()) throw ModelError(pre + ": com must be finite");
    if (!l.inertia_rot.allFinite() ||
        max_abs_asym(l.inertia_rot) > 1e-9 * std::max(1.0, max_abs(l.inertia_rot)))
      throw ModelError(pre + ": rotational inertia must be symmetric");
    if (!(sym3_min_eig(l.inertia_rot) > 0.0))
      throw ModelError(pre + ": rotational inertia must be positive definite");
    if (!l.joint_screw.allFinite()) throw ModelError(pre + ": joint_screw must be finite");
    const double nrm = l.joint_screw.norm();
    if (std::fabs(nrm - 1.0) > 1e-9)
      throw ModelError(pre + ": joint_screw must have unit norm (got " + std::to_string(nrm) + ")");
    if (!l.home.is_valid(1e-9))
      throw ModelError(pre + ": home_transform rotation must be orthonormal with determinant +1");
  }
}

// model.cpp:26-56. Uniform draws on the raw mt19937_64 stream.
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  Vec3 unit_vector() {
    const double z = uniform(-1.0, 1.0);
    const double phi = uniform(0.0, 2.0 * M_PI);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    return v3(r * std::cos(phi), r * std::sin(phi), z);
  }
  // Shoemake uniform quaternion -> Eigen::Quaterniond::toRotationMatrix
  // (Eigen 3.3/3.4 Quaternion.h formula).
  Mat3 rotation() {
    const double u1 = uniform();
    const double a2 = uniform(0.0, 2.0 * M_PI);
    const double a3 = uniform(0.0, 2.0 * M_PI);
    const double s1 = std::sqrt(1.0 - u1), s2 = std::sqrt(u1);
    const double w = s2 * std::cos(a3), x = s1 * std::sin(a2), y = s1 * std::cos(a2),
                 z = s2 * std::sin(a3);
    const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    Mat3 r;
    r(0, 0) = 1 - (tyy + tzz); r(0, 1) = txy - twz;       r(0, 2) = txz + twy;
    r(1, 0) = txy + twz;       r(1, 1) = 1 - (txx + tzz); r(1, 2) = tyz - twx;
    r(2, 0) = txz - twy;       r(2, 1) = tyz + twx;       r(2, 2) = 1 - (txx + tyy);
    return r;
  }

 private:
  std::mt19937_64 eng_;
};

// model.cpp:157-185. Draw order is the one GCC 13 produces for the
// reference source: constructor / operator arguments evaluate right to left
// (probed in this container), so com draws z,y,x; moments z,y,x; and the
// home translation draws unit_vector() before its magnitude.
inline RobotChain random_chain(int n, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("random_chain: n must be at least 1");
  Rng rng(seed);
  RobotChain chain;
  chain.links.resize(n);
  for (LinkSpec& link : chain.links) {
    link.mass = rng.uniform(0.1, 10.0);
    const double cz = rng.uniform(-0.3, 0.3), cy = rng.uniform(-0.3, 0.3), cx = rng.uniform(-0.3, 0.3);
    link.com = v3(cx, cy, cz);
    const Mat3 axes = rng.rotation();
    const double mz = rng.uniform(0.1, 1.0), my = rng.uniform(0.1, 1.0), mx = rng.uniform(0.1, 1.0);
    Mat3 d = Mat3::Zero();
    d(0, 0) = mx;
    d(1, 1) = my;
    d(2, 2) = mz;
    const Mat3 inertia = (axes * d) * axes.T();
    link.inertia_rot = 0.5 * (inertia + inertia.T());
    link.joint_screw = stack(rng.unit_vector(), Vec3::Zero());
    link.home.R = rng.rotation();
    const Vec3 dir = rng.unit_vector();
    const double mag = rng.uniform(0.1, 1.0);
    link.home.p = mag * dir;
  }
  validate_chain(chain);
  return chain;
}

// ---------------------------------------------------------------------------
// Scan + block bi-diagonal solvers (include/pardyn/scan.hpp).

// scan.hpp:32-65: Hillis-Steele, identity padded to m = 2^L, exactly L rounds.
template <class T, class Combine>
std::vector<T> scan_inclusive(const std::vector<T>& items, const T& identity, Combine combine,
                              ScanTrace* trace = nullptr) {
  const size_t n = items.size();
  if (trace) trace->rounds = 0;
  if (n == 0) return {};
  size_t m = 1;
  while (m < n) m <<= 1;
  std::vector<T> cur(m, identity);
  std::copy(items.begin(), items.end(), cur.begin());
  std::vector<T> next(m, identity);
  for (size_t dist = 1; dist < m; dist <<= 1) {
    if (trace) ++trace->rounds;
    for (size_t i = 0; i < m; ++i) next[i] = (i >= dist) ? combine(cur[i - dist], cur[i]) : cur[i];
    cur.swap(next);
  }
  cur.resize(n);
  return cur;
}

// scan.hpp:82-97
template <int D>
struct AffineElement {
  Mat<D, D> coeff = Mat<D, D>::Identity();
  Mat<D, 1> offset = Mat<D, 1>::Zero();
  static AffineElement compose(const AffineElement& first, const AffineElement& second) {
    AffineElement o;
    o.coeff = second.coeff * first.coeff;
    o.offset = second.coeff * first.offset;
    o.offset += second.offset;
    return o;
  }
};

// scan.hpp:115-140. lower: x[0]=rhs[0], x[k]=coupling[k-1] x[k-1] + rhs[k]
template <int D>
std::vector<Mat<D, 1>> solve_lower_bidiag(const std::vector<Mat<D, D>>& coupling,
                                          const std::vector<Mat<D, 1>>& rhs, ScanTrace* trace = nullptr) {
  const size_t n = rhs.size();
  if (n == 0) {
    if (trace) trace->rounds = 0;
    return {};
  }
  std::vector<AffineElement<D>> steps(n);
  steps[0].offset = rhs[0];
  for (size_t k = 1; k < n; ++k) {
    steps[k].coeff = coupling[k - 1];
    steps[k].offset = rhs[k];
  }
  auto pre = scan_inclusive(steps, AffineElement<D>(), &AffineElement<D>::compose, trace);
  std::vector<Mat<D, 1>> x(n);
  for (size_t k = 0; k < n; ++k) x[k] = pre[k].offset;
  return x;
}

// scan.hpp:143-168. upper: x[n-1]=rhs[n-1], x[k]=coupling[k] x[k+1] + rhs[k]
template <int D>
std::vector<Mat<D, 1>> solve_upper_bidiag(const std::vector<Mat<D, D>>& coupling,
                                          const std::vector<Mat<D, 1>>& rhs, ScanTrace* trace = nullptr) {
  const size_t n = rhs.size();
  if (n == 0) {
    if (trace) trace->rounds = 0;
    return {};
  }
  std::vector<AffineElement<D>> steps(n);
  steps[0].offset = rhs[n - 1];
  for (size_t k = 1; k < n; ++k) {
    steps[k].coeff = coupling[n - 1 - k];
    steps[k].offset = rhs[n - 1 - k];
  }
  auto pre = scan_inclusive(steps, AffineElement<D>(), &AffineElement<D>::compose, trace);
  std::vector<Mat<D, 1>> x(n);
  for (size_t k = 0; k < n; ++k) x[n - 1 - k] = pre[k].offset;
  return x;
}

// ---------------------------------------------------------------------------
// Full-pivot LU with Eigen::FullPivLU semantics (used by oee.hpp:40-51,
// 194-233): pivot = largest |a| in the trailing corner (first in column-major
// order on ties), rank = #pivots with |p| > (B * eps) * |max pivot|,
// isInvertible <=> full rank.

template <int B>
struct FullPivLU {
  Mat<B, B> lu;
  int rowt[B], colt[B];
  int nonzero = B;
  double maxpivot = 0.0;
  explicit FullPivLU(const Mat<B, B>& m) : lu(m) {
    nonzero = B;
    maxpivot = 0.0;
    for (int k = 0; k < B; ++k) {
      double big = -1.0;
      int br = k, bc = k;
      for (int c = k; c < B; ++c)
        for (int r = k; r < B; ++r) {
          const double v = std::fabs(lu(r, c));
          if (v > big) {
            big = v;
            br = r;
            bc = c;
          }
        }
      if (big == 0.0) {
        nonzero = k;
        for (int i = k; i < B; ++i) rowt[i] = colt[i] = i;
        break;
      }
      if (big > maxpivot) maxpivot = big;
      rowt[k] = br;
      colt[k] = bc;
      if (br != k)
        for (int c = 0; c < B; ++c) std::swap(lu(k, c), lu(br, c));
      if (bc != k)
        for (int r = 0; r < B; ++r) std::swap(lu(r, k), lu(r, bc));
      for (int r = k + 1; r < B; ++r) lu(r, k) /= lu(k, k);
      for (int r = k + 1; r < B; ++r)
        for (int c = k + 1; c < B; ++c) lu(r, c) -= lu(r, k) * lu(k, c);
    }
  }
  int rank() const {
    const double thr = std::numeric_limits<double>::epsilon() * B;
    int r = 0;
    for (int i = 0; i < nonzero; ++i)
      if (std::fabs(lu(i, i)) > thr * std::fabs(maxpivot)) ++r;
    return r;
  }
  bool isInvertible() const { return rank() == B; }
  template <int M>
  Mat<B, M> solve(const Mat<B, M>& rhs) const {
    Mat<B, M> c = rhs;
    for (int k = 0; k < B; ++k)  // row permutation P
      if (rowt[k] != k)
        for (int j = 0; j < M; ++j) std::swap(c(k, j), c(rowt[k], j));
    for (int j = 0; j < M; ++j) {
      for (int r = 0; r < B; ++r)  // unit lower
        for (int k = 0; k < r; ++k) c(r, j) -= lu(r, k) * c(k, j);
      for (int r = B - 1; r >= 0; --r) {  // upper
        for (int k = r + 1; k < B; ++k) c(r, j) -= lu(r, k) * c(k, j);
        c(r, j) /= lu(r, r);
      }
    }
    for (int k = B - 1; k >= 0; --k)  // column permutation Q
      if (colt[k] != k)
        for (int j = 0; j < M; ++j) std::swap(c(k, j), c(colt[k], j));
    return c;
  }
};

// Cholesky with Eigen::LLT semantics: failure iff a pivot x <= 0 (Eigen's
// llt_inplace test -- a NaN pivot does not fail, the NaN propagates).
inline bool llt_inplace(double* a, int n) {  // row-major n x n; lower L on return
  for (int k = 0; k < n; ++k) {
    double x = a[k * n + k];
    for (int j = 0; j < k; ++j) x -= a[k * n + j] * a[k * n + j];
    if (x <= 0.0) return false;
    x = std::sqrt(x);
    a[k * n + k] = x;
    for (int i = k + 1; i < n; ++i) {
      double s = a[i * n + k];
      for (int j = 0; j < k; ++j) s -= a[i * n + j] * a[k * n + j];
      a[i * n + k] = s / x;
    }
  }
  return true;
}
inline void llt_solve(const double* L, int n, double* b) {
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i * n + k] * b[k];
    b[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * b[k];
    b[i] = s / L[i * n + i];
  }
}

// ---------------------------------------------------------------------------
// Odd-even elimination (include/pardyn/oee.hpp).

template <int B>
struct SymBlockTriDiag {  // oee.hpp:28-32
  std::vector<Mat<B, B>> diag, upper;
};

template <int B, int M>
Mat<B, M> coefficient_solve(const Mat<B, B>& pivot, const Mat<B, M>& rhs, int round, int index) {
  FullPivLU<B> lu(pivot);  // oee.hpp:40-51
  if (!lu.isInvertible())
    throw SingularBlockError(round, index,
                             "odd-even elimination: singular pivot block (round " + std::to_string(round) +
                                 ", block " + std::to_string(index) + ")");
  return lu.solve(rhs);
}

template <int B, int M = 1>
struct OeeState {  // oee.hpp:57-67
  std::vector<Mat<B, B>> diag, coupling;
  std::vector<Mat<B, M>> rhs;
  int distance = 1;
  int round = 0;
};

// oee.hpp:73-145 (row-centric Eq. 17; smallest failing row reported).
template <int B, int M>
void oee_eliminate_round(OeeState<B, M>& st) {
  const long n = static_cast<long>(st.diag.size());
  const long h = st.distance;
  const int round = st.round + 1;
  std::vector<Mat<B, B>> nd(n), nc(std::max<long>(n - 2 * h, 0));
  std::vector<Mat<B, M>> nr(n);
  long bad_row = n;
  int bad_pivot = 0;
  for (long i = 0; i < n; ++i) {
    try {
      Mat<B, B> d = st.diag[i];
      Mat<B, M> r = st.rhs[i];
      if (i < n - h) {
        const Mat<B, B> up = coefficient_solve<B, B>(st.diag[i + h], st.coupling[i].T(), round, (int)(i + h));
        d -= up.T() * st.coupling[i].T();
        r -= up.T() * st.rhs[i + h];
        if (i < n - 2 * h) nc[i] = -(up.T() * st.coupling[i + h]);
      }
      if (i >= h) {
        const Mat<B, B> dn = coefficient_solve<B, B>(st.diag[i - h], st.coupling[i - h], round, (int)(i - h));
        d -= dn.T() * st.coupling[i - h];
        r -= dn.T() * st.rhs[i - h];
      }
      nd[i] = d;
      nr[i] = r;
    } catch (const SingularBlockError& e) {
      if (i < bad_row) {
        bad_row = i;
        bad_pivot = e.index();
      }
    }
  }
  if (bad_row < n)
    throw SingularBlockError(round, bad_pivot,
                             "odd-even elimination: singular pivot block (round " + std::to_string(round) +
                                 ", block " + std::to_string(bad_pivot) + ")");
  st.diag.swap(nd);
  st.rhs.swap(nr);
  st.coupling.swap(nc);
  st.distance = static_cast<int>(2 * h);
  st.round = round;
}

// oee.hpp:149-189
template <int B, int M = 1>
std::vector<Mat<B, M>> oee_solve(const SymBlockTriDiag<B>& sys, const std::vector<Mat<B, M>>& rhs,
                                 OeeTrace* trace = nullptr) {
  const long n = static_cast<long>(sys.diag.size());
  if (trace) trace->rounds = 0;
  if (n == 0) return {};
  OeeState<B, M> st{sys.diag, sys.upper, rhs, 1, 0};
  const int rounds = ceil_log2(static_cast<size_t>(n));
  for (int j = 0; j < rounds; ++j) oee_eliminate_round(st);
  if (trace) trace->rounds = st.round;
  std::vector<Mat<B, M>> x(n);
  long bad_row = n;
  for (long i = 0; i < n; ++i) {
    try {
      x[i] = coefficient_solve<B, M>(st.diag[i], st.rhs[i], st.round, (int)i);
    } catch (const SingularBlockError&) {
      if (i < bad_row) bad_row = i;
    }
  }
  if (bad_row < n)
    throw SingularBlockError(st.round, (int)bad_row,
                             "odd-even elimination: singular diagonal block after elimination (block " +
                                 std::to_string(bad_row) + ")");
  return x;
}

// oee.hpp:194-233 (sequential oracle).
template <int B, int M = 1>
std::vector<Mat<B, M>> block_thomas_solve(const SymBlockTriDiag<B>& sys, const std::vector<Mat<B, M>>& rhs) {
  const long n = static_cast<long>(sys.diag.size());
  if (n == 0) return {};
  std::vector<Mat<B, B>> d = sys.diag;
  std::vector<Mat<B, M>> r = rhs;
  for (long i = 1; i < n; ++i) {
    FullPivLU<B> lu(d[i - 1]);
    if (!lu.isInvertible()) throw DynamicsError("block Thomas: singular pivot at row " + std::to_string(i - 1));
    const Mat<B, B> factor = lu.solve(sys.upper[i - 1]);
    d[i] -= sys.upper[i - 1].T() * factor;
    r[i] -= factor.T() * r[i - 1];
  }
  std::vector<Mat<B, M>> x(n);
  for (long i = n - 1; i >= 0; --i) {
    Mat<B, M> b = r[i];
    if (i < n - 1) b -= sys.upper[i] * x[i + 1];
    FullPivLU<B> lu(d[i]);
    if (!lu.isInvertible()) throw DynamicsError("block Thomas: singular pivot at row " + std::to_string(i));
    x[i] = lu.solve(b);
  }
  return x;
}

// ---------------------------------------------------------------------------
// Inverse dynamics (include/pardyn/inverse_dynamics.hpp, src/inverse_dynamics.cpp).

struct IdOptions {  // inverse_dynamics.hpp:23-28
  Vec6 base_velocity = Vec6::Zero();
  Vec6 base_acceleration = Vec6::Zero();
  Vec6 tip_wrench = Vec6::Zero();
  bool apply_gravity = true;
};

inline void check_joint_size(const ChainKinematics& kin, const VecX& v, const char* name) {
  if (static_cast<int>(v.size()) != kin.size())
    throw std::invalid_argument(std::string(name) + " has length " + std::to_string(v.size()) +
                                " but the chain has " + std::to_string(kin.size()) + " joints");
}

// inverse_dynamics.cpp:27-51
inline std::vector<Vec6> propagate_velocities(const ChainKinematics& kin, const VecX& qd, const Vec6& base_v,
                                              ScanTrace* trace = nullptr) {
  check_joint_size(kin, qd, "qdot");
  const int n = kin.size();
  if (n == 0) {
    if (trace) trace->rounds = 0;
    return {};
  }
  std::vector<Mat6> coupling(n - 1);
  std::vector<Vec6> rhs(n);
  for (int i = 0; i < n; ++i) {
    rhs[i] = qd[i] * kin.screw[i];
    if (i >= 1) coupling[i - 1] = kin.transport[i - 1];
  }
  rhs[0] += kin.base_transport * base_v;
  return solve_lower_bidiag<6>(coupling, rhs, trace);
}

// inverse_dynamics.cpp:53-84
inline std::vector<Vec6> propagate_accelerations(const ChainKinematics& kin, const std::vector<Vec6>& vel,
                                                 const VecX& qd, const VecX& qdd, const Vec6& base_a,
                                                 ScanTrace* trace = nullptr) {
  check_joint_size(kin, qd, "qdot");
  check_joint_size(kin, qdd, "qddot");
  const int n = kin.size();
  if (n == 0) {
    if (trace) trace->rounds = 0;
    return {};
  }
  std::vector<Mat6> coupling(n - 1);
  std::vector<Vec6> rhs(n);
  for (int i = 0; i < n; ++i) {
    const Vec6 rate = qd[i] * kin.screw[i];
    rhs[i] = qdd[i] * kin.screw[i] + small_adjoint(vel[i]) * rate;
    if (i >= 1) coupling[i - 1] = kin.transport[i - 1];
  }
  rhs[0] += kin.base_transport * base_a;
  return solve_lower_bidiag<6>(coupling, rhs, trace);
}

// inverse_dynamics.cpp:86-120
inline std::vector<Vec6> propagate_forces(const ChainKinematics& kin, const std::vector<Vec6>& vel,
                                          const std::vector<Vec6>& acc, const std::vector<Mat6>& inertia,
                                          const Vec6& tip_wrench, ScanTrace* trace = nullptr) {
  const int n = kin.size();
  if (n == 0) {
    if (trace) trace->rounds = 0;
    return {};
  }
  std::vector<Mat6> coupling(n - 1);
  std::vector<Vec6> rhs(n);
  for (int i = 0; i < n; ++i) {
    const Vec6 momentum = inertia[i] * vel[i];
    rhs[i] = inertia[i] * acc[i] - small_adjoint(vel[i]).T() * momentum;
    if (i + 1 < n) coupling[i] = kin.transport[i].T();
  }
  rhs[n - 1] += tip_wrench;
  return solve_upper_bidiag<6>(coupling, rhs, trace);
}

// inverse_dynamics.cpp:122-164
inline VecX inverse_dynamics_assembled(const ChainKinematics& kin, const std::vector<Mat6>& inertia,
                                       const Vec3& gravity, const VecX& qd, const VecX& qdd,
                                       const IdOptions& opts = {}, ExecTrace* trace = nullptr) {
  const int n = kin.size();
  ScanTrace sv, sa, sf;
  const auto vel = propagate_velocities(kin, qd, opts.base_velocity, &sv);
  Vec6 base_acc = opts.base_acceleration;
  if (opts.apply_gravity)
    for (int k = 0; k < 3; ++k) base_acc[3 + k] -= gravity[k];
  const auto acc = propagate_accelerations(kin, vel, qd, qdd, base_acc, &sa);
  const auto frc = propagate_forces(kin, vel, acc, inertia, opts.tip_wrench, &sf);
  VecX tau(n);
  for (int i = 0; i < n; ++i) tau[i] = dot(kin.screw[i], frc[i]);
  if (trace) {
    trace->note_scan(sv);
    trace->note_scan(sa);
    trace->note_scan(sf);
    for (int k = 0; k < 5; ++k) trace->note_parallel_stage();
  }
  return tau;
}

// inverse_dynamics.cpp:166-173
inline VecX inverse_dynamics(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& qdd,
                             const IdOptions& opts = {}, ExecTrace* trace = nullptr) {
  const ChainKinematics kin = assemble_kinematics(chain, q);
  const auto inertia = link_inertias(chain);
  return inverse_dynamics_assembled(kin, inertia, chain.gravity, qd, qdd, opts, trace);
}

// inverse_dynamics.cpp:175-179
inline VecX bias_torque(const RobotChain& chain, const VecX& q, const VecX& qd, ExecTrace* trace = nullptr) {
  return inverse_dynamics(chain, q, qd, VecX(chain.size(), 0.0), {}, trace);
}

struct LinkStates {
  std::vector<Vec6> velocity, acceleration, force;
};
// inverse_dynamics.cpp:181-196
inline LinkStates link_states(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& qdd,
                              const IdOptions& opts = {}) {
  const ChainKinematics kin = assemble_kinematics(chain, q);
  const auto inertia = link_inertias(chain);
  LinkStates s;
  s.velocity = propagate_velocities(kin, qd, opts.base_velocity);
  Vec6 base_acc = opts.base_acceleration;
  if (opts.apply_gravity)
    for (int k = 0; k < 3; ++k) base_acc[3 + k] -= chain.gravity[k];
  s.acceleration = propagate_accelerations(kin, s.velocity, qd, qdd, base_acc);
  s.force = propagate_forces(kin, s.velocity, s.acceleration, inertia, opts.tip_wrench);
  return s;
}

// ---------------------------------------------------------------------------
// Forward dynamics (include/pardyn/forward_dynamics.hpp, src/forward_dynamics.cpp).

enum class FdAlgo { jsiia = 0, abia = 1, cfa = 2 };

// forward_dynamics.cpp:19-31
inline void check_sizes(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& tau) {
  const size_t n = chain.links.size();
  if (n == 0) throw std::invalid_argument("forward dynamics: chain has no links");
  if (q.size() != n || qd.size() != n || tau.size() != n)
    throw std::invalid_argument(
        "forward dynamics: q, qdot and tau must each have one entry per joint (chain has " +
        std::to_string(n) + ")");
}

// forward_dynamics.cpp:35-42
inline VecX torque_surplus(const ChainKinematics& kin, const std::vector<Mat6>& inertia, const Vec3& gravity,
                           const VecX& qd, const VecX& tau, ExecTrace* trace) {
  const VecX zero(qd.size(), 0.0);
  const VecX id = inverse_dynamics_assembled(kin, inertia, gravity, qd, zero, IdOptions{}, trace);
  VecX out(tau.size());
  for (size_t i = 0; i < tau.size(); ++i) out[i] = tau[i] - id[i];
  return out;
}

// forward_dynamics.cpp:44-66
inline MatX joint_space_inertia_assembled(const ChainKinematics& kin, const std::vector<Mat6>& inertia,
                                          ExecTrace* trace) {
  const int n = kin.size();
  MatX m(n);
  if (trace) trace->note_parallel_stage();
  const VecX zero(n, 0.0);
  IdOptions opts;
  opts.apply_gravity = false;
  for (int j = 0; j < n; ++j) {
    VecX unit(n, 0.0);
    unit[j] = 1.0;
    const VecX col = inverse_dynamics_assembled(kin, inertia, Vec3::Zero(), zero, unit, opts,
                                                j == 0 ? trace : nullptr);
    for (int i = 0; i < n; ++i) m(i, j) = col[i];
  }
  MatX s(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) s(i, j) = 0.5 * (m(i, j) + m(j, i));
  return s;
}

// forward_dynamics.cpp:70-80
inline MatX joint_space_inertia(const RobotChain& chain, const VecX& q, ExecTrace* trace = nullptr) {
  if (static_cast<int>(q.size()) != chain.size())
    throw std::invalid_argument("joint_space_inertia: q must have one entry per joint");
  const ChainKinematics kin = assemble_kinematics(chain, q);
  return joint_space_inertia_assembled(kin, link_inertias(chain), trace);
}

// forward_dynamics.cpp:82-118
inline VecX jsiia_forward_dynamics(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& tau,
                                   ExecTrace* trace = nullptr) {
  check_sizes(chain, q, qd, tau);
  const ChainKinematics kin = assemble_kinematics(chain, q);
  const auto inertia = link_inertias(chain);
  const VecX surplus = torque_surplus(kin, inertia, chain.gravity, qd, tau, trace);
  const MatX m = joint_space_inertia_assembled(kin, inertia, trace);
  const int n = m.n;
  std::vector<double> L = m.a;
  if (!llt_inplace(L.data(), n))
    throw DynamicsError("joint-space inertia is not positive definite; the chain model is degenerate");
  VecX qdd = surplus;
  llt_solve(L.data(), n, qdd.data());
  const double scale = std::max(vnorm(surplus), std::numeric_limits<double>::min());
  auto residual_of = [&](const VecX& x) {
    VecX r(n);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += m(i, j) * x[j];
      r[i] = surplus[i] - s;
    }
    return r;
  };
  VecX res = residual_of(qdd);
  if (vnorm(res) > 1e-9 * scale) {
    llt_solve(L.data(), n, res.data());
    for (int i = 0; i < n; ++i) qdd[i] += res[i];
    res = residual_of(qdd);
    if (vnorm(res) > 1e-9 * scale)
      throw DynamicsError(
          "joint-space inertia solve failed to reach the required residual; the inertia matrix is too "
          "ill-conditioned");
  }
  return qdd;
}

struct ArticulatedBodyInertias {  // forward_dynamics.hpp:48-52
  std::vector<Mat6> inertia;
  VecX joint_inertia;
  std::vector<Vec6> gain;
};

// forward_dynamics.cpp:120-163 (sequential tip-to-base recursion).
inline ArticulatedBodyInertias articulated_body_inertias(const ChainKinematics& kin,
                                                         const std::vector<Mat6>& inertia,
                                                         ExecTrace* trace = nullptr) {
  const size_t n = kin.size();
  ArticulatedBodyInertias out;
  if (n == 0) return out;
  out.inertia.resize(n);
  out.joint_inertia.resize(n);
  out.gain.resize(n);
  out.inertia[n - 1] = inertia[n - 1];
  for (size_t i = n; i-- > 0;) {
    const Vec6& s = kin.screw[i];
    const Vec6 Is = out.inertia[i] * s;
    const double lambda = dot(s, Is);
    if (!(lambda > 1e-14 * mtrace(out.inertia[i])))
      throw DynamicsError("degenerate articulation at joint " + std::to_string(i) +
                          ": projected articulated inertia vanishes");
    out.joint_inertia[i] = lambda;
    for (int k = 0; k < 6; ++k) out.gain[i][k] = Is[k] / lambda;
    if (i > 0) {
      // projected = I - (I s)(I s)^T / lambda, carried across joint i-1.
      const Mat6 outer = Is * Is.T();
      Mat6 proj;
      for (int k = 0; k < 36; ++k) proj[k] = out.inertia[i][k] - outer[k] / lambda;
      const Mat6 carried = kin.transport[i - 1].T() * proj * kin.transport[i - 1];
      const Mat6 assembled = inertia[i - 1] + carried;
      out.inertia[i - 1] = 0.5 * (assembled + assembled.T());
    }
  }
  if (trace) trace->note_sequential_chain(static_cast<int>(n));
  return out;
}

// forward_dynamics.cpp:165-243
inline VecX abia_forward_dynamics(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& tau,
                                  ExecTrace* trace = nullptr) {
  check_sizes(chain, q, qd, tau);
  const size_t n = chain.links.size();
  const ChainKinematics kin = assemble_kinematics(chain, q);
  const auto inertia = link_inertias(chain);
  const VecX surplus = torque_surplus(kin, inertia, chain.gravity, qd, tau, trace);
  const ArticulatedBodyInertias ab = articulated_body_inertias(kin, inertia, trace);

  std::vector<Mat6> fc(n - 1);
  std::vector<Vec6> fr(n, Vec6::Zero());
  for (size_t i = 0; i + 1 < n; ++i) {
    const Vec6& ns = kin.screw[i + 1];
    const Mat6 yield = Mat6::Identity() - ab.gain[i + 1] * ns.T();
    fc[i] = kin.transport[i].T() * yield;
    fr[i] = kin.transport[i].T() * (surplus[i + 1] * ab.gain[i + 1]);
  }
  ScanTrace fs;
  const auto z = solve_upper_bidiag<6>(fc, fr, trace ? &fs : nullptr);

  std::vector<Mat6> ac(n - 1);
  std::vector<Vec6> ar(n);
  for (size_t i = 0; i < n; ++i) {
    const Vec6& s = kin.screw[i];
    const double free_rate = (surplus[i] - dot(s, z[i])) / ab.joint_inertia[i];
    ar[i] = free_rate * s;
    if (i > 0) {
      const Mat6 yield = Mat6::Identity() - s * ab.gain[i].T();
      ac[i - 1] = yield * kin.transport[i - 1];
    }
  }
  ScanTrace as;
  const auto accel = solve_lower_bidiag<6>(ac, ar, trace ? &as : nullptr);

  VecX qdd(n);
  for (size_t i = 0; i < n; ++i) {
    const Vec6& s = kin.screw[i];
    double value = (surplus[i] - dot(s, z[i])) / ab.joint_inertia[i];
    if (i > 0) {
      const Vec6 pa = kin.transport[i - 1] * accel[i - 1];
      value -= dot(ab.gain[i], pa);
    }
    qdd[i] = value;
  }
  if (trace) {
    trace->note_scan(fs);
    trace->note_scan(as);
    trace->note_parallel_stage();
  }
  return qdd;
}

// Eigen::HouseholderQR of a 6x1 column, then householderQ() * Identity
// (forward_dynamics.cpp:245-259): makeHouseholder + applyHouseholderOnTheLeft.
inline Mat6 householder_q_of(const Vec6& s) {
  double tail_sq = 0.0;
  for (int i = 1; i < 6; ++i) tail_sq += s[i] * s[i];
  const double c0 = s[0];
  double tau, beta;
  double ess[5];
  if (tail_sq <= std::numeric_limits<double>::min()) {
    tau = 0.0;
    beta = c0;
    for (double& e : ess) e = 0.0;
  } else {
    beta = std::sqrt(c0 * c0 + tail_sq);
    if (c0 >= 0.0) beta = -beta;
    for (int i = 0; i < 5; ++i) ess[i] = s[i + 1] / (c0 - beta);
    tau = (beta - c0) / beta;
  }
  (void)beta;
  Mat6 Q = Mat6::Identity();
  if (tau != 0.0) {
    for (int c = 0; c < 6; ++c) {
      double tmp = 0.0;  // essential^T * bottom
      for (int r = 1; r < 6; ++r) tmp += ess[r - 1] * Q(r, c);
      tmp += Q(0, c);
      Q(0, c) -= tau * tmp;
      for (int r = 1; r < 6; ++r) Q(r, c) -= tau * ess[r - 1] * tmp;
    }
  }
  return Q;
}

struct ConstraintBasis {
  std::vector<Mat65> basis;
};
inline ConstraintBasis build_constraint_basis(const RobotChain& chain) {
  ConstraintBasis out;
  out.basis.resize(chain.links.size());
  for (size_t k = 0; k < chain.links.size(); ++k) {
    const Mat6 Q = householder_q_of(chain.links[k].joint_screw);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 5; ++c) out.basis[k](r, c) = Q(r, c + 1);
  }
  return out;
}

struct CfaOperators {  // forward_dynamics.hpp:80-91
  SymBlockTriDiag<5> constraint_op;
  std::vector<Vec5> cross_sub, cross_diag, cross_super;
  VecX joint_diag, joint_off;

  std::vector<Vec5> apply_cross(const VecX& v) const {  // :359-376
    const size_t n = cross_diag.size();
    std::vector<Vec5> out(n);
    for (size_t i = 0; i < n; ++i) {
      Vec5 val = v[i] * cross_diag[i];
      if (i > 0) val += v[i - 1] * cross_sub[i - 1];
      if (i + 1 < n) val += v[i + 1] * cross_super[i];
      out[i] = val;
    }
    return out;
  }
  VecX apply_cross_transpose(const std::vector<Vec5>& f) const {  // :378-399
    const size_t n = cross_diag.size();
    if (f.size() != n)
      throw std::invalid_argument("apply_cross_transpose: one constraint block per link expected");
    VecX out(n);
    for (size_t i = 0; i < n; ++i) {
      double val = dot(cross_diag[i], f[i]);
      if (i + 1 < n) val += dot(cross_sub[i], f[i + 1]);
      if (i > 0) val += dot(cross_super[i - 1], f[i - 1]);
      out[i] = val;
    }
    return out;
  }
  VecX apply_joint(const VecX& v) const {  // :401-416
    const size_t n = joint_diag.size();
    VecX out(n);
    for (size_t k = 0; k < n; ++k) {
      double val = joint_diag[k] * v[k];
      if (k > 0) val += joint_off[k - 1] * v[k - 1];
      if (k + 1 < n) val += joint_off[k] * v[k + 1];
      out[k] = val;
    }
    return out;
  }
};

// Solve J x = b column-wise with a precomputed 6x6 Cholesky factor.
template <int M>
inline Mat<6, M> llt6_solve(const Mat6& L, const Mat<6, M>& b) {
  Mat<6, M> x = b;
  for (int c = 0; c < M; ++c) {
    double col[6];
    for (int r = 0; r < 6; ++r) col[r] = x(r, c);
    llt_solve(L.a, 6, col);
    for (int r = 0; r < 6; ++r) x(r, c) = col[r];
  }
  return x;
}

// forward_dynamics.cpp:261-357
inline CfaOperators build_cfa_operators(const RobotChain& chain, const ChainKinematics& kin,
                                        const ConstraintBasis& basis, ExecTrace* trace = nullptr) {
  const size_t n = chain.links.size();
  if (n == 0) throw std::invalid_argument("build_cfa_operators: chain has no links");
  if (basis.basis.size() != n || static_cast<size_t>(kin.size()) != n)
    throw std::invalid_argument("build_cfa_operators: kinematics and basis must match the chain");
  const auto inertia = link_inertias(chain);
  CfaOperators ops;
  ops.constraint_op.diag.resize(n);
  ops.constraint_op.upper.resize(n - 1);
  ops.cross_sub.resize(n - 1);
  ops.cross_diag.resize(n);
  ops.cross_super.resize(n - 1);
  ops.joint_diag.resize(n);
  ops.joint_off.resize(n - 1);

  std::vector<Mat65> sb(n), cb(n - 1), scb(n - 1);
  std::vector<Vec6> ss(n), cs(n - 1), scs(n - 1);
  bool llt_failed = false;
  for (size_t i = 0; i < n; ++i) {
    Mat6 L = inertia[i];
    if (!llt_inplace(L.a, 6)) {
      llt_failed = true;
      continue;
    }
    sb[i] = llt6_solve<5>(L, basis.basis[i]);
    ss[i] = llt6_solve<1>(L, kin.screw[i]);
    if (i + 1 < n) {
      cb[i] = kin.transport[i].T() * basis.basis[i + 1];
      cs[i] = kin.transport[i].T() * kin.screw[i + 1];
      scb[i] = llt6_solve<5>(L, cb[i]);
      scs[i] = llt6_solve<1>(L, cs[i]);
    }
  }
  if (llt_failed) throw DynamicsError("constraint-force assembly: a link inertia is not positive definite");
  if (trace) trace->note_parallel_stage();

  for (size_t i = 0; i < n; ++i) {
    const Mat65& w = basis.basis[i];
    const Vec6& s = kin.screw[i];
    Mat5 a_diag = w.T() * sb[i];
    Vec5 b_diag = w.T() * ss[i];
    double c_diag = dot(s, ss[i]);
    if (i > 0) {
      a_diag += cb[i - 1].T() * scb[i - 1];
      b_diag += cb[i - 1].T() * scs[i - 1];
      c_diag += dot(cs[i - 1], scs[i - 1]);
    }
    ops.constraint_op.diag[i] = 0.5 * (a_diag + a_diag.T());
    ops.cross_diag[i] = b_diag;
    ops.joint_diag[i] = c_diag;
    if (i + 1 < n) {
      ops.constraint_op.upper[i] = -(w.T() * scb[i]);
      ops.cross_super[i] = -(w.T() * scs[i]);
      ops.cross_sub[i] = -(cb[i].T() * ss[i]);
      ops.joint_off[i] = -dot(s, scs[i]);
    }
  }
  if (trace) trace->note_parallel_stage();
  return ops;
}

// forward_dynamics.cpp:418-450 (Algorithm 1 of the paper).
inline VecX cfa_forward_dynamics(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& tau,
                                 ExecTrace* trace = nullptr) {
  check_sizes(chain, q, qd, tau);
  const ChainKinematics kin = assemble_kinematics(chain, q);
  const auto inertia = link_inertias(chain);
  const VecX surplus = torque_surplus(kin, inertia, chain.gravity, qd, tau, trace);
  const ConstraintBasis basis = build_constraint_basis(chain);
  const CfaOperators ops = build_cfa_operators(chain, kin, basis, trace);
  std::vector<Vec5> rhs = ops.apply_cross(surplus);
  for (Vec5& b : rhs) b = -b;
  OeeTrace ot;
  const auto fcon = oee_solve<5, 1>(ops.constraint_op, rhs, trace ? &ot : nullptr);
  VecX qdd = ops.apply_joint(surplus);
  const VecX extra = ops.apply_cross_transpose(fcon);
  for (size_t i = 0; i < qdd.size(); ++i) qdd[i] += extra[i];
  if (trace) {
    trace->note_oee(ot);
    trace->note_parallel_stage();
    trace->note_parallel_stage();
  }
  return qdd;
}

// forward_dynamics.cpp:452-464
inline VecX forward_dynamics(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& tau, FdAlgo algo,
                             ExecTrace* trace = nullptr) {
  switch (algo) {
    case FdAlgo::jsiia:
      return jsiia_forward_dynamics(chain, q, qd, tau, trace);
    case FdAlgo::abia:
      return abia_forward_dynamics(chain, q, qd, tau, trace);
    case FdAlgo::cfa:
      return cfa_forward_dynamics(chain, q, qd, tau, trace);
  }
  throw std::invalid_argument("forward_dynamics: unknown algorithm");
}

// ---------------------------------------------------------------------------
// Sequential / dense oracles of the reference test suite
// (tests/support/oracles.hpp), used to pin this restatement.

// oracles.hpp:203-255 (sequential Newton-Euler, no scans).
inline LinkStates newton_euler(const RobotChain& chain, const VecX& q, const VecX& qd, const VecX& qdd,
                               bool apply_gravity, VecX* torque) {
  const int n = chain.size();
  LinkStates st;
  st.velocity.resize(n);
  st.acceleration.resize(n);
  st.force.resize(n);
  std::vector<Mat6> ad(n), inertia(n);
  std::vector<Vec6> screw(n);
  for (int i = 0; i < n; ++i) {
    const LinkSpec& l = chain.links[i];
    ad[i] = adjoint_of(screw_exp(l.joint_screw, -q[i]) * l.home);
    screw[i] = l.joint_screw;
    inertia[i] = spatial_inertia_from(l.mass, l.com, l.inertia_rot);
  }
  Vec6 bv = Vec6::Zero(), ba = Vec6::Zero();
  if (apply_gravity)
    for (int k = 0; k < 3; ++k) ba[3 + k] = -chain.gravity[k];
  for (int i = 0; i < n; ++i) {
    const Vec6 pv = i == 0 ? bv : st.velocity[i - 1];
    const Vec6 pa = i == 0 ? ba : st.acceleration[i - 1];
    const Vec6 v = ad[i] * pv + qd[i] * screw[i];
    const Vec6 a = ad[i] * pa + qdd[i] * screw[i] + small_adjoint(v) * (qd[i] * screw[i]);
    st.velocity[i] = v;
    st.acceleration[i] = a;
  }
  if (torque) torque->assign(n, 0.0);
  for (int i = n - 1; i >= 0; --i) {
    Vec6 f = inertia[i] * st.acceleration[i] - small_adjoint(st.velocity[i]).T() * (inertia[i] * st.velocity[i]);
    if (i + 1 < n) f += ad[i + 1].T() * st.force[i + 1];
    st.force[i] = f;
    if (torque) (*torque)[i] = dot(screw[i], f);
  }
  return st;
}

}  // namespace oracle
