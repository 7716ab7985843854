// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
// extern "C" surface of the CPU oracle (oracle.hpp) for the Python tests and
// for bench.py's CPU-baseline / --impl reference arm (ctypes). All arrays are
// flat row-major doubles; a chain is n x 31 LinkSpec records (see
// oracle.hpp kLinkFields). Return value = status code with the same meaning
// as the product C-ABI's pd_status (include/pardyn_c.h).
#include <omp.h>

#include <cstdio>
#include <cstring>

#include "oracle.hpp"

using namespace oracle;

namespace {

enum {
  ST_OK = 0,
  ST_INVALID_ARGUMENT = 1,
  ST_MODEL_ERROR = 2,
  ST_DYNAMICS_ERROR = 3,
  ST_SINGULAR_BLOCK = 4,
  ST_INTERNAL = 7,
};

void put_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
  }
}

// Maps the reference's exception classes to status codes.
template <class F>
int guarded(F&& f, char* err, int errlen, int* err_round = nullptr, int* err_index = nullptr) {
  try {
    f();
    put_err(err, errlen, "");
    return ST_OK;
  } catch (const SingularBlockError& e) {
    if (err_round) *err_round = e.round();
    if (err_index) *err_index = e.index();
    put_err(err, errlen, e.what());
    return ST_SINGULAR_BLOCK;
  } catch (const DynamicsError& e) {
    put_err(err, errlen, e.what());
    return ST_DYNAMICS_ERROR;
  } catch (const ModelError& e) {
    put_err(err, errlen, e.what());
    return ST_MODEL_ERROR;
  } catch (const std::invalid_argument& e) {
    put_err(err, errlen, e.what());
    return ST_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return ST_INTERNAL;
  }
}

VecX vec(const double* p, int n) { return p ? VecX(p, p + n) : VecX(n, 0.0); }
void out_vec(const VecX& v, double* p) { std::copy(v.begin(), v.end(), p); }
template <int R, int C>
void out_mat(const Mat<R, C>& m, double* p) {
  std::memcpy(p, m.a, sizeof(double) * R * C);
}
template <int R, int C>
Mat<R, C> in_mat(const double* p) {
  Mat<R, C> m;
  std::memcpy(m.a, p, sizeof(double) * R * C);
  return m;
}

// bench.cpp:42-47
uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace

extern "C" {

int orc_num_threads(void) { return omp_get_max_threads(); }

uint64_t orc_mt19937_64_nth(uint64_t seed, int64_t nth) {
  std::mt19937_64 e(seed);
  uint64_t v = 0;
  for (int64_t i = 0; i < nth; ++i) v = e();
  return v;
}

uint64_t orc_mix(uint64_t x) { return mix(x); }

// bench.cpp:350-355
uint64_t orc_workload_seed(uint64_t seed, int n_links, int n_groups) {
  uint64_t h = mix(seed);
  h = mix(h ^ static_cast<uint64_t>(n_links));
  h = mix(h ^ (static_cast<uint64_t>(n_groups) << 20));
  return h;
}

int orc_random_chain(int n, uint64_t seed, double* links, double* gravity3, char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = random_chain(n, seed);
        for (int i = 0; i < n; ++i) link_to_flat(c.links[i], links + static_cast<size_t>(i) * kLinkFields);
        if (gravity3)
          for (int k = 0; k < 3; ++k) gravity3[k] = c.gravity[k];
      },
      err, errlen);
}

// bench.cpp:357-366 -- chains [g0, g0+count) of the cell, OpenMP over chains
// (each chain has its own seed, so the result is thread-count independent).
int orc_workload_chains(uint64_t cell_seed, int n_links, int64_t g0, int64_t count, double* links) {
  int status = ST_OK;
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < count; ++g) {
    try {
      const RobotChain c = random_chain(n_links, mix(cell_seed ^ (0xC0FFEEULL + static_cast<uint64_t>(g0 + g))));
      double* dst = links + static_cast<size_t>(g) * n_links * kLinkFields;
      for (int i = 0; i < n_links; ++i) link_to_flat(c.links[i], dst + static_cast<size_t>(i) * kLinkFields);
    } catch (...) {
#pragma omp critical
      status = ST_INTERNAL;
    }
  }
  return status;
}

// bench.cpp:368-383 -- q, qdot, drive for every group member, [group][link].
void orc_workload_inputs(uint64_t cell_seed, int n_links, int64_t n_groups, int64_t repeat, double* q,
                         double* qd, double* drive) {
  std::mt19937_64 eng(mix(cell_seed ^ (0x5EEDULL + static_cast<uint64_t>(repeat) * 0x9e3779b97f4a7c15ULL)));
  auto sym = [&] { return 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0; };
  for (int64_t g = 0; g < n_groups; ++g) {
    for (int i = 0; i < n_links; ++i) q[g * n_links + i] = sym();
    for (int i = 0; i < n_links; ++i) qd[g * n_links + i] = sym();
    for (int i = 0; i < n_links; ++i) drive[g * n_links + i] = sym();
  }
}

int orc_validate_chain(int n, const double* links, const double* gravity, char* err, int errlen) {
  return guarded([&] { validate_chain(chain_from_flat(n, links, gravity)); }, err, errlen);
}

int orc_spatial_inertia(double mass, const double* com, const double* Ic, double* out36, char* err, int errlen) {
  return guarded([&] { out_mat(spatial_inertia_from(mass, in_mat<3, 1>(com), in_mat<3, 3>(Ic)), out36); },
                 err, errlen);
}

void orc_screw_exp(const double* s6, double q, double* R9, double* p3) {
  const SE3 t = screw_exp(in_mat<6, 1>(s6), q);
  out_mat(t.R, R9);
  out_mat(t.p, p3);
}

void orc_small_adjoint(const double* v6, double* out36) { out_mat(small_adjoint(in_mat<6, 1>(v6)), out36); }

void orc_adjoint_of(const double* R9, const double* p3, double* out36) {
  SE3 t;
  t.R = in_mat<3, 3>(R9);
  t.p = in_mat<3, 1>(p3);
  out_mat(adjoint_of(t), out36);
}

// rel: n x 12 (R row-major, p); transport: (n-1) x 36; base: 36.
int orc_assemble_kinematics(int n, const double* links, const double* q, double* rel, double* transport,
                            double* base36, char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, nullptr);
        const ChainKinematics k = assemble_kinematics(c, vec(q, n));
        for (int i = 0; i < n; ++i) {
          out_mat(k.rel[i].R, rel + 12 * i);
          out_mat(k.rel[i].p, rel + 12 * i + 9);
        }
        for (int i = 0; i + 1 < n; ++i) out_mat(k.transport[i], transport + 36 * i);
        if (n > 0) out_mat(k.base_transport, base36);
      },
      err, errlen);
}

// opts: base_velocity[6], base_acceleration[6], tip_wrench[6] (nullable).
int orc_inverse_dynamics(int n, const double* links, const double* gravity, const double* q, const double* qd,
                         const double* qdd, const double* base_v, const double* base_a, const double* tip,
                         int apply_gravity, double* tau, int* trace4, char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, gravity);
        IdOptions o;
        if (base_v) o.base_velocity = in_mat<6, 1>(base_v);
        if (base_a) o.base_acceleration = in_mat<6, 1>(base_a);
        if (tip) o.tip_wrench = in_mat<6, 1>(tip);
        o.apply_gravity = apply_gravity != 0;
        ExecTrace tr;
        out_vec(inverse_dynamics(c, vec(q, n), vec(qd, n), vec(qdd, n), o, trace4 ? &tr : nullptr), tau);
        if (trace4) {
          trace4[0] = tr.parallel_link_stages;
          trace4[1] = tr.longest_sequential_link_chain;
          trace4[2] = tr.scan_rounds_max;
          trace4[3] = tr.oee_rounds;
        }
      },
      err, errlen);
}

int orc_link_states(int n, const double* links, const double* gravity, const double* q, const double* qd,
                    const double* qdd, const double* base_v, const double* base_a, const double* tip,
                    int apply_gravity, double* vel, double* acc, double* frc, char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, gravity);
        IdOptions o;
        if (base_v) o.base_velocity = in_mat<6, 1>(base_v);
        if (base_a) o.base_acceleration = in_mat<6, 1>(base_a);
        if (tip) o.tip_wrench = in_mat<6, 1>(tip);
        o.apply_gravity = apply_gravity != 0;
        const LinkStates s = link_states(c, vec(q, n), vec(qd, n), vec(qdd, n), o);
        for (int i = 0; i < n; ++i) {
          out_mat(s.velocity[i], vel + 6 * i);
          out_mat(s.acceleration[i], acc + 6 * i);
          out_mat(s.force[i], frc + 6 * i);
        }
      },
      err, errlen);
}

// oracles.hpp:203-263 sequential Newton-Euler (states + torque).
int orc_newton_euler(int n, const double* links, const double* gravity, const double* q, const double* qd,
                     const double* qdd, int apply_gravity, double* vel, double* acc, double* frc, double* tau,
                     char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, gravity);
        VecX t;
        const LinkStates s = newton_euler(c, vec(q, n), vec(qd, n), vec(qdd, n), apply_gravity != 0, &t);
        for (int i = 0; i < n; ++i) {
          if (vel) out_mat(s.velocity[i], vel + 6 * i);
          if (acc) out_mat(s.acceleration[i], acc + 6 * i);
          if (frc) out_mat(s.force[i], frc + 6 * i);
        }
        out_vec(t, tau);
      },
      err, errlen);
}

int orc_joint_space_inertia(int n, const double* links, const double* gravity, const double* q, double* M,
                            char* err, int errlen) {
  return guarded(
      [&] {
        const MatX m = joint_space_inertia(chain_from_flat(n, links, gravity), vec(q, n));
        std::copy(m.a.begin(), m.a.end(), M);
      },
      err, errlen);
}

// nq / nqd / ntau are the vector lengths (check_sizes sees the true lengths).
int orc_forward_dynamics(int algo, int n, const double* links, const double* gravity, const double* q, int nq,
                         const double* qd, int nqd, const double* tau, int ntau, double* qdd, int* trace4,
                         int* err_round, int* err_index, char* err, int errlen) {
  return guarded(
      [&] {
        if (algo < 0 || algo > 2) throw std::invalid_argument("forward_dynamics: unknown algorithm");
        const RobotChain c = chain_from_flat(n, links, gravity);
        ExecTrace tr;
        const VecX out = forward_dynamics(c, vec(q, nq), vec(qd, nqd), vec(tau, ntau), static_cast<FdAlgo>(algo),
                                          trace4 ? &tr : nullptr);
        out_vec(out, qdd);
        if (trace4) {
          trace4[0] = tr.parallel_link_stages;
          trace4[1] = tr.longest_sequential_link_chain;
          trace4[2] = tr.scan_rounds_max;
          trace4[3] = tr.oee_rounds;
        }
      },
      err, errlen, err_round, err_index);
}

// forward_dynamics.cpp:466-481: OpenMP dynamic over problems, per-slot
// status. Uniform n. Problem p uses model (n_models == 1 ? 0 : p); models are
// [model][link][31], gravity [model][3]; q/qd/tau/qdd are [problem][link].
// nthreads <= 0 keeps the OpenMP default.
void orc_batch_forward_dynamics(int algo, int64_t n_problems, int n, int64_t n_models, const double* links,
                                const double* gravity, const double* q, const double* qd, const double* tau,
                                double* qdd, int* status, int nthreads) {
  std::vector<RobotChain> chains(static_cast<size_t>(n_models));
  for (int64_t m = 0; m < n_models; ++m)
    chains[m] = chain_from_flat(n, links + static_cast<size_t>(m) * n * kLinkFields, gravity + 3 * m);
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic) num_threads(nt)
  for (int64_t p = 0; p < n_problems; ++p) {
    const RobotChain& c = chains[n_models == 1 ? 0 : p];
    int st = guarded(
        [&] {
          const VecX out = forward_dynamics(c, vec(q + p * n, n), vec(qd + p * n, n), vec(tau + p * n, n),
                                            static_cast<FdAlgo>(algo));
          out_vec(out, qdd + p * n);
        },
        nullptr, 0);
    if (status) status[p] = st;
  }
}

// Articulated-body inertias: inertia n x 36, joint_inertia n, gain n x 6.
int orc_articulated_body_inertias(int n, const double* links, const double* q, double* inertia, double* lam,
                                  double* gain, char* err, int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, nullptr);
        const ChainKinematics k = assemble_kinematics(c, vec(q, n));
        const auto ab = articulated_body_inertias(k, link_inertias(c));
        for (int i = 0; i < n; ++i) {
          out_mat(ab.inertia[i], inertia + 36 * i);
          lam[i] = ab.joint_inertia[i];
          out_mat(ab.gain[i], gain + 6 * i);
        }
      },
      err, errlen);
}

void orc_constraint_basis(int n, const double* links, double* basis /* n x 6 x 5 */) {
  const ConstraintBasis b = build_constraint_basis(chain_from_flat(n, links, nullptr));
  for (int i = 0; i < n; ++i) out_mat(b.basis[i], basis + 30 * i);
}

int orc_cfa_operators(int n, const double* links, const double* q, double* diag, double* upper, double* cross_sub,
                      double* cross_diag, double* cross_super, double* joint_diag, double* joint_off, char* err,
                      int errlen) {
  return guarded(
      [&] {
        const RobotChain c = chain_from_flat(n, links, nullptr);
        const ChainKinematics k = assemble_kinematics(c, vec(q, n));
        const CfaOperators ops = build_cfa_operators(c, k, build_constraint_basis(c));
        for (int i = 0; i < n; ++i) {
          out_mat(ops.constraint_op.diag[i], diag + 25 * i);
          out_mat(ops.cross_diag[i], cross_diag + 5 * i);
          joint_diag[i] = ops.joint_diag[i];
          if (i + 1 < n) {
            out_mat(ops.constraint_op.upper[i], upper + 25 * i);
            out_mat(ops.cross_sub[i], cross_sub + 5 * i);
            out_mat(ops.cross_super[i], cross_super + 5 * i);
            joint_off[i] = ops.joint_off[i];
          }
        }
      },
      err, errlen);
}

// Block bi-diagonal solve via the Hillis-Steele scan (D in {1,2,6}).
int orc_bidiag_solve(int D, int upper, int n, const double* coupling, const double* rhs, double* x, int* rounds) {
  ScanTrace tr;
  auto run = [&](auto tag) {
    constexpr int DD = decltype(tag)::value;
    std::vector<Mat<DD, DD>> c(n > 0 ? n - 1 : 0);
    std::vector<Mat<DD, 1>> r(n);
    for (int k = 0; k + 1 < n; ++k) c[k] = in_mat<DD, DD>(coupling + DD * DD * k);
    for (int k = 0; k < n; ++k) r[k] = in_mat<DD, 1>(rhs + DD * k);
    auto out = upper ? solve_upper_bidiag<DD>(c, r, &tr) : solve_lower_bidiag<DD>(c, r, &tr);
    for (int k = 0; k < n; ++k) out_mat(out[k], x + DD * k);
  };
  if (D == 1)
    run(std::integral_constant<int, 1>{});
  else if (D == 2)
    run(std::integral_constant<int, 2>{});
  else if (D == 6)
    run(std::integral_constant<int, 6>{});
  else
    return ST_INVALID_ARGUMENT;
  if (rounds) *rounds = tr.rounds;
  return ST_OK;
}

// Integer prefix sum through the same scan (test_scan.cpp:11-26).
void orc_scan_int64(int n, const int64_t* items, int64_t* out, int* rounds) {
  ScanTrace tr;
  std::vector<int64_t> v(items, items + n);
  auto r = scan_inclusive(v, int64_t{0}, [](int64_t a, int64_t b) { return a + b; }, &tr);
  std::copy(r.begin(), r.end(), out);
  if (rounds) *rounds = tr.rounds;
}

}  // extern "C"

namespace {
template <int B, int M>
int oee_dispatch(int n, const double* diag, const double* upper, const double* rhs, double* x, int* rounds,
                 int* err_round, int* err_index, char* err, int errlen, bool thomas) {
  return guarded(
      [&] {
        SymBlockTriDiag<B> s;
        s.diag.resize(n);
        s.upper.resize(n > 0 ? n - 1 : 0);
        std::vector<Mat<B, M>> r(n);
        for (int k = 0; k < n; ++k) s.diag[k] = in_mat<B, B>(diag + B * B * k);
        for (int k = 0; k + 1 < n; ++k) s.upper[k] = in_mat<B, B>(upper + B * B * k);
        for (int k = 0; k < n; ++k) r[k] = in_mat<B, M>(rhs + B * M * k);
        OeeTrace tr;
        auto out = thomas ? block_thomas_solve<B, M>(s, r) : oee_solve<B, M>(s, r, &tr);
        for (int k = 0; k < n; ++k) out_mat(out[k], x + B * M * k);
        if (rounds) *rounds = tr.rounds;
      },
      err, errlen, err_round, err_index);
}
template <int B, int M>
int oee_round_dispatch(int n, int distance, int round, double* diag, double* coupling, double* rhs) {
  OeeState<B, M> st;
  st.distance = distance;
  st.round = round;
  const int nc = std::max(n - distance, 0);
  st.diag.resize(n);
  st.coupling.resize(nc);
  st.rhs.resize(n);
  for (int k = 0; k < n; ++k) st.diag[k] = in_mat<B, B>(diag + B * B * k);
  for (int k = 0; k < nc; ++k) st.coupling[k] = in_mat<B, B>(coupling + B * B * k);
  for (int k = 0; k < n; ++k) st.rhs[k] = in_mat<B, M>(rhs + B * M * k);
  return guarded(
      [&] {
        oee_eliminate_round(st);
        for (int k = 0; k < n; ++k) out_mat(st.diag[k], diag + B * B * k);
        for (size_t k = 0; k < st.coupling.size(); ++k) out_mat(st.coupling[k], coupling + B * B * k);
        for (int k = 0; k < n; ++k) out_mat(st.rhs[k], rhs + B * M * k);
      },
      nullptr, 0);
}
}  // namespace

extern "C" {

// OEE (thomas=0) or block Thomas (thomas=1) for B in {1,2,5}, M in {1,3}.
int orc_tridiag_solve(int B, int M, int thomas, int n, const double* diag, const double* upper, const double* rhs,
                      double* x, int* rounds, int* err_round, int* err_index, char* err, int errlen) {
#define PD_OEE_CASE(BB, MM) \
  if (B == BB && M == MM)   \
    return oee_dispatch<BB, MM>(n, diag, upper, rhs, x, rounds, err_round, err_index, err, errlen, thomas != 0);
  PD_OEE_CASE(1, 1)
  PD_OEE_CASE(2, 1)
  PD_OEE_CASE(5, 1)
  PD_OEE_CASE(5, 3)
#undef PD_OEE_CASE
  return ST_INVALID_ARGUMENT;
}

// One elimination round in place (coupling array sized n - distance in,
// n - 2*distance valid out).
int orc_oee_round(int B, int n, int distance, int round, double* diag, double* coupling, double* rhs) {
  if (B == 2) return oee_round_dispatch<2, 1>(n, distance, round, diag, coupling, rhs);
  if (B == 5) return oee_round_dispatch<5, 1>(n, distance, round, diag, coupling, rhs);
  return ST_INVALID_ARGUMENT;
}

// Full-pivot LU rank (oee.hpp:43 isInvertible semantics) for B = 5.
int orc_fullpivlu_rank5(const double* m25) { return FullPivLU<5>(in_mat<5, 5>(m25)).rank(); }

}  // extern "C"
